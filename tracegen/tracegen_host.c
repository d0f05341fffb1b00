/*
 * tracegen_host.c -- host build of the seeded trace generator (tcm_tracegen.h).
 * Input preparation for tests, smoke() and bench.py's host-buffer (e2e) leg.  Holds
 * none of the scheduling arithmetic.  Build: gcc -O2 -ffp-contract=off -fopenmp.
 */
#include "tcm_tracegen.h"

tg_replica tcmgen_make_replica(uint64_t base_seed, uint64_t replica, uint32_t n_requests,
                               double rate_per_s, double mix_text, double mix_image,
                               uint64_t kv_capacity, uint32_t flags)
{
    return tg_make_replica(base_seed, replica, n_requests, rate_per_s, mix_text, mix_image,
                           kv_capacity, flags);
}

/* Fill R replicas; replica r occupies [offset[r], offset[r+1]) of the SoA arrays.
 * Requires offset[r+1] - offset[r] == reps[r].n_requests. */
int tcmgen_fill(const tg_replica* reps, uint32_t R, const uint64_t* offset,
                uint64_t* arrival_us, uint32_t* footprint, uint32_t* inline_us,
                uint16_t* out_tokens, uint8_t* modality)
{
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(| : bad)
    for (long r = 0; r < (long)R; ++r) {
        uint64_t base = offset[r];
        if (offset[r + 1] - base != reps[r].n_requests) { bad |= 1; continue; }
        uint64_t t = 0;
        for (uint32_t i = 0; i < reps[r].n_requests; ++i) {
            tg_request q = tg_draw(&reps[r], i);
            if (i > 0) t += q.gap_us;
            arrival_us[base + i] = t;
            footprint[base + i] = q.footprint;
            inline_us[base + i] = q.inline_us;
            out_tokens[base + i] = q.out_tokens;
            modality[base + i] = q.modality;
        }
    }
    return bad ? -1 : 0;
}
