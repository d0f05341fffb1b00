// tcm_api.cu -- the C ABI of libtcm (include/tcm.h): context, trace binding, workspace,
// engine dispatch, statistics.  Host-side orchestration only; every step of the
// scheduling path runs in the kernels of tcm_fused.cu / tcm_stepwise.cu / tcm_aux.cu.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "tcm_aux.cuh"
#include "tcm_internal.cuh"
#include "tcm_stepwise.cuh"

using namespace tcm;

struct tcm_ctx {
    tcm_config cfg{};
    ModelConst m{};
    cudaStream_t s = nullptr;
    int device = 0;
    std::string err;
    bool loaded = false;
    TraceDev t{};
    std::vector<std::pair<void*, size_t>> allocs;   // workspace + HOST mirrors
    std::vector<std::pair<void*, size_t>> spare;    // the previous trace's, reused by size on reload
    bool host_results = false;
    tcm_results_view host_res{};
    uint32_t* d_active = nullptr;        // [1]
    unsigned long long* d_acc = nullptr; // [kAccN]
    uint32_t* d_val = nullptr;           // [3] worst status, first bad replica, any TCM_KV_GROWTH (16 bytes)
    StepwiseWorkspace sw{};
    uint64_t launches = 0;
    // device timing of the library's launches (tcm_stats_host.*_ms)
    cudaEvent_t ev[9] = {};              // reset begin/end, engine begin/end, stamp end, k_step begin/end,
                                         // tcm_run_async: engine done, results copied
    bool async_pending = false;          // a tcm_run_async not yet completed by tcm_wait(TCM_WAIT_ALL)
    bool reset_pending = false;          // ev[0..1] recorded, not yet read
    double reset_ms = 0, engine_ms = 0, stamp_ms = 0;
    // tcm_step(n <= kGraphMaxIters): the call's launches (k_step, or k_fused + stamp with the
    // events and the active-count copy) replayed as one CUDA graph per n, captured on the second
    // call with that n (the first one runs eagerly: it also initialises per-device launch caches)
    struct Graph { uint32_t iters; cudaGraphExec_t exec; uint64_t launches; bool deferred; };
    std::vector<Graph> graphs;
    std::vector<uint32_t> graph_seen;
    std::vector<uint32_t> graph_never;   // n whose capture failed: always eager
    uint32_t* h_active = nullptr;        // pinned: the graphs' active-count target
    uint32_t* h_active_dev = nullptr;    // its mapped device address (stepwise graphs: k_step writes it)
    unsigned long long* h_acc = nullptr; // pinned mapped copy of the k_reduce accumulators
    unsigned long long* h_acc_dev = nullptr;
    cudaStream_t xs = nullptr;           // tcm_run_async's copy-back stream (after the engine's event)
    cudaStream_t cs = nullptr;           // capture stream (the caller's may be the legacy stream,
                                         // which cannot be captured; a graph launches into any stream)
};

namespace {

thread_local std::string g_err;

tcm_status fail(tcm_ctx* c, tcm_status code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    g_err = buf;
    return code;
}

#define TCM_CUDA(ctx, call)                                                                   \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail((ctx), TCM_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));    \
    } while (0)

// keep: park the buffers for reuse by the next tcm_load_trace (reloading a trace of the same
// shape then allocates nothing); otherwise free everything.
void free_allocs(tcm_ctx* c, bool keep = false) {
    for (auto& a : c->allocs) {
        if (keep) c->spare.push_back(a);
        else cudaFree(a.first);
    }
    c->allocs.clear();
    if (!keep) {
        for (auto& a : c->spare) cudaFree(a.first);
        c->spare.clear();
    }
    c->loaded = false;
    c->sw = StepwiseWorkspace{};
    for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);   // they captured the old trace's pointers
    c->graphs.clear();
    c->graph_seen.clear();
    c->graph_never.clear();
}

tcm_status dalloc(tcm_ctx* c, void** p, size_t bytes) {
    if (bytes == 0) bytes = 16;
    for (size_t i = 0; i < c->spare.size(); ++i) {
        if (c->spare[i].second == bytes) {
            *p = c->spare[i].first;
            c->spare.erase(c->spare.begin() + i);
            c->allocs.push_back({*p, bytes});
            return TCM_OK;
        }
    }
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess && !c->spare.empty()) {      // the parked buffers may be in the way
        cudaGetLastError();
        for (auto& a : c->spare) cudaFree(a.first);
        c->spare.clear();
        e = cudaMalloc(p, bytes);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(c, TCM_E_OOM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
    }
    c->allocs.push_back({*p, bytes});
    return TCM_OK;
}

tcm_status validate_config(const tcm_config* cfg) {
    if (!cfg) return fail(nullptr, TCM_E_ARG, "config is NULL");
    if (cfg->abi_version != TCM_ABI_VERSION)
        return fail(nullptr, TCM_E_VERSION, "abi_version %u != %u", cfg->abi_version, TCM_ABI_VERSION);
    if (cfg->engine > TCM_ENGINE_STEPWISE) return fail(nullptr, TCM_E_ARG, "bad engine %u", cfg->engine);
    if (cfg->slo_den == 0 || cfg->n_cells == 0 || cfg->reserved != 0)
        return fail(nullptr, TCM_E_ARG, "slo_den and n_cells must be >= 1, reserved 0");
    for (int c = 0; c < 3; ++c) {
        if (!(cfg->k[c] >= 0.0) || !(cfg->p[c] > 0.0) || !(cfg->S[c] >= 0.0))
            return fail(nullptr, TCM_E_ARG, "priority constants must be finite, k,S >= 0, p > 0");
    }
    return TCM_OK;
}

ModelConst to_model(const tcm_config& c) {
    ModelConst m{};
    m.c0 = c.c0_us;
    m.cp = c.cp_us;
    m.cd = c.cd_us;
    for (int i = 0; i < 3; ++i) {
        m.S[i] = c.S[i];
        m.k[i] = c.k[i];
        m.p[i] = c.p[i];
        m.thr_mc[i] = c.thr_mc[i];
        m.thr_ct[i] = c.thr_ct[i];
    }
    m.slo_num = c.slo_num;
    m.slo_den = c.slo_den;
    m.n_cells = c.n_cells;
    return m;
}

size_t ws_bytes(const tcm_config* cfg, uint32_t R, uint64_t N, int host_mirror) {
    size_t b = 0;
    if (cfg && cfg->engine == TCM_ENGINE_STEPWISE) {
        b += 4 * N;                              // link
        b += (size_t)R * kCalSlots * 4;          // calendar slot list heads
    } else {
        b += (sizeof(FRec) + 32 + 8) * N;        // class-segment records, event log, finish iterations
        b += sizeof(FRec) * 6ull * R;            // segment sentinels
        b += (size_t)R * kCalSlots * 8;          // calendar slot counters
    }
    b += (size_t)R * kCalWords * 4;              // occupancy
    b += (size_t)R * sizeof(ReplicaState);
    b += (size_t)R * sizeof(ClassPack);
    b += 20 * N;                                 // results kept on device when not supplied
    if (cfg && cfg->engine == TCM_ENGINE_STEPWISE) b += stepwise_workspace_bytes(R, N) + 8 * N;
    if (cfg && cfg->engine == TCM_ENGINE_STEPWISE) b += 40 * N;   // NEXT-1 per-request state + results
    if (host_mirror) b += (size_t)(R + 1) * 8 + 19 * N + (size_t)R * sizeof(tcm_replica_params);
    return b;
}

tcm_status copy_results_to_host(tcm_ctx* c, cudaStream_t s = nullptr) {
    if (!c->host_results) return TCM_OK;
    if (!s) s = c->s;
    const uint64_t N = c->t.N;
    if (c->host_res.admit_seq)
        TCM_CUDA(c, cudaMemcpyAsync(c->host_res.admit_seq, c->t.admit_seq, 4 * N, cudaMemcpyDeviceToHost, s));
    if (c->host_res.first_token_us)
        TCM_CUDA(c, cudaMemcpyAsync(c->host_res.first_token_us, c->t.first_token, 8 * N, cudaMemcpyDeviceToHost, s));
    if (c->host_res.done_us)
        TCM_CUDA(c, cudaMemcpyAsync(c->host_res.done_us, c->t.done, 8 * N, cudaMemcpyDeviceToHost, s));
    if (c->host_res.preempt_count && c->t.pcount)
        TCM_CUDA(c, cudaMemcpyAsync(c->host_res.preempt_count, c->t.pcount, 4 * N, cudaMemcpyDeviceToHost, s));
    if (c->host_res.preempted_us && c->t.ptime)
        TCM_CUDA(c, cudaMemcpyAsync(c->host_res.preempted_us, c->t.ptime, 8 * N, cudaMemcpyDeviceToHost, s));
    return TCM_OK;
}

tcm_status reduce_stats(tcm_ctx* c, unsigned long long* h) {
    TCM_CUDA(c, cudaMemsetAsync(c->d_acc, 0, kAccN * 8, c->s));
    TCM_CUDA(c, cudaMemsetAsync(c->d_acc + kAccBadReplica, 0xFF, 8, c->s));
    launch_reduce(c->t, c->d_acc, c->s);
    c->launches++;
    TCM_CUDA(c, cudaGetLastError());
    if (c->h_acc_dev) {                  // stores into mapped memory: never waits behind a copy-back in flight
        launch_copy_words(c->d_acc, c->h_acc_dev, kAccN, c->s);
        c->launches++;
        TCM_CUDA(c, cudaStreamSynchronize(c->s));
        memcpy(h, c->h_acc, kAccN * 8);
        return TCM_OK;
    }
    TCM_CUDA(c, cudaMemcpyAsync(h, c->d_acc, kAccN * 8, cudaMemcpyDeviceToHost, c->s));
    TCM_CUDA(c, cudaStreamSynchronize(c->s));
    return TCM_OK;
}

// Initial state of every replica (clock 0, empty queues, all KV free).
tcm_status reset_state(tcm_ctx* c) {
    const TraceDev& t = c->t;
    cudaStream_t s = c->s;
    c->reset_ms = c->engine_ms = c->stamp_ms = 0;
    TCM_CUDA(c, cudaEventRecord(c->ev[0], s));
    const uint32_t R = t.R;
    const uint64_t N = t.N;
    if (t.cal) TCM_CUDA(c, cudaMemsetAsync(t.cal, 0xFF, (size_t)R * kCalSlots * 4, s));
    if (t.fw.cal) TCM_CUDA(c, cudaMemsetAsync(t.fw.cal, 0, (size_t)R * kCalSlots * 8, s));
    if (t.fw.fin) TCM_CUDA(c, cudaMemsetAsync(t.fw.fin, 0, 8 * (N ? N : 1), s));
    TCM_CUDA(c, cudaMemsetAsync(t.occ, 0, (size_t)R * kCalWords * 4, s));
    TCM_CUDA(c, cudaMemsetAsync(t.first_token, 0, 8 * N, s));
    TCM_CUDA(c, cudaMemsetAsync(t.done, 0, 8 * N, s));
    TCM_CUDA(c, cudaMemsetAsync(t.admit_seq, 0xFF, 4 * N, s));
    if (t.req_state) TCM_CUDA(c, cudaMemsetAsync(t.req_state, 0, N ? N : 1, s));
    if (t.pcount) TCM_CUDA(c, cudaMemsetAsync(t.pcount, 0, 4 * (N ? N : 1), s));
    if (t.ptime) TCM_CUDA(c, cudaMemsetAsync(t.ptime, 0, 8 * (N ? N : 1), s));
    if (t.genp) TCM_CUDA(c, cudaMemsetAsync(t.genp, 0, 4 * (N ? N : 1), s));
    if (t.fg.pfin) {
        const uint64_t P = N + 6ull * R;
        TCM_CUDA(c, cudaMemsetAsync(t.fg.pfin, 0, 8 * P, s));
        TCM_CUDA(c, cudaMemsetAsync(t.fg.pflag, 0, P, s));
    }
    launch_init(t, s);
    c->launches++;
    if (c->cfg.engine == TCM_ENGINE_STEPWISE) {
        stepwise_init(t, c->sw, s);
        c->launches++;
    } else {
        launch_fused_prologue(c->m, t, s);      // a1: class segments
        c->launches++;
    }
    TCM_CUDA(c, cudaGetLastError());
    TCM_CUDA(c, cudaEventRecord(c->ev[1], s));
    c->reset_pending = true;
    return TCM_OK;
}

constexpr uint32_t kGraphMaxIters = 64;

// Everything one engine call enqueues, ending with the active-count copy to `active_dst`.
// timed = false (graph capture): no event records -- events recorded by graph nodes cannot be timed
tcm_status enqueue_engine(tcm_ctx* c, uint32_t max_iters, uint32_t* active_dst, uint64_t* launches, bool* deferred,
                          bool timed = true) {
    *deferred = false;
    if (c->cfg.engine == TCM_ENGINE_FUSED) TCM_CUDA(c, cudaMemsetAsync(c->d_active, 0, 4, c->s));
    if (timed) TCM_CUDA(c, cudaEventRecord(c->ev[2], c->s));
    if (c->cfg.engine == TCM_ENGINE_FUSED) {
        launch_fused(c->m, c->t, max_iters, c->d_active, c->s);
        if (timed) TCM_CUDA(c, cudaEventRecord(c->ev[3], c->s));
        launch_fused_stamp(c->t, c->s);
        *launches += 2;
    } else {
        double kms = 0;
        // captured (graph) calls: the last k_step CTA writes the count straight into the mapped
        // host word, so the graph is the k_step launch alone
        const bool direct = !timed && active_dst == c->h_active && c->h_active_dev;
        tcm_status st = stepwise_run(c->m, c->t, c->sw, max_iters, direct ? c->h_active_dev : c->d_active, c->s,
                                     launches, timed ? c->ev[5] : nullptr, timed ? c->ev[6] : nullptr, &kms, deferred);
        c->engine_ms += kms;
        if (st != TCM_OK) return fail(c, st, "stepwise engine failed: %s", cudaGetErrorString(cudaGetLastError()));
        TCM_CUDA(c, cudaGetLastError());
        if (direct) return TCM_OK;
    }
    TCM_CUDA(c, cudaGetLastError());
    if (timed && c->cfg.engine != TCM_ENGINE_FUSED) TCM_CUDA(c, cudaEventRecord(c->ev[3], c->s));
    if (timed) TCM_CUDA(c, cudaEventRecord(c->ev[4], c->s));
    TCM_CUDA(c, cudaMemcpyAsync(active_dst, c->d_active, 4, cudaMemcpyDeviceToHost, c->s));
    return TCM_OK;
}

// The graph of a short call (max_iters <= kGraphMaxIters, one k_step chunk), or nullptr.
const tcm_ctx::Graph* step_graph(tcm_ctx* c, uint32_t max_iters) {
    if (max_iters > kGraphMaxIters || !c->h_active) return nullptr;
    if (const char* g = getenv("TCM_GRAPHS"))                 // development knob: "0" = always eager
        if (g[0] == '0') return nullptr;
    for (auto& g : c->graphs)
        if (g.iters == max_iters) return &g;
    bool seen = false;
    for (uint32_t k : c->graph_seen) seen |= k == max_iters;
    if (!seen) {                                   // first call with this n: eager
        c->graph_seen.push_back(max_iters);
        return nullptr;
    }
    for (uint32_t k : c->graph_never)
        if (k == max_iters) return nullptr;
    cudaGraph_t graph = nullptr;
    uint64_t l = 0;
    bool deferred = false;
    const std::string err0 = c->err;
    if (!c->cs && cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking) != cudaSuccess) {
        c->cs = nullptr;
        cudaGetLastError();
        return nullptr;
    }
    cudaStream_t user = c->s;
    c->s = c->cs;
    cudaError_t e = cudaStreamBeginCapture(c->s, cudaStreamCaptureModeRelaxed);
    tcm_status st = e == cudaSuccess ? enqueue_engine(c, max_iters, c->h_active, &l, &deferred, false) : TCM_E_CUDA;
    const cudaError_t ecap = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamEndCapture(c->s, &graph);
    c->s = user;
    cudaGraphExec_t exec = nullptr;
    cudaError_t einst = cudaSuccess;
    const bool one_chunk = c->cfg.engine == TCM_ENGINE_FUSED || deferred;   // stepwise: no mid-call synchronisation
    if (st == TCM_OK && e == cudaSuccess && graph && one_chunk) einst = cudaGraphInstantiate(&exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (st != TCM_OK || e != cudaSuccess || !one_chunk || einst != cudaSuccess || !exec) {
        if (getenv("TCM_GRAPH_DEBUG"))
            fprintf(stderr, "libtcm: no graph for tcm_step(%u): status %d, capture %s / %s, instantiate %s\n", max_iters,
                    (int)st, cudaGetErrorString(ecap), cudaGetErrorString(e), cudaGetErrorString(einst));
        cudaGetLastError();
        c->err = err0;                             // the eager path below is the call's result
        c->graph_never.push_back(max_iters);
        return nullptr;
    }
    c->graphs.push_back({max_iters, exec, l, deferred});
    return &c->graphs.back();
}

tcm_status run_engine(tcm_ctx* c, uint32_t max_iters, uint32_t* active) {
    if (const tcm_ctx::Graph* g = step_graph(c, max_iters)) {
        // engine_ms of a replayed call is the whole graph (its launches and the active-count copy)
        TCM_CUDA(c, cudaEventRecord(c->ev[2], c->s));
        TCM_CUDA(c, cudaGraphLaunch(g->exec, c->s));
        TCM_CUDA(c, cudaEventRecord(c->ev[3], c->s));
        TCM_CUDA(c, cudaStreamSynchronize(c->s));
        *active = *c->h_active;
        c->launches += g->launches;
        float ms = 0;
        if (c->reset_pending) {
            TCM_CUDA(c, cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
            c->reset_ms += ms;
            c->reset_pending = false;
        }
        TCM_CUDA(c, cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]));
        c->engine_ms += ms;
        return TCM_OK;
    }
    bool deferred = false;      // stepwise: k_step events still to be read after the sync below
    uint64_t l = 0;
    tcm_status st = enqueue_engine(c, max_iters, active, &l, &deferred);
    c->launches += l;
    if (st != TCM_OK) return st;
    TCM_CUDA(c, cudaStreamSynchronize(c->s));
    float ms = 0;
    if (c->reset_pending) {
        TCM_CUDA(c, cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
        c->reset_ms += ms;
        c->reset_pending = false;
    }
    if (c->cfg.engine == TCM_ENGINE_FUSED || deferred) {
        TCM_CUDA(c, cudaEventElapsedTime(&ms, deferred ? c->ev[5] : c->ev[2], deferred ? c->ev[6] : c->ev[3]));
        c->engine_ms += ms;
    }
    TCM_CUDA(c, cudaEventElapsedTime(&ms, c->ev[3], c->ev[4]));
    c->stamp_ms += ms;
    return TCM_OK;
}

}  // namespace

extern "C" {

tcm_status tcm_create(const tcm_config* cfg, void* cuda_stream, tcm_ctx** out) {
    if (!out) return fail(nullptr, TCM_E_ARG, "out is NULL");
    *out = nullptr;
    tcm_status st = validate_config(cfg);
    if (st != TCM_OK) return st;
    tcm_ctx* c = new (std::nothrow) tcm_ctx();
    if (!c) return fail(nullptr, TCM_E_OOM, "context allocation failed");
    c->cfg = *cfg;
    c->m = to_model(*cfg);
    c->s = reinterpret_cast<cudaStream_t>(cuda_stream);
    cudaError_t e = cudaGetDevice(&c->device);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_active, 4);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_acc, kAccN * 8);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_val, 16);
    for (int i = 0; i < 9 && e == cudaSuccess; ++i) e = cudaEventCreate(&c->ev[i]);
    if (e == cudaSuccess && cudaMallocHost(&c->h_active, 4) != cudaSuccess) {
        c->h_active = nullptr;                      // no pinned word: short calls run eagerly
        cudaGetLastError();
    }
    if (c->h_active && cudaHostGetDevicePointer((void**)&c->h_active_dev, c->h_active, 0) != cudaSuccess) {
        c->h_active_dev = nullptr;                  // not mapped: the graph copies the count instead
        cudaGetLastError();
    }
    if (e == cudaSuccess && (cudaMallocHost(&c->h_acc, kAccN * 8) != cudaSuccess ||
                             cudaHostGetDevicePointer((void**)&c->h_acc_dev, c->h_acc, 0) != cudaSuccess)) {
        c->h_acc_dev = nullptr;                     // the stats read back with a copy instead
        cudaGetLastError();
    }
    if (e != cudaSuccess) {
        fail(nullptr, TCM_E_CUDA, "tcm_create: %s", cudaGetErrorString(e));
        cudaFree(c->d_active);
        cudaFree(c->d_acc);
        cudaFree(c->d_val);
        for (auto& ev : c->ev)
            if (ev) cudaEventDestroy(ev);
        delete c;
        return TCM_E_CUDA;
    }
    *out = c;
    return TCM_OK;
}

tcm_status tcm_load_trace(tcm_ctx* c, const tcm_trace_view* tv, const tcm_results_view* rv) {
    if (!c) return fail(nullptr, TCM_E_ARG, "ctx is NULL");
    if (c->async_pending) return fail(c, TCM_E_STATE, "tcm_load_trace while a tcm_run_async is pending (tcm_wait first)");
    if (!tv) return fail(c, TCM_E_ARG, "trace is NULL");
    if (tv->n_replicas == 0) return fail(c, TCM_E_ARG, "n_replicas must be >= 1");
    if (!tv->req_offset || !tv->params || (tv->n_requests > 0 && (!tv->arrival_us || !tv->footprint ||
        !tv->inline_us || !tv->out_tokens || !tv->modality)))
        return fail(c, TCM_E_ARG, "trace arrays must be non-NULL");
    if (tv->mem > TCM_MEM_HOST || (rv && rv->mem > TCM_MEM_HOST)) return fail(c, TCM_E_ARG, "bad mem kind");
    free_allocs(c, true);
    const uint32_t R = tv->n_replicas;
    const uint64_t N = tv->n_requests;
    TraceDev t{};
    t.R = R;
    t.N = N;
    cudaStream_t s = c->s;
    tcm_status st;

    if (tv->mem == TCM_MEM_HOST) {
        if (tv->req_offset[R] != N || tv->req_offset[0] != 0)
            return fail(c, TCM_E_ARG, "req_offset[R] (%llu) != n_requests (%llu)",
                        (unsigned long long)tv->req_offset[R], (unsigned long long)N);
        void *o, *a, *f, *il, *ou, *md, *pp;
        if ((st = dalloc(c, &o, (R + 1) * 8ull)) || (st = dalloc(c, &a, 8 * N)) || (st = dalloc(c, &f, 4 * N)) ||
            (st = dalloc(c, &il, 4 * N)) || (st = dalloc(c, &ou, 2 * N)) || (st = dalloc(c, &md, N)) ||
            (st = dalloc(c, &pp, R * sizeof(tcm_replica_params))))
            return st;
        TCM_CUDA(c, cudaMemcpyAsync(o, tv->req_offset, (R + 1) * 8ull, cudaMemcpyHostToDevice, s));
        TCM_CUDA(c, cudaMemcpyAsync(a, tv->arrival_us, 8 * N, cudaMemcpyHostToDevice, s));
        TCM_CUDA(c, cudaMemcpyAsync(f, tv->footprint, 4 * N, cudaMemcpyHostToDevice, s));
        TCM_CUDA(c, cudaMemcpyAsync(il, tv->inline_us, 4 * N, cudaMemcpyHostToDevice, s));
        TCM_CUDA(c, cudaMemcpyAsync(ou, tv->out_tokens, 2 * N, cudaMemcpyHostToDevice, s));
        TCM_CUDA(c, cudaMemcpyAsync(md, tv->modality, N, cudaMemcpyHostToDevice, s));
        TCM_CUDA(c, cudaMemcpyAsync(pp, tv->params, R * sizeof(tcm_replica_params), cudaMemcpyHostToDevice, s));
        t.offset = (const uint64_t*)o;
        t.arrival = (const uint64_t*)a;
        t.footprint = (const uint32_t*)f;
        t.inl = (const uint32_t*)il;
        t.out = (const uint16_t*)ou;
        t.mod = (const uint8_t*)md;
        t.params = (const tcm_replica_params*)pp;
    } else {
        uint64_t lastoff = 0;
        TCM_CUDA(c, cudaMemcpyAsync(&lastoff, tv->req_offset + R, 8, cudaMemcpyDeviceToHost, s));
        TCM_CUDA(c, cudaStreamSynchronize(s));
        if (lastoff != N)
            return fail(c, TCM_E_ARG, "req_offset[R] (%llu) != n_requests (%llu)",
                        (unsigned long long)lastoff, (unsigned long long)N);
        t.offset = tv->req_offset;
        t.arrival = tv->arrival_us;
        t.footprint = tv->footprint;
        t.inl = tv->inline_us;
        t.out = tv->out_tokens;
        t.mod = tv->modality;
        t.params = tv->params;
    }

    // results: caller DEVICE buffers, or device workspace (+ copy-back for HOST buffers)
    c->host_results = rv && rv->mem == TCM_MEM_HOST;
    if (c->host_results) c->host_res = *rv;
    const bool dev_res = rv && rv->mem == TCM_MEM_DEVICE;
    void* p;
    if (dev_res && rv->admit_seq) t.admit_seq = rv->admit_seq;
    else { if ((st = dalloc(c, &p, 4 * N))) return st; t.admit_seq = (uint32_t*)p; }
    if (dev_res && rv->first_token_us) t.first_token = rv->first_token_us;
    else { if ((st = dalloc(c, &p, 8 * N))) return st; t.first_token = (uint64_t*)p; }
    if (dev_res && rv->done_us) t.done = rv->done_us;
    else { if ((st = dalloc(c, &p, 8 * N))) return st; t.done = (uint64_t*)p; }

    // workspace
    if (c->cfg.engine == TCM_ENGINE_STEPWISE) {
        if ((st = dalloc(c, &p, 4 * N))) return st;
        t.link = (uint32_t*)p;
        if ((st = dalloc(c, &p, (size_t)R * kCalSlots * 4))) return st;
        t.cal = (uint32_t*)p;
    } else {
        if ((st = dalloc(c, &p, sizeof(FRec) * (N + 6ull * R)))) return st;
        t.fw.rec = (FRec*)p;
        if ((st = dalloc(c, &p, 32 * N))) return st;
        t.fw.log = (uint64_t*)p;
        if ((st = dalloc(c, &p, 8 * N))) return st;
        t.fw.fin = (uint64_t*)p;
        if ((st = dalloc(c, &p, (size_t)R * kCalSlots * 8))) return st;
        t.fw.cal = (uint64_t*)p;
    }
    if ((st = dalloc(c, &p, (size_t)R * kCalWords * 4))) return st;
    t.occ = (uint32_t*)p;
    if ((st = dalloc(c, &p, (size_t)R * sizeof(ReplicaState)))) return st;
    t.state = (ReplicaState*)p;
    if ((st = dalloc(c, &p, (size_t)R * sizeof(ClassPack)))) return st;
    t.kpack = (ClassPack*)p;
    if (c->cfg.engine == TCM_ENGINE_STEPWISE) {
        if ((st = dalloc(c, &p, N ? N : 1))) return st;
        t.req_state = (uint8_t*)p;
        if ((st = dalloc(c, &p, stepwise_extra_bytes(R, N)))) return st;
        c->sw = stepwise_bind(p, R, N);
        if ((st = dalloc(c, &p, 8 * (N ? N : 1)))) return st;
        t.deadline = (uint64_t*)p;
        // NEXT-1 (TCM_KV_GROWTH) per-request state and results
        const uint64_t Nn = N ? N : 1;
        if ((st = dalloc(c, &p, 4 * Nn))) return st;
        t.kvres = (uint32_t*)p;
        if ((st = dalloc(c, &p, 4 * Nn))) return st;
        t.kvfin = (uint32_t*)p;
        if ((st = dalloc(c, &p, 8 * Nn))) return st;
        t.fin = (uint64_t*)p;
        if ((st = dalloc(c, &p, 4 * Nn))) return st;
        t.genp = (uint32_t*)p;
        if ((st = dalloc(c, &p, 8 * Nn))) return st;
        t.pstart = (uint64_t*)p;
        if (dev_res && rv->preempt_count) t.pcount = rv->preempt_count;
        else { if ((st = dalloc(c, &p, 4 * Nn))) return st; t.pcount = (uint32_t*)p; }
        if (dev_res && rv->preempted_us) t.ptime = rv->preempted_us;
        else { if ((st = dalloc(c, &p, 8 * Nn))) return st; t.ptime = (uint64_t*)p; }
    }

    c->t = t;

    // validate on the device (R18) before any kernel reads the trace
    uint32_t hv[3] = {0, 0xFFFFFFFFu, 0};
    TCM_CUDA(c, cudaMemcpyAsync(c->d_val, hv, 12, cudaMemcpyHostToDevice, s));
    launch_validate(t, c->d_val, c->cfg.engine == TCM_ENGINE_STEPWISE, s);
    c->launches++;
    TCM_CUDA(c, cudaGetLastError());
    if (c->h_acc_dev) {                  // through mapped memory (see reduce_stats)
        launch_copy_words(reinterpret_cast<const unsigned long long*>(c->d_val), c->h_acc_dev, 2, s);
        c->launches++;
        TCM_CUDA(c, cudaStreamSynchronize(s));
        memcpy(hv, c->h_acc, 12);
    } else {
        TCM_CUDA(c, cudaMemcpyAsync(hv, c->d_val, 12, cudaMemcpyDeviceToHost, s));
        TCM_CUDA(c, cudaStreamSynchronize(s));
    }
    c->t.any_growth = t.any_growth = hv[2] & 1u;
    c->t.all_growth = t.all_growth = (hv[2] & 2u) == 0;
    c->t.all_tcm = t.all_tcm = (hv[2] & 4u) == 0;
    if (c->cfg.engine == TCM_ENGINE_FUSED && t.any_growth && hv[0] == ST_OK) {
        // NEXT-1 on the fused engine (k_fgrow): per-position state, per-class stacks, preemption results
        const uint64_t P = N + 6ull * R;
        if ((st = dalloc(c, &p, 8 * P))) return st;
        t.fg.pfin = (uint64_t*)p;
        if ((st = dalloc(c, &p, 4 * P))) return st;
        t.fg.pkv = (uint32_t*)p;
        if ((st = dalloc(c, &p, 4 * P))) return st;
        t.fg.prem = (uint32_t*)p;
        if ((st = dalloc(c, &p, 4 * P))) return st;
        t.fg.pgen = (uint32_t*)p;
        if ((st = dalloc(c, &p, 4 * P))) return st;
        t.fg.pnext = (uint32_t*)p;
        if ((st = dalloc(c, &p, P))) return st;
        t.fg.pflag = (uint8_t*)p;
        if ((st = dalloc(c, &p, 12ull * R))) return st;
        t.fg.top = (uint32_t*)p;
        if ((st = dalloc(c, &p, 12ull * R))) return st;
        t.fg.seg = (uint32_t*)p;
        if ((st = dalloc(c, &p, 12ull * R))) return st;
        t.fg.hres = (uint32_t*)p;
        const uint64_t Nn = N ? N : 1;
        if ((st = dalloc(c, &p, 8 * Nn))) return st;
        t.pstart = (uint64_t*)p;
        if (dev_res && rv->preempt_count) t.pcount = rv->preempt_count;
        else { if ((st = dalloc(c, &p, 4 * Nn))) return st; t.pcount = (uint32_t*)p; }
        if (dev_res && rv->preempted_us) t.ptime = rv->preempted_us;
        else { if ((st = dalloc(c, &p, 8 * Nn))) return st; t.ptime = (uint64_t*)p; }
        c->t = t;
    }
    if (hv[0] == ST_CAPACITY)
        return fail(c, TCM_E_CAPACITY, "replica %u: a footprint (with TCM_KV_GROWTH: footprint + out - 1) exceeds kv_capacity (R18, R28)", hv[1]);
    if (hv[0] != ST_OK)
        return fail(c, TCM_E_ARG, "replica %u: malformed trace or params (footprint/out/modality/"
                    "arrival order/policy/budget/kv/alpha/flags; EDF, TCM_ADMIT_SKIP, TCM_KV_GROWTH and replicas of "
                    ">= 2^24 requests need the "
                    "stepwise engine)", hv[1]);
    launch_kpack(c->m, t, s);                 // params are validated: K1 class constants once
    c->launches++;
    TCM_CUDA(c, cudaGetLastError());
    {
        tcm_status rs = reset_state(c);
        if (rs != TCM_OK) return rs;
    }
    for (auto& a : c->spare) cudaFree(a.first);     // what this trace did not reuse
    c->spare.clear();
    c->loaded = true;
    c->err.clear();
    return TCM_OK;
}

tcm_status tcm_reset(tcm_ctx* c) {
    if (!c) return fail(nullptr, TCM_E_ARG, "ctx is NULL");
    if (c->async_pending) return fail(c, TCM_E_STATE, "tcm_reset while a tcm_run_async is pending (tcm_wait first)");
    if (!c->loaded) return fail(c, TCM_E_STATE, "tcm_reset before tcm_load_trace");
    return reset_state(c);
}

tcm_status tcm_step(tcm_ctx* c, uint32_t max_iterations, uint32_t* active_replicas) {
    if (!c) return fail(nullptr, TCM_E_ARG, "ctx is NULL");
    if (c->async_pending) return fail(c, TCM_E_STATE, "tcm_step while a tcm_run_async is pending (tcm_wait first)");
    if (!c->loaded) return fail(c, TCM_E_STATE, "tcm_step before tcm_load_trace");
    uint32_t active = 0;
    tcm_status st = run_engine(c, max_iterations, &active);
    if (st != TCM_OK) return st;
    if (c->host_results) {     // DEVICE results need no copy and no second synchronisation
        if ((st = copy_results_to_host(c)) != TCM_OK) return st;
        TCM_CUDA(c, cudaStreamSynchronize(c->s));
    }
    if (active_replicas) *active_replicas = active;
    return TCM_OK;
}

tcm_status tcm_run(tcm_ctx* c) {
    if (!c) return fail(nullptr, TCM_E_ARG, "ctx is NULL");
    if (c->async_pending) return fail(c, TCM_E_STATE, "tcm_run while a tcm_run_async is pending (tcm_wait first)");
    if (!c->loaded) return fail(c, TCM_E_STATE, "tcm_run before tcm_load_trace");
    uint32_t active = 1;
    while (active > 0) {
        tcm_status st = run_engine(c, 0xFFFFFFFFu, &active);
        if (st != TCM_OK) return st;
    }
    unsigned long long h[kAccN];
    tcm_status st = reduce_stats(c, h);
    if (st != TCM_OK) return st;
    if ((st = copy_results_to_host(c)) != TCM_OK) return st;
    TCM_CUDA(c, cudaStreamSynchronize(c->s));
    if (h[kAccBadStatus] != 0)
        return fail(c, TCM_E_REPLICA, "replica %llu reported status %llu (deadlock assertion)",
                    h[kAccBadReplica], h[kAccBadStatus]);
    return TCM_OK;
}

tcm_status tcm_run_async(tcm_ctx* c) {
    if (!c) return fail(nullptr, TCM_E_ARG, "ctx is NULL");
    if (!c->loaded) return fail(c, TCM_E_STATE, "tcm_run_async before tcm_load_trace");
    if (c->cfg.engine != TCM_ENGINE_FUSED) return fail(c, TCM_E_ARG, "tcm_run_async: FUSED engine only");
    if (c->async_pending) return fail(c, TCM_E_STATE, "tcm_run_async: the previous run is still pending (tcm_wait)");
    if (!c->h_active) return fail(c, TCM_E_STATE, "tcm_run_async: no pinned host word");
    // one engine launch runs every replica to completion (the iteration budget never binds), then the
    // stamping; the active count lands in the pinned word and is checked by tcm_wait
    uint64_t l = 0;
    bool deferred = false;
    tcm_status st = enqueue_engine(c, 0xFFFFFFFFu, c->h_active, &l, &deferred);
    c->launches += l;
    if (st != TCM_OK) return st;
    TCM_CUDA(c, cudaEventRecord(c->ev[7], c->s));
    // the copy-back runs on a stream of its own once the kernels are done, so tcm_stats (kernels on
    // the context's stream) need not wait for it
    if (!c->xs) TCM_CUDA(c, cudaStreamCreateWithFlags(&c->xs, cudaStreamNonBlocking));
    TCM_CUDA(c, cudaStreamWaitEvent(c->xs, c->ev[7], 0));
    if ((st = copy_results_to_host(c, c->xs)) != TCM_OK) return st;
    TCM_CUDA(c, cudaEventRecord(c->ev[8], c->xs));
    c->async_pending = true;                 // load / reset / step / run wait for tcm_wait(TCM_WAIT_ALL)
    return TCM_OK;
}

tcm_status tcm_wait(tcm_ctx* c, int what) {
    if (!c) return fail(nullptr, TCM_E_ARG, "ctx is NULL");
    if (what != TCM_WAIT_ENGINE && what != TCM_WAIT_ALL) return fail(c, TCM_E_ARG, "tcm_wait: bad what (%d)", what);
    if (!c->async_pending) return TCM_OK;
    if (what == TCM_WAIT_ENGINE) {
        TCM_CUDA(c, cudaEventSynchronize(c->ev[7]));
        return TCM_OK;
    }
    TCM_CUDA(c, cudaEventSynchronize(c->ev[8]));
    c->async_pending = false;
    float ms = 0;
    if (c->reset_pending) {
        TCM_CUDA(c, cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
        c->reset_ms += ms;
        c->reset_pending = false;
    }
    TCM_CUDA(c, cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]));
    c->engine_ms += ms;
    TCM_CUDA(c, cudaEventElapsedTime(&ms, c->ev[3], c->ev[4]));
    c->stamp_ms += ms;
    if (*c->h_active != 0) return fail(c, TCM_E_STATE, "tcm_wait: %u replicas unfinished", *c->h_active);
    unsigned long long h[kAccN];
    tcm_status st = reduce_stats(c, h);
    if (st != TCM_OK) return st;
    if (h[kAccBadStatus] != 0)
        return fail(c, TCM_E_REPLICA, "replica %llu reported status %llu (deadlock assertion)",
                    h[kAccBadReplica], h[kAccBadStatus]);
    return TCM_OK;
}

tcm_status tcm_stats(tcm_ctx* c, tcm_stats_host* out, int64_t* dev_hist, int64_t* dev_cnt) {
    if (!c) return fail(nullptr, TCM_E_ARG, "ctx is NULL");
    if (!c->loaded) return fail(c, TCM_E_STATE, "tcm_stats before tcm_load_trace");
    unsigned long long h[kAccN];
    tcm_status st = reduce_stats(c, h);
    if (st != TCM_OK) return st;
    if (out) {
        out->iterations = h[kAccIter];
        out->decisions = h[kAccDecisions];
        out->ff_iterations = h[kAccFF];
        out->idle_jumps = h[kAccIdle];
        out->sum_pending = h[kAccSumPending];
        out->max_pending = h[kAccMaxPending];
        out->requests_done = h[kAccDone];
        out->replicas_done = h[kAccReplicasDone];
        out->replicas_active = h[kAccReplicasActive];
        out->scanned_decisions = h[kAccScanned];
        out->preemptions = h[kAccPreempt];
        out->forced_preemptions = h[kAccForced];
        out->first_bad_replica = h[kAccBadStatus] ? (int32_t)h[kAccBadReplica] : -1;
        out->first_bad_status = (int32_t)h[kAccBadStatus];
        if (c->reset_pending) {
            float ms = 0;
            TCM_CUDA(c, cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
            c->reset_ms += ms;
            c->reset_pending = false;
        }
        out->reset_ms = c->reset_ms;
        out->engine_ms = c->engine_ms;
        out->stamp_ms = c->stamp_ms;
    }
    if (dev_hist || dev_cnt) {
        if (h[kAccReplicasActive] != 0)
            return fail(c, TCM_E_STATE, "aggregation needs every replica finished (%llu active)",
                        h[kAccReplicasActive]);
        if (!dev_hist || !dev_cnt) return fail(c, TCM_E_ARG, "dev_hist and dev_cnt go together");
        const size_t hb = (size_t)c->m.n_cells * kGroups * kHistBins * 8;
        const size_t cb = (size_t)c->m.n_cells * kGroups * kNcnt * 8;
        TCM_CUDA(c, cudaMemsetAsync(dev_hist, 0, hb, c->s));
        TCM_CUDA(c, cudaMemsetAsync(dev_cnt, 0, cb, c->s));
        launch_aggregate(c->m, c->t, reinterpret_cast<unsigned long long*>(dev_hist),
                         reinterpret_cast<unsigned long long*>(dev_cnt), c->s);
        c->launches++;
        TCM_CUDA(c, cudaGetLastError());
        TCM_CUDA(c, cudaStreamSynchronize(c->s));
    }
    if (out) out->kernel_launches = c->launches;
    return TCM_OK;
}

tcm_status tcm_replica_counters(tcm_ctx* c, uint64_t* dev_out) {
    if (!c) return fail(nullptr, TCM_E_ARG, "ctx is NULL");
    if (!c->loaded) return fail(c, TCM_E_STATE, "tcm_replica_counters before tcm_load_trace");
    if (!dev_out) return fail(c, TCM_E_ARG, "dev_out is NULL");
    launch_replica_counters(c->t, reinterpret_cast<unsigned long long*>(dev_out), c->s);
    c->launches++;
    TCM_CUDA(c, cudaGetLastError());
    TCM_CUDA(c, cudaStreamSynchronize(c->s));
    return TCM_OK;
}

tcm_status tcm_preemption_stats(tcm_ctx* c, int64_t* dev_out) {
    if (!c) return fail(nullptr, TCM_E_ARG, "ctx is NULL");
    if (!c->loaded) return fail(c, TCM_E_STATE, "tcm_preemption_stats before tcm_load_trace");
    if (!dev_out) return fail(c, TCM_E_ARG, "dev_out is NULL");
    TCM_CUDA(c, cudaMemsetAsync(dev_out, 0, (size_t)c->m.n_cells * kGroups * 3 * 8, c->s));
    if (c->t.pcount) {                  // NEXT-1 results exist (some replica runs TCM_KV_GROWTH)
        launch_preempt_stats(c->m, c->t, reinterpret_cast<unsigned long long*>(dev_out), c->s);
        c->launches++;
        TCM_CUDA(c, cudaGetLastError());
    }
    TCM_CUDA(c, cudaStreamSynchronize(c->s));
    return TCM_OK;
}

void tcm_destroy(tcm_ctx* c) {
    if (!c) return;
    free_allocs(c);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    cudaFree(c->d_active);
    cudaFree(c->d_acc);
    cudaFree(c->d_val);
    if (c->h_active) cudaFreeHost(c->h_active);
    if (c->h_acc) cudaFreeHost(c->h_acc);
    if (c->cs) cudaStreamDestroy(c->cs);
    if (c->xs) cudaStreamDestroy(c->xs);
    delete c;
}

const char* tcm_last_error(const tcm_ctx* c) {
    return c ? c->err.c_str() : g_err.c_str();
}

size_t tcm_workspace_bytes(const tcm_config* cfg, uint32_t n_replicas, uint64_t n_requests, int host_mirror) {
    return ws_bytes(cfg, n_replicas, n_requests, host_mirror);
}

tcm_status tcm_generate_trace(const tcm_gen_replica* reps, uint32_t R, const uint64_t* off,
                              uint64_t* arrival, uint32_t* footprint, uint32_t* inl, uint16_t* out,
                              uint8_t* mod, void* stream) {
    if (!reps || !off || R == 0) return fail(nullptr, TCM_E_ARG, "bad generator arguments");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    uint32_t* bad = nullptr;
    cudaError_t e = cudaMalloc(&bad, 4);
    if (e != cudaSuccess) return fail(nullptr, TCM_E_CUDA, "cudaMalloc: %s", cudaGetErrorString(e));
    uint32_t hb = 0;
    cudaMemsetAsync(bad, 0, 4, s);
    launch_generate(reps, R, off, arrival, footprint, inl, out, mod, bad, s);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(bad);
    if (e != cudaSuccess) return fail(nullptr, TCM_E_CUDA, "generator: %s", cudaGetErrorString(e));
    if (hb) return fail(nullptr, TCM_E_ARG, "req_offset does not match n_requests");
    return TCM_OK;
}

tcm_status tcm_k1_eval(const tcm_config* cfg, const uint8_t* cls, const uint64_t* w, const double* alpha,
                       double* outp, uint64_t n, void* stream) {
    tcm_status st = validate_config(cfg);
    if (st != TCM_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    launch_k1_eval(to_model(*cfg), cls, w, alpha, outp, n, s);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(nullptr, TCM_E_CUDA, "k1_eval: %s", cudaGetErrorString(e));
    return TCM_OK;
}

tcm_status tcm_k1_audit(const tcm_config* cfg, uint32_t cls, double alpha, uint64_t lo, uint64_t hi,
                        uint64_t* first, void* stream) {
    tcm_status st = validate_config(cfg);
    if (st != TCM_OK) return st;
    if (cls > 2 || hi <= lo || !first) return fail(nullptr, TCM_E_ARG, "bad audit arguments");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(first, 0xFF, 8, s);
    if (e == cudaSuccess) {
        launch_k1_audit(to_model(*cfg), cls, alpha, lo, hi, reinterpret_cast<unsigned long long*>(first), s);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(nullptr, TCM_E_CUDA, "k1_audit: %s", cudaGetErrorString(e));
    return TCM_OK;
}

tcm_status tcm_k1_filter_error(const tcm_config* cfg, uint32_t cls, double alpha, uint64_t lo, uint64_t hi,
                               uint64_t step, double* max_err, void* stream) {
    tcm_status st = validate_config(cfg);
    if (st != TCM_OK) return st;
    if (cls > 2 || hi <= lo || step == 0 || !max_err) return fail(nullptr, TCM_E_ARG, "bad filter-audit arguments");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    unsigned long long* d = nullptr;
    cudaError_t e = cudaMalloc(&d, 8);
    if (e == cudaSuccess) e = cudaMemsetAsync(d, 0, 8, s);
    if (e == cudaSuccess) {
        launch_filter_audit(to_model(*cfg), cls, alpha, lo, hi, step, d, s);
        e = cudaGetLastError();
    }
    unsigned long long h = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(d);
    if (e != cudaSuccess) return fail(nullptr, TCM_E_CUDA, "k1_filter_error: %s", cudaGetErrorString(e));
    memcpy(max_err, &h, 8);
    return TCM_OK;
}

}  // extern "C"
