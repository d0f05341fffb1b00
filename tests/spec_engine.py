"""A second, declarative statement of the scheduling step, used ONLY to pin the oracle.

Written from PAPER.md:315, 447-461, 572, 580 and SPEC.md:131-144, 394-403, 455 with the
readings R1-R25, in a deliberately different shape from oracle/tcm_oracle.c:
per-request dicts, Python's sorted() with a tuple key, and the paper's priority formula
evaluated with Python's math library (not K1).  Because math.exp/pow differ from K1 in the
last bits, callers must discard traces whose order depends on a near-tie
(`near_tie` is set when two keys of different classes are within 1e-11 of each other).
"""
from __future__ import annotations

import math

S = (0.1, 0.05, 0.0)
K = (0.05, 0.003, 0.00075)
P = (3.5, 2.5, 1.1)


def paper_priority(c, w_us, alpha):
    if w_us == 0 or alpha == 0.0:
        return S[c]
    return S[c] + (1.0 - math.exp(-alpha * K[c] * (w_us / 1e6) ** P[c]))


def classify(mod, f, thr):
    mc, ct = thr[mod]
    return 0 if f < mc else (1 if f < ct else 2)


def iso_e2e(f, inl, out, B, c0=5000, cp=20, cd=500):
    return inl + -(-f // B) * c0 + cp * f + (out - 1) * (c0 + cd)


def run(reqs, policy, alpha=1.0, kv=131072, B=2048, c0=5000, cp=20, cd=500,
        thr=((4096, 2**32 - 1), (0, 2**32 - 1), (0, 8192)), skip=False, slo=5, growth=False):
    """reqs: list of (arrival_us, footprint, inline_us, out, modality); policy: 0 FCFS, 1 TCM,
    2 EDF (deadline = arrival + slo x isolated E2E), 3 naive aging.  growth=True: NEXT-1 decode
    KV growth and preemption by recomputation (R28-R32).  Returns dict of lists."""
    n = len(reqs)
    R = [dict(id=i, arr=a, f=f, inl=il, out=o, cls=classify(m, f, thr), state="future",
              rem=f, gen=0, admit=None, first=None, done=None, held=0, npre=0, tpre=0, since=None)
         for i, (a, f, il, o, m) in enumerate(reqs)]
    clock, free, seq = 0, kv, 0
    near_tie = False
    it_no = 0                                             # engine iterations (R34 marks victims)
    while True:
        for r in R:                                       # step 1: ingest
            if r["state"] == "future" and r["arr"] <= clock:
                r["state"] = "waiting"
        pend = [r for r in R if r["state"] in ("waiting", "partial")]
        dec = [r for r in R if r["state"] == "decoding"]
        if not pend and not dec:                          # step 2: idle jump
            fut = [r["arr"] for r in R if r["state"] == "future"]
            if not fut:
                break
            clock = min(fut)
            continue
        if growth:
            # R28/R29: the decode tokens of this iteration need len(dec) free KV tokens; the
            # victim is the running request that comes LAST in the policy's order (TCM: by
            # priority among non-motorcycles first; otherwise: latest arrival)
            while free < len(dec):
                running = [r for r in R if r["state"] in ("partial", "decoding")]
                if policy == 1:
                    pool = [r for r in running if r["cls"] != 0] or running
                    keyed = sorted(((max(paper_priority(r["cls"], clock - r["arr"], alpha), 1e-12), r)
                                    for r in pool), key=lambda t: (-t[0], t[1]["arr"], t[1]["id"]))
                    if len(keyed) > 1 and keyed[-2][1]["cls"] != keyed[-1][1]["cls"] and \
                            abs(keyed[-2][0] - keyed[-1][0]) < 1e-11:
                        near_tie = True
                    v = keyed[-1][1]
                else:
                    v = max(running, key=lambda r: (r["arr"], r["id"]))
                free += v["held"]
                v["rem"], v["held"] = v["held"], 0          # R30: recompute what it held
                v["state"], v["since"] = "waiting", clock
                v["npre"] += 1
                dec = [r for r in R if r["state"] == "decoding"]
            pend = [r for r in R if r["state"] in ("waiting", "partial")]
            free -= len(dec)
            for r in dec:
                r["held"] += 1
        budget = max(0, B - len(dec))                     # step 3 (R8)
        if policy == 1:                                   # steps 4-5 (R2-R5)
            keyed = [(max(paper_priority(r["cls"], clock - r["arr"], alpha), 1e-12), r) for r in pend]
            vals = sorted(keyed, key=lambda t: -t[0])
            for (pa, ra), (pb, rb) in zip(vals, vals[1:]):
                if ra["cls"] != rb["cls"] and abs(pa - pb) < 1e-11:
                    near_tie = True
            order = [r for _, r in sorted(keyed, key=lambda t: (-t[0], t[1]["arr"], t[1]["id"]))]
        elif policy == 2:
            dl = lambda r: r["arr"] + slo * iso_e2e(r["f"], r["inl"], r["out"], B, c0, cp, cd)
            order = sorted(pend, key=lambda r: (dl(r), r["arr"], r["id"]))
        elif policy == 3:
            order = sorted(pend, key=lambda r: (-(clock - r["arr"]), r["arr"], r["id"]))
        else:
            order = sorted(pend, key=lambda r: (r["arr"], r["id"]))
        left, blocked, tok, inl = budget, False, 0, 0     # step 6 (R6, R7)
        it_no += 1
        for r in order:
            if left == 0:
                break
            if r["state"] == "waiting":
                need = r["rem"] if growth else r["f"]
                if blocked or r.get("pre_it") == it_no:
                    continue
                if need > free and growth and policy == 2:
                    # R34: EDF preempts running requests with a later deadline (deadline, arrival, id),
                    # latest first, until the earlier-deadline request fits -- if they can make it fit
                    ek = lambda x: (dl(x), x["arr"], x["id"])
                    later = sorted((x for x in R if x["state"] in ("partial", "decoding") and ek(x) > ek(r)),
                                   key=ek, reverse=True)
                    if free + sum(x["held"] for x in later) >= need:
                        for v in later:
                            if need <= free:
                                break
                            free += v["held"]
                            v["rem"] = v["held"] - 1 if v["state"] == "decoding" else v["held"]
                            v["held"], v["state"], v["since"], v["pre_it"] = 0, "waiting", clock, it_no
                            v["npre"] += 1
                        dec = [x for x in dec if x["state"] == "decoding"]
                if need > free:
                    blocked = not skip
                    continue
                r["state"] = "partial"
                free -= need
                r["held"] = need
                if r["admit"] is None:
                    r["admit"] = seq
                    seq += 1
                    inl += r["inl"]
                else:                                     # R31: back from preemption
                    r["tpre"] += clock - r["since"]
            chunk = min(r["rem"], left)
            r["rem"] -= chunk
            left -= chunk
            tok += chunk
        assert tok > 0 or dec, "deadlock"
        clock += c0 + cp * tok + cd * len(dec) + inl      # step 8
        for r in dec:                                     # step 9
            r["gen"] += 1
            if r["gen"] == r["out"]:
                r["state"], r["done"] = "finished", clock
                free += r["held"] if growth else r["f"]
        for r in pend:                                    # step 10 (R12; R30 after a re-prefill)
            if r["state"] == "partial" and r["rem"] == 0:
                if r["first"] is None:
                    r["first"] = clock
                r["gen"] += 1
                if r["gen"] == r["out"]:
                    r["state"], r["done"] = "finished", clock
                    free += r["held"] if growth else r["f"]
                else:
                    r["state"] = "decoding"
    return dict(admit_seq=[r["admit"] for r in R], first=[r["first"] for r in R],
                done=[r["done"] for r in R], preempt_count=[r["npre"] for r in R],
                preempted_us=[r["tpre"] for r in R], near_tie=near_tie)
