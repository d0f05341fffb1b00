"""Summarise an ncu report (--set full) or a launch list (--metrics gpu__time_duration.sum --csv)
into a small JSON + markdown file under profiles/ (run here, on the CPU box, with `ncu -i`).

usage: python tools/ncu_summary.py report.ncu-rep out_prefix [--alg-bytes N] [--units N]
       python tools/ncu_summary.py --launches launches.csv out_prefix
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

RAW = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__warps_eligible.avg.per_cycle_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "lts__t_sector_hit_rate.pct",
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        res.append({"kernel": d.get("Kernel Name", "")[:80],
                    **{k: (d.get(k), u.get(k)) for k in RAW if k in d}})
    return res


def stall_top(rep, n=8):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    d = dict(zip(hdr, rows[2]))
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", "") or 0)
          for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(st.values()) or 1
    return sorted(((k, v / tot) for k, v in st.items()), key=lambda x: -x[1])[:n]


def to_float(x):
    try:
        return float(str(x).replace(",", ""))
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("out")
    ap.add_argument("--launches", action="store_true")
    ap.add_argument("--alg-bytes", type=float, default=None, help="algorithmic bytes per launch")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    if a.launches:
        rows = list(csv.reader(open(a.src)))
        for i, r in enumerate(rows):
            if "Kernel Name" in r:
                hdr, start = r, i + 1
                break
        ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
        agg = defaultdict(lambda: [0, 0.0])
        for r in rows[start:]:
            if len(r) > vi and r[mi] == "gpu__time_duration.sum":
                name = r[ki].split("(")[0].replace("void ", "")
                agg[name][0] += 1
                agg[name][1] += float(r[vi].replace(",", ""))
        tot = sum(v[1] for v in agg.values())
        res = [{"kernel": k, "launches": v[0], "total_ns": v[1], "share": v[1] / tot}
               for k, v in sorted(agg.items(), key=lambda x: -x[1][1])]
        json.dump({"source": a.src, "note": a.note, "kernels": res}, open(a.out + ".json", "w"), indent=1)
        with open(a.out + ".md", "w") as f:
            f.write(f"# Launch list: {a.note}\n\n| kernel | launches | total ms | share |\n|---|---|---|---|\n")
            for r in res:
                f.write(f"| {r['kernel']} | {r['launches']} | {r['total_ns'] / 1e6:.3f} | {r['share']:.2%} |\n")
        return
    ms = raw_metrics(a.src)
    stalls = stall_top(a.src)
    m = ms[0]
    dur = to_float(m["gpu__time_duration.sum"][0])
    dur_unit = m["gpu__time_duration.sum"][1]
    nob = ("0", "byte")          # a capture without the memory sections has no DRAM byte counts
    rd, rdu = to_float(m.get("dram__bytes_read.sum", nob)[0]), m.get("dram__bytes_read.sum", nob)[1]
    wr, wru = to_float(m.get("dram__bytes_write.sum", nob)[0]), m.get("dram__bytes_write.sum", nob)[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tscale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
    traffic = rd * scale.get(rdu, 1) + wr * scale.get(wru, 1)
    secs = dur * tscale.get(dur_unit, 1e-9)
    summary = {"source": a.src, "note": a.note, "kernel": m["kernel"], "duration_s": secs,
               "dram_bytes": traffic, "dram_GBps": traffic / secs / 1e9,
               "metrics": {k: v for k, v in m.items() if k != "kernel"}, "stall_top": stalls}
    if a.alg_bytes:
        summary["alg_bytes"] = a.alg_bytes
        summary["traffic_over_alg"] = traffic / a.alg_bytes
    json.dump(summary, open(a.out + ".json", "w"), indent=1)
    with open(a.out + ".md", "w") as f:
        f.write(f"# ncu --set full: {m['kernel']}\n\n{a.note}\n\n")
        f.write(f"- duration: {secs * 1e3:.3f} ms (cold-cache, serialised replay)\n")
        if traffic:
            f.write(f"- DRAM traffic: {traffic / 1e6:.1f} MB ({traffic / secs / 1e9:.1f} GB/s)\n")
        if a.alg_bytes and traffic:
            f.write(f"- algorithmic bytes: {a.alg_bytes / 1e6:.1f} MB (traffic / algorithmic = {traffic / a.alg_bytes:.2f})\n")
        f.write("\n| metric | value | unit |\n|---|---|---|\n")
        for k, (v, u) in summary["metrics"].items():
            f.write(f"| {k} | {v} | {u} |\n")
        f.write("\nTop stall reasons (share of PC samples):\n\n")
        for k, v in stalls:
            f.write(f"- {k}: {v:.1%}\n")


if __name__ == "__main__":
    main()
