"""Group an ncu source page (cuda,sass) by line ranges: warp / thread instructions, active lanes,
stall samples (development tool).  usage: ncu_regions.py report.ncu-rep file.cu start:end:name ..."""
import csv, io, subprocess, sys
rep, fn = sys.argv[1], sys.argv[2]
regs = [(int(a), int(b), n) for a, b, n in (x.split(":", 2) for x in sys.argv[3:])]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, agg = None, {}
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit():
        try:
            agg[(fname, int(r[0]))] = (int(r[7] or 0), int(r[8] or 0), int(r[4] or 0))
        except ValueError:
            pass
T = sum(v[0] for v in agg.values()) or 1
TT = sum(v[1] for v in agg.values()) or 1
S = sum(v[2] for v in agg.values()) or 1
print(f"warp inst {T:.3e}  thread inst {TT:.3e}  avg lanes {TT / T:.2f}")
used = set()
for a, b, n in regs + [(0, 10**9, "rest of " + fn)]:
    sel = [k for k in agg if k[0] == fn and a <= k[1] <= b and k not in used]
    used.update(sel)
    i = sum(agg[k][0] for k in sel); t = sum(agg[k][1] for k in sel); s = sum(agg[k][2] for k in sel)
    print(f"{n:26s} warp {i / T * 100:5.1f}%  thread {t / TT * 100:5.1f}%  lanes {t / max(i, 1):5.2f}  stalls {s / S * 100:5.1f}%")
rest = [k for k in agg if k[0] != fn]
for f in sorted({k[0] for k in rest}):
    sel = [k for k in rest if k[0] == f]
    i = sum(agg[k][0] for k in sel); t = sum(agg[k][1] for k in sel); s = sum(agg[k][2] for k in sel)
    print(f"{f:26s} warp {i / T * 100:5.1f}%  thread {t / TT * 100:5.1f}%  lanes {t / max(i, 1):5.2f}  stalls {s / S * 100:5.1f}%")
