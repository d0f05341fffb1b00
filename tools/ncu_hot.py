"""Per-source-line warp instructions, active lanes and stall samples of an ncu report, sorted by
instructions (development tool).  usage: ncu_hot.py report.ncu-rep units [top]"""
import csv, io, subprocess, sys
rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, fname = {}, None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 9 or not r[0].isdigit():
        continue
    try:
        agg[(fname, int(r[0]))] = (int(r[7] or 0), int(r[8] or 0), int(r[4] or 0), r[1][:90])
    except ValueError:
        pass
T = sum(v[0] for v in agg.values()) or 1
S = sum(v[2] for v in agg.values()) or 1
print(f"total warp inst {T} ({T / units:.0f} per unit), stall samples {S}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0][:12]}:{k[1]:4d} {v[0] / T * 100:5.1f}% inst lanes {v[1] / max(v[0], 1):5.1f} samp {v[2] / S * 100:5.1f}%  {v[3]}")
