"""Per-source-line instruction / stall-sample breakdown of an ncu report (development tool).
usage: python tools/ncu_lines.py report.ncu-rep [units] [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, fname = {}, None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] in ("Line No", "Function Name") or r[0] == "":
        continue
    try:
        agg[(fname, int(r[0]))] = [int(r[7]), int(r[4]), r[1][:90]]
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total inst {tot} ({tot / units:.0f} per unit), samples {ts}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]}:{k[1]:4d} inst {v[0] / tot * 100:5.1f}% samp {v[1] / ts * 100:5.1f}%  {v[2]}")
