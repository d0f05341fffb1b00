"""Write profiles/fused_issue.json and profiles/fused_dram_bytes.json (the bench's k_fused roofline
`issue` and `traffic` inputs) from the CSV of
  ncu --metrics smsp__inst_executed.sum,smsp__thread_inst_executed.sum,gpu__time_duration.sum,
      dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fused -c 1 --csv
      python tools/run_fused_once.py 65536
(development tool; usage: fused_counters.py launches.csv [tag])."""
import csv, io, json, os, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path, tag = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
text = open(path).read()
text = text[text.index('"ID"'):]
vals, units = {}, {}
for r in csv.DictReader(io.StringIO(text)):
    if "k_fused" in r.get("Kernel Name", ""):
        vals[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        units[r["Metric Name"]] = r["Metric Unit"]
requests = 65536 * 10000
inst, tinst = vals["smsp__inst_executed.sum"], vals["smsp__thread_inst_executed.sum"]
to_ms = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}[units["gpu__time_duration.sum"]]
src = ("ncu --metrics smsp__inst_executed.sum,smsp__thread_inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,"
       "dram__bytes_write.sum --clock-control none -k regex:k_fused -c 1 python tools/run_fused_once.py 65536 "
       f"(the bench's C4 workload{', ' + tag if tag else ''}); raw: profiles/{os.path.basename(path)}")
issue = {"inst_executed": int(inst), "thread_inst_executed": int(tinst), "thread_inst_per_inst": tinst / inst,
         "sm_clock_hz": 1965e6, "ncu_duration_ms": vals["gpu__time_duration.sum"] * to_ms,
         "source": src}
rd, wr = vals["dram__bytes_read.sum"], vals["dram__bytes_write.sum"]
dram = {"kernel": "k_fused", "workload": "C4 bench workload, 65,536 replicas x 10,000 requests (tools/run_fused_once.py)",
        "dram_bytes_read": int(rd), "dram_bytes_write": int(wr), "dram_bytes_per_request": (rd + wr) / requests,
        "requests": requests, "algorithmic_bytes_per_request": 55, "traffic_over_algorithmic": (rd + wr) / requests / 55,
        "source": "same ncu pass as profiles/fused_issue.json"}
json.dump(issue, open(os.path.join(ROOT, "profiles", "fused_issue.json"), "w"), indent=1)
json.dump(dram, open(os.path.join(ROOT, "profiles", "fused_dram_bytes.json"), "w"), indent=1)
print(json.dumps(issue), json.dumps(dram), sep="\n")
