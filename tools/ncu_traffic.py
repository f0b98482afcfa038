"""Captures DRAM traffic of bench.py's batch-mode saturation launches under
ncu (first k_worker launch of each; --clock-control none) and writes
profiles/ncu_traffic_r02.json entries (bench.ncu_traffic reads them),
keeping the live fig7 entry. Run on the GPU box:
    python tools/ncu_traffic.py [stream gemv gemm conv]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")
METRICS = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"

doc = json.load(open(OUT)) if os.path.exists(OUT) else {}
for name in sys.argv[1:] or ["stream", "gemv", "gemm", "conv"]:
    cmd = ["ncu", "--metrics", METRICS, "--clock-control", "none", "--print-units", "base", "-k",
           "regex:k_worker", "-c", "1", "--csv",
           sys.executable, os.path.join(ROOT, "tools", "sat_once.py"), name]
    p = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=900)
    lines = p.stdout.splitlines()
    info = json.loads(next(l for l in lines if l.startswith("{") and '"name"' in l))
    rows = [r for r in csv.DictReader(io.StringIO("\n".join(l for l in lines if l.startswith('"'))))
            if "k_worker" in r.get("Kernel Name", "")]
    vals = {r["Metric Name"]: float(r["Metric Value"].replace(",", "")) for r in rows}
    doc[name] = {"cmd": " ".join(cmd[-2:]), "config": info["config"],
                 "dram_read": int(vals["dram__bytes_read.sum"]), "dram_write": int(vals["dram__bytes_write.sum"]),
                 "duration_ns": int(vals["gpu__time_duration.sum"]),
                 "algorithmic_bytes": info["algorithmic_bytes"]}
    print(name, doc[name], flush=True)
doc["how_batch"] = ("ncu --metrics " + METRICS + " --clock-control none -k regex:k_worker -c 1: the first "
                    "batch-mode k_worker launch of bench.py's saturation measurement with its exact shapes "
                    "(tools/sat_once.py), 1 x B200")
json.dump(doc, open(OUT, "w"), indent=1)
