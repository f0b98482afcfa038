"""One of bench.py's batch-mode saturation measurements (stream | gemv |
gemm | conv) with the bench's exact shapes, for an ncu capture of its first
k_worker launch (tools/ncu_traffic.py). Prints the bench's config string."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2504_15465_b200 import api  # noqa: E402

CONFIGS = {}  # name -> config string, recorded through bench.ncu_traffic


def record(name, config):
    CONFIGS[name] = config
    return None


bench.ncu_traffic = record
name = sys.argv[1]
args = argparse.Namespace(workers_per_sm=2, time_scale=10.0)
fn = {"stream": bench.saturation, "gemv": bench.gemv_saturation, "gemm": bench.gemm_saturation,
      "conv": bench.conv_saturation}[name]
r = fn(api, 0, args)
print(json.dumps({"name": name, "config": CONFIGS.get(name), "algorithmic_bytes": r.get("algorithmic_bytes"),
                  "achieved": r["achieved"], "unit": r["unit"]}))
