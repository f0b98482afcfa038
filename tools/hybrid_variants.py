"""Config #3 (hybrid decode + training) under scheduler variants: decode p99
vs alone and training throughput vs its static partition per variant.

    python tools/hybrid_variants.py [--horizon-ms 1000] [--reps 3] [--only A,B]"""
import argparse
import json
import sys

sys.path.insert(0, ".")
from paper_2504_15465_b200 import configs  # noqa: E402

RS = {"rightsizer": True, "rightsizer_plateau": True, "dvfs": False}
VARIANTS = {
    "A": ({}, {}),
    "B": (RS, {}),
    "C": (dict(RS, slip_k=1.04), {}),
    "D": (dict(RS, slip_k=1.2), {}),
    "E": ({"atom_lookahead": True}, {}),
    "F": ({"be_coexist": True}, {}),
    "G": ({"atom_lookahead": True, "be_coexist": True}, {}),
    "H": ({"be_coexist": True, "hp_pair_reserve": True}, {}),
    "I": ({"be_coexist": True, "hp_pair_reserve": True, "atom_lookahead": True}, {}),
    "J": ({"be_coexist": True, "hp_pair_reserve": True, "hp_quota_full": True}, {}),
    "L": ({"chain_best_effort": True}, {}),
    "P": ({"hp_steal_busy_be": False}, {}),
    "R": ({"hp_pair_reserve": True, "hp_quota_full": True}, {}),
    "S": ({"hp_pair_reserve": True}, {}),
    "Q": ({"hp_steal_busy_be": False, "atom_lookahead": True}, {}),
    "N": ({"atom_duration_us": 500.0}, {}),
    "O": ({"atom_duration_us": 2000.0}, {}),
    "K": ({"be_coexist": True, "hp_pair_reserve": True, "hp_quota_full": True, "chain_best_effort": True}, {}),
}

ap = argparse.ArgumentParser()
ap.add_argument("--horizon-ms", type=float, default=1000.0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--only", default=",".join(VARIANTS))
ap.add_argument("--config", default="hybrid")
ap.add_argument("--splits", default=None, help="decode GEMV K splits, e.g. 6,8,1,9")
ap.add_argument("--be-batch", type=int, default=None, help="infer4: best-effort training batch")
ap.add_argument("--attention", action="store_true", help="hybrid: decode attention as the tenant body")
args = ap.parse_args()
cfg = None
if args.attention:
    from paper_2504_15465_b200 import workloads  # noqa: E402
    cfg = workloads.hybrid(args.horizon_ms, real_attention=True)
if args.be_batch is not None:
    from paper_2504_15465_b200 import workloads  # noqa: E402
    cfg = workloads.infer4(args.horizon_ms, be_batch=args.be_batch)
if args.splits:
    from paper_2504_15465_b200 import workloads  # noqa: E402
    cfg = workloads.hybrid(args.horizon_ms, decode_splits=tuple(int(x) for x in args.splits.split(",")))
for name in args.only.split(","):
    knobs, b200 = VARIANTS[name]
    r = configs.run(args.config, horizon_ms=args.horizon_ms, reps=args.reps, knobs=knobs, b200=b200, cfg=cfg)
    row = {"variant": name, "knobs": knobs, "b200": b200, "tpc_utilization": r["tpc_utilization"],
           "rightsizer": r.get("rightsizer")}
    for app, a in r["apps"].items():
        row[app] = {k: a.get(k) for k in ("p99_vs_alone", "throughput_vs_static", "iterations_vs_static", "slo_attainment")}
        row[app].update({"p99_ms": a["stacked"].get("p99_ms"), "alone_p99": a["alone"].get("p99_ms"),
                         "per_s": a["stacked"].get("per_s"), "static_per_s": a["static"].get("per_s"),
                         "alone_per_s": a["alone"].get("per_s")})
    print(json.dumps(row), flush=True)
