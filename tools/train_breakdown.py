"""Where a best-effort training iteration's time goes on the live path
(BASELINE config #3's ResNet-50 training tenant, alone, at a given width).

Per kernel (from the per-atom device timeline): device span (first block
start .. last block end), the gap before it (previous kernel's last block
end -> this kernel's first block start: host completion round trip,
scheduling, submit, ingest, wake-up), its width in TPCs and its body.
Prints the totals per body kind and the widest gaps / longest spans.

    python tools/train_breakdown.py [--batch 64] [--quota 37] [--horizon-ms 600]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2504_15465_b200 import api, models  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--quota", type=int, default=74)
    ap.add_argument("--horizon-ms", type=float, default=600.0)
    ap.add_argument("--set", default="{}", help="extra scheduler knobs (JSON)")
    ap.add_argument("--brief", action="store_true", help="one summary line")
    args = ap.parse_args()
    kern = models.resnet50_train(args.batch, ws_base=100_000)
    cfg = {"name": "train-alone", "device": {"gpc_count": 2, "tpcs_per_gpc": 37},
           "policy": "full_system", "horizon_ms": args.horizon_ms, "seed": 3,
           "scheduler": {"rightsizer": False, "dvfs": False, "stealing": args.quota < 74, "atomizer": True,
                         "atom_duration_us": 1000.0, "steal_horizon_us": 0.0},
           "apps": [{"id": "rn50_train", "priority": "be", "quota": args.quota, "arrival": "closed_loop",
                     "kernels": kern}]}
    knobs = {"block_revocation": True} | json.loads(args.set)
    with api.Session({"scenario": {"config": cfg}, "backend": "b200", "device": "b200", "requests": True,
                      "b200": {"chunk_cap": 256}, "set": knobs, "warm_start": True}) as s:
        s.run()
        s.run()
        r = s.run(timeline=True)
    tl = r["b200"]["timeline"]
    n = len(tl["lo"])
    by_kernel: dict[int, dict] = {}
    for i in range(n):
        k = tl["kernel"][i]
        e = by_kernel.setdefault(k, {"first": tl["dev_first"][i], "last": tl["dev_last"][i], "atoms": 0,
                                     "width": 0, "blocks": 0, "submit": tl["submit"][i]})
        e["first"] = min(e["first"], tl["dev_first"][i])
        e["last"] = max(e["last"], tl["dev_last"][i])
        e["submit"] = min(e["submit"], tl["submit"][i])
        e["atoms"] += 1
        e["blocks"] += tl["hi"][i] - tl["lo"][i]
        e["width"] = max(e["width"], bin(tl["mask0"][i]).count("1") + bin(tl["mask1"][i]).count("1"))
    order = sorted(by_kernel, key=lambda k: by_kernel[k]["first"])
    kinds: dict[str, dict] = {}
    rows = []
    for a, b in zip(order, order[1:] + [None]):
        e = by_kernel[a]
        body = kern[a % len(kern)]["body"]["kind"]
        span = e["last"] - e["first"]
        gap = (by_kernel[b]["first"] - e["last"]) if b is not None else 0
        kd = kinds.setdefault(body, {"kernels": 0, "span_ms": 0.0, "gap_after_ms": 0.0})
        kd["kernels"] += 1
        kd["span_ms"] += span / 1e6
        kd["gap_after_ms"] += max(0, gap) / 1e6
        rows.append((span, gap, body, e["width"], e["blocks"], e["atoms"], kern[a % len(kern)]["body"]["p"]))
    wall = (by_kernel[order[-1]]["last"] - by_kernel[order[0]]["first"]) / 1e6
    iters = sum(1 for x in r["request_log"].splitlines() if json.loads(x)["completed"])
    summary = {"batch": args.batch, "quota": args.quota, "kernels": len(order), "iterations": iters,
               "iters_per_s": iters / (wall * 1e-3), "device_span_ms": wall,
               "kinds": {k: {kk: round(vv, 2) for kk, vv in v.items()} for k, v in kinds.items()},
               "span_ms": sum(x[0] for x in rows) / 1e6,
               "gap_ms": sum(max(0, x[1]) for x in rows) / 1e6,
               "gap_p50_us": sorted(x[1] for x in rows)[len(rows) // 2] / 1e3}
    if args.brief:
        print(json.dumps(summary))
        return
    print(json.dumps(summary, indent=1))
    print("longest spans:")
    for x in sorted(rows, key=lambda x: -x[0])[:12]:
        print(f"  {x[0] / 1e3:8.1f} us  {x[2]:10s} w={x[3]:2d} blocks={x[4]:5d} atoms={x[5]} p={x[6]}")


if __name__ == "__main__":
    main()
