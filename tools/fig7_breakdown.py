"""Where the headline run's HBM time goes (BASELINE config #1, live).

Runs the bench's stacked fig7-b200 scenario once with the per-atom device
timeline and decomposes the dispatcher kernel's time T:

  * achieved HBM rate = algorithmic STREAM bytes / T (the bench's roofline);
  * the workload's own ceiling: each worker streams at the calibrated
    per-worker rate (B200Options::stream_words_per_us) while it runs a
    block, and the BE tenant is capped at tpc_cap TPCs by the scenario
    (scheduler filter_cap, rightsizer.cpp:21-26), so at most
    (BE TPCs + LC TPCs in use) x workers x rate can stream at any time;
  * TPC-time: running >= 1 block (device sampler, reference definition),
    held by an atom but idle (dispatch / claim / tail of a wave), and not
    held by any atom (scheduler: caps, quotas, host round trips);
  * BE atom boundaries: gap between one BE atom's last block and the next
    BE atom's first block (host poll -> scheduler -> ring -> ingest).

    python tools/fig7_breakdown.py [--horizon-ms 2000] [--out profiles/x.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2504_15465_b200 import api, workloads  # noqa: E402


def union_len(iv):
    tot, cur_s, cur_e = 0, None, None
    for s, e in sorted(iv):
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--horizon-ms", type=float, default=2000.0)
    ap.add_argument("--time-scale", type=float, default=10.0)
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-lookahead", action="store_true")
    ap.add_argument("--quantum-us", type=float, default=None, help="default: 250 / time-scale (bench)")
    args = ap.parse_args()
    cfg = workloads.fig7_b200(args.time_scale, args.horizon_ms)
    q = 250.0 / args.time_scale if args.quantum_us is None else args.quantum_us
    b200 = {"device": 0, "workers_per_sm": 2, "chunk_cap": 256, "quantum_us": q}
    sess = api.Session({"scenario": {"config": cfg}, "backend": "b200", "b200": b200,
                        "requests": True, "set": {"block_revocation": True, "chain_launches": True,
                                "atom_lookahead": not args.no_lookahead}})
    prev = None
    for _ in range(args.runs - 1):
        prev = sess.run()
    r = sess.run(timeline=True)
    b = r["b200"]
    wbusy = b["worker_busy_ns_total"] - (prev["b200"]["worker_busy_ns_total"] if prev else 0)
    tbusy = b["tpc_busy_ns_total"] - (prev["b200"]["tpc_busy_ns_total"] if prev else 0)
    tl = b["timeline"]
    T_ns = b["kernel_ms"] * 1e6
    n = len(tl["lo"])
    app_ids = [a["app_id"] for a in r["report"]["apps"]]
    hp = {i for i, a in enumerate(r["report"]["apps"]) if a["high_priority"]}
    words = tl["kernel_words"]
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    rate_worker = 2750.0 * 8 * 1e6 / 1e9  # GB/s per streaming worker (calibration)
    tpcs = b["logical_tpcs"]
    wpt = b["workers_per_tpc"]

    def popc(i):
        return bin(tl["mask0"][i]).count("1") + bin(tl["mask1"][i]).count("1")

    bytes_app = {}
    held = {}
    active = {}
    for i in range(n):
        app = tl["tag"][i]
        k = tl["kernel"][i]
        by = 8.0 * words[k] * (tl["hi"][i] - tl["lo"][i])
        bytes_app[app] = bytes_app.get(app, 0.0) + by
        d = max(0, tl["dev_last"][i] - tl["dev_first"][i])
        held[app] = held.get(app, 0.0) + popc(i) * max(0, tl["complete"][i] - tl["submit"][i])
        active.setdefault(app, []).append((tl["dev_first"][i], tl["dev_last"][i]))
    t0 = min(tl["dev_first"])
    t1 = max(tl["dev_last"])
    span = t1 - t0
    be = [i for i in range(n) if tl["tag"][i] not in hp]
    be.sort(key=lambda i: tl["dev_first"][i])
    gaps = []
    for a, c in zip(be, be[1:]):
        gaps.append(tl["dev_first"][c] - tl["dev_last"][a])
    pos_gaps = [g for g in gaps if g > 0]
    be_tpcs = [popc(i) for i in be]
    # Held TPC-time by BE / LC atoms (submit -> completion on the host clock)
    total_bytes = sum(bytes_app.values())
    out = {
        "workload": cfg["name"],
        "kernel_ms": b["kernel_ms"],
        "device_span_ms": span / 1e6,
        "atoms": n,
        "achieved_gbs": total_bytes / T_ns,
        "roofline_frac": total_bytes / T_ns / pk,
        "per_app_gbs": {app_ids[a]: v / T_ns for a, v in bytes_app.items()},
        "quantum_us": q,
        "atom_lookahead": not args.no_lookahead,
        "tpc_busy_frac_sampled": tbusy / (tpcs * T_ns),
        "avg_running_workers": wbusy / T_ns,
        "gbs_per_running_worker": total_bytes / wbusy if wbusy else None,
        "be_device_held_tpc_frac": sum(popc(i) * max(0, tl["dev_last"][i] - tl["dev_first"][i]) for i in be)
        / (tpcs * T_ns),
        "be_blocks_per_atom_mean": sum(tl["hi"][i] - tl["lo"][i] for i in be) / len(be),
        "lc_p99_ms": sorted(json.loads(l)["latency_us"] for l in r["request_log"].splitlines()
                            if json.loads(l)["app"] in [app_ids[h] for h in hp]
                            and json.loads(l)["completed"])[-1] / 1e3 if r.get("request_log") else None,
        "held_tpc_frac": {app_ids[a]: v / (tpcs * T_ns) for a, v in held.items()},
        "active_frac": {app_ids[a]: union_len(v) / T_ns for a, v in active.items()},
        "be_tpcs_per_atom": {"min": min(be_tpcs), "max": max(be_tpcs),
                             "mean": sum(be_tpcs) / len(be_tpcs)},
        "be_tpc_cap": [a.get("tpc_cap") for a in cfg["apps"] if a["priority"] == "be"][0],
        "worker_rate_gbs": rate_worker,
        "ceiling_be_cap_gbs": [a.get("tpc_cap") for a in cfg["apps"] if a["priority"] == "be"][0]
        * wpt * rate_worker,
        "be_boundary_gaps_us": {"count": len(pos_gaps),
                                "p50": sorted(pos_gaps)[len(pos_gaps) // 2] / 1e3 if pos_gaps else 0,
                                "sum_ms": sum(pos_gaps) / 1e6,
                                "frac_of_T": sum(pos_gaps) / T_ns},
        "ingest_to_first_block_us_p50": sorted(
            tl["dev_first"][i] - tl["dev_ingest"][i] for i in range(n))[n // 2] / 1e3,
        "submit_to_first_block_us_p50": sorted(
            tl["dev_first"][i] - tl["submit"][i] for i in range(n))[n // 2] / 1e3,
        "backpressure_waits": b.get("backpressure_waits"),
    }
    print(json.dumps(out, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
