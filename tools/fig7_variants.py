"""Config #1 (fig7-b200-x10, the bench's headline workload) under live-mode
knob variants, with the bench's own session settings: BE atoms/s and
blocks/s on the device clock, live HBM GB/s, LC p99.

    python tools/fig7_variants.py [reps]"""
import json
import sys

sys.path.insert(0, ".")
from paper_2504_15465_b200 import api, workloads  # noqa: E402


def p99(xs):
    s = sorted(xs)
    return s[max(0, -(-99 * len(s) // 100) - 1)] if s else None


reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
cfg = workloads.fig7_b200(10.0, 2000.0)
base = {"block_revocation": True, "chain_launches": True}
variants = {"bench": ({}, 25.0), "lookahead": ({"atom_lookahead": True}, 25.0),
            "chain_be": ({"chain_best_effort": True}, 25.0),
            "both": ({"atom_lookahead": True, "chain_best_effort": True}, 25.0),
            "lookahead_q15": ({"atom_lookahead": True}, 15.0), "lookahead_q10": ({"atom_lookahead": True}, 10.0),
            "alone": ({}, 25.0), "alone_q10": ({}, 10.0)}
for name, (knobs, q) in variants.items():
    if only and name not in only:
        continue
    scen = workloads.without_apps(cfg, "be") if name.startswith("alone") else cfg
    with api.Session({"scenario": {"config": scen}, "backend": "b200", "b200": {"chunk_cap": 256, "quantum_us": q},
                      "requests": True, "set": base | knobs}) as s:
        s.run()
        s.run()
        rs = [s.run() for _ in range(reps)]
    ms = sum(r["b200"]["kernel_ms"] for r in rs)
    lat = [json.loads(x)["latency_us"] / 1e3 for r in rs for x in r["request_log"].splitlines()
           if json.loads(x)["app"] == "hp" and json.loads(x)["completed"]]
    print(json.dumps({"variant": name, "be_atoms_per_s": sum(r["atoms"]["be"] for r in rs) / (ms * 1e-3),
                      "be_blocks_per_s": sum(r["blocks_per_app"][-1] for r in rs) / (ms * 1e-3),
                      "live_gbs": sum(r["b200"]["stream_bytes"] for r in rs) / (ms * 1e-3) / 1e9,
                      "lc_p99_ms": p99(lat), "util": sum(r["report"]["tpc_utilization"] for r in rs) / reps}),
          flush=True)
