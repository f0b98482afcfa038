"""Live fig7-on-B200 variants: LC p99 / BE throughput / live HBM bandwidth
for the scheduler and dispatcher options (block revocation, preemption
quantum). Usage: python tools/live_variants.py [time_scale] [reps]"""
import json
import sys

sys.path.insert(0, ".")
from oracle.policy import percentile  # noqa: E402  (checker only: nearest-rank)
from paper_2504_15465_b200 import api, workloads  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = workloads.fig7_b200(scale, 2000.0)
alone = workloads.without_apps(cfg, "be")
static = workloads.variant(cfg, stealing=False, atomizer=False)


def lat(r):
    out = []
    for line in r["request_log"].splitlines():
        j = json.loads(line)
        if j["app"] == "hp" and j["completed"]:
            out.append(j["latency_us"])
    return out


variants = [
    ("base", {}, {}),
    ("rev", {"set": {"block_revocation": True}}, {}),
    ("q25", {}, {"quantum_us": 25.0}),
    ("q25_rev", {"set": {"block_revocation": True}}, {"quantum_us": 25.0}),
    ("q10_rev", {"set": {"block_revocation": True}}, {"quantum_us": 10.0}),
    ("alone", {"scenario": {"config": alone}}, {}),
    ("alone_q25", {"scenario": {"config": alone}}, {"quantum_us": 25.0}),
    ("static", {"scenario": {"config": static}}, {}),
]
by_b200 = {}
for name, kw, b in variants:
    key = json.dumps(b, sort_keys=True)
    if key not in by_b200:
        by_b200[key] = api.Session({"scenario": {"config": cfg}, "backend": "b200", "requests": True,
                                    "b200": dict(b, chunk_cap=256)})
        by_b200[key].run()
        by_b200[key].run()
    s = by_b200[key]
    rs = [s.run(**kw) for _ in range(reps)]
    L = sum((lat(r) for r in rs), [])
    ms = sum(r["b200"]["kernel_ms"] for r in rs)
    print(json.dumps({"variant": name, "lc_p50_us": percentile(L, 50), "lc_p99_us": percentile(L, 99),
                      "be_atoms_per_s": sum(r["atoms"]["be"] for r in rs) / (ms * 1e-3),
                      "be_blocks_per_s": sum(r["blocks_per_app"][-1] for r in rs) / (ms * 1e-3),
                      "live_GBps": sum(r["b200"]["stream_bytes"] for r in rs) / (ms * 1e-3) / 1e9,
                      "kernel_ms": ms / reps}), flush=True)
for s in by_b200.values():
    s.close()
