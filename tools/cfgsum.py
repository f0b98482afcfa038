"""Summarise tools/hybrid_variants.py JSON lines for any config."""
import json
import sys

for line in sys.stdin:
    try:
        d = json.loads(line)
    except Exception:
        print(line.strip()[:200])
        continue
    parts = [d["variant"], f"util {d['tpc_utilization']:.3f}"]
    for k, v in d.items():
        if isinstance(v, dict) and ("p99_vs_alone" in v or "throughput_vs_static" in v):
            if v.get("p99_vs_alone") is not None:
                parts.append(f"{k} p99x {v['p99_vs_alone']:.3f} ({v['p99_ms']:.2f}/{v['alone_p99']:.2f} ms, "
                             f"slo {v.get('slo_attainment')})")
            if v.get("throughput_vs_static") is not None:
                parts.append(f"{k} work x {v['throughput_vs_static']:.3f}")
    print(" | ".join(parts))
