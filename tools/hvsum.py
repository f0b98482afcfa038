import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    dd, t = d["llama_decode"], d["rn50_train"]
    print(d["variant"], "util", round(d["tpc_utilization"],3), "decode p99x", round(dd["p99_vs_alone"],3), dd["p99_ms"], dd["alone_p99"], "train work x", round(t["throughput_vs_static"],3), "iters x", round(t.get("iterations_vs_static") or 0,3))
