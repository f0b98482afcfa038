"""Where config #3's decode tail comes from: Llama-3-8B decode stacked with
ResNet-50 training vs decode alone, per kernel kind, from the per-atom
device timeline.

For each decode kernel: device span (first block start .. last block end),
gap before it (previous decode kernel's last end -> this first start), and,
stacked, how many best-effort atoms overlapped it on a shared TPC. Per
token: latency split into spans and gaps.

    python tools/hybrid_breakdown.py [--horizon-ms 1000] [--set '{...}']
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2504_15465_b200 import api, models, workloads  # noqa: E402


def pct(xs, p):
    s = sorted(xs)
    return s[min(len(s) - 1, int(p / 100.0 * len(s)))] if s else 0.0


def kernels_of(tl, app):
    n = len(tl["lo"])
    ks: dict[int, dict] = {}
    for i in range(n):
        if tl["tag"][i] != app:
            continue
        k = tl["kernel"][i]
        e = ks.setdefault(k, {"first": tl["dev_first"][i], "last": tl["dev_last"][i],
                              "armed": tl["dev_armed"][i], "mask": 0, "atoms": 0})
        e["first"] = min(e["first"], tl["dev_first"][i])
        e["last"] = max(e["last"], tl["dev_last"][i])
        e["armed"] = min(e["armed"], tl["dev_armed"][i])
        e["mask"] |= tl["mask0"][i] | (tl["mask1"][i] << 64)
        e["atoms"] += 1
    return ks


def analyse(r, trace, decode_app=0, be_app=1, label=""):
    tl = r["b200"]["timeline"]
    ks = kernels_of(tl, decode_app)
    ids = sorted(ks)
    per = len(trace)
    # BE atom intervals for overlap counting
    be = [(tl["dev_first"][i], tl["dev_last"][i], tl["mask0"][i] | (tl["mask1"][i] << 64))
          for i in range(len(tl["lo"])) if tl["tag"][i] == be_app]
    kinds: dict[str, dict] = {}
    tokens = []
    for t0 in range(0, len(ids) - per + 1, per):
        tok = ids[t0:t0 + per]
        if any(ks[k]["last"] <= 0 for k in tok):
            continue
        span_sum = gap_sum = 0.0
        prev_last = None
        for j, k in enumerate(tok):
            e = ks[k]
            kind = trace[j]["body"]["kind"] + " " + str(tuple(trace[j]["body"]["p"]))
            span = (e["last"] - e["first"]) / 1e3
            gap = (e["first"] - prev_last) / 1e3 if prev_last is not None else 0.0
            prev_last = e["last"]
            ov = sum(1 for (f, l, m) in be if f < e["last"] and l > e["first"] and (m & e["mask"]))
            d = kinds.setdefault(kind, {"n": 0, "span": [], "gap": [], "overlap_be": 0,
                                         "width": bin(e["mask"]).count("1")})
            d["n"] += 1
            d["span"].append(span)
            d["gap"].append(gap)
            d["overlap_be"] += ov
            span_sum += span
            gap_sum += max(0.0, gap)
        tokens.append(((ks[tok[-1]]["last"] - ks[tok[0]]["first"]) / 1e3, span_sum, gap_sum))
    out = {"label": label, "tokens": len(tokens),
           "token_us_p50": pct([t[0] for t in tokens], 50), "token_us_p99": pct([t[0] for t in tokens], 99),
           "span_us_mean": sum(t[1] for t in tokens) / max(1, len(tokens)),
           "gap_us_mean": sum(t[2] for t in tokens) / max(1, len(tokens)), "kinds": {}}
    for kind, d in kinds.items():
        out["kinds"][kind] = {"n": d["n"], "width": d["width"],
                              "span_p50": round(pct(d["span"], 50), 2), "span_p90": round(pct(d["span"], 90), 2),
                              "span_mean": round(sum(d["span"]) / d["n"], 2),
                              "gap_p50": round(pct(d["gap"], 50), 2), "gap_mean": round(sum(d["gap"]) / d["n"], 2),
                              "be_overlaps_per_kernel": round(d["overlap_be"] / d["n"], 2)}
    lat = [json.loads(x)["latency_us"] / 1e3 for x in r["request_log"].splitlines()
           if json.loads(x)["completed"] and json.loads(x)["app"] == "llama_decode"]
    out["req_p50_ms"] = pct(lat, 50)
    out["req_p99_ms"] = pct(lat, 99)
    return out


def be_rate(r, be_trace, decode_app=0, be_app=1):
    """Best-effort work rate (sum of calibrated block_us per device second)
    inside and outside the decode tenant's busy windows: each BE atom's work
    is spread evenly over its device span."""
    tl = r["b200"]["timeline"]
    n = len(tl["lo"])
    ks = kernels_of(tl, decode_app)
    win = sorted((e["first"], e["last"]) for e in ks.values() if e["last"] > 0)
    merged = []
    for f, l in win:
        if merged and f <= merged[-1][1] + 20_000:  # join windows closer than 20 us
            merged[-1][1] = max(merged[-1][1], l)
        else:
            merged.append([f, l])
    be_ids = sorted({tl["kernel"][i] for i in range(n) if tl["tag"][i] == be_app})
    pos = {k: j % len(be_trace) for j, k in enumerate(be_ids)}
    t0 = min(tl["dev_first"][i] for i in range(n) if tl["dev_first"][i] > 0)
    t1 = max(tl["dev_last"][i] for i in range(n))
    busy = sum(l - f for f, l in merged)
    w_in = w_out = 0.0
    for i in range(n):
        if tl["tag"][i] != be_app or tl["dev_last"][i] <= 0:
            continue
        k = be_trace[pos[tl["kernel"][i]]]
        work = (tl["hi"][i] - tl["lo"][i]) * k["block_us"]
        f, l = tl["dev_first"][i], tl["dev_last"][i]
        span = max(1, l - f)
        ov = sum(max(0, min(l, b) - max(f, a)) for a, b in merged)
        w_in += work * ov / span
        w_out += work * (span - ov) / span
    return {"decode_busy_frac": busy / (t1 - t0), "be_work_us_per_ms_in_decode": w_in / max(1, busy) * 1e6,
            "be_work_us_per_ms_outside": w_out / max(1, (t1 - t0) - busy) * 1e6}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--horizon-ms", type=float, default=1000.0)
    ap.add_argument("--set", default="{}", help="extra scheduler knobs (JSON)")
    ap.add_argument("--b200", default="{}", help="extra B200Options (JSON)")
    ap.add_argument("--splits", default="3,4,1,4", help="decode GEMV K splits (QKV, O, gate-up, down)")
    ap.add_argument("--train-alone", action="store_true")
    ap.add_argument("--attention", action="store_true", help="decode attention as the tenant body")
    args = ap.parse_args()
    splits = tuple(int(x) for x in args.splits.split(","))
    cfg = workloads.hybrid(args.horizon_ms, decode_splits=splits, real_attention=args.attention)
    trace = models.llama3_8b_decode(1024, ws_base=0, splits=splits, attention=args.attention)
    knobs = {"block_revocation": True, "chain_launches": True} | json.loads(args.set)
    req = {"scenario": {"config": cfg}, "backend": "b200", "device": "b200", "requests": True,
           "b200": {"chunk_cap": 256} | json.loads(args.b200), "set": knobs, "warm_start": True}
    with api.Session(req) as s:
        s.run()
        s.run()
        st = s.run(timeline=True)
        solo = workloads.silence_apps(cfg, "rn50_train")
        s.run(scenario={"config": solo})
        al = s.run(scenario={"config": solo}, timeline=True)
        if args.train_alone:
            tcfg = workloads.silence_apps(cfg, "llama_decode")
            ta = s.run(scenario={"config": tcfg}, timeline=True)
    a = analyse(al, trace, label="alone")
    b = analyse(st, trace, label="stacked")
    for x in (a, b):
        print(json.dumps({k: v for k, v in x.items() if k != "kinds"}))
    be_trace = models.resnet50_train(256, ws_base=100_000)
    print(json.dumps({"be_rate_stacked": be_rate(st, be_trace)}))
    if args.train_alone:
        print(json.dumps({"be_rate_alone": be_rate(ta, be_trace, decode_app=-1, be_app=1)}))
    print(f"{'kind':40s} {'w':>3s} | {'alone span50':>12s} {'span_mean':>9s} {'gap_mean':>8s} | "
          f"{'stack span50':>12s} {'span_mean':>9s} {'gap_mean':>8s} {'be_ov':>6s}")
    for kind in a["kinds"]:
        x, y = a["kinds"][kind], b["kinds"].get(kind, {})
        print(f"{kind:40s} {x['width']:3d} | {x['span_p50']:12.2f} {x['span_mean']:9.2f} {x['gap_mean']:8.2f} | "
              f"{y.get('span_p50', 0):12.2f} {y.get('span_mean', 0):9.2f} {y.get('gap_mean', 0):8.2f} "
              f"{y.get('be_overlaps_per_kernel', 0):6.2f}")


if __name__ == "__main__":
    main()
