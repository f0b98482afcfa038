"""Scenario configurations for B200 runs, as scenario JSON (the reference's
own config format, sim.cpp:164-244) so that the identical file drives the
B200 library and the unmodified reference (oracle/_ref/ref_bench).

fig7_b200(): BASELINE.json config #1, "SPEC.md default two-tenant trace (one
LC + one BE kernel stream), TPC scheduler + atomization on". SPEC defines no
literal default trace; the reference's Figure-7 preset (sim.cpp:266-291) is
it. Here it is mapped onto the B200: 74 TPCs (2 x 37), quotas and the BE
width cap scaled by 74/54, and every duration (arrivals, block times, SLO,
atom_duration, default prediction, horizon) divided by `time_scale` so that
a 10 s reference run becomes a 1 s live run with 100 us atoms.
"""
from __future__ import annotations

import math


def fig7_b200(time_scale: float = 10.0, horizon_ms: float = 10_000.0, tpcs: int = 74) -> dict:
    s = float(time_scale)
    q = tpcs / 54.0
    n_bursts = int(math.ceil(horizon_ms / 100.0))
    return {
        "name": f"fig7-b200-x{time_scale:g}",
        "device": {"gpc_count": 2, "tpcs_per_gpc": tpcs // 2},
        "policy": "full_system",
        "horizon_ms": horizon_ms / s,
        "seed": 1,
        "switch_latency_ms": 50.0 / s,
        "scheduler": {"rightsizer": False, "dvfs": False, "stealing": True, "atomizer": True,
                      "atom_duration_us": 1000.0 / s, "default_unknown_us": 10_000.0 / s,
                      "time_slice_window_us": 2000.0 / s, "steal_horizon_us": 0.0},
        "apps": [
            {"id": "hp", "priority": "hp", "quota": int(18 * q), "slo_ms": 80.0 / s,
             "arrival": {"times_ms": [k * 100.0 / s for k in range(n_bursts) for _ in range(5)]},
             "kernels": [{"blocks": 360, "block_us": 500.0 / s, "s": 0.6, "occ": 2}] * 2},
            {"id": "be", "priority": "be", "quota": int(9 * q), "tpc_cap": int(36 * q),
             "arrival": {"times_ms": [(k * 100.0 + 95.0) / s for k in range(n_bursts)
                                      if k * 100.0 + 95.0 < horizon_ms]},
             "kernels": [{"blocks": 2160, "block_us": 2000.0 / s, "s": 0.3, "occ": 4}] * 6},
        ],
    }


def variant(cfg: dict, **sched) -> dict:
    """Copy with scheduler knobs overridden (e.g. stealing=False)."""
    out = dict(cfg)
    out["scheduler"] = dict(cfg["scheduler"], **sched)
    return out


def silence_apps(cfg: dict, *ids: str) -> dict:
    """Copy in which tenants `ids` issue no requests but keep their place
    (and quota): the other tenants' app indices -- the predictor's and
    right-sizer's keys, which warm-started sessions carry from run to run --
    stay those of the stacked run, so an `alone` baseline is the same
    scheduler state minus the competition."""
    out = dict(cfg)
    never = {"times_ms": [1e3 * (cfg["horizon_ms"] + 1e6)]}  # (an arrival past the horizon)
    out["apps"] = [dict(a, arrival=never) if a["id"] in ids else a for a in cfg["apps"]]
    return out


def without_apps(cfg: dict, *ids: str) -> dict:
    out = dict(cfg)
    out["apps"] = [a for a in cfg["apps"] if a["id"] not in ids]
    return out


def tenant_set(rank: int, time_scale: float = 10.0, horizon_ms: float = 2000.0,
               tpcs: int = 74) -> dict:
    """BASELINE config #5: one independent 8-tenant set per GPU (64 tenants
    on 8 GPUs). Two latency-critical tenants (Figure-7-shaped bursts,
    phase-shifted per rank) and six best-effort tenants with mixed kernel
    shapes (long / short / cap-limited / wide), quotas summing to 66 of 74
    TPCs. Deterministic in `rank`."""
    s = float(time_scale)
    off = (rank * 13) % 50

    def times(period_ms, phase_ms, per_burst=1):
        return [(k * period_ms + phase_ms) / s for k in range(int(horizon_ms // period_ms))
                for _ in range(per_burst) if k * period_ms + phase_ms < horizon_ms]

    lc = lambda i, q, phase: {  # noqa: E731
        "id": f"lc{i}", "priority": "hp", "quota": q, "slo_ms": 40.0 / s,
        "arrival": {"times_ms": times(50.0, phase, 2)},
        "kernels": [{"blocks": 288, "block_us": 400.0 / s, "s": 0.6, "occ": 2},
                    {"blocks": 144, "block_us": 300.0 / s, "s": 0.5, "occ": 2}]}
    be_shapes = [
        [{"blocks": 2160, "block_us": 2000.0 / s, "s": 0.3, "occ": 4}] * 3,
        [{"blocks": 540, "block_us": 200.0 / s, "s": 0.4, "occ": 1}] * 10,
        [{"blocks": 48, "block_us": 1000.0 / s, "s": 0.2, "occ": 4}] * 6,
        [{"blocks": 2880, "block_us": 50.0 / s, "s": 0.7, "occ": 4}] * 4,
        [{"blocks": 1080, "block_us": 500.0 / s, "s": 0.5, "occ": 2}] * 4,
        [{"blocks": 720, "block_us": 1000.0 / s, "s": 0.3, "occ": 1}] * 2,
    ]
    apps = [lc(0, 14, off), lc(1, 14, off + 25)]
    for i, kernels in enumerate(be_shapes):
        apps.append({"id": f"be{i}", "priority": "be", "quota": 6 if i < 2 else 7,
                     "arrival": "closed_loop", "kernels": kernels})
    assert sum(a["quota"] for a in apps) <= tpcs
    return {
        "name": f"box8-rank{rank}-x{time_scale:g}",
        "device": {"gpc_count": 2, "tpcs_per_gpc": tpcs // 2},
        "policy": "full_system", "horizon_ms": horizon_ms / s, "seed": 1 + rank,
        "switch_latency_ms": 50.0 / s,
        "scheduler": {"rightsizer": False, "dvfs": False, "atom_duration_us": 1000.0 / s,
                      "default_unknown_us": 10_000.0 / s, "time_slice_window_us": 2000.0 / s},
        "apps": apps,
    }


def infer4(horizon_ms: float = 2000.0, rps: tuple = (150.0, 150.0, 100.0, 100.0),
           slo_ms: tuple = (10.0, 10.0, 25.0, 25.0), tpcs: int = 74, be_batch: int = 256) -> dict:
    """BASELINE config #2, inference stacking: four latency-critical tenants
    on one B200 -- two ResNet-50 at batch 1 and two BERT-base at batch 8
    (random-init kernel traces, models.py) -- with Poisson arrivals, equal
    quotas (18 TPCs each) and TPC stealing (atomizer on, right-sizer off),
    plus a best-effort ResNet-50 training tenant (batch `be_batch`, closed
    loop, 2-TPC quota; 0 drops it) that soaks up every TPC the inference
    tenants leave idle -- the contention the stacking must survive."""
    from . import models

    traces = [models.resnet50_infer(1, ws_base=0), models.resnet50_infer(1, ws_base=10_000),
              models.bert_base_infer(8, ws_base=20_000), models.bert_base_infer(8, ws_base=30_000)]
    names = ["rn50_a", "rn50_b", "bert_a", "bert_b"]
    quota = tpcs // 4
    apps = [{"id": nm, "priority": "hp", "quota": quota, "slo_ms": slo_ms[i],
             "arrival": {"poisson_rps": rps[i], "seed_offset": i}, "kernels": traces[i]}
            for i, nm in enumerate(names)]
    if be_batch:
        apps.append({"id": "train_be", "priority": "be", "quota": tpcs - 4 * quota, "arrival": "closed_loop",
                     "kernels": models.resnet50_train(be_batch, ws_base=40_000)})
    return {
        "name": "infer4-b200", "device": {"gpc_count": 2, "tpcs_per_gpc": tpcs // 2},
        "policy": "full_system", "horizon_ms": horizon_ms, "seed": 2,
        "scheduler": {"rightsizer": False, "dvfs": False, "stealing": True, "atomizer": True,
                      "atom_duration_us": 1000.0, "steal_horizon_us": 0.0},
        "apps": apps,
    }


def hybrid(horizon_ms: float = 2000.0, tokens_per_s: float = 60.0, slo_ms: float = 25.0,
           train_batch: int = 256, tpcs: int = 74, decode_splits: tuple = (3, 4, 1, 4),
           real_attention: bool = False) -> dict:
    """BASELINE config #3, hybrid stacking: Llama-3-8B bf16 decode at batch 1
    (latency-critical, Poisson token requests, one request = one token's 258
    kernels over 15 GB of weights) with ResNet-50 training (best-effort,
    closed loop, forward + backward + SGD, batch 256 -- the per-GPU ImageNet
    batch; at batch 64 most kernels have too few tiles to use more than
    the tenant's quota: 1.26x from 37 to 74 TPCs alone vs 1.52x at 256,
    tools/train_breakdown.py) on one B200; mid-kernel reallocation through
    TPC stealing, atomization and block revocation."""
    from . import models

    return {
        "name": "hybrid-b200", "device": {"gpc_count": 2, "tpcs_per_gpc": tpcs // 2},
        "policy": "full_system", "horizon_ms": horizon_ms, "seed": 3,
        "scheduler": {"rightsizer": False, "dvfs": False, "stealing": True, "atomizer": True,
                      "atom_duration_us": 1000.0, "steal_horizon_us": 0.0},
        "apps": [
            {"id": "llama_decode", "priority": "hp", "quota": tpcs // 2, "slo_ms": slo_ms,
             "arrival": {"poisson_rps": tokens_per_s, "seed_offset": 0},
             "kernels": models.llama3_8b_decode(1024, ws_base=0, splits=decode_splits,
                                                attention=real_attention)},
            {"id": "rn50_train", "priority": "be", "quota": tpcs - tpcs // 2,
             "arrival": "closed_loop", "kernels": models.resnet50_train(train_batch, ws_base=100_000)},
        ],
    }
