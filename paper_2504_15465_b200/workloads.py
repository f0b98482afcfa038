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
