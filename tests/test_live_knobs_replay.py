"""Live-mode scheduler knobs on the replay engine (host logic only, no GPU):
off by default they leave the reference's dispatch log untouched; on, they
change placement decisions the way tpc_scheduler.hpp documents.

* be_coexist: a best-effort thief keeps stealing while an HP tenant has
  work (the reference backs off, scheduler.cpp:245-249);
* hp_steal_busy_be (with block_revocation): an HP thief may take a busy
  best-effort tenant's quota; off, it keeps to idle TPCs.
"""
from __future__ import annotations

import json


def _cfg(knobs=None, horizon_ms=300.0):
    from paper_2504_15465_b200 import workloads

    cfg = workloads.fig7_b200(10.0, horizon_ms * 10.0)
    cfg = workloads.variant(cfg, **(knobs or {}))
    return cfg


def _dispatches(api, cfg, knobs=None):
    r = api.run({"scenario": {"config": cfg}, "backend": "replay", "log": True, "set": knobs or {}})
    out = []
    for line in r["log"].splitlines():
        f = line.split()
        if f and f[0] == "D":
            out.append(f)
    return r, out


def test_knobs_off_keep_the_reference_log(api):
    base, _ = _dispatches(api, _cfg())
    explicit, _ = _dispatches(api, _cfg(), {"be_coexist": False, "hp_pair_reserve": False,
                                              "hp_quota_full": False, "hp_steal_busy_be": True})
    assert base["log"] == explicit["log"]


def _tpcs(runs: str) -> set[int]:
    out = set()
    for part in runs.split(","):
        a, _, b = part.partition("-")
        out.update(range(int(a), int(b or a) + 1))
    return out


def test_be_coexist_steals_while_hp_busy(api):
    """With be_coexist the best-effort tenant dispatches onto TPCs beyond its
    quota while the LC tenant has a request in flight; without it (the
    reference's back-off), never."""
    cfg = _cfg()
    quota_be = set(range(24, 36))  # fig7-b200: LC quota 0-23, BE 24-35

    def stolen_while_hp_busy(knobs):
        r = api.run({"scenario": {"config": cfg}, "backend": "replay", "log": True, "requests": True,
                     "set": knobs})
        busy = [(q["arrival_us"] * 1e3, (q["arrival_us"] + q["latency_us"]) * 1e3)
                for q in map(json.loads, r["request_log"].splitlines()) if q["app"] == "hp" and q["completed"]]
        n = 0
        for line in r["log"].splitlines():
            f = line.split()
            if f[0] != "D" or int(f[3]) != 1:
                continue
            t = int(f[1])
            if any(a < t < b for a, b in busy) and not _tpcs(f[9]) <= quota_be:
                n += 1
        return n

    assert stolen_while_hp_busy({"be_coexist": True}) > 0
    assert stolen_while_hp_busy({}) == 0
