"""The B200 measured-curve right-sizer (RightsizerConfig::plateau, off in
replay so the reference's logs stay bit-exact): a third probe at half width
and l(t) = max(m/t + b, floor) through l(1), l(T/2) and the plateau l(T).

Pins: (1) with floor 0 the chooser IS the reference's choose_tpcs_wave on
every known-answer vector the reference produced; (2) an HBM-bound curve
(latency flat from 48 of 74 TPCs) gets the plateau's start instead of 74;
(3) a compute-bound curve keeps the reference's answer; (4) the scheduler
runs the three-probe sequence end to end on the replay backend."""
from __future__ import annotations

import gzip
import json
import os

from conftest import GOLDEN


def vectors(kind):
    with gzip.open(os.path.join(GOLDEN, "vectors.jsonl.gz"), "rt") as f:
        for line in f:
            j = json.loads(line)
            if j.get("fn") == kind:
                yield j


def test_floor_zero_is_the_reference_chooser(api):
    n = 0
    for a in vectors("choose_tpcs_wave"):
        ref = api.choose_tpcs_wave(a["m"], a["b"], a["valid"], a["t_alloc"], a["slip"], a["blocks"], a["occ"])
        got = api.choose_tpcs_wave_floor(a["m"], a["b"], 0.0, a["valid"], a["t_alloc"], a["slip"], a["blocks"],
                                          a["occ"])
        assert got == ref == a["out"], (a, got, ref)
        n += 1
    assert n > 0


def test_hbm_plateau_gets_the_plateau_start(api):
    # STREAM 512 MiB as measured in round 1: 178 us from 48 TPCs on.
    lat = lambda t: int(max(178_000 * 48 / t, 178_000))  # noqa: E731
    m, b, floor, valid = api.fit_scaling_plateau(lat(1), 37, lat(37), lat(74), 74)
    assert valid and floor == lat(74)
    t = api.choose_tpcs_wave_floor(m, b, floor, valid, 74, 1.04, 512, 4)
    assert 46 <= t <= 48, t
    # The reference's two-point fit keeps it at full width.
    m2, b2, v2 = api.fit_scaling(lat(1), lat(74), 74)
    assert api.choose_tpcs_wave(m2, b2, v2, 74, 1.04, 512, 4) == 74


def test_compute_bound_curve_matches_the_two_point_answer(api):
    lat = lambda t: int(4_000_000 / t + 20_000)  # noqa: E731
    m, b, floor, valid = api.fit_scaling_plateau(lat(1), 37, lat(37), lat(74), 74)
    got = api.choose_tpcs_wave_floor(m, b, floor, valid, 74, 1.04, 148, 2)
    m2, b2, v2 = api.fit_scaling(lat(1), lat(74), 74)
    assert got == api.choose_tpcs_wave(m2, b2, v2, 74, 1.04, 148, 2)


def test_no_speedup_falls_back_to_two_point(api):
    m, b, floor, valid = api.fit_scaling_plateau(1000, 37, 2000, 900, 74)
    assert floor == 0.0


def test_scheduler_runs_the_mid_probe_in_replay(api):
    base = {"scenario": {"preset": "inf-train"}, "backend": "replay", "horizon_ms": 3000,
            "set": {"rightsizer": True, "dvfs": False}}
    ref = api.run(base)
    plat = api.run(dict(base, set={"rightsizer": True, "dvfs": False, "rightsizer_plateau": True}))
    for r in (ref, plat):
        assert all(a["completed"] > 0 for a in r["report"]["apps"])
    # (the replay engine's latency model has no plateau: same choices after
    # one extra half-width probe per kernel, so nearly the same throughput)
    done = lambda r: sum(a["completed"] for a in r["report"]["apps"])  # noqa: E731
    assert abs(done(plat) - done(ref)) <= 0.1 * done(ref)


def test_measured_search_converges_to_the_plateau_start(api):
    """Bisection on a smooth HBM-shaped curve (flat from ~48 TPCs): every
    probe is a width the search asks for; the answer is within the slip and
    the bracket below it is not."""
    lat = lambda t: 167_000.0 * max(1.0, 48.0 / t) * (1.0 + 0.06 * max(0.0, 60 - t) / 60)  # noqa: E731
    seen = {74: lat(74), 1: lat(1)}
    probes = 0
    while True:
        ok, probe = api.choose_measured(seen, 1.04)
        if not probe:
            break
        assert 1 < probe < 74 and probe not in seen
        seen[probe] = lat(probe)
        probes += 1
    assert probes <= 8
    assert lat(ok) <= 1.04 * lat(74)
    assert 40 <= ok <= 64, ok
    assert all(lat(t) > 1.04 * lat(74) for t in seen if t < ok)


def test_measured_search_keeps_a_compute_bound_kernel_wide(api):
    lat = lambda t: 4_000_000.0 / t + 20_000  # noqa: E731
    seen = {74: lat(74), 1: lat(1)}
    while True:
        ok, probe = api.choose_measured(seen, 1.04)
        if not probe:
            break
        seen[probe] = lat(probe)
    assert ok >= 70, ok


def test_warm_start_carries_learned_state_across_runs(api):
    """A B200 session with warm_start: the second run's scheduler starts with
    the first run's predictor tables (no cold first kernel confined to its
    quota), keyed by app id, so a run without the BE tenant still finds
    the LC tenant's tables."""
    req = {"scenario": {"preset": "fig7"}, "backend": "replay", "horizon_ms": 300, "requests": True,
           "warm_start": True}
    with api.Session(req) as s:
        cold = s.run()
        warm = s.run()
        lc_only = s.run(drop_apps=["be"])

    def first_latency(r):
        import json as _j
        rows = [_j.loads(x) for x in r["request_log"].splitlines()]
        return min((x for x in rows if x["app"] == "hp"), key=lambda x: x["arrival_us"])["latency_us"]

    assert first_latency(warm) < first_latency(cold)
    assert first_latency(lc_only) <= first_latency(cold)
    # Off: every run starts cold (the reference's single-run semantics).
    with api.Session(dict(req, warm_start=False)) as s:
        a, b = s.run(), s.run()
    assert a["request_log"] == b["request_log"]
