"""Pins the CPU oracle (oracle/policy.py, oracle/engine.py) and the B200
library's policy functions against the known-answer vectors the UNMODIFIED
reference produced (tests/golden/vectors.jsonl.gz), plus the reference's
own unit-test vectors (proj/tests/test_*.cpp)."""
from __future__ import annotations

import gzip
import json
import os
import random

import pytest

from conftest import GOLDEN
from oracle import policy as P
from oracle.engine import Engine


def vectors():
    with gzip.open(os.path.join(GOLDEN, "vectors.jsonl.gz"), "rt") as f:
        return [json.loads(line) for line in f]


VEC = vectors()


def by_fn(name):
    return [v for v in VEC if v["fn"] == name]


def test_vector_file_covers_every_function():
    fns = {v["fn"] for v in VEC}
    assert fns == {"plan_atoms", "should_atomize", "filter_cap", "fit_scaling", "choose_tpcs",
                   "choose_tpcs_wave", "block_latency", "predictor", "select_frequency"}


# ------------------------------------------------------------- oracle pinning
def test_oracle_plan_atoms():
    for v in by_fn("plan_atoms"):
        assert P.plan_atoms(v["n"], v["pred"], v["atom"], v["min"]) == [tuple(x) for x in v["out"]]


def test_oracle_should_atomize():
    for v in by_fn("should_atomize"):
        assert P.should_atomize(v["pred"], v["n"], v["atom"], v["df"]) == bool(v["out"])


def test_oracle_filter_cap():
    for v in by_fn("filter_cap"):
        assert P.filter_cap(v["n"], v["occ"], v["total"]) == v["out"]


def test_oracle_fit_and_choose():
    for v in by_fn("fit_scaling"):
        m, b, valid = P.fit_scaling(v["l1"], v["lT"], v["T"])
        assert (m, b, int(valid)) == (v["m"], v["b"], v["valid"])  # bit-exact doubles
    for v in by_fn("choose_tpcs"):
        assert P.choose_tpcs(v["m"], v["b"], v["valid"], v["t_alloc"], v["slip"], v["cap"]) == v["out"]
    for v in by_fn("choose_tpcs_wave"):
        assert P.choose_tpcs_wave(v["m"], v["b"], v["valid"], v["t_alloc"], v["slip"], v["blocks"],
                                  v["occ"]) == v["out"]


def test_oracle_latency_model():
    for v in by_fn("block_latency"):
        assert P.block_latency(v["d0"], v["s"], v["f"]) == v["lat"]
        assert P.reference_kernel_latency(v["blocks"], v["d0"], v["s"], v["occ"], v["t"], v["f"]) == v["ref"]


def test_oracle_predictor():
    for v in by_fn("predictor"):
        p = P.Predictor()
        for t, f, b, obs in v["records"]:
            p.record(t, f, b, obs)
        for t, f, b, lat, conf in v["queries"]:
            assert p.predict(t, f, b) == (lat, conf)


def test_oracle_select_frequency():
    for v in by_fn("select_frequency"):
        assert P.select_frequency(v["S"], v["slip"]) == v["out"]


def test_oracle_reference_unit_vectors():
    """Known answers quoted from the reference's own unit tests."""
    # test_atomizer.cpp:10-19, :38-47
    assert P.plan_atoms(10, 3_000_000, 1_000_000, 1) == [(0, 4), (4, 7), (7, 10)]
    assert [h - lo for lo, h in P.plan_atoms(100, 10_000_000, 1_000_000, 48)] == [50, 50]
    sizes = [h - lo for lo, h in P.plan_atoms(64, 10_000_000, 1_000_000, 1)]
    assert sizes == [7] * 4 + [6] * 6
    # test_device.cpp:50-60
    assert P.block_latency(1_000_000, 0.5, 705, 1410) == 1_500_000
    # test_rightsizer.cpp:11-19, :97-112
    m, b, ok = P.fit_scaling(38_000_000, 3_000_000, 36)
    assert ok and abs(m - 36e6) < 1e-3 and abs(b - 2e6) < 1e-3
    fit = P.fit_scaling(12_000_000, 1_000_000, 12)
    assert P.choose_tpcs(*fit, 36, 1.1, 12) == 11
    assert P.choose_tpcs_wave(*fit, 36, 1.1, 48, 4) == 12
    assert P.choose_tpcs_wave(*P.fit_scaling(36_000_000, 1_000_000, 36), 36, 1.1, 2880, 4) == 33
    # test_predictor.cpp:21-43
    p = P.Predictor()
    p.record(8, 1410, 100, 8_000_000)
    assert p.predict(4, 1410, 100) == (16_000_000, 1)
    assert p.predict(8, 705, 100) == (16_000_000, 1)
    # test_metrics.cpp: nearest rank
    assert P.percentile(list(range(1, 1001)), 99) == 990


def test_oracle_engine_reference_cases():
    # Priority refill: HP done at 3 ms, LP at 6 ms (test_device.cpp:101-115).
    e = Engine(1)
    lo = e.register_kernel(4, 1_000_000, 1.0, 1)
    hi = e.register_kernel(2, 1_000_000, 1.0, 1)
    e.submit(lo, 0, 4, [0], 5, False, 0)
    e.submit(hi, 0, 2, [0], 20, False, 1)
    e.run()
    assert {tag: t for _, tag, t in e.completions} == {1: 3_000_000, 0: 6_000_000}
    # Prelude: two waves of (1 ms + 500 ns) (test_device.cpp:159-169).
    e = Engine(1)
    k = e.register_kernel(4, 1_000_000, 1.0, 2)
    e.submit(k, 0, 4, [0], 10, True, 0)
    e.run()
    assert e.completions[-1][2] == 2 * 1_000_500
    # Pause: resumes at 5 ms -> done at 7 ms (test_device.cpp:117-129).
    e = Engine(1)
    k = e.register_kernel(3, 1_000_000, 1.0, 1)
    a = e.submit(k, 0, 3, [0], 10, False, 0)
    e.call(500_000, lambda: e.pause(a, True))
    e.call(5_000_000, lambda: e.pause(a, False))
    e.run()
    assert e.completions[-1][2] == 7_000_000


def test_oracle_engine_matches_closed_form():
    rng = random.Random(11)
    for _ in range(60):
        blocks, d0 = rng.randint(1, 500), rng.randint(1, 1_000_000)
        occ, t = rng.randint(1, 4), rng.randint(1, 54)
        e = Engine(54)
        k = e.register_kernel(blocks, d0, 1.0, occ)
        e.submit(k, 0, blocks, list(range(t)), 10, False, 0)
        e.run()
        assert e.completions[0][2] == P.reference_kernel_latency(blocks, d0, 1.0, occ, t, 1410)


# ------------------------------------------- B200 library vs the same vectors
def test_library_policy_functions_match_reference(api):
    for v in by_fn("plan_atoms"):
        assert api.plan_atoms(v["n"], v["pred"], v["atom"], v["min"]) == [tuple(x) for x in v["out"]]
    for v in by_fn("should_atomize"):
        assert api.should_atomize(v["pred"], v["n"], v["atom"], v["df"]) == bool(v["out"])
    for v in by_fn("filter_cap"):
        assert api.filter_cap(v["n"], v["occ"], v["total"]) == v["out"]
    for v in by_fn("fit_scaling"):
        m, b, valid = api.fit_scaling(v["l1"], v["lT"], v["T"])
        assert (m, b, int(valid)) == (v["m"], v["b"], v["valid"])
    for v in by_fn("choose_tpcs"):
        assert api.choose_tpcs(v["m"], v["b"], v["valid"], v["t_alloc"], v["slip"], v["cap"]) == v["out"]
    for v in by_fn("choose_tpcs_wave"):
        assert api.choose_tpcs_wave(v["m"], v["b"], v["valid"], v["t_alloc"], v["slip"], v["blocks"],
                                    v["occ"]) == v["out"]
    for v in by_fn("block_latency"):
        assert api.block_latency(v["d0"], v["s"], v["f"]) == v["lat"]
        assert api.reference_kernel_latency(v["blocks"], v["d0"], v["s"], v["occ"], v["t"], v["f"]) == v["ref"]
    for v in by_fn("select_frequency"):
        assert api.select_frequency(v["S"], v["slip"]) == v["out"]
    for v in by_fn("predictor"):
        got = api.predictor_replay(v["records"], [q[:3] for q in v["queries"]])
        assert got == [(q[3], q[4]) for q in v["queries"]]


def test_library_rejects_bad_inputs(api):
    with pytest.raises(api.GpuosError):
        api.plan_atoms(0, 1, 1, 1)
    assert api.filter_cap(0, 1, 54) == -2
    with pytest.raises(api.GpuosError):
        api.fit_scaling(1, 1, 1)


def test_rightsize_r_squared_matches_reference_semantics():
    """paper_2504_15465_b200.rightsize.r_squared restates rightsizer.cpp:105-119:
    exact fit -> 1, constant data with a perfect fit -> 1, constant data
    with residual -> -ss_res, and the ordinary 1 - ss_res / ss_tot."""
    from paper_2504_15465_b200.rightsize import r_squared

    m, b = 36e6, 2e6
    pts = [(t, m / t + b) for t in (1, 2, 4, 8, 36)]
    assert r_squared(m, b, pts) == 1.0
    assert r_squared(0.0, 5.0, [(1, 5.0), (2, 5.0)]) == 1.0
    assert r_squared(0.0, 4.0, [(1, 5.0), (2, 5.0)]) == -2.0
    pts = [(1, 10.0), (2, 7.0), (4, 4.0)]
    mean = 7.0
    ss_res = sum((l - (8.0 / t + 2.0)) ** 2 for t, l in pts)
    ss_tot = sum((l - mean) ** 2 for _, l in pts)
    assert abs(r_squared(8.0, 2.0, pts) - (1 - ss_res / ss_tot)) < 1e-12
