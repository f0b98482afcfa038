"""The gpuos:: scheduler driving the B200 through the C ABI.

* Mirror backend: the replay clock drives every decision (so the
  dispatch/completion log must equal the reference's golden log byte for
  byte) while every atom is also executed on the B200 on exactly the TPC
  set the scheduler chose; then every block is checked: executed once, on
  an SM of its atom's TPC set, body output equal to the CPU oracle.
* Live backend: the persistent dispatcher executes a time-scaled stacked
  scenario in real time with per-block verification.
"""
from __future__ import annotations

import gzip
import json
import os

import pytest

from conftest import GOLDEN
from oracle.policy import percentile

pytestmark = pytest.mark.gpu
CASES = json.load(open(os.path.join(GOLDEN, "cases.json")))["cases"]

MIRROR = {
    "fig7_2s": {"scenario": {"preset": "fig7"}, "horizon_ms": 2000},
    "inf-inf_2s": {"scenario": {"preset": "inf-inf"}, "horizon_ms": 2000},
    "inf-train_2s": {"scenario": {"preset": "inf-train"}, "horizon_ms": 2000},
    "inf-inf_mps_like_1s": {"scenario": {"preset": "inf-inf"}, "horizon_ms": 1000, "policy": "mps_like"},
    "inf-inf_time_slice_1s": {"scenario": {"preset": "inf-inf"}, "horizon_ms": 1000, "policy": "time_slice"},
    "inf-inf_mig_like_1s": {"scenario": {"preset": "inf-inf"}, "horizon_ms": 1000, "policy": "mig_like"},
    "inf-inf_priority_only_1s": {"scenario": {"preset": "inf-inf"}, "horizon_ms": 1000,
                                 "policy": "priority_only"},
    "inf-inf_reef_like_1s": {"scenario": {"preset": "inf-inf"}, "horizon_ms": 1000, "policy": "reef_like"},
    "cli_smoke": {"scenario": {"config_path": os.path.join(GOLDEN, "scenarios", "cli_smoke.json")}},
    "random_7": {"scenario": {"config_path": os.path.join(GOLDEN, "scenarios", "random_7.json")}},
    "random_3": {"scenario": {"config_path": os.path.join(GOLDEN, "scenarios", "random_3.json")}},
    # B200-form BASELINE configs: #1 and one rank of #5 (STREAM bodies), #2
    # and #3 on model traces (tensor-core bodies, values checked in float64).
    "fig7_b200_x10": {"scenario": {"config_path": os.path.join(GOLDEN, "scenarios", "fig7_b200_x10.json")}},
    "box8_rank0": {"scenario": {"config_path": os.path.join(GOLDEN, "scenarios", "box8_rank0.json")}},
    "infer4_300ms": {"scenario": {"config_path": os.path.join(GOLDEN, "scenarios", "infer4_300ms.json")}},
    "hybrid_300ms": {"scenario": {"config_path": os.path.join(GOLDEN, "scenarios", "hybrid_300ms.json")}},
}
TENSOR_CASES = {"infer4_300ms", "hybrid_300ms"}


@pytest.mark.parametrize("name", sorted(MIRROR))
def test_mirror_executes_reference_schedule_on_b200(api, cuda_device, name):
    req = dict(MIRROR[name], backend="mirror", log=True,
               b200={"min_words": 256, "words_per_us": 0.0, "chunk_cap": 64})
    r = api.run(req)
    ref = gzip.open(os.path.join(GOLDEN, "logs", name + ".log.gz")).read().decode()
    assert r["log"].splitlines() == [line for line in ref.splitlines() if line[:1] in "DC"]
    v = r["verify"]
    assert v["ok"], v
    assert v["missing"] == v["duplicated"] == v["misplaced"] == v["bad_words"] == 0
    assert r["gpu_atoms"] == r["atoms"]["hp"] + r["atoms"]["be"]
    if name in TENSOR_CASES:
        assert v["tensor_kernels"] > 0 and v["tensor_checked"] > 0 and v["tensor_bad"] == 0, v
    else:
        assert v["checked_words"] > 0


def live_request(**kw):
    req = {"scenario": {"preset": "fig7"}, "backend": "b200", "device": "b200",
           "quota_scale": 74 / 54, "time_scale": 10.0, "horizon_ms": 1000,
           "b200": {"chunk_cap": 64}, "requests": True}
    req.update(kw)
    return req


def hp_latencies(r):
    lat = []
    for line in r["request_log"].splitlines():
        j = json.loads(line)
        if j["app"] == "hp" and j["completed"]:
            lat.append(j["latency_us"])
    return lat


def test_live_fig7_verified(api, cuda_device):
    with api.Session(live_request(verify=True, timeline=True,
                                  b200={"chunk_cap": 64, "trace": True})) as s:
        s.run()  # warm: creates workspaces
        r = s.run()
    v = r["verify"]
    assert v["ok"], v
    hp, be = r["report"]["apps"]
    assert hp["completed"] == hp["offered"] > 0
    assert be["completed"] > 0
    # Every atom ran only on TPCs of its set and touched at least one.
    tl = r["b200"]["timeline"]
    for m0, m1, t0, t1 in zip(tl["mask0"], tl["mask1"], tl["touched0"], tl["touched1"]):
        assert (t0 & ~m0) == 0 and (t1 & ~m1) == 0 and (t0 | t1) != 0
    # HP requests meet their (scaled) 8 ms SLO.
    assert percentile(hp_latencies(r), 99) <= 8000


def test_live_mechanisms_lc_tail_and_be_throughput(api, cuda_device):
    """Block-granular revocation + 25 us preemption quanta: the LC tenant's
    p99 stays near its alone p99 while BE runs far faster than a static
    partition (the north-star targets, 1.2x and 1.3x, asserted as such)."""
    import sys

    sys.path.insert(0, os.path.dirname(GOLDEN))
    from paper_2504_15465_b200 import workloads

    cfg = workloads.fig7_b200(10.0, 2000.0)
    req = {"scenario": {"config": cfg}, "backend": "b200", "requests": True,
           "b200": {"chunk_cap": 256, "quantum_us": 25.0},
           "set": {"block_revocation": True, "chain_launches": True}}

    def measure():
        with api.Session(req) as s:
            s.run()
            s.run()
            # 4 runs (400 LC requests): p99 is the 4th-worst request, so one
            # burst caught by a host-side stall does not decide the test.
            live = [s.run() for _ in range(4)]
            alone = [s.run(scenario={"config": workloads.without_apps(cfg, "be")}) for _ in range(4)]
            static = [s.run(scenario={"config": workloads.variant(cfg, stealing=False, atomizer=False)})
                      for _ in range(2)]
        p_live = percentile(sum((hp_latencies(r) for r in live), []), 99)
        p_alone = percentile(sum((hp_latencies(r) for r in alone), []), 99)
        return live, static, p_live, p_alone

    live, static, p_live, p_alone = measure()
    if p_live > 1.2 * p_alone:  # one re-measurement: the host loop shares the CPU with the test
        live, static, p_live, p_alone = measure()
    assert p_live <= 1.2 * p_alone, (p_live, p_alone)
    be = sum(r["blocks_per_app"][1] for r in live) / sum(r["b200"]["kernel_ms"] for r in live)
    be_static = sum(r["blocks_per_app"][1] for r in static) / sum(r["b200"]["kernel_ms"] for r in static)
    assert be >= 1.3 * be_static, (be, be_static)
    for r in live:
        hp = r["report"]["apps"][0]
        assert hp["completed"] == hp["offered"]


def test_baseline_policies_run_live(api, cuda_device):
    """Every reference policy (scheduler.cpp:111-121, 199-226, 494-521) drives
    the live dispatcher: all LC requests complete; full_system has the lowest
    LC tail and mps_like the highest (the paper's ordering)."""
    from paper_2504_15465_b200 import configs

    r = configs.policy_comparison(horizon_ms=200.0, reps=1)
    assert set(r) == set(configs.POLICIES)
    for row in r.values():
        assert row["lc_completed"] > 0 and row["be_atoms"] > 0
    assert r["full_system"]["lc_p99_ms"] < r["mps_like"]["lc_p99_ms"]


def test_inference_stacking_keeps_every_lc_tail(api, cuda_device):
    """BASELINE config #2 under contention (configs.run("infer4")): four LC
    inference tenants beside a training tenant, TPC utilisation >= 0.5, every
    LC tenant's p99 within 1.2x of its alone p99 (~400-600 requests each), 100 %
    SLO attainment."""
    import sys

    sys.path.insert(0, os.path.dirname(GOLDEN))
    from paper_2504_15465_b200 import configs

    r = configs.run("infer4", horizon_ms=2000.0, reps=2)
    assert r["tpc_utilization"] >= 0.5, r["tpc_utilization"]
    for app, row in r["apps"].items():
        if row["priority"] != "hp":
            continue
        assert row["stacked"]["completed"] >= 350, (app, row["stacked"]["completed"])
        assert row["p99_vs_alone"] <= 1.2, (app, row["p99_vs_alone"])
        assert row["slo_attainment"] == 1.0, (app, row["slo_attainment"])
