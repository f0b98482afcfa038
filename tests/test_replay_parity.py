"""Replay-mode parity: the B200 library's scheduler + replay engine must
reproduce the reference's dispatch/completion logs and reports byte for
byte (atom partitioning, TPC assignments, completion order, accounting).

Fixtures come from the UNMODIFIED reference (tests/golden/make_golden.py);
when oracle/_ref is available the same comparison also runs live on fresh
randomized scenarios."""
from __future__ import annotations

import gzip
import hashlib
import json
import os
import random
import subprocess
import sys

import pytest

from conftest import GOLDEN

CASES = json.load(open(os.path.join(GOLDEN, "cases.json")))


def replay_tool(built, args, cwd=GOLDEN):
    return subprocess.run([built["gpuos_replay"]] + args, cwd=cwd, capture_output=True, check=True).stdout


@pytest.mark.parametrize("name", sorted(CASES["cases"]))
def test_log_and_report_match_reference(built, name):
    args = CASES["cases"][name]
    ref_log = gzip.open(os.path.join(GOLDEN, "logs", name + ".log.gz")).read()
    assert replay_tool(built, args) == ref_log
    ref_rep = open(os.path.join(GOLDEN, "reports", name + ".txt"), "rb").read()
    assert replay_tool(built, args + ["--report"]) == ref_rep


@pytest.mark.parametrize("name", sorted(CASES["digests"]))
def test_full_length_log_digest(built, name):
    d = CASES["digests"][name]
    assert hashlib.sha256(replay_tool(built, d["args"])).hexdigest() == d["sha256"]


def test_capi_session_log_matches_reference(api):
    """Same parity through the C ABI a reference-side binding would use."""
    ref_log = gzip.open(os.path.join(GOLDEN, "logs", "fig7_2s.log.gz")).read().decode()
    r = api.run({"scenario": {"preset": "fig7"}, "backend": "replay", "horizon_ms": 2000, "log": True})
    dc = [line for line in ref_log.splitlines() if line[:1] in "DC"]
    assert r["log"].splitlines() == dc
    ref_rep = open(os.path.join(GOLDEN, "reports", "fig7_2s.txt")).read()
    report_json = ref_rep[: ref_rep.index("\n}\n") + 2]
    assert r["report"] == json.loads(report_json)


def test_live_random_scenarios_against_reference(built, oracle_ref, tmp_path):
    sys.path.insert(0, GOLDEN)
    from make_golden import random_scenario  # noqa: E402

    for seed in random.Random(2024).sample(range(100, 10_000), 6):
        cfg = random_scenario(seed)
        path = tmp_path / f"s{seed}.json"
        path.write_text(json.dumps(cfg))
        args = ["--config", str(path)]
        ref = subprocess.run([os.path.join(oracle_ref, "ref_golden")] + args, capture_output=True,
                             check=True).stdout
        assert replay_tool(built, args, cwd=str(tmp_path)) == ref, f"seed {seed}"


def test_config_errors_exit_2(built, tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"device": {"gpc_count": 1, "tpcs_per_gpc": 2},
                               "apps": [{"id": "x", "priority": "hp", "quota": 1,
                                         "arrival": "closed_loop",
                                         "kernels": [{"blocks": 1, "block_us": 10}]}]}))
    for args in (["--config", str(bad)], ["--config", str(tmp_path / "missing.json")],
                 ["--preset", "no-such-preset"], ["--config", str(bad), "--preset", "fig7"]):
        assert subprocess.run([built["gpuos_replay"]] + args, capture_output=True).returncode == 2
    bad.write_text("{ not json")
    assert subprocess.run([built["gpuos_replay"], "--config", str(bad)], capture_output=True).returncode == 2


def test_model_traces_run_on_replay(api):
    """Model kernel traces are reference kernel records plus a body the
    reference ignores: they run on the replay engine (conv bodies carry nine
    parameters)."""
    from paper_2504_15465_b200 import models

    for kernels in (models.resnet50_infer(1), models.llama3_8b_decode(256)):
        cfg = {"name": "m", "device": {"gpc_count": 2, "tpcs_per_gpc": 37}, "policy": "full_system",
               "horizon_ms": 20.0, "seed": 1, "scheduler": {"dvfs": False},
               "apps": [{"id": "t", "priority": "hp", "quota": 74, "slo_ms": 100.0,
                         "arrival": {"times_ms": [0.0]}, "kernels": kernels}]}
        r = api.run({"scenario": {"config": cfg}, "backend": "replay"})
        assert r["report"]["apps"][0]["completed"] == 1
    conv = [k for k in models.resnet50_infer(1) if k["body"]["kind"] == "conv_bf16"][0]
    assert len(conv["body"]["p"]) == 9


def _dispatch_log(text):
    disp, comp = {}, {}
    for line in text.splitlines():
        f = line.split()
        if f[0] == "D":
            disp[int(f[2])] = int(f[1])
        elif f[0] == "C":
            comp[int(f[2])] = int(f[1])
    return disp, comp


def test_chained_launches_on_replay(api):
    """chain_launches (live-mode extension, off by default): an HP tenant's
    next kernel is submitted while the current one runs and starts the
    instant it retires. On the zero-latency replay engine that is timing-
    neutral for a lone tenant -- same request latencies as host-paced
    launches -- and every kernel but each request's first is dispatched
    before its predecessor completes."""
    from paper_2504_15465_b200 import models

    kernels = models.llama3_8b_decode(256)[:40]
    out = {}
    for chain in (False, True):
        cfg = {"name": "m", "device": {"gpc_count": 2, "tpcs_per_gpc": 37}, "policy": "full_system",
               "horizon_ms": 200.0, "seed": 1, "scheduler": {"dvfs": False, "chain_launches": chain},
               "apps": [{"id": "t", "priority": "hp", "quota": 74, "slo_ms": 100.0,
                         "arrival": {"times_ms": [0.0, 50.0, 100.0]}, "kernels": kernels}]}
        out[chain] = api.run({"scenario": {"config": cfg}, "backend": "replay", "log": True})
    for r in out.values():
        assert r["report"]["apps"][0]["completed"] == 3
    plain, chained = (out[c]["report"]["apps"][0] for c in (False, True))
    assert (plain["p50_ns"], plain["p99_ns"]) == (chained["p50_ns"], chained["p99_ns"])
    disp, comp = _dispatch_log(out[True]["log"])
    early = sum(1 for a in disp if a - 1 in comp and disp[a] < comp[a - 1])
    assert early == 3 * (len(kernels) - 1)


def test_chained_launches_with_contention_on_replay(api):
    """Two HP tenants and a BE tenant with stealing and revocation: every
    request still completes and the run is deterministic."""
    req = {"scenario": {"preset": "inf-inf"}, "backend": "replay", "horizon_ms": 400,
           "set": {"chain_launches": True, "block_revocation": True}}
    a, b = api.run(req), api.run(req)
    assert a["report"] == b["report"]
    for app in a["report"]["apps"][:2]:
        assert app["completed"] >= app["offered"] - 1


def test_chain_depth_limits_and_validation(api):
    """chain_depth bounds how many kernels ride behind the running one; it
    is validated like the reference's other knobs (ConfigError, code 2)."""
    from paper_2504_15465_b200 import models

    kernels = models.llama3_8b_decode(256)[:12]
    cfg = {"name": "m", "device": {"gpc_count": 2, "tpcs_per_gpc": 37}, "policy": "full_system",
           "horizon_ms": 50.0, "seed": 1, "scheduler": {"dvfs": False, "chain_launches": True},
           "apps": [{"id": "t", "priority": "hp", "quota": 74, "slo_ms": 100.0,
                     "arrival": {"times_ms": [0.0]}, "kernels": kernels}]}
    outstanding = {}
    for depth in (1, 4):
        r = api.run({"scenario": {"config": cfg}, "backend": "replay", "log": True,
                     "set": {"chain_depth": depth}})
        assert r["report"]["apps"][0]["completed"] == 1
        # Dispatched but not yet completed atoms at every dispatch: the
        # running kernel plus at most `depth` chained behind it.
        live, worst = set(), 0
        for line in r["log"].splitlines():
            f = line.split()
            if f[0] == "D":
                live.add(int(f[2]))
                worst = max(worst, len(live))
            elif f[0] == "C":
                live.discard(int(f[2]))
        outstanding[depth] = worst
    assert outstanding[1] == 2 and outstanding[4] == 5
    with pytest.raises(api.GpuosError) as e:
        api.run({"scenario": {"config": cfg}, "backend": "replay", "set": {"chain_depth": 0}})
    assert e.value.code == 2
