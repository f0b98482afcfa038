"""bench.py's N>1 path on CPU: `--gpus N` outside torchrun starts N ranks
itself (RANK / WORLD_SIZE / LOCAL_RANK / MASTER_ADDR=127.0.0.1), they
rendezvous over gloo, and rank 0 alone prints one JSON line. The reference
arm is the part that runs without a GPU; the repo arm's rank logic is the
same launcher."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def run_bench(*args, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=240, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.strip()]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.timeout(300)
def test_self_launch_two_ranks_prints_one_line(oracle_ref):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    line = run_bench("--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
                     "--sample-s", "0.3", env=env)
    assert line["n_gpus"] == 2
    assert line["impl"] == "reference"
    assert line["config"]["parallelism"] == "replicas x2"
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["cpu_model"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0


@pytest.mark.timeout(300)
def test_reference_arm_config_matches_single_rank(oracle_ref):
    """Both arms print their `config` from bench_config(); at N = 1 the
    reference arm's dict is exactly what the repo arm prints."""
    sys.path.insert(0, ROOT)
    import argparse

    import bench
    from paper_2504_15465_b200 import workloads

    args = argparse.Namespace(workload="fig7", time_scale=10.0)
    cfg = workloads.fig7_b200(10.0, 2000.0)
    line = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0", "--sample-s", "0.3")
    assert line["config"] == json.loads(json.dumps(bench.bench_config(cfg, args, 1)))
