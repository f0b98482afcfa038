"""The N>1 path: one independent tenant set per rank, scalar results reduced
over gloo (sum of throughput counters, max of time, pooled latency samples).
world_size 2 on CPU with the replay backend; the GPU path differs only in
the backend each rank's session uses."""
from __future__ import annotations

import json
import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def worker(rank: int, world: int, port: int, out_dir: str) -> None:
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    from paper_2504_15465_b200 import api, replicas, workloads

    me = replicas.init_from_env()
    cfg = workloads.tenant_set(me.rank, 10.0, 500.0)
    r = api.run({"scenario": {"config": cfg}, "backend": "replay", "requests": True})
    wall = r["wall_ns"] * 1e-9
    replicas.barrier()
    atoms, = replicas.reduce([float(r["atoms"]["be"])], "sum")
    slowest, = replicas.reduce([wall], "max")
    lat = [json.loads(x)["latency_us"] for x in r["request_log"].splitlines()
           if json.loads(x)["app"].startswith("lc") and json.loads(x)["completed"]]
    pooled = replicas.gather_samples(lat)
    with open(os.path.join(out_dir, f"rank{me.rank}.json"), "w") as f:
        json.dump({"atoms_sum": atoms, "wall_max": slowest, "pooled": len(pooled),
                   "own_atoms": r["atoms"]["be"], "own_wall": wall, "own_lat": len(lat)}, f)
    import torch.distributed as dist

    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_replicas_reduce_like_independent_runs(api, tmp_path):
    mp.spawn(worker, args=(2, free_port(), str(tmp_path)), nprocs=2, join=True)
    r0 = json.load(open(tmp_path / "rank0.json"))
    r1 = json.load(open(tmp_path / "rank1.json"))
    assert r0["atoms_sum"] == r1["atoms_sum"] == r0["own_atoms"] + r1["own_atoms"]
    assert r0["wall_max"] == r1["wall_max"] == max(r0["own_wall"], r1["own_wall"])
    assert r0["pooled"] == r0["own_lat"] + r1["own_lat"]
    # Different ranks run different tenant sets (phase-shifted LC bursts).
    from paper_2504_15465_b200 import workloads

    assert workloads.tenant_set(0) != workloads.tenant_set(1)
