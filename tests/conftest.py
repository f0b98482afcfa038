"""Shared fixtures. Markers: `gpu` tests need a B200 (run under gpurun);
everything else runs on CPU in the build container."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE = "/root/reference/proj"
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU (run under gpurun)")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def built():
    """Builds the native library and tools in-tree (incremental)."""
    from paper_2504_15465_b200 import build as b

    return b.build()


@pytest.fixture(scope="session")
def api(built):
    from paper_2504_15465_b200 import api as a

    a.library()
    return a


@pytest.fixture(scope="session")
def oracle_ref():
    """The unmodified reference built by oracle/Makefile (needs /root/reference
    here, or a prebuilt oracle/_ref/ shipped with the snapshot)."""
    ref = os.path.join(ROOT, "oracle", "_ref")
    if os.path.isdir(REFERENCE):
        r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], capture_output=True, text=True)
        if r.returncode != 0:
            pytest.fail("oracle build failed:\n" + r.stderr[-2000:])
    if not os.path.exists(os.path.join(ref, "ref_golden")):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return ref


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def run_atoms(api, dev, atoms, workers, body, args, trace=None, timeout=60.0):
    """Executes (lo, hi, tpcs, prio) atoms of one body: live (ring + ingest
    warp) with W = 2 workers per SM, batch mode with W = 1 (live mode needs
    W = 2: the ingest cluster takes one of a TPC's two worker pairs)."""
    import time

    if workers == 2:
        dev.start()
        for lo, hi, tpcs, prio in atoms:
            dev.submit(lo, hi, tpcs, prio, body, args, trace=trace)
    else:
        dev.run_batch([api.Device.desc(lo, hi, tpcs, prio, body, args, trace=trace)
                       for lo, hi, tpcs, prio in atoms])
    done = []
    t0 = time.time()
    while len(done) < len(atoms):
        done += dev.poll()
        assert time.time() - t0 < timeout, f"only {len(done)}/{len(atoms)} atoms completed"
    if workers == 2:
        dev.stop()
    return done
