"""GEMV atom body (decode y = W . x, HBM-bound: TMA-streamed W, tensor-core
MACs on the TPC pair) on the persistent dispatcher, checked against a
float64 CPU product of the same bf16 inputs.
Tolerance: fp32 accumulation, max |y - ref| <= 1e-3 max |ref| and relative
Frobenius error <= 1e-5; bf16 y within one rounding (2^-8 |ref| + 1e-4 max).
Every block runs exactly once and only on its atom's TPCs."""
from __future__ import annotations

import random
import time

import numpy as np
import pytest

from conftest import run_atoms

pytestmark = pytest.mark.gpu


def wait_all(dev, n, timeout=60.0):
    done = []
    t0 = time.time()
    while len(done) < n:
        done += dev.poll()
        assert time.time() - t0 < timeout, f"only {len(done)}/{n} atoms completed"
    return done


@pytest.mark.parametrize("n,k,bf16_out,workers,splits,packed", [
    (6144, 4096, False, 2, 1, False),   # Llama-3-8B QKV projection
    (4096, 14336, True, 2, 1, False),   # down projection, bf16 y
    (4096, 14336, True, 2, 16, False),  # down projection, split-K, bf16 y
    (1000, 264, False, 1, 3, False),    # ragged last tile, K not a multiple of 64, split-K
    (6144, 4096, False, 2, 3, True),    # packed W (gpuos_dev_gemv_pack), split-K
    (1000, 264, True, 2, 3, True),      # packed W, ragged N and K (zero-padded tiles)
])
def test_gemv_atoms_match_reference(api, cuda_device, n, k, bf16_out, workers, splits, packed):
    import torch

    g = torch.Generator().manual_seed(n + k)
    w = (torch.rand(n, k, generator=g) * 2 - 1).to(torch.bfloat16)
    x = (torch.rand(k, generator=g) * 2 - 1).to(torch.bfloat16)
    ref = w.double().numpy() @ x.double().numpy()
    W, X = w.cuda(), x.cuda()
    y = torch.full((n,), float("nan"), device="cuda",
                   dtype=torch.bfloat16 if bf16_out else torch.float32)
    rng = random.Random(k)
    with api.Device(workers_per_sm=workers) as dev:
        if packed:
            Wp = torch.full((dev.gemv_packed_bytes(n, k) // 2,), float("nan"), device="cuda", dtype=torch.bfloat16)
            dev.gemv_pack(Wp.data_ptr(), W.data_ptr(), n, k)
            W = Wp
        desc, blocks = dev.gemv_desc(W.data_ptr(), X.data_ptr(), y.data_ptr(), n, k, bf16_out=bf16_out,
                                     k_splits=splits, packed=packed)
        assert blocks == -(-n // 256) * min(splits, -(-k // 64))
        trace = torch.zeros(blocks, dtype=torch.int32, device="cuda")
        cuts = sorted(rng.sample(range(1, blocks), min(6, blocks - 1)))
        atoms = [(lo, hi, sorted(rng.sample(range(74), rng.choice([1, 5, 74]))), rng.choice([10, 20, 30]))
                 for lo, hi in zip([0] + cuts, cuts + [blocks])]
        x2 = (torch.rand(k, generator=g) * 2 - 1).to(torch.bfloat16)
        if workers == 2:
            dev.start()
            for lo, hi, tpcs, prio in atoms:
                dev.submit(lo, hi, tpcs, prio, api.GPUOS_BODY_GEMV_BF16, [desc], trace=trace.data_ptr())
            wait_all(dev, len(atoms))
            # The same descriptor serves the next decode step: new x, same pointers.
            X.copy_(x2.cuda())
            torch.cuda.current_stream().synchronize()  # not the device: the dispatcher is resident
            dev.submit(0, blocks, list(range(74)), 20, api.GPUOS_BODY_GEMV_BF16, [desc])
            wait_all(dev, 1)
            dev.stop()
        else:  # W = 1: batch mode (see conftest.run_atoms)
            run_atoms(api, dev, atoms, workers, api.GPUOS_BODY_GEMV_BF16, [desc], trace=trace.data_ptr())
            X.copy_(x2.cuda())
            torch.cuda.synchronize()
            run_atoms(api, dev, [(0, blocks, list(range(74)), 20)], workers, api.GPUOS_BODY_GEMV_BF16, [desc])
        dev.free(desc)
    tr = trace.cpu().numpy().view(np.uint32)
    assert ((tr >> 16) == 1).all()
    sm = (tr & 0xFFFF).astype(np.int64) - 1
    for lo, hi, tpcs, _ in atoms:
        assert set((sm[lo:hi] >> 1).tolist()) <= set(tpcs)
    ref = w.double().numpy() @ x2.double().numpy()
    got = y.float().cpu().numpy().astype(np.float64)
    err = np.abs(got - ref)
    if bf16_out:
        assert (err <= np.abs(ref) * 2.0 ** -8 + 1e-4 * np.abs(ref).max()).all()
    else:
        assert err.max() <= 1e-3 * np.abs(ref).max()
        assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref)


def test_gemv_rejects_bad_shapes(api, cuda_device):
    import torch

    w = torch.zeros(256, 100, dtype=torch.bfloat16, device="cuda")
    with api.Device() as dev:
        with pytest.raises(api.GpuosError):  # K % 8 != 0: rows not 16-byte aligned
            dev.gemv_desc(w.data_ptr(), w.data_ptr(), w.data_ptr(), 256, 100)
        dev.start()
        with pytest.raises(api.GpuosError):  # no descriptor
            dev.submit(0, 1, [0], 20, api.GPUOS_BODY_GEMV_BF16, [0])
        dev.stop()
