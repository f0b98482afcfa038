"""GEMM atom body (tcgen05.mma + TMEM + TMA) on the persistent dispatcher.

C = A . B^T with bf16 operands and fp32 accumulation, checked against a
float64 CPU product of the same bf16 inputs. Tolerances (the north star's
"1e-3 relative for bf16 GEMM"):
  * fp32 output: max |C - ref| <= 1e-3 * max |ref| and relative Frobenius
    error <= 1e-5 (accumulation order only);
  * bf16 output: |C - ref| <= 2^-8 |ref| + 1e-4 max|ref| per element (one
    round-to-nearest of the fp32 accumulator, which itself may differ from
    the exact product by accumulation order).
Every block (output tile) must run exactly once and only on its atom's TPCs.
"""
from __future__ import annotations

import random
import time

import numpy as np
import pytest

from conftest import run_atoms
from oracle.policy import stream_expect

pytestmark = pytest.mark.gpu


def wait_all(dev, n, timeout=60.0):
    done = []
    t0 = time.time()
    while len(done) < n:
        done += dev.poll()
        assert time.time() - t0 < timeout, f"only {len(done)}/{n} atoms completed"
    return done


def operands(torch, m, n, k, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    a = (torch.rand(m, k, generator=g) * 2 - 1).to(torch.bfloat16)
    b = (torch.rand(n, k, generator=g) * 2 - 1).to(torch.bfloat16)
    ref = a.double().numpy() @ b.double().numpy().T
    return a.cuda(), b.cuda(), ref


def check(c, ref, bf16_out):
    got = c.float().cpu().numpy().astype(np.float64)
    err = np.abs(got - ref)
    if bf16_out:
        bound = np.abs(ref) * 2.0 ** -8 + 1e-4 * np.abs(ref).max()
        assert (err <= bound).all(), float((err - bound).max())
    else:
        assert err.max() <= 1e-3 * np.abs(ref).max(), float(err.max())
        assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref)


def random_atoms(rng, blocks, n_atoms):
    cuts = sorted(rng.sample(range(1, blocks), min(n_atoms - 1, blocks - 1)))
    out = []
    for lo, hi in zip([0] + cuts, cuts + [blocks]):
        k = rng.choice([1, 3, 16, 74])
        tpcs = sorted(rng.sample(range(74), k)) if k < 74 else list(range(74))
        out.append((lo, hi, tpcs, rng.choice([10, 20, 30])))
    return out


@pytest.mark.parametrize("m,n,k,bf16_out,workers", [
    (512, 1024, 768, False, 2),
    (300, 200, 72, True, 2),      # ragged M / N tiles, K not a multiple of 64
    (1024, 768, 1024, False, 1),  # 1 worker per SM: deeper ring
    (640, 384, 520, True, 1),
    (1000, 64, 384, False, 2),    # 64-wide tiles (attention-head output)
    (520, 100, 128, True, 2),     # 128-wide tiles, ragged N
])
def test_gemm_atoms_match_reference(api, cuda_device, m, n, k, bf16_out, workers):
    import torch

    a, b, ref = operands(torch, m, n, k, seed=m + n + k)
    c = torch.full((m, n), float("nan"), device="cuda",
                   dtype=torch.bfloat16 if bf16_out else torch.float32)
    rng = random.Random(k)
    with api.Device(workers_per_sm=workers) as dev:
        desc, blocks, tm, tn = dev.gemm_desc(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k,
                                             bf16_out=bf16_out)
        assert tm == 256 and tn == (64 if n <= 64 else 128 if n <= 128 else 256)
        assert blocks == -(-m // tm) * -(-n // tn)
        trace = torch.zeros(blocks, dtype=torch.int32, device="cuda")
        atoms = random_atoms(rng, blocks, min(blocks, 7))
        run_atoms(api, dev, atoms, workers, api.GPUOS_BODY_GEMM_BF16, [desc], trace=trace.data_ptr())
        dev.free(desc)
    tr = trace.cpu().numpy().view(np.uint32)
    assert ((tr >> 16) == 1).all(), "a tile did not run exactly once"
    sm = (tr & 0xFFFF).astype(np.int64) - 1
    for lo, hi, tpcs, _ in atoms:
        assert set((sm[lo:hi] >> 1).tolist()) <= set(tpcs)
    check(c, ref, bf16_out)


def test_workers_per_sm_bounded(api, cuda_device):
    """At most two TMEM-owning worker CTAs fit on an SM: W > 2 is refused."""
    with pytest.raises(api.GpuosError):
        api.Device(workers_per_sm=3)


def test_gemm_and_stream_share_workers(api, cuda_device):
    """GEMM tiles and STREAM blocks interleaved on the same TPCs: the two
    shared-memory pipelines keep independent phases inside one worker."""
    import torch

    m, n, k = 768, 512, 640
    a, b, ref = operands(torch, m, n, k, seed=7)
    c = torch.zeros(m, n, device="cuda")
    words, sblocks, salt = 2048, 400, 0xABCDEF
    src = torch.randint(-2**31, 2**31 - 1, (sblocks * words,), dtype=torch.int32, device="cuda")
    dst = torch.zeros_like(src)
    with api.Device(workers_per_sm=2) as dev:
        desc, blocks, _, _ = dev.gemm_desc(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k)
        dev.start()
        tpcs = list(range(0, 8))
        n_atoms = 0
        for i in range(blocks):
            dev.submit(i, i + 1, tpcs, 20, api.GPUOS_BODY_GEMM_BF16, [desc])
            lo = i * sblocks // blocks
            hi = (i + 1) * sblocks // blocks
            dev.submit(lo, hi, tpcs, 20, api.GPUOS_BODY_STREAM,
                       [src.data_ptr(), dst.data_ptr(), words, salt, 0])
            n_atoms += 2
        wait_all(dev, n_atoms)
        dev.stop()
        dev.free(desc)
    check(c, ref, False)
    assert np.array_equal(dst.cpu().numpy().view(np.uint32),
                          stream_expect(src.cpu().numpy().view(np.uint32), salt, 0))


def test_gemm_batch_large(api, cuda_device):
    """A 4096^3 GEMM as 32 atoms on all 74 TPCs in one batch-mode launch;
    checked against torch's fp32 GEMM of the same bf16 inputs (TF32 off)."""
    import torch

    torch.backends.cuda.matmul.allow_tf32 = False
    m = n = k = 4096
    g = torch.Generator(device="cuda").manual_seed(3)
    a = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    b = (torch.rand(n, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    c = torch.zeros(m, n, device="cuda")
    ref = a.float() @ b.float().T
    with api.Device(workers_per_sm=2) as dev:
        desc, blocks, _, _ = dev.gemm_desc(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k)
        per = blocks // 32
        descs = [api.Device.desc(i * per, (i + 1) * per if i < 31 else blocks, range(74), 20,
                                 api.GPUOS_BODY_GEMM_BF16, [desc]) for i in range(32)]
        ms = dev.run_batch(descs)
        dev.free(desc)
    err = (c - ref).abs().max().item()
    assert err <= 1e-3 * ref.abs().max().item(), err
    tflops = 2 * m * n * k / (ms * 1e-3) / 1e12
    print(f"batch GEMM 4096^3: {ms:.3f} ms, {tflops:.0f} TFLOP/s")
    assert tflops > 100  # sanity: the tensor-core path ran


@pytest.mark.parametrize("m,n,k,splits,bf16_out,workers", [
    (576, 64, 12544, 6, True, 2),     # stage-1 3x3 weight gradient shape (transposed), 64-wide tiles
    (300, 200, 4160, 5, False, 2),    # ragged M / N, K split unevenly (65 slices over 5 splits)
    (1024, 512, 8192, 16, False, 1),  # 1 worker per SM
    (256, 1000, 2048, 3, True, 2),
])
def test_gemm_split_k_matches_reference(api, cuda_device, m, n, k, splits, bf16_out, workers):
    """Split-K GEMM (gpuos_dev_gemm_desc_splitk): block b = (tile b % tiles,
    split b / tiles); the tile's last split sums the fp32 partials in split
    order. Random atoms over random TPC sets, run twice (the arrival
    counters reset themselves), every block exactly once."""
    import torch

    a, b, ref = operands(torch, m, n, k, seed=m + n + k + splits)
    rng = random.Random(splits)
    with api.Device(workers_per_sm=workers) as dev:
        c = torch.full((m, n), float("nan"), device="cuda",
                       dtype=torch.bfloat16 if bf16_out else torch.float32)
        desc, blocks, tm, tn = dev.gemm_desc(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k,
                                             bf16_out=bf16_out, k_splits=splits)
        tiles = -(-m // tm) * -(-n // tn)
        nk = -(-k // 64)
        per = -(-nk // splits)
        assert blocks == tiles * -(-nk // per)
        for rep in range(2):
            c.fill_(float("nan"))
            trace = torch.zeros(blocks, dtype=torch.int32, device="cuda")
            atoms = random_atoms(rng, blocks, min(blocks, 9))
            run_atoms(api, dev, atoms, workers, api.GPUOS_BODY_GEMM_BF16, [desc], trace=trace.data_ptr())
            torch.cuda.synchronize()
            tr = trace.cpu().numpy().view(np.uint32)
            assert ((tr >> 16) == 1).all(), "a block did not run exactly once"
            sm = (tr & 0xFFFF).astype(np.int64) - 1
            for lo, hi, tpcs, _ in atoms:
                assert set((sm[lo:hi] >> 1).tolist()) <= set(tpcs)
            check(c, ref, bf16_out)
        dev.free(desc)
