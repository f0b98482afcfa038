"""Tenant-supplied bodies (include/gpuos_body.cuh) on the persistent
dispatcher: the prelude's blockIdx recovery from the linear block index
 and two real tenant kernels (RMSNorm,
SiLU-mul, csrc/bodies/llama_elementwise.cu) atomized over random TPC sets,
checked against float64 CPU references of the same bf16 inputs (tolerance:
one bf16 rounding of the result, 2^-8 |ref|, plus 1e-3 max |ref| for fp32
accumulation order). Every block runs exactly once and on its atom's TPCs."""
from __future__ import annotations

import random
import struct
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def wait_all(dev, n, timeout=60.0):
    done = []
    t0 = time.time()
    while len(done) < n:
        done += dev.poll()
        assert time.time() - t0 < timeout, f"only {len(done)}/{n} atoms completed"
    return done


def atoms_for(blocks, seed):
    rng = random.Random(seed)
    cuts = sorted(rng.sample(range(1, blocks), min(5, blocks - 1))) if blocks > 1 else []
    return [(lo, hi, sorted(rng.sample(range(74), rng.choice([1, 3, 74]))), rng.choice([10, 20, 30]))
            for lo, hi in zip([0] + cuts, cuts + [blocks])]


def run(api, body, args, blocks, seed, trace):
    with api.Device() as dev:
        atoms = atoms_for(blocks, seed)
        dev.start()
        for lo, hi, tpcs, prio in atoms:
            dev.submit(lo, hi, tpcs, prio, body, args, trace=trace.data_ptr())
        wait_all(dev, len(atoms))
        dev.stop()
    tr = trace.cpu().numpy().view(np.uint32)
    assert ((tr >> 16) == 1).all(), "a block did not run exactly once"
    sm = (tr & 0xFFFF).astype(np.int64) - 1
    for lo, hi, tpcs, _ in atoms:
        assert set((sm[lo:hi] >> 1).tolist()) <= set(tpcs)


def test_unknown_body_name_is_rejected(api):
    with pytest.raises(api.GpuosError):
        api.body_id("no_such_body")


def test_prelude_recovers_block_index(api, cuda_device):
    import torch

    gx, gy, gz = 7, 5, 3
    n = gx * gy * gz
    out = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    trace = torch.zeros(n, dtype=torch.int32, device="cuda")
    run(api, api.body_id("grid_probe"), [out.data_ptr(), 0, 0, 0, api.grid(gx, gy, gz)], n, 1, trace)
    got = out.cpu().numpy().view(np.uint32)
    lin = np.arange(n)
    want = (lin % gx) | (((lin // gx) % gy) << 10) | ((lin // (gx * gy)) << 20)
    assert np.array_equal(got, want.astype(np.uint32))


@pytest.mark.parametrize("rows,d", [(37, 4096), (3, 14336)])
def test_rmsnorm_body_matches_reference(api, cuda_device, rows, d):
    import torch

    g = torch.Generator().manual_seed(rows + d)
    x = ((torch.rand(rows, d, generator=g) * 2 - 1) * 3).to(torch.bfloat16)
    w = (torch.rand(d, generator=g) + 0.5).to(torch.bfloat16)
    y = torch.full((rows, d), float("nan"), dtype=torch.bfloat16, device="cuda")
    X, Wt = x.cuda(), w.cuda()
    eps = 1e-5
    a3 = d | (struct.unpack("<I", struct.pack("<f", eps))[0] << 32)
    trace = torch.zeros(rows, dtype=torch.int32, device="cuda")
    run(api, api.body_id("rmsnorm_bf16"), [X.data_ptr(), Wt.data_ptr(), y.data_ptr(), a3, api.grid(rows)],
        rows, 2, trace)
    xd, wd = x.double().numpy(), w.double().numpy()
    ref = xd / np.sqrt((xd * xd).mean(axis=1, keepdims=True) + eps) * wd
    got = y.float().cpu().numpy().astype(np.float64)
    assert (np.abs(got - ref) <= np.abs(ref) * 2.0 ** -8 + 1e-3 * np.abs(ref).max()).all()


def test_silu_mul_body_matches_reference(api, cuda_device):
    import torch

    n, chunk = 2 * 14336 + 5, 2048
    blocks = -(-n // chunk)
    g = torch.Generator().manual_seed(9)
    gate = ((torch.rand(n, generator=g) * 2 - 1) * 6).to(torch.bfloat16)
    up = ((torch.rand(n, generator=g) * 2 - 1) * 2).to(torch.bfloat16)
    # 16-byte aligned buffers with the ragged tail inside them
    G = torch.zeros(n + 8, dtype=torch.bfloat16, device="cuda")
    U = torch.zeros_like(G)
    O = torch.full_like(G, float("nan"))
    G[:n].copy_(gate.cuda())
    U[:n].copy_(up.cuda())
    trace = torch.zeros(blocks, dtype=torch.int32, device="cuda")
    run(api, api.body_id("silu_mul_bf16"), [G.data_ptr(), U.data_ptr(), O.data_ptr(), n | (chunk << 32),
                                            api.grid(blocks)], blocks, 3, trace)
    gd, ud = gate.double().numpy(), up.double().numpy()
    ref = gd / (1 + np.exp(-gd)) * ud
    got = O[:n].float().cpu().numpy().astype(np.float64)
    assert (np.abs(got - ref) <= np.abs(ref) * 2.0 ** -8 + 1e-3 * np.abs(ref).max()).all()
    assert torch.isnan(O[n:].float()).all()  # nothing written past n


@pytest.mark.parametrize("ctx,chunk", [(1024, 32), (300, 24), (2000, 32)])
def test_attention_body_matches_reference(api, cuda_device, ctx, chunk):
    """attn_decode_bf16: Llama-3 GQA decode attention (32 query / 8 KV heads of
    128, RoPE base 500000 on interleaved pairs at position ctx) split over the
    context in chunks, merged by each KV head's last block; against a float64
    restatement. The merge is deterministic (chunk order), so a second run of
    the same kernel reproduces the result bit for bit."""
    import torch

    chunks = -(-ctx // chunk)
    blocks = chunks * 8
    g = torch.Generator().manual_seed(ctx)
    q = (torch.rand(32, 128, generator=g) * 2 - 1).to(torch.bfloat16)
    kv = (torch.rand(2, ctx, 8, 128, generator=g) * 2 - 1).to(torch.bfloat16)
    Q, KV = q.cuda(), kv.cuda()
    ws = torch.zeros((8448 + 32 * chunks * 130 * 4) // 4, dtype=torch.float32, device="cuda")
    args = [Q.data_ptr(), KV.data_ptr(), ws.data_ptr(), ctx | (chunk << 32), api.grid(chunks, 8)]
    outs = []
    for seed in (4, 5):
        trace = torch.zeros(blocks, dtype=torch.int32, device="cuda")
        run(api, api.body_id("attn_decode_bf16"), args, blocks, seed, trace)
        outs.append(ws[:2048].view(torch.bfloat16)[:4096].cpu().clone())
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    got = outs[0].view(32, 128).double().numpy()
    qd, k, v = q.double().numpy(), kv[0].double().numpy(), kv[1].double().numpy()
    j = np.arange(64)
    ang = ctx * 500000.0 ** (-2.0 * j / 128)
    qr = np.empty_like(qd)
    qr[:, 0::2] = qd[:, 0::2] * np.cos(ang) - qd[:, 1::2] * np.sin(ang)
    qr[:, 1::2] = qd[:, 0::2] * np.sin(ang) + qd[:, 1::2] * np.cos(ang)
    for h in range(32):
        s = k[:, h // 4, :] @ qr[h] / np.sqrt(128.0)
        e = np.exp(s - s.max())
        ref = (e[:, None] * v[:, h // 4, :]).sum(0) / e.sum()
        mag = (e[:, None] * np.abs(v[:, h // 4, :])).sum(0) / e.sum()
        assert (np.abs(got[h] - ref) <= np.abs(ref) * 2.0 ** -8 + 2e-3 * mag + 1e-4).all(), h
