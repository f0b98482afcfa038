"""Convolution atom body (NHWC implicit GEMM on the TPC pair's tensor cores,
TMA im2col loads per filter tap, padding = TMA zero fill) checked against
torch's float64 conv2d of the same bf16 inputs. Tolerance: fp32 output
max |y - ref| <= 1e-3 max |ref|, relative Frobenius <= 1e-5; bf16 output
within one rounding. Shapes cover ResNet-50 stages (3x3 and 1x1, stride 1
and 2, 56/28/14/7 feature maps, the 7x7 stem with C padded to 8)."""
from __future__ import annotations

import random
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


CASES = [
    # n, h, w, c, k, r, s, pad, stride, bf16_out
    (2, 14, 14, 64, 128, 3, 3, 1, 1, False),
    (1, 56, 56, 64, 64, 3, 3, 1, 1, True),
    (2, 28, 28, 128, 256, 1, 1, 0, 1, False),
    (2, 28, 28, 128, 128, 3, 3, 1, 2, False),     # stride 2: 28 -> 14
    (4, 7, 7, 512, 512, 3, 3, 1, 1, True),        # 7x7 maps: tiles span images
    (1, 32, 32, 8, 64, 7, 7, 3, 2, False),        # stem-like: C = 3 padded to 8, 7x7 s2
    (3, 10, 12, 72, 300, 3, 3, 1, 1, False),      # ragged everything
    (1, 7, 7, 256, 256, 3, 3, 1, 1, False),       # 49 pixels: the peer's rows are all past the end
    (2, 28, 28, 256, 512, 1, 1, 0, 2, True),      # 1x1 stride-2 downsample
    (2, 56, 56, 64, 64, 3, 3, 1, 1, False),       # 64-wide channel tiles
    (2, 28, 28, 128, 96, 3, 3, 1, 1, True),       # 128-wide tiles, ragged K
]


@pytest.mark.parametrize("case", CASES, ids=[str(c[:9]) for c in CASES])
def test_conv_atoms_match_reference(api, cuda_device, case):
    import torch

    n, h, w, c, k, r, s, pad, stride, bf16_out = case
    g = torch.Generator().manual_seed(sum(case[:9]))
    x = (torch.rand(n, h, w, c, generator=g) * 2 - 1).to(torch.bfloat16)
    wt = (torch.rand(k, r, s, c, generator=g) * 2 - 1).to(torch.bfloat16)
    cb = -(-c // 64) * 64
    wpad = torch.zeros(k, r, s, cb, dtype=torch.bfloat16)
    wpad[..., :c] = wt
    ref = torch.nn.functional.conv2d(x.double().permute(0, 3, 1, 2), wt.double().permute(0, 3, 1, 2),
                                     padding=pad, stride=stride).permute(0, 2, 3, 1).numpy()
    X, Wd = x.cuda(), wpad.cuda()
    p, q = ref.shape[1], ref.shape[2]
    y = torch.full((n, p, q, k), float("nan"), device="cuda",
                   dtype=torch.bfloat16 if bf16_out else torch.float32)
    rng = random.Random(k)
    with api.Device() as dev:
        desc, blocks, P, Q = dev.conv_desc(X.data_ptr(), Wd.data_ptr(), y.data_ptr(), n, h, w, c, k, r, s,
                                           pad, stride, bf16_out=bf16_out)
        assert (P, Q) == (p, q)
        trace = torch.zeros(blocks, dtype=torch.int32, device="cuda")
        cuts = sorted(rng.sample(range(1, blocks), min(4, blocks - 1))) if blocks > 1 else []
        atoms = [(lo, hi, sorted(rng.sample(range(74), rng.choice([1, 8, 74]))), 20)
                 for lo, hi in zip([0] + cuts, cuts + [blocks])]
        dev.start()
        for lo, hi, tpcs, prio in atoms:
            dev.submit(lo, hi, tpcs, prio, api.GPUOS_BODY_CONV_BF16, [desc], trace=trace.data_ptr())
        wait_all(dev, len(atoms))
        dev.stop()
        dev.free(desc)
    tr = trace.cpu().numpy().view(np.uint32)
    assert ((tr >> 16) == 1).all()
    got = y.float().cpu().numpy().astype(np.float64)
    err = np.abs(got - ref)
    if bf16_out:
        assert (err <= np.abs(ref) * 2.0 ** -8 + 1e-4 * np.abs(ref).max()).all(), float(err.max())
    else:
        assert err.max() <= 1e-3 * np.abs(ref).max(), float(err.max())
        assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref)
