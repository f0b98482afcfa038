"""Batch-mode launches of the worker kernel executing an NHWC implicit-GEMM
convolution (tcgen05 pair tiles, TMA im2col loads per filter tap) atomized over
all 74 TPCs; prints ms and TFLOP/s (algorithmic: 2 N P Q K R S C).

usage: conv_batch.py N H W C K R S pad stride [launches]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_15465_b200 import api  # noqa: E402

n, h, w, c, k, r, s, pad, stride = (int(v) for v in sys.argv[1:10])
reps = int(sys.argv[10]) if len(sys.argv) > 10 else 3
cb = -(-c // 64) * 64
x = (torch.rand(n, h, w, c, device="cuda") * 2 - 1).to(torch.bfloat16)
wt = (torch.rand(k, r, s, cb, device="cuda") * 2 - 1).to(torch.bfloat16)
p = (h + 2 * pad - r) // stride + 1
q = (w + 2 * pad - s) // stride + 1
y = torch.empty(n, p, q, k, device="cuda", dtype=torch.bfloat16)
torch.cuda.synchronize()
with api.Device() as dev:
    desc, blocks, P, Q = dev.conv_desc(x.data_ptr(), wt.data_ptr(), y.data_ptr(), n, h, w, c, k, r, s,
                                       pad, stride, bf16_out=True)
    n_atoms = min(32, blocks)
    descs = [api.Device.desc(i * blocks // n_atoms, (i + 1) * blocks // n_atoms, range(74), 20,
                             api.GPUOS_BODY_CONV_BF16, [desc]) for i in range(n_atoms)]
    flops = 2.0 * n * P * Q * k * r * s * c
    for _ in range(reps):
        ms = dev.run_batch(descs)
        while dev.in_flight():
            dev.poll()
        st = dev.stats()
        print(f"conv n{n} {h}x{w}x{c} -> {P}x{Q}x{k} {r}x{s}/{stride} ({blocks} blocks): {ms:.3f} ms, "
              f"{flops / ms / 1e9:.0f} TFLOP/s (device span {st.worker_span_ns / 1e3:.1f} us: "
              f"{flops / st.worker_span_ns / 1e3:.0f} TFLOP/s)", flush=True)
    dev.free(desc)
