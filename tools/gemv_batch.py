"""Batch-mode launches of the worker kernel executing a decode GEMV
(y = W . x, bf16 W [N, K]) atomized over all 74 TPCs; prints ms and HBM GB/s
(algorithmic bytes: W + x + y).

usage: gemv_batch.py N K [launches] [atoms] [k_splits]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_15465_b200 import api  # noqa: E402

n, k = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n_atoms = int(sys.argv[4]) if len(sys.argv) > 4 else 32
splits = int(sys.argv[5]) if len(sys.argv) > 5 else 1
w = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
x = torch.randn(k, device="cuda", dtype=torch.bfloat16)
y = torch.empty(n, device="cuda")
torch.cuda.synchronize()
with api.Device() as dev:
    desc, blocks = dev.gemv_desc(w.data_ptr(), x.data_ptr(), y.data_ptr(), n, k, k_splits=splits)
    n_atoms = min(n_atoms, blocks)
    descs = [api.Device.desc(i * blocks // n_atoms, (i + 1) * blocks // n_atoms, range(74), 20,
                             api.GPUOS_BODY_GEMV_BF16, [desc]) for i in range(n_atoms)]
    for _ in range(reps):
        ms = dev.run_batch(descs)
        while dev.in_flight():
            dev.poll()
        nbytes = n * k * 2 + k * 2 + n * 4
        st = dev.stats()
        print(f"gemv {n}x{k} ({blocks} blocks of 256 rows, {n_atoms} atoms): {ms:.3f} ms, "
              f"{nbytes / ms / 1e6:.0f} GB/s (device span {st.worker_span_ns / 1e3:.1f} us: "
              f"{nbytes / st.worker_span_ns:.0f} GB/s, claim retries {st.claim_retries})", flush=True)
    dev.free(desc)
ref = (w.float() @ x.float())
print("max rel err", ((y - ref).abs().max() / ref.abs().max()).item())
