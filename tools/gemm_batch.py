"""Batch-mode launches of the dispatcher's worker kernel executing a bf16
GEMM (C = A . B^T, tcgen05) atomized over all 74 TPCs; prints ms and
TFLOP/s per launch. Single self-contained launches, so ncu can replay them:

  ncu --set full --clock-control none --import-source on -k regex:k_worker \
      -s 2 -c 1 -o gpurun_out/prof_gemm python tools/gemm_batch.py 4096 4096 4096 3

usage: gemm_batch.py M N K [launches] [workers_per_sm] [atoms] [bf16_out]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_15465_b200 import api  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
workers = int(sys.argv[5]) if len(sys.argv) > 5 else 2
n_atoms = int(sys.argv[6]) if len(sys.argv) > 6 else 32
bf16_out = len(sys.argv) > 7 and sys.argv[7] == "1"
a = (torch.rand(m, k, device="cuda") * 2 - 1).to(torch.bfloat16)
b = (torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16)
c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16 if bf16_out else torch.float32)
torch.cuda.synchronize()
with api.Device(workers_per_sm=workers) as dev:
    desc, blocks, tm, tn = dev.gemm_desc(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k,
                                         bf16_out=bf16_out)
    n_atoms = min(n_atoms, blocks)
    descs = [api.Device.desc(i * blocks // n_atoms, (i + 1) * blocks // n_atoms, range(74), 20,
                             api.GPUOS_BODY_GEMM_BF16, [desc]) for i in range(n_atoms)]
    for _ in range(reps):
        ms = dev.run_batch(descs)
        while dev.in_flight():
            dev.poll()
        st = dev.stats()
        print(f"gemm {m}x{n}x{k} W={workers} tiles {tm}x{tn} ({blocks}) atoms {n_atoms}: "
              f"{ms:.3f} ms, {2 * m * n * k / ms / 1e9:.0f} TFLOP/s "
              f"(device span {st.worker_span_ns / 1e3:.1f} us, first block after "
              f"{st.first_block_ns / 1e3:.1f} us)", flush=True)
    dev.free(desc)
