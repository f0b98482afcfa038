"""Batch-mode latency of GEMM shapes (optionally split-K) on t TPCs.

    python tools/gemm_shapes.py "M,N,K,splits" ... [--tpcs 37,74]"""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_15465_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("shapes", nargs="+")
ap.add_argument("--tpcs", default="37,74")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
with api.Device() as dev:
    for sh in args.shapes:
        m, n, k, sp = (int(x) for x in sh.split(","))
        a = (torch.rand(m, k, device="cuda") * 2 - 1).to(torch.bfloat16)
        b = (torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16)
        c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        torch.cuda.synchronize()
        desc, blocks, tm, tn = dev.gemm_desc(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, bf16_out=True,
                                             k_splits=sp)
        for t in (int(x) for x in args.tpcs.split(",")):
            best = 1e9
            for _ in range(args.reps):
                dev.run_batch([api.Device.desc(0, blocks, range(t), 20, api.GPUOS_BODY_GEMM_BF16, [desc])])
                done = []
                while not done:
                    done = dev.poll()
                best = min(best, (done[0].dev_last_end_ns - done[0].dev_first_start_ns) / 1e3)
            byts = 2 * (m * k + n * k + m * n)
            print(f"{m}x{n}x{k} splits {sp} blocks {blocks} tile {tm}x{tn} t={t}: {best:.1f} us, "
                  f"{2 * m * n * k / best / 1e6:.0f} TF/s, {byts / best / 1e3:.0f} GB/s", flush=True)
        dev.free(desc)
        del a, b, c
