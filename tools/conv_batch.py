"""Batch-mode launches of the worker kernel executing an NHWC implicit-GEMM
convolution (tcgen05 pair tiles, TMA im2col loads per filter tap) atomized over
all 74 TPCs; prints ms and TFLOP/s (algorithmic: 2 N P Q K R S C).

usage: conv_batch.py N H W C K R S pad stride [launches] [atoms]"""
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
    n_atoms = min(int(sys.argv[11]) if len(sys.argv) > 11 else 32, blocks)
    timing = len(sys.argv) > 12 and sys.argv[12] == "timing"
    stamps = torch.zeros(4 * blocks, dtype=torch.int64, device="cuda")
    trace = torch.zeros(blocks, dtype=torch.int32, device="cuda")
    if timing:  # ConvDesc::timing (offset 336): 4 stamps per tile
        import ctypes
        ptr = ctypes.c_uint64(stamps.data_ptr())
        dev._check(dev._lib.gpuos_dev_copy(dev._h, ctypes.c_void_p(desc + 336), ctypes.byref(ptr), 8, 1))
    descs = [api.Device.desc(i * blocks // n_atoms, (i + 1) * blocks // n_atoms, range(74), 20,
                             api.GPUOS_BODY_CONV_BF16, [desc], trace=trace.data_ptr() if timing else None)
             for i in range(n_atoms)]
    flops = 2.0 * n * P * Q * k * r * s * c
    for _ in range(reps):
        ms = dev.run_batch(descs)
        while dev.in_flight():
            dev.poll()
        st = dev.stats()
        print(f"conv n{n} {h}x{w}x{c} -> {P}x{Q}x{k} {r}x{s}/{stride} ({blocks} blocks): {ms:.3f} ms, "
              f"{flops / ms / 1e9:.0f} TFLOP/s (device span {st.worker_span_ns / 1e3:.1f} us: "
              f"{flops / st.worker_span_ns / 1e3:.0f} TFLOP/s)", flush=True)
    if timing:
        # per tile: fill (start -> first MMA), main loop (-> accumulator
        # ready), epilogue (-> end); per TPC: share of the span during which
        # at least one of its pairs is in a main loop.
        t = stamps.view(blocks, 4).cpu().double()
        tpc = ((trace.cpu().numpy().view("uint32") & 0xFFFF).astype("int64") - 1) >> 1
        t0 = t[:, 0].min().item()
        span = t[:, 3].max().item() - t0
        fill, main, epi = (t[:, 1] - t[:, 0]), (t[:, 2] - t[:, 1]), (t[:, 3] - t[:, 2])
        cover = []
        for tp in range(74):
            iv = sorted((t[i, 1].item(), t[i, 2].item()) for i in range(blocks) if tpc[i] == tp)
            tot, cur = 0.0, None
            for a, b in iv:
                if cur is None or a > cur[1]:
                    if cur: tot += cur[1] - cur[0]
                    cur = [a, b]
                else:
                    cur[1] = max(cur[1], b)
            if cur: tot += cur[1] - cur[0]
            cover.append(tot / span)
        gaps = []
        for tp in range(74):  # tile start after the previous tile end on the same TPC (either pair)
            ends = sorted(t[i, 3].item() for i in range(blocks) if tpc[i] == tp)
            starts = sorted(t[i, 0].item() for i in range(blocks) if tpc[i] == tp)
        print(f"span {span / 1e3:.1f} us; per tile median: fill {fill.median() / 1e3:.2f} us, main loop "
              f"{main.median() / 1e3:.2f} us (p10 {main.quantile(0.1) / 1e3:.2f}, p90 {main.quantile(0.9) / 1e3:.2f}),"
              f" epilogue {epi.median() / 1e3:.2f} us; tiles per TPC {blocks / 74:.1f}; TPC main-loop coverage "
              f"mean {sum(cover) / 74:.3f} min {min(cover):.3f}; first tile start skew "
              f"{(t[:, 0].kthvalue(min(148, blocks)).values.item() - t0) / 1e3:.1f} us", flush=True)
    dev.free(desc)
