"""Decode GEMV beside best-effort tensor work on the same TPCs: device time
of one GEMV atom (armed -> last block end) on all 74 TPCs, alone and with a
background of conv / GEMM pair tiles (priority 20) keeping every TPC busy,
and with a background of 1-SM SPIN blocks.

    python tools/corun_probe.py [--reps 40]
"""
from __future__ import annotations

import argparse
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2504_15465_b200 import api  # noqa: E402

ALL = list(range(74))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=40)
    ap.add_argument("--shape", default="6144,4096,6")
    ap.add_argument("--only", default="none,conv,gemm,spin")
    ap.add_argument("--timing", action="store_true", help="per-block stamps (GemvDesc::timing)")
    ap.add_argument("--gemv-tpcs", default="0-73")
    ap.add_argument("--workers", type=int, default=2)
    ap.add_argument("--packed", action="store_true", help="W pre-packed (GPUOS_GEMV_W_PACKED)")
    ap.add_argument("--bg-tpcs", default="0-73")
    args = ap.parse_args()
    n, k, splits = (int(x) for x in args.shape.split(","))
    rng = lambda r: list(range(int(r.split("-")[0]), int(r.split("-")[1]) + 1))  # noqa: E731
    gt, bt = rng(args.gemv_tpcs), rng(args.bg_tpcs)
    g = torch.Generator(device="cuda").manual_seed(1)
    w = (torch.rand(n, k, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    x = (torch.rand(k, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    y = torch.zeros(n, device="cuda")
    # ResNet-50 stage-2 conv at batch 256 (the training tenant's shape class)
    cn, ch, cw, cc, ck = 256, 28, 28, 256, 256
    X = (torch.rand(cn, ch, cw, cc, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    Wc = (torch.rand(ck, 3, 3, cc, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    Y = torch.zeros(cn, ch, cw, ck, device="cuda", dtype=torch.bfloat16)
    A = (torch.rand(8192, 4096, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    B = (torch.rand(4096, 4096, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    Cm = torch.zeros(8192, 4096, device="cuda", dtype=torch.bfloat16)
    torch.cuda.synchronize()
    ref = w.cpu().double() @ x.cpu().double()
    with api.Device(workers_per_sm=args.workers) as dev:
        wsrc = w
        if args.packed:
            wsrc = torch.empty(dev.gemv_packed_bytes(n, k) // 2, device="cuda", dtype=torch.bfloat16)
            dev.gemv_pack(wsrc.data_ptr(), w.data_ptr(), n, k)
        gd, gblocks = dev.gemv_desc(wsrc.data_ptr(), x.data_ptr(), y.data_ptr(), n, k, k_splits=splits,
                                    packed=args.packed)
        cd, cblocks, _, _ = dev.conv_desc(X.data_ptr(), Wc.data_ptr(), Y.data_ptr(), cn, ch, cw, cc, ck, 3, 3, 1, 1,
                                          bf16_out=True)
        md, mblocks, _, _ = dev.gemm_desc(A.data_ptr(), B.data_ptr(), Cm.data_ptr(), 8192, 4096, 4096, bf16_out=True)
        bgs = {"none": None, "conv": (api.GPUOS_BODY_CONV_BF16, [cd], cblocks),
               "gemm": (api.GPUOS_BODY_GEMM_BF16, [md], mblocks),
               "spin": (api.GPUOS_BODY_SPIN, [20_000], 4 * 74 * 8)}
        stamps = torch.zeros(4 * gblocks, dtype=torch.int64, device="cuda")
        if args.timing:
            import ctypes
            ptr = ctypes.c_uint64(stamps.data_ptr())
            dev._check(dev._lib.gpuos_dev_copy(dev._h, ctypes.c_void_p(gd + 312), ctypes.byref(ptr), 8, 1))
        dev.start()
        for name in args.only.split(","):
            bg = bgs[name]
            phases = []
            bg_live: set[int] = set()
            spans, totals = [], []
            for rep in range(args.reps + 3):
                if bg is not None:
                    while len(bg_live) < 2:
                        bg_live.add(dev.submit(0, bg[2], bt, 20, bg[0], bg[1], tag=1))
                    time.sleep(0.0003)
                aid = dev.submit(0, gblocks, gt, 30, api.GPUOS_BODY_GEMV_BF16, [gd], tag=2)
                got = None
                while got is None:
                    for c in dev.poll():
                        if c.atom_id == aid:
                            got = c
                        else:
                            bg_live.discard(c.atom_id)
                if rep >= 3 and args.timing:
                    t = stamps.view(gblocks, 4).cpu().double()
                    t0 = t[:, 0].min()
                    phases.append([(t[:, 0].max() - t0).item(), (t[:, 1] - t[:, 0]).median().item(),
                                   (t[:, 2] - t[:, 1]).median().item(), (t[:, 3] - t[:, 2]).median().item(),
                                   (t[:, 3].max() - t0).item(), (got.dev_first_start_ns - got.dev_armed_ns)])
                if rep >= 3:
                    spans.append((got.dev_last_end_ns - got.dev_first_start_ns) / 1e3)
                    totals.append((got.dev_last_end_ns - got.dev_armed_ns) / 1e3)
            while bg_live:
                for c in dev.poll():
                    bg_live.discard(c.atom_id)
            # (CPU check: no kernel runs beside the resident dispatcher)
            err = ((y.cpu().double() - ref).abs().max() / ref.abs().max()).item()
            assert err < 1e-3, err
            gb = n * k * 2 / 1e3
            print(f"{name:5s} W{args.workers} {'packed ' if args.packed else ''}tpcs {args.gemv_tpcs} bg {args.bg_tpcs} gemv {n}x{k}/{splits} ({gblocks} blocks): armed->end p50 {statistics.median(totals):7.2f} us"
                  f" ({gb / statistics.median(totals):6.0f} GB/s)  span p50 {statistics.median(spans):7.2f} us"
                  f"  p90 {sorted(totals)[int(0.9 * len(totals))]:7.2f}", flush=True)
            if phases:
                med = [statistics.median(p[i] for p in phases) / 1e3 for i in range(6)]
                print(f"      armed->first {med[5]:6.2f} | start skew {med[0]:6.2f}  first load {med[1]:6.2f}"
                      f"  stream {med[2]:6.2f}  epilogue+reduce {med[3]:6.2f}  first start->last end {med[4]:6.2f} us",
                      flush=True)
        dev.stop()
        for d in (gd, cd, md):
            dev.free(d)


if __name__ == "__main__":
    main()
