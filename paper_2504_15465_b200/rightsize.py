"""Hardware right-sizing sweep on measured per-TPC scaling curves
(BASELINE.json config #4).

For each atomized body the tenant kernel runs as ONE atom on TPCs 0..t-1 of
the persistent dispatcher (batch mode) for t over a grid up to all 74 TPCs;
the latency is the atom's device span (first block start .. last block end,
%globaltimer, from its completion record), median of `reps` runs. Then the
reference's right-sizer runs on those measurements, through the library's
C ABI (the same functions the gpuos:: Rightsizer calls):

  fit  = fit_scaling(l(1), l(74), 74)                  rightsizer.cpp:8-19
  t*   = choose_tpcs_wave(fit, 74, slip, blocks, occ)  rightsizer.cpp:40-60
  R^2 of the fit over every measured t                 rightsizer.cpp:105-119

and l(t*) is measured to report the real slowdown against the full width and
the capacity saved (1 - t*/74). Beside it, the B200 measured-curve chooser
(RightsizerConfig::plateau, the live scheduler's mode) runs its search on
the same body: from l(74) and l(1) it bisects the width, measuring what it
asks for, and picks the narrowest measured width within the slip of l(74)
-- HBM-bound bodies, whose latency stops falling once enough TPCs saturate
the memory system, get the width where the plateau starts instead of 74. occ = blocks a TPC advances at once: 2W
worker slots for 1-SM bodies (STREAM); 1 for pair bodies (GEMM, GEMV): a
TPC has one pair of tensor cores, which its W pairs share.

    python -m paper_2504_15465_b200.rightsize [--slip 1.04] [--quick]
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
from typing import Any, Callable

from . import api

FULL = 74
GRID = [1, 2, 4, 8, 12, 16, 24, 32, 40, 48, 56, 64, 74]
GRID_QUICK = [1, 4, 16, 37, 74]


def r_squared(m: float, b: float, points: list[tuple[int, float]]) -> float:
    """Coefficient of determination of l = m / t + b over measured points
    (restates rightsizer.cpp:105-119 exactly, including its degenerate cases)."""
    if len(points) < 2:
        raise ValueError("r_squared needs >= 2 points")
    mean = sum(l for _, l in points) / len(points)
    ss_res = sum((l - (m / t + b)) ** 2 for t, l in points)
    ss_tot = sum((l - mean) ** 2 for _, l in points)
    if ss_tot == 0.0:
        return 1.0 if ss_res == 0.0 else -ss_res
    return 1.0 - ss_res / ss_tot


class Body:
    """A tenant kernel: its descriptor args, grid and per-TPC slot count."""

    def __init__(self, name: str, kind: int, args: list[int], blocks: int, occ: int,
                 work: str, reset: Callable[[], None] | None = None):
        self.name, self.kind, self.args, self.blocks, self.occ = name, kind, args, blocks, occ
        self.work = work
        self.reset = reset


def atom_latency_ns(dev: api.Device, body: Body, t: int, reps: int) -> float:
    spans = []
    for _ in range(reps):
        if body.reset:
            body.reset()
        dev.run_batch([api.Device.desc(0, body.blocks, range(t), 20, body.kind, body.args)])
        done = []
        while not done:
            done = dev.poll()
        c = done[0]
        spans.append(c.dev_last_end_ns - c.dev_first_start_ns)
    return float(statistics.median(spans))


def default_bodies(dev: api.Device, torch, keep: list) -> list[Body]:
    """The config #4 mix: tensor-core GEMMs of several shapes, a decode GEMV
    and an HBM stream; operands random-initialised on the device."""
    W = dev.topology.workers_per_sm
    out = []

    def bf16(*shape):
        x = (torch.rand(*shape, device="cuda") * 2 - 1).to(torch.bfloat16)
        keep.append(x)
        return x

    for m, n, k in ((4096, 4096, 4096), (2048, 2048, 2048), (8192, 1024, 4096), (1024, 1024, 8192)):
        a, b = bf16(m, k), bf16(n, k)
        c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        keep.append(c)
        desc, blocks, _, _ = dev.gemm_desc(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k,
                                           bf16_out=True)
        keep.append(("desc", desc))
        out.append(Body(f"gemm_bf16 {m}x{n}x{k}", api.GPUOS_BODY_GEMM_BF16, [desc], blocks, 1,
                        f"{2 * m * n * k / 1e9:.1f} GFLOP"))
    # ResNet-50 training-batch 3x3 convolutions (stage 2 and stage 3), NHWC
    for (cn, h, w_, c, kk) in ((64, 28, 28, 128, 128), (64, 14, 14, 256, 256)):
        x, wt = bf16(cn, h, w_, c), bf16(kk, 3, 3, c)
        yv = torch.empty(cn, h, w_, kk, device="cuda", dtype=torch.bfloat16)
        keep.append(yv)
        desc, blocks, P, Q = dev.conv_desc(x.data_ptr(), wt.data_ptr(), yv.data_ptr(), cn, h, w_, c, kk, 3, 3,
                                           1, 1, bf16_out=True)
        keep.append(("desc", desc))
        out.append(Body(f"conv_bf16 n{cn} {h}x{w_}x{c} k{kk} 3x3", api.GPUOS_BODY_CONV_BF16, [desc], blocks, 1,
                        f"{2 * cn * P * Q * kk * 9 * c / 1e9:.1f} GFLOP"))
    n, k = 28672, 4096  # Llama-3-8B gate+up projection at batch 1
    w, x = bf16(n, k), bf16(k)
    y = torch.zeros(n, device="cuda")
    keep.append(y)
    desc, blocks = dev.gemv_desc(w.data_ptr(), x.data_ptr(), y.data_ptr(), n, k, k_splits=4)
    keep.append(("desc", desc))
    out.append(Body(f"gemv_bf16 {n}x{k} (split-K 4)", api.GPUOS_BODY_GEMV_BF16, [desc], blocks, 1,
                    f"{n * k * 2 / 1e6:.0f} MB of W"))
    words = 256 * 1024  # 1 MiB per block in, 1 MiB out
    nblocks = 512
    src = torch.randint(-2**31, 2**31 - 1, (nblocks * words,), dtype=torch.int32, device="cuda")
    dst = torch.empty_like(src)
    keep += [src, dst]
    out.append(Body("stream 512 MiB", api.GPUOS_BODY_STREAM,
                    [src.data_ptr(), dst.data_ptr(), words, 7, 0], nblocks, 2 * W,
                    f"{nblocks * words * 8 / 1e6:.0f} MB moved"))
    return out


def sweep(device: int = 0, slip: float = 1.04, quick: bool = False, reps: int = 3,
          workers_per_sm: int = 2) -> dict[str, Any]:
    import torch

    grid = GRID_QUICK if quick else GRID
    keep: list = []
    rows = []
    with api.Device(device=device, workers_per_sm=workers_per_sm) as dev:
        bodies = default_bodies(dev, torch, keep)
        torch.cuda.synchronize()
        for body in bodies:
            lat = {t: atom_latency_ns(dev, body, t, reps) for t in grid}
            m, b, valid = api.fit_scaling(int(round(lat[1])), int(round(lat[FULL])), FULL)
            r2 = r_squared(m, b, sorted(lat.items())) if valid else None
            t_star = api.choose_tpcs_wave(m, b, valid, FULL, slip, body.blocks, body.occ)
            if t_star not in lat:
                lat[t_star] = atom_latency_ns(dev, body, t_star, reps)
            # The live scheduler's measured-curve search (RightsizerConfig::
            # plateau), run on this body: starting from the full-width and
            # one-TPC probes, measure the width it asks for until it converges.
            seen = {FULL: lat[FULL], 1: lat[1]}
            probes = []
            while True:
                t_b200, probe = api.choose_measured(seen, slip)
                if probe == 0 or len(probes) >= 8:
                    break
                if probe not in lat:
                    lat[probe] = atom_latency_ns(dev, body, probe, reps)
                seen[probe] = lat[probe]
                probes.append(probe)
            rows.append({
                "body": body.name, "work": body.work, "blocks": body.blocks, "occ": body.occ,
                "latency_us": {str(t): round(v / 1e3, 2) for t, v in sorted(lat.items())},
                "fit": {"m_us": m / 1e3, "b_us": b / 1e3, "valid": valid},
                "r2": r2, "t_star": t_star,
                "slowdown": lat[t_star] / lat[FULL],
                "capacity_savings": 1.0 - t_star / FULL,
                "b200": {"probes": probes,
                         "t_star": t_b200, "slowdown": lat[t_b200] / lat[FULL],
                         "capacity_savings": 1.0 - t_b200 / FULL},
            })
        for item in keep:
            if isinstance(item, tuple):
                dev.free(item[1])
    # Execution-time-weighted R^2 over bodies, as Rightsizer::weighted_r_squared
    # (rightsizer.cpp:121-139): weight = total measured latency of the body.
    def exec_time(r):
        return sum(r["latency_us"].values())

    wsum = sum(exec_time(r) for r in rows if r["r2"] is not None)
    return {
        "slip": slip, "grid": grid, "reps": reps, "bodies": rows,
        "mean_capacity_savings": statistics.mean(r["capacity_savings"] for r in rows),
        "max_slowdown": max(r["slowdown"] for r in rows),
        "b200_mean_capacity_savings": statistics.mean(r["b200"]["capacity_savings"] for r in rows),
        "b200_max_slowdown": max(r["b200"]["slowdown"] for r in rows),
        "weighted_r2": (sum(r["r2"] * exec_time(r) for r in rows if r["r2"] is not None) / wsum)
        if wsum else None,
    }


def main(argv: list[str] | None = None) -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--slip", type=float, default=1.04)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--device", type=int, default=0)
    args = ap.parse_args(argv)
    json.dump(sweep(args.device, args.slip, args.quick, args.reps), sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
