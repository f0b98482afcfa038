"""Device gaps inside a chain: a decode-shaped GEMV on all 74 TPCs followed
by a one-block kernel, repeated. Median gap GEMV last end -> one-block first
start (and back), with the one-block kernel's TPC set one TPC or all TPCs
(the latter lets the GEMV's finisher run it at once), against a chain of
one-block kernels on one TPC.

    python tools/chain_gap_probe.py [--n 200]
"""
from __future__ import annotations

import argparse
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_15465_b200 import api  # noqa: E402

ALL = list(range(74))


def run_chain(dev, kinds, n, batch=False):
    if batch:
        # Every link in place before the dispatcher starts serving it (atom
        # ids of a batch are consecutive from the handle's next id).
        out = []
        for r in range(0, n, 24):
            dev.run_batch([api.Device.desc(0, 1, [0], 30, api.GPUOS_BODY_SPIN, [0])])
            (c,) = wait(dev, 1)
            base = c.atom_id + 1
            descs = []
            for i in range(min(24, n - r)):
                lo_hi, tpcs, body, args = kinds[i % len(kinds)]
                descs.append(api.Device.desc(0, lo_hi, tpcs, 30, body, args, chain_head=True))
                if i:
                    descs[-1].after = base + i - 1 + 1
            dev.run_batch(descs)
            got = {c.atom_id: c for c in wait(dev, len(descs))}
            out += [got[base + i] for i in range(len(descs))]
        return out
    ids, done = [], []
    for i in range(n):
        while len(ids) - len(done) >= 20:
            done += dev.poll()
        lo_hi, tpcs, body, args = kinds[i % len(kinds)]
        ids.append(dev.submit(0, lo_hi, tpcs, 30, body, args, after=ids[-1] if ids else None, chain_head=True))
    while len(done) < n:
        done += dev.poll()
    by = {c.atom_id: c for c in done}
    return [by[i] for i in ids]


def probe_rows(dev):
    """(count, rows) of the GPUOS_PROBE_HANDOFF ring, or None in a normal build."""
    import ctypes as C
    import numpy as np
    fn = getattr(dev._lib, "gpuos_dev_probe_read", None)
    if fn is None:
        return None
    buf = np.zeros((4096, 12), dtype=np.uint64)
    n = C.c_uint()
    fn(C.c_void_p(buf.ctypes.data), C.byref(n))
    return n.value, buf


STAMPS = ["body end", "acct start", "fields", "exch", "succ loaded", "armed", "pre-flush", "flushed",
          "acct end", "loop top", "t_start"]
ORDER = [10, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9]


def wait(dev, n):
    got = []
    while len(got) < n:
        got += dev.poll()
    return got


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200)
    ap.add_argument("--shape", default="4096,4096,4")
    args = ap.parse_args()
    n, k, splits = (int(x) for x in args.shape.split(","))
    g = torch.Generator(device="cuda").manual_seed(1)
    w = (torch.rand(n, k, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    x = (torch.rand(k, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    y = torch.zeros(n, device="cuda")
    torch.cuda.synchronize()
    with api.Device(workers_per_sm=2) as dev:
        gd, gblocks = dev.gemv_desc(w.data_ptr(), x.data_ptr(), y.data_ptr(), n, k, k_splits=splits)
        dev.start()
        spin = lambda tp: (1, tp, api.GPUOS_BODY_SPIN, [1000])  # noqa: E731
        gemv = (gblocks, ALL, api.GPUOS_BODY_GEMV_BF16, [gd])
        cases = {"spin->spin tpc3": [spin([3])],
                 "gemv->spin tpc3": [gemv, spin([3])],
                 "gemv->spin all": [gemv, spin(ALL)],
                 "gemv->gemv": [gemv]}
        prev = probe_rows(dev)
        running = True
        for (name, kinds), batch in [(c, b) for b in (False, True) for c in cases.items()]:
            if batch:
                name += " batch"
                if running:
                    dev.stop()
                    running = False
            else:
                run_chain(dev, kinds, 40)  # warm
            cs = run_chain(dev, kinds, args.n, batch)
            gaps = {}
            for a, b in zip(cs, cs[1:]):
                key = ("G" if a.blocks > 1 else "s") + ">" + ("G" if b.blocks > 1 else "s")
                gaps.setdefault(key, []).append((b.dev_first_start_ns - a.dev_last_end_ns) / 1e3)
            spans = {}
            for c in cs:
                spans.setdefault("G" if c.blocks > 1 else "s", []).append(
                    (c.dev_last_end_ns - c.dev_first_start_ns) / 1e3)
            txt = "  ".join(f"gap {kk} p50 {statistics.median(v):6.2f} p90 {sorted(v)[int(0.9 * len(v))]:6.2f}"
                            for kk, v in sorted(gaps.items()))
            txt += "  " + "  ".join(f"span {kk} p50 {statistics.median(v):6.2f}" for kk, v in sorted(spans.items()))
            print(f"{name:24s} {txt}", flush=True)
            cur = probe_rows(dev)
            if cur is not None:
                n0, n1 = prev[0], cur[0]
                rows = cur[1][[i & 4095 for i in range(n0, n1)]].astype("int64") if n1 > n0 else []
                prev = cur
                full = [r for r in rows if all(r[i] != 0 for i in (0, 2, 3, 4, 5, 6, 7, 8, 9, 10))]
                if full:
                    import numpy as np
                    segs = []
                    for a, b in zip(ORDER, ORDER[1:]):
                        d = [int(r[b] - r[a]) for r in full if r[a] and r[b]]
                        if d:
                            segs.append(f"{STAMPS[ORDER.index(a)]}->{STAMPS[ORDER.index(b)]} {np.median(d):.0f}")
                    print(f"    handoffs {len(full)} (SM cycles, median): " + " | ".join(segs), flush=True)
        dev.free(gd)


if __name__ == "__main__":
    main()
