"""First GPU run of the dispatcher: device-level checks, a replay mirror of
fig7, and a live time-scaled fig7. Prints one JSON object per stage.
Run under gpurun with a timeout; every stage has its own bounded wait."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_15465_b200 import api  # noqa: E402


def stream_expect(src: np.ndarray, salt: int, base: int) -> np.ndarray:
    idx = (np.arange(src.size, dtype=np.uint64) + np.uint64(base)).astype(np.uint32)
    return ((src ^ np.uint32(salt)) * np.uint32(0x9E3779B1) + idx).astype(np.uint32)


def stage_device():
    with api.Device(workers_per_sm=2) as dev:
        return _stage_device(dev)


def _stage_device(dev):
    out = {}
    topo = dev.topology
    out["topology"] = {f: getattr(topo, f) for f, _ in topo._fields_}
    words, blocks = 4096, 2000
    src = torch.randint(0, 2**31 - 1, (blocks * words,), dtype=torch.int64, device="cuda").to(torch.int32)
    dst = torch.zeros_like(src)
    trace = torch.zeros(blocks, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    dev.start()
    t0 = time.time()
    salt = 0x1234567
    # Three atoms on overlapping TPC sets at different priorities.
    ranges = [(0, 700, list(range(0, 10)), 20), (700, 1500, list(range(5, 40)), 30),
              (1500, 2000, [70, 71, 72, 73], 10)]
    ids = []
    for lo, hi, tpcs, prio in ranges:
        ids.append(dev.submit(lo, hi, tpcs, prio, api.GPUOS_BODY_STREAM,
                              [src.data_ptr(), dst.data_ptr(), words, salt, 0], tag=prio,
                              trace=trace.data_ptr()))
    done = []
    while len(done) < len(ids) and time.time() - t0 < 20:
        done += dev.poll()
    ms = dev.stop(drain=True)
    out["completions"] = len(done)
    out["kernel_ms"] = ms
    tr = trace.cpu().numpy().astype(np.uint32)
    counts = tr >> 16
    sm = (tr & 0xFFFF).astype(np.int64) - 1
    misplaced = 0
    for lo, hi, tpcs, _ in ranges:
        allowed = set(tpcs)
        misplaced += int(sum(1 for b in range(lo, hi) if (sm[b] >> 1) not in allowed))
    out["exactly_once"] = bool((counts == 1).all())
    out["misplaced"] = misplaced
    exp = stream_expect(src.cpu().numpy().view(np.uint32), salt, 0)
    out["bit_exact"] = bool((dst.cpu().numpy().view(np.uint32) == exp).all())
    out["atoms"] = [{"id": c.atom_id, "blocks": c.blocks, "tag": c.tag,
                     "host_lat_us": (c.host_complete_ns - c.host_submit_ns) / 1e3,
                     "dev_us": (c.dev_last_end_ns - c.dev_first_start_ns) / 1e3,
                     "touched": bin(c.tpc_touched[0]).count("1") + bin(c.tpc_touched[1]).count("1")}
                    for c in done]
    # Bandwidth: one big atom over all TPCs, drained, CUDA-event timed.
    words2, blocks2 = 65536, 4096  # 256 KiB per block, 1 GiB per buffer
    src2 = torch.randint(0, 2**31 - 1, (blocks2 * words2,), dtype=torch.int32, device="cuda")
    dst2 = torch.zeros_like(src2)
    torch.cuda.synchronize()
    bw = []
    for rep in range(3):
        dev.start()
        dev.submit(0, blocks2, list(range(topo.logical_tpcs)), 20, api.GPUOS_BODY_STREAM,
                   [src2.data_ptr(), dst2.data_ptr(), words2, salt, 0])
        ms = dev.stop(drain=True)
        dev.poll()
        bw.append(blocks2 * words2 * 8 / (ms * 1e-3) / 1e9)
    out["stream_GBps_event"] = bw
    # Spin atoms: dispatch overhead (device side), N one-block atoms back to back.
    dev.start()
    t0 = time.time()
    n = 2000
    got = 0
    sub = 0
    while got < n and time.time() - t0 < 20:
        if sub < n and dev.in_flight() < 16:
            dev.submit(0, 1, [0], 20, api.GPUOS_BODY_SPIN, [1000, 0, 0, 0, 0])
            sub += 1
        got += len(dev.poll())
    wall = time.time() - t0
    dev.stop(drain=True)
    while dev.in_flight():
        dev.poll()
    out["spin_1us_atoms_per_s_pipelined16"] = got / wall
    # Serial round trip: submit, wait, repeat.
    dev.start()
    lat = []
    for i in range(300):
        t1 = dev.now_ns()
        dev.submit(0, 1, [1], 20, api.GPUOS_BODY_SPIN, [0, 0, 0, 0, 0])
        while True:
            c = dev.poll()
            if c:
                break
        lat.append(dev.now_ns() - t1)
    dev.stop(drain=True)
    lat = np.array(lat[20:]) / 1e3
    out["serial_roundtrip_us"] = {"p50": float(np.median(lat)), "p90": float(np.percentile(lat, 90)),
                                  "p99": float(np.percentile(lat, 99))}
    return out


def stage_mirror():
    r = api.run({"scenario": {"preset": "fig7"}, "backend": "mirror", "horizon_ms": 1000,
                 "b200": {"min_words": 256, "words_per_us": 0.0, "chunk_cap": 64}})
    return {"verify": r["verify"], "gpu_atoms": r["gpu_atoms"], "gpu_kernel_ms": r["gpu_kernel_ms"],
            "atoms": r["atoms"]}


def stage_live():
    req = {"scenario": {"preset": "fig7"}, "backend": "b200", "device": "b200",
           "quota_scale": 74 / 54, "time_scale": 10.0, "horizon_ms": 2000,
           "b200": {"chunk_cap": 64}}
    s = api.Session(req)
    res = []
    for i in range(2):
        t0 = time.time()
        r = s.run()
        r["py_wall_s"] = time.time() - t0
        apps = r["report"]["apps"]
        res.append({"apps": [{k: a[k] for k in ("app_id", "completed", "offered", "p50_ns", "p99_ns")} for a in apps],
                    "atoms": r["atoms"], "b200": r["b200"], "util": r["report"]["tpc_utilization"],
                    "py_wall_s": r["py_wall_s"]})
    s.close()
    return res


if __name__ == "__main__":
    for name in sys.argv[1:] or ["device", "mirror", "live"]:
        t0 = time.time()
        try:
            res = globals()["stage_" + name]()
            print(json.dumps({"stage": name, "ok": True, "s": time.time() - t0, "result": res}), flush=True)
        except Exception as e:  # report and continue with the next stage
            print(json.dumps({"stage": name, "ok": False, "error": repr(e)}), flush=True)
