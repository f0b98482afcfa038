"""Benchmark: LC p99 latency + BE atoms/s per B200 under stacking, with the
HBM roofline of the dispatcher kernel (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--time-scale 10] [--horizon-ms 10000]

Workload (config.workload): BASELINE.json config #1, the SPEC two-tenant
trace = the reference's Figure-7 preset (one bursty LC tenant + one
backlogged BE tenant), mapped onto the B200's 74 TPCs and time-scaled
(paper_2504_15465_b200/workloads.py). The SAME scenario JSON drives both
arms. A step = one complete scenario run (all arrivals over the horizon,
drained) on the live persistent dispatcher.

ours:      gpuos:: scheduler (C++) -> C ABI -> persistent sm_100a dispatcher;
           value = BE atoms completed / device time (CUDA events around the
           dispatcher kernel, summed over steps, max over ranks).
           e2e = same metric through the C-ABI session call with host
           buffers: tenant inputs copied H2D from pinned memory before each
           step and an output digest read back D2H after it, wall clock.
reference: the UNMODIFIED reference simulator (oracle/_ref/ref_bench, built
           from /root/reference) on the box's host cores (rank 0 only),
           same scenario JSON; value = BE atoms completed / wall second.
Multi-GPU: replicas only (no collective on this path): each
rank runs its own tenant set; atoms summed, time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2504_15465_b200 import replicas, workloads  # noqa: E402

METRIC = "LC p99 latency + BE atoms/sec per B200 under stacking; HBM/TC roofline %"


def peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        p = json.load(open(path))
        return {"hbm_gbs": p["hbm_gbs"], "bf16_tflops": p["bf16_tflops"], "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


def nearest_rank(samples, p):
    s = sorted(samples)
    if not s:
        return None
    import math

    return s[max(1, math.ceil(p / 100.0 * len(s))) - 1]


def be_blocks_of(result) -> int:
    flags = [a["high_priority"] for a in result["report"]["apps"]]
    return sum(b for b, hp in zip(result["blocks_per_app"], flags) if not hp)


def hp_latencies_us(result) -> list[float]:
    out = []
    hp_ids = {a["app_id"] for a in result["report"]["apps"] if a["high_priority"]}
    for line in result["request_log"].splitlines():
        j = json.loads(line)
        if j["app"] in hp_ids and j["completed"]:
            out.append(j["latency_us"])
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in self.rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(self.rows[0][1]), "reasons": reasons,
                "samples": len(self.rows)}


def dist_init():
    r = replicas.init_from_env("gloo")
    return r.rank, r.world, r.local


def allreduce(values: list[float], op: str) -> list[float]:
    return replicas.reduce(values, op)


def barrier():
    replicas.barrier()


def reference_arm(args, cfgs: list[dict], rank: int, world: int) -> None:
    """The unmodified reference on this box's host cores (rank 0 only): every
    rank's scenario, each as parallel replicas over an equal share of cores;
    each step a bounded ~5 s sample."""
    if rank != 0:
        return
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    if not os.path.exists(exe) and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    if not os.path.exists(exe):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_bench not built"}))
        return
    for _ in range(args.warmup):
        cpu_baseline(cfgs, seconds=0.0)
    steps = [cpu_baseline(cfgs, seconds=args.sample_s) for _ in range(args.steps)]
    be = sum(s["value"] * s["wall_s"] for s in steps)
    wall = sum(s["wall_s"] for s in steps)
    value = be / wall
    cb = dict(steps[-1], value=value, wall_s=wall)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "BE atoms/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": bench_config(cfgs[0], args, world),
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "BE atoms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def host_cores() -> int:
    """Cores this process may run on (the affinity mask, not the machine)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def bench_config(cfg: dict, args, world: int) -> dict:
    """The `config` object both arms print (identical dicts: same scenario,
    same replica layout)."""
    return {"workload": cfg["name"] + (" (BASELINE config #5, per GPU)" if args.workload == "box8"
                                       else " (BASELINE config #1)"),
            "tenants": [a["id"] + (" (LC)" if a["priority"] == "hp" else " (BE)") for a in cfg["apps"]],
            "tpcs": 74, "time_scale": args.time_scale, "horizon_ms": cfg["horizon_ms"],
            "l2": "inputs larger than L2 (STREAM workspaces >> 126 MB)",
            "parallelism": f"replicas x{world}"}


def cpu_baseline(cfgs: list[dict], cores: int | None = None, seconds: float = 10.0) -> dict:
    """Bounded sample of the reference on this box's host (rank 0, N=1): the
    compiled reference simulator (oracle/_ref/ref_bench) on the same
    scenario(s), `cores` independent replicas in parallel (one per core)."""
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    if not os.path.exists(exe):
        return {"value": None, "unit": "BE atoms/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}
    cores = cores or host_cores()
    per = max(1, cores // len(cfgs))
    paths = []
    for c in cfgs:
        with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
            json.dump(c, f)
            paths.append(f.name)

    def run(reps):
        procs = [subprocess.Popen([exe, "--config", p, "--threads", str(per), "--reps", str(reps)],
                                  stdout=subprocess.PIPE, text=True) for p in paths]
        outs = [json.loads(p.communicate()[0]) for p in procs]
        return {"be_atoms": sum(o["be_atoms"] for o in outs), "wall_s": max(o["wall_s"] for o in outs),
                "hp_p99_ns": max(o["hp_p99_ns"] for o in outs)}

    one = run(1)
    reps = max(1, int(seconds / max(one["wall_s"], 1e-3)))
    r = run(reps)
    return {"value": r["be_atoms"] / r["wall_s"], "unit": "BE atoms/s", "cores": per * len(cfgs),
            "kind": "reference", "cpu_model": cpu_model(), "wall_s": r["wall_s"], "reps": reps,
            "sample": f"{reps} runs of each of {len(cfgs)} scenario(s) on each of {per} parallel "
                      f"replica threads ({r['wall_s']:.1f} s; reference discrete-event simulator, "
                      f"simulated LC p99 {r['hp_p99_ns'] / 1e6:.3f} ms)"}


def ours(args, cfg: dict, rank: int, world: int, local: int) -> None:
    import torch

    from paper_2504_15465_b200 import api

    torch.cuda.set_device(local)
    pk = peaks()
    # B200-native live mechanisms: block-granular revocation (fences + HP
    # preemption of best-effort TPCs), a preemption quantum of a quarter
    # atom (blocks run as independently claimed slices) and LC kernels
    # chained on the device (no host round trip between dependent kernels).
    quantum_us = 250.0 / args.time_scale
    b200 = {"device": local, "workers_per_sm": args.workers_per_sm, "chunk_cap": args.chunk_cap,
            "quantum_us": quantum_us}
    live_set = {"block_revocation": True, "chain_launches": True}
    sess = api.Session({"scenario": {"config": cfg}, "backend": "b200", "b200": b200,
                        "requests": True, "set": live_set})
    for _ in range(max(args.warmup, 1)):  # the first run creates the tenant workspaces
        sess.run()

    # ---- timed region: stacked LC + BE, device-timed
    barrier()
    steps = []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            steps.append(sess.run())
    barrier()
    dev_ms = sum(s["b200"]["kernel_ms"] for s in steps)
    be_atoms = sum(s["atoms"]["be"] for s in steps)
    be_blocks = sum(be_blocks_of(s) for s in steps)
    stream_bytes = sum(s["b200"]["stream_bytes"] for s in steps)
    lat = replicas.gather_samples(sum((hp_latencies_us(s) for s in steps), []))
    max_ms, = allreduce([dev_ms], "max")
    be_atoms_all, be_blocks_all = allreduce([float(be_atoms), float(be_blocks)], "sum")
    value = be_atoms_all / (max_ms * 1e-3)

    # ---- comparisons on the same device: LC alone, static partition
    alone_cfg = workloads.without_apps(cfg, *[a["id"] for a in cfg["apps"] if a["priority"] == "be"])
    static_cfg = workloads.variant(cfg, stealing=False, atomizer=False)
    alone = [sess.run(scenario={"config": alone_cfg}) for _ in range(args.steps)]
    static = [sess.run(scenario={"config": static_cfg}) for _ in range(args.steps)]
    # Ablation: the reference's semantics on the same dispatcher (atom-
    # boundary revocation, whole blocks).
    ref_sem = [sess.run(set={"block_revocation": False, "chain_launches": False},
                        b200=dict(b200, quantum_us=0.0))
               for _ in range(args.steps)]
    lat_alone = replicas.gather_samples(sum((hp_latencies_us(s) for s in alone), []))
    lat_ref_sem = replicas.gather_samples(sum((hp_latencies_us(s) for s in ref_sem), []))
    ref_sem_ms = sum(s["b200"]["kernel_ms"] for s in ref_sem)
    static_blocks = sum(be_blocks_of(s) for s in static)
    static_ms = sum(s["b200"]["kernel_ms"] for s in static)

    # ---- end to end through the C-ABI session call with host buffers
    barrier()
    e2e = [sess.run(e2e=True) for _ in range(args.steps)]
    barrier()
    e2e_s = sum(s["b200"]["e2e_wall_ns"] for s in e2e) * 1e-9
    e2e_atoms = sum(s["atoms"]["be"] for s in e2e)
    e2e_s_max, = allreduce([e2e_s], "max")
    e2e_atoms_all, = allreduce([float(e2e_atoms)], "sum")

    # ---- saturated roofline: the BE tenant's atomized kernel alone at full width
    sat = saturation(api, local, args)
    sat_tc = gemm_saturation(api, local, args)
    sat_gemv = guarded(lambda: gemv_saturation(api, local, args))
    sat_conv = guarded(lambda: conv_saturation(api, local, args))
    rsz = guarded(lambda: right_sizing_summary(local, args)) if rank == 0 else None
    cfgs = guarded(lambda: model_configs_isolated(local)) if (rank == 0 and not args.skip_configs) else None
    pols = guarded(lambda: policy_rows(local)) if (rank == 0 and not args.skip_configs) else None
    probe = api.probe_dispatch(device=local, workers_per_sm=args.workers_per_sm, serial=2000,
                               pipelined=20000, depth=16)

    if rank != 0:
        return
    lc_p99 = nearest_rank(lat, 99) / 1e3
    lc_alone = nearest_rank(lat_alone, 99) / 1e3
    achieved = stream_bytes / (dev_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "BE atoms/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (reference Figure-7 trace, time-scaled; STREAM bodies over seeded u32 workspaces)",
        "config": bench_config(cfg, args, world),
        "workers_per_sm": args.workers_per_sm,
        "lc_p99_ms": lc_p99, "lc_p99_alone_ms": lc_alone, "lc_p99_vs_alone": lc_p99 / lc_alone,
        "lc_slo_ms": cfg["apps"][0]["slo_ms"],
        "be_blocks_per_s": be_blocks_all / (max_ms * 1e-3),
        "be_blocks_per_s_static": static_blocks / (static_ms * 1e-3),
        "be_vs_static": (be_blocks / dev_ms) / (static_blocks / static_ms),
        "tpc_utilization": sum(s["report"]["tpc_utilization"] for s in steps) / len(steps),
        "live_mechanisms": {"block_revocation": True, "chain_launches": True, "quantum_us": quantum_us},
        "ablation_reference_semantics": {
            "lc_p99_ms": nearest_rank(lat_ref_sem, 99) / 1e3,
            "lc_p99_vs_alone": nearest_rank(lat_ref_sem, 99) / nearest_rank(lat_alone, 99),
            "be_atoms_per_s": sum(s["atoms"]["be"] for s in ref_sem) / (ref_sem_ms * 1e-3),
            "be_blocks_per_s": sum(be_blocks_of(s) for s in ref_sem) / (ref_sem_ms * 1e-3)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"], "traffic": live_traffic(),
                     "traffic_note": "DRAM read+write of one live k_worker launch of this scenario "
                                     "under ncu (profiles/ncu_traffic_r02.json); algorithmic bytes "
                                     "of that launch in traffic_algorithmic",
                     "traffic_algorithmic": live_traffic("algorithmic_bytes"),
                     "kernel": "k_worker (persistent dispatcher, stacked run, CUDA events)",
                     "peak_source": pk["source"]},
        "roofline_saturated": sat,
        "roofline_tensor": sat_tc,
        "roofline_gemv": sat_gemv,
        "roofline_conv": sat_conv,
        "right_sizing": rsz,
        "model_configs": cfgs,
        "policy_comparison": pols,
        "dispatcher_overhead": {
            "serial_roundtrip_us_p50": probe["serial_roundtrip_ns"]["p50"] / 1e3,
            "publish_to_first_block_us_p50": probe["publish_to_first_block_ns"]["p50"] / 1e3,
            "pipelined_ns_per_atom": probe["pipelined_ns_per_atom"],
            # publish -> first block split on the device clock: ring entry seen by
            # the ingest warp -> armed (slot, keys, wake-ups) -> first block start
            "ingest_to_armed_us_p50": probe["device_ingest_to_armed_ns_p50"] / 1e3,
            "armed_to_first_block_us_p50": probe["device_armed_to_first_block_ns_p50"] / 1e3,
            "publish_to_ingest_us_p50": probe["host_submit_to_device_ingest_ns_p50_offset_sensitive"] / 1e3,
            "last_block_to_host_us_p50": probe["last_block_to_host_ns"]["p50"] / 1e3,
            "note": "empty one-block atoms through the live ring (gpuos_probe_dispatch)"},
        "cpu_baseline": cpu_baseline([cfg]) if world == 1 else None,
        "e2e": {"value": e2e_atoms_all / e2e_s_max, "unit": "BE atoms/s",
                "h2d_bytes_per_step": e2e[0]["b200"]["h2d_bytes"],
                "d2h_bytes_per_step": e2e[0]["b200"]["d2h_bytes"]},
        "gpu_launches": args.steps,  # one self-contained k_worker launch per step
        "clocks": clocks.summary(),
    }
    print(json.dumps(line))


def saturation(api, local: int, args) -> dict:
    """k_worker executing the BE tenant's kernel shape atomized at full width,
    staged first so the CUDA events cover execution only."""
    import torch

    pk = peaks()
    words = (int(round(2000.0 / args.time_scale * 2750.0)) + 3) & ~3
    blocks = 2160 * 4
    chunks = 256
    src = torch.randint(-2**31, 2**31 - 1, (chunks * words,), dtype=torch.int32, device=f"cuda:{local}")
    dst = torch.empty_like(src)
    torch.cuda.synchronize()
    best = 0.0
    n_atoms = 32  # resident-list capacity per TPC
    per = blocks // n_atoms
    descs = [api.Device.desc(i * per, (i + 1) * per, range(74), 20, api.GPUOS_BODY_STREAM,
                             [src.data_ptr(), dst.data_ptr(), words, 7, chunks]) for i in range(n_atoms)]
    with api.Device(device=local, workers_per_sm=args.workers_per_sm) as dev:
        for _ in range(3):
            ms = dev.run_batch(descs)  # single k_worker launch, CUDA events
            while dev.in_flight():
                dev.poll()
            best = max(best, blocks * words * 8 / (ms * 1e-3) / 1e9)
    return {"bound": "hbm", "achieved": best, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": best / pk["hbm_gbs"], "traffic": ncu_traffic("stream", f"{blocks} blocks x {words} words"),
            "algorithmic_bytes": blocks * words * 8,
            "note": f"{blocks} blocks x {words * 4} B read + write, {n_atoms} atoms on all 74 TPCs, "
                    f"single batch-mode k_worker launch"}


def ncu_traffic(name: str, config: str):
    """DRAM bytes (read + write) of one launch of the same shape from the
    committed ncu capture (profiles/ncu_traffic_r02.json, tools/ncu_traffic.py),
    else None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")))[name]
    except (OSError, KeyError, ValueError):
        return None
    return t["dram_read"] + t["dram_write"] if t.get("config") == config else None


def live_traffic(key: str = "dram"):
    """The live stacked run's DRAM bytes per k_worker launch from the committed
    ncu capture of the same scenario (profiles/ncu_traffic_r02.json)."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")))["fig7_live"]
    except (OSError, KeyError, ValueError):
        return None
    return t["dram_read"] + t["dram_write"] if key == "dram" else t[key]


def isolated(fn_name: str, local: int, timeout_s: float, *extra):
    """Runs bench.<fn_name>(local, *extra) in a child process bounded by
    timeout_s (the model-config runs are the longest secondary measurements;
    a hang there must not cost the bench line). The parent holds no
    dispatcher meanwhile, so the child has the GPU."""
    call_args = ", ".join([repr(local)] + [repr(x) for x in extra])
    code = (f"import json, sys; sys.path.insert(0, {ROOT!r}); import bench; "
            f"print('@@' + json.dumps(bench.{fn_name}({call_args})))")
    try:
        p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=timeout_s,
                           cwd=ROOT)
    except subprocess.TimeoutExpired:
        return {"error": f"{fn_name} exceeded {timeout_s:.0f} s"}
    for line in p.stdout.splitlines()[::-1]:
        if line.startswith("@@"):
            return json.loads(line[2:])
    return {"error": f"{fn_name} failed (rc {p.returncode}): {p.stderr.strip()[-400:]}"}


def guarded(fn):
    """Secondary measurements never take the bench line down."""
    try:
        return fn()
    except Exception as e:  # noqa: BLE001
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def gemv_saturation(api, local: int, args) -> dict:
    """The decode GEMV body (TMA-streamed W, tensor-core MACs) on a weight
    matrix far larger than L2, one atom on all 74 TPCs, batch mode."""
    import torch

    pk = peaks()
    n, k = 262144, 8192
    dev_name = f"cuda:{local}"
    w = torch.randn(n, k, device=dev_name, dtype=torch.bfloat16)
    x = torch.randn(k, device=dev_name, dtype=torch.bfloat16)
    y = torch.empty(n, device=dev_name)
    torch.cuda.synchronize()
    best = 0.0
    nbytes = n * k * 2 + k * 2 + n * 4
    with api.Device(device=local, workers_per_sm=args.workers_per_sm) as dev:
        desc, blocks = dev.gemv_desc(w.data_ptr(), x.data_ptr(), y.data_ptr(), n, k)
        descs = [api.Device.desc(0, blocks, range(74), 20, api.GPUOS_BODY_GEMV_BF16, [desc])]
        for _ in range(3):
            ms = dev.run_batch(descs)
            while dev.in_flight():
                dev.poll()
            best = max(best, nbytes / (ms * 1e-3) / 1e9)
        dev.free(desc)
    return {"bound": "hbm", "achieved": best, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": best / pk["hbm_gbs"], "traffic": ncu_traffic("gemv", f"{n}x{k}"),
            "algorithmic_bytes": nbytes,
            "note": f"GEMV y = W x, W bf16 {n}x{k} ({nbytes / 1e9:.1f} GB) as {blocks} 256-row pair "
                    f"tiles on all 74 TPCs, single batch-mode k_worker launch, CUDA events"}


def right_sizing_summary(local: int, args) -> dict:
    """BASELINE config #4 on the quick grid (paper_2504_15465_b200.rightsize)."""
    from paper_2504_15465_b200 import rightsize

    r = rightsize.sweep(device=local, slip=1.04, quick=True, reps=2, workers_per_sm=args.workers_per_sm)
    return {"slip": r["slip"], "grid": r["grid"], "mean_capacity_savings": r["mean_capacity_savings"],
            "max_slowdown": r["max_slowdown"], "weighted_r2": r["weighted_r2"],
            "b200_mean_capacity_savings": r["b200_mean_capacity_savings"],
            "b200_max_slowdown": r["b200_max_slowdown"],
            "bodies": [{k: b[k] for k in ("body", "t_star", "slowdown", "capacity_savings", "r2")}
                       | {"b200_t_star": b["b200"]["t_star"], "b200_slowdown": b["b200"]["slowdown"],
                          "b200_capacity_savings": b["b200"]["capacity_savings"]}
                       for b in r["bodies"]],
            "note": "t* = choose_tpcs_wave(fit_scaling(l(1), l(74)), slip 1.04) on device-timed "
                    "single-atom runs (the reference's right-sizer); b200_t_star = the measured-curve "
                    "chooser (l(1), l(37), plateau l(74)); slowdown = measured l(t*) / l(74)"}


def policy_rows(local: int) -> dict:
    """The reference's baseline policies on the live dispatcher, config #1
    workload."""
    from paper_2504_15465_b200 import configs

    r = configs.policy_comparison(horizon_ms=500.0, reps=2, device=local)
    r["note"] = ("fig7-b200 (time-scaled /10) under each scheduling policy, live; "
                 "be_blocks_per_s over device time")
    return r


MODEL_CONFIGS = ("infer4", "hybrid", "hybrid_real_attention")
MODEL_CONFIGS_NOTE = (
    "#2: 2x ResNet-50 b1 (150 rps) + 2x BERT-base b8 (100 rps), LC, Poisson, beside a "
    "ResNet-50 b256 training tenant (BE, closed loop), 2 s x 4 runs; #3: Llama-3-8B decode LC "
    "(60 tokens/s Poisson) + ResNet-50 b256 training BE (closed loop), 1 s x 10 runs (~580 tokens; 6 for the real-attention line); decode "
    "RMSNorm / SiLU-mul as tenant bodies, attention as a byte-equivalent STREAM kernel "
    "(hybrid) or the attn_decode_bf16 tenant body (hybrid_real_attention); "
    "alone = the same scenario with the other tenants silent; static = each tenant on its "
    "quota (no stealing, atomizer or sharing); BE throughput = executed work (blocks x "
    "calibrated block time) per second; random-init weights, live on the persistent dispatcher")


def model_config(local: int, name: str) -> dict:
    """One of BASELINE configs #2 / #3 on model kernel traces (configs.py)."""
    from paper_2504_15465_b200 import configs
    from paper_2504_15465_b200 import workloads as wl

    # infer4: 2 s x 4 runs = 1200 / 800 requests per ResNet / BERT tenant
    # (nearest-rank p99 over >= 800 samples), alone runs likewise.
    horizon, reps, cfg = {"infer4": (2000.0, 4, None), "hybrid": (1000.0, 10, None),
                          "hybrid_real_attention": (1000.0, 6, wl.hybrid(1000.0, real_attention=True))}[name]
    r = configs.run("hybrid" if cfg is not None else name, horizon_ms=horizon, reps=reps, device=local, cfg=cfg)
    return {"tpc_utilization": r["tpc_utilization"], "apps": {
        a: {k: v for k, v in row.items() if k in ("priority", "p99_vs_alone", "slo_attainment",
                                                    "throughput_vs_static", "iterations_vs_static")}
        | {"p99_ms": row["stacked"].get("p99_ms"), "alone_p99_ms": row["alone"].get("p99_ms"),
           "per_s": row["stacked"].get("per_s"), "completed": row["stacked"].get("completed")}
        for a, row in r["apps"].items()}, "knobs": r["knobs"]}


def model_configs(local: int) -> dict:
    """BASELINE configs #2 and #3, in this process (tools/hang_hunt2.py)."""
    out = {name: model_config(local, name) for name in MODEL_CONFIGS}
    out["note"] = MODEL_CONFIGS_NOTE
    return out


def model_configs_isolated(local: int) -> dict:
    """Each config in its own child process (~50-70 s each); a config whose
    run fails (a device fault aborts that process's runs) is measured once
    more in a fresh process, and the first error is kept beside the result."""
    out = {}
    for name in MODEL_CONFIGS:
        r = isolated("model_config", local, 300, name)
        if "error" in r and "exceeded" not in r["error"]:  # (a hang is not retried)
            first = r["error"]
            again = isolated("model_config", local, 300, name)
            r = ({"error": first, "retry_error": again["error"]} if "error" in again
                 else dict(again, first_attempt_error=first))
        out[name] = r
    out["note"] = MODEL_CONFIGS_NOTE
    return out


def gemm_saturation(api, local: int, args) -> dict:
    """k_worker executing a bf16 GEMM tenant kernel (C = A . B^T, tcgen05
    pair tiles) atomized over all 74 TPCs, staged in batch mode so the CUDA
    events cover one self-contained launch."""
    import torch

    pk = peaks()
    m = n = k = 8192
    dev_name = f"cuda:{local}"
    a = (torch.rand(m, k, device=dev_name) * 2 - 1).to(torch.bfloat16)
    b = (torch.rand(n, k, device=dev_name) * 2 - 1).to(torch.bfloat16)
    c = torch.empty(m, n, device=dev_name, dtype=torch.bfloat16)
    torch.cuda.synchronize()
    best, span = 0.0, 0.0
    # The reference's atomizer leaves a kernel whole unless its predicted
    # latency reaches 2 x the 1 ms atom duration (atomizer.cpp:33-40); this
    # one runs < 1 ms, so it is one atom, as the scheduler would submit it.
    n_atoms = 1
    with api.Device(device=local, workers_per_sm=args.workers_per_sm) as dev:
        desc, blocks, tm, tn = dev.gemm_desc(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k,
                                             bf16_out=True)
        # One kernel per launch: at 8192^3 (~0.7 ms) the dispatcher's ~13 us
        # start is ~2 %; two back-to-back copies measured lower (1484 vs
        # 1540 TF/s: the second atom's tiles interleave with the first's and
        # break the grouped raster's L2 reuse -- DRAM 2.07 GB for 0.81 GB).
        kernels = int(os.environ.get("GPUOS_BENCH_GEMM_KERNELS", "1"))
        descs = [api.Device.desc(i * blocks // n_atoms, (i + 1) * blocks // n_atoms, range(74), 20,
                                 api.GPUOS_BODY_GEMM_BF16, [desc]) for i in range(n_atoms)] * kernels
        for _ in range(5):  # best of 5 (MEASURED_PEAKS' cuBLAS figure is a best of 10)
            ms = dev.run_batch(descs)
            while dev.in_flight():
                dev.poll()
            tf = kernels * 2.0 * m * n * k / (ms * 1e-3) / 1e12
            if tf > best:
                best, span = tf, dev.stats().worker_span_ns * 1e-9
        dev.free(desc)
    return {"bound": "tensor", "achieved": best, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
            "frac": best / pk["bf16_tflops"], "traffic": ncu_traffic("gemm", f"{m}x{n}x{k} bf16 out x{kernels}"),
            "algorithmic_bytes": kernels * 2 * (m * k + n * k + m * n),
            "note": f"bf16 GEMM {m}x{n}x{k} (bf16 out) as {blocks} 256x256 pair tiles "
                    f"(tcgen05.mma.cta_group::2), {kernels} such kernels of {n_atoms} atom(s) each on all 74 "
                    f"TPCs in one batch-mode k_worker launch, CUDA events; peak = measured cuBLAS burst; "
                    f"device-clock span {kernels * 2.0 * m * n * k / span / 1e12:.0f} TFLOP/s",
            "peak_source": pk["source"]}


def conv_saturation(api, local: int, args) -> dict:
    """k_worker executing a ResNet-50 stage-2 3x3 convolution at batch 256
    (NHWC implicit GEMM, TMA im2col, tcgen05 pair tiles) atomized over all
    74 TPCs in batch mode."""
    import torch

    pk = peaks()
    n, h, w, c, k, r, s_, pad, st = 256, 28, 28, 256, 256, 3, 3, 1, 1
    dev_name = f"cuda:{local}"
    x = (torch.rand(n, h, w, c, device=dev_name) * 2 - 1).to(torch.bfloat16)
    wt = (torch.rand(k, r, s_, c, device=dev_name) * 2 - 1).to(torch.bfloat16)
    y = torch.empty(n, h, w, k, device=dev_name, dtype=torch.bfloat16)
    torch.cuda.synchronize()
    best, span = 0.0, 0.0
    # The reference's atomizer leaves a kernel whole unless its predicted
    # latency reaches 2 x the 1 ms atom duration (atomizer.cpp:33-40); this
    # one runs < 1 ms, so it is one atom, as the scheduler would submit it.
    n_atoms = 1
    with api.Device(device=local, workers_per_sm=args.workers_per_sm) as dev:
        desc, blocks, P, Q = dev.conv_desc(x.data_ptr(), wt.data_ptr(), y.data_ptr(), n, h, w, c, k, r, s_,
                                           pad, st, bf16_out=True)
        flops = 2.0 * n * P * Q * k * r * s_ * c
        # Four back-to-back kernels (a training step's convolutions) in one
        # launch: the dispatcher's one-time start (cluster launch, TMEM
        # allocation, ~13 us) is paid once per persistent-kernel lifetime in
        # live mode, not per tenant kernel.
        kernels = 4
        descs = [api.Device.desc(i * blocks // n_atoms, (i + 1) * blocks // n_atoms, range(74), 20,
                                 api.GPUOS_BODY_CONV_BF16, [desc]) for i in range(n_atoms)] * kernels
        for _ in range(5):  # best of 5 (MEASURED_PEAKS' cuBLAS figure is a best of 10)
            ms = dev.run_batch(descs)
            while dev.in_flight():
                dev.poll()
            tf = kernels * flops / (ms * 1e-3) / 1e12
            if tf > best:
                best, span = tf, dev.stats().worker_span_ns * 1e-9
        dev.free(desc)
    return {"bound": "tensor", "achieved": best, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
            "frac": best / pk["bf16_tflops"],
            "traffic": ncu_traffic("conv", f"n{n} {h}x{w}x{c} k{k} {r}x{s_}/{st} x{kernels}"),
            "algorithmic_bytes": kernels * 2 * (n * h * w * c + k * r * s_ * c + n * P * Q * k),
            "note": f"conv n{n} {h}x{w}x{c} -> {P}x{Q}x{k} {r}x{s_}/{st} (bf16 out) as {blocks} pair tiles "
                    f"of 256 pixels x 256 channels (TMA im2col, tcgen05.mma.cta_group::2), {kernels} such "
                    f"kernels of {n_atoms} atom(s) each on all 74 TPCs in one batch-mode k_worker launch, CUDA "
                    f"events; device-clock span {kernels * flops / span / 1e12:.0f} TFLOP/s",
            "peak_source": pk["source"]}


def self_launch(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: start N ranks of this same
    command line, one per GPU (RANK / LOCAL_RANK / WORLD_SIZE /
    MASTER_ADDR=127.0.0.1 / MASTER_PORT in the environment, exactly what
    torchrun would set). Rank 0's stdout is the bench line; the others'
    stdout is discarded. Returns the worst exit code."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    return max(abs(p.wait()) for p in procs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--time-scale", type=float, default=10.0)
    ap.add_argument("--horizon-ms", type=float, default=2000.0, help="reference-scale horizon")
    ap.add_argument("--workers-per-sm", type=int, default=2)
    ap.add_argument("--chunk-cap", type=int, default=256)
    ap.add_argument("--skip-configs", action="store_true",
                    help="skip the model-trace runs of configs #2/#3")
    ap.add_argument("--workload", choices=["fig7", "box8"], default="fig7",
                    help="fig7: BASELINE config #1; box8: config #5 (8 tenants per GPU)")
    ap.add_argument("--sample-s", type=float, default=5.0,
                    help="reference arm: seconds of simulator work per step")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args.gpus))
    rank, world, local = dist_init()
    if world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; using {world}", file=sys.stderr)
    if args.workload == "box8":
        cfg = workloads.tenant_set(rank, args.time_scale, args.horizon_ms)
    else:
        cfg = workloads.fig7_b200(args.time_scale, args.horizon_ms)
    if args.impl == "reference":
        cfgs = ([workloads.tenant_set(r, args.time_scale, args.horizon_ms) for r in range(world)]
                if args.workload == "box8" else [cfg] * world)
        reference_arm(args, cfgs, rank, world)
    else:
        ours(args, cfg, rank, world, local)


if __name__ == "__main__":
    main()
