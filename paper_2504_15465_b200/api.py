"""ctypes bindings of the B200 dispatcher's C ABI (include/gpuos_dev.h,
include/gpuos_sim.h).

The product is the native library ``lib/libgpuos_b200.so`` (host scheduler in
C++, persistent sm_100a dispatcher in CUDA). Python only drives it: there is
no Python or CPU fallback for any device operation — if the library is
missing, every entry point raises.

Scenario requests (``Session``) are JSON objects::

    {"scenario": {"preset": "fig7"} | {"config": {...}} | {"config_path": "..."},
     "backend": "replay" | "b200" | "mirror",
     "horizon_ms": float, "policy": str, "seed": int, "device": "b200",
     "quota_scale": float, "drop_apps": [ids], "time_scale": float,
     "set": {scheduler knob: value},            # scenario-JSON knob names
     "b200": {"workers_per_sm", "idle_sleep_ns", "trace", "synth",
              "words_per_us", "min_words", "chunk_cap"},
     "log": bool, "requests": bool, "timeline": bool, "e2e": bool,
     "verify": bool}
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Any

PKG = os.path.dirname(os.path.abspath(__file__))
# GPUOS_LIB overrides the in-tree library (A/B builds of the same tree).
LIB_PATH = os.environ.get("GPUOS_LIB") or os.path.join(PKG, "lib", "libgpuos_b200.so")

GPUOS_BODY_STREAM = 1
GPUOS_BODY_GEMM_BF16 = 2
GPUOS_BODY_SPIN = 3
GPUOS_BODY_GEMV_BF16 = 4
GPUOS_BODY_CONV_BF16 = 5
GPUOS_GEMM_OUT_BF16 = 1
GPUOS_GEMV_OUT_BF16 = 1
GPUOS_GEMV_W_PACKED = 2
GPUOS_BODY_USER0 = 64


def grid(gx: int, gy: int = 1, gz: int = 1) -> int:
    """args[4] of a tenant body (GPUOS_GRID)."""
    return gx | (gy << 21) | (gz << 42)


def body_id(name: str) -> int:
    """Id of the tenant body GPUOS_USER_BODY(name) compiled into the library."""
    lib = library()
    out = C.c_uint32()
    rc = lib.gpuos_dev_body_id(name.encode(), C.byref(out))
    if rc != 0:
        raise GpuosError(rc, lib.gpuos_dev_last_error().decode())
    return out.value
GPUOS_E_FULL = -5
GPUOS_DEV_DEFER_WORKERS = 1

# Every symbol the C headers declare (tests check the library exports them).
DEV_SYMBOLS = [
    "gpuos_dev_open", "gpuos_dev_close", "gpuos_dev_get_topology", "gpuos_dev_start",
    "gpuos_dev_stop", "gpuos_dev_submit_atom", "gpuos_dev_set_atom_paused",
    "gpuos_dev_set_tpc_fence", "gpuos_dev_poll", "gpuos_dev_now_ns", "gpuos_dev_in_flight",
    "gpuos_dev_get_stats", "gpuos_dev_alloc", "gpuos_dev_free", "gpuos_dev_copy",
    "gpuos_dev_memset", "gpuos_dev_last_error", "gpuos_dev_launch_workers", "gpuos_dev_consumed",
    "gpuos_dev_host_alloc", "gpuos_dev_host_free", "gpuos_dev_run_batch", "gpuos_dev_set_fence_mask", "gpuos_dev_set_tpc_owner",
    "gpuos_dev_gemm_desc", "gpuos_dev_gemm_desc_splitk", "gpuos_dev_gemv_desc", "gpuos_dev_conv_desc", "gpuos_dev_fill_bf16",
    "gpuos_dev_gemv_pack", "gpuos_dev_set_pair_fence", "gpuos_power_sample", "gpuos_power_lock_sm_clock",
    "gpuos_dev_body_id", "gpuos_dev_debug_dump",
]
SIM_SYMBOLS = [
    "gpuos_session_open", "gpuos_session_run", "gpuos_session_close", "gpuos_run_json",
    "gpuos_free_text", "gpuos_sim_last_error", "gpuos_plan_atoms", "gpuos_should_atomize",
    "gpuos_filter_cap", "gpuos_fit_scaling", "gpuos_choose_tpcs", "gpuos_choose_tpcs_wave",
    "gpuos_fit_scaling_plateau", "gpuos_choose_tpcs_wave_floor", "gpuos_choose_measured",
    "gpuos_block_latency", "gpuos_reference_kernel_latency", "gpuos_select_frequency",
    "gpuos_predictor_replay", "gpuos_probe_dispatch",
]


class GpuosError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class DevConfig(C.Structure):
    _fields_ = [("device_ordinal", C.c_int32), ("workers_per_sm", C.c_int32),
                ("logical_tpcs", C.c_int32), ("atom_slots", C.c_int32),
                ("ring_entries", C.c_int32), ("idle_sleep_ns", C.c_int32),
                ("flags", C.c_uint32), ("pipeline_timeout_ms", C.c_int32)]


class DevTopology(C.Structure):
    _fields_ = [("sm_count", C.c_int32), ("physical_tpcs", C.c_int32),
                ("logical_tpcs", C.c_int32), ("workers_per_sm", C.c_int32),
                ("workers_per_tpc", C.c_int32), ("threads_per_worker", C.c_int32),
                ("smem_per_worker", C.c_int32), ("reserved", C.c_int32)]


class AtomDesc(C.Structure):
    _fields_ = [("lo", C.c_int64), ("hi", C.c_int64), ("tpc_mask", C.c_uint64 * 2),
                ("priority", C.c_int32), ("body", C.c_uint32), ("args", C.c_uint64 * 5),
                ("tag", C.c_uint64), ("trace", C.c_void_p), ("atomized", C.c_int32),
                ("parts", C.c_uint32), ("after", C.c_uint32), ("flags", C.c_uint32),
                ("tenant", C.c_uint32), ("reserved", C.c_uint32)]


GPUOS_ATOM_CHAIN_HEAD = 1
GPUOS_ATOM_NO_EARLY = 2


class Completion(C.Structure):
    _fields_ = [("atom_id", C.c_uint32), ("blocks", C.c_uint32), ("tag", C.c_uint64),
                ("host_submit_ns", C.c_int64), ("host_complete_ns", C.c_int64),
                ("dev_first_start_ns", C.c_int64), ("dev_last_end_ns", C.c_int64),
                ("tpc_touched", C.c_uint64 * 2), ("dev_ingest_ns", C.c_int64),
                ("dev_armed_ns", C.c_int64)]


class DevStats(C.Structure):
    _fields_ = [("blocks_executed", C.c_uint64), ("atoms_completed", C.c_uint64),
                ("worker_busy_ns", C.c_uint64), ("claim_retries", C.c_uint64),
                ("kernel_elapsed_ns", C.c_int64), ("ingest_entries", C.c_int64),
                ("worker_span_ns", C.c_int64), ("first_block_ns", C.c_int64),
                ("tpc_busy_ns", C.c_uint64), ("fault", C.c_uint32), ("reserved", C.c_uint32)]


_lib: C.CDLL | None = None


def library() -> C.CDLL:
    """Loads the native library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(
            f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    sig = {
        "gpuos_dev_open": (C.c_int, [C.POINTER(DevConfig), C.POINTER(P)]),
        "gpuos_dev_close": (C.c_int, [P]),
        "gpuos_dev_get_topology": (C.c_int, [P, C.POINTER(DevTopology)]),
        "gpuos_dev_start": (C.c_int, [P]),
        "gpuos_dev_stop": (C.c_int, [P, C.c_int, C.POINTER(C.c_float)]),
        "gpuos_dev_submit_atom": (C.c_int, [P, C.POINTER(AtomDesc), C.POINTER(C.c_uint32)]),
        "gpuos_dev_set_atom_paused": (C.c_int, [P, C.c_uint32, C.c_int]),
        "gpuos_dev_set_tpc_fence": (C.c_int, [P, C.c_int32, C.c_int32]),
        "gpuos_dev_set_fence_mask": (C.c_int, [P, C.POINTER(C.c_uint64), C.c_int32]),
        "gpuos_dev_set_tpc_owner": (C.c_int, [P, C.POINTER(C.c_uint64), C.c_uint32, C.c_int32]),
        "gpuos_dev_poll": (C.c_int, [P, C.POINTER(Completion), C.c_int32]),
        "gpuos_dev_now_ns": (C.c_int64, [P]),
        "gpuos_dev_in_flight": (C.c_int32, [P]),
        "gpuos_dev_get_stats": (C.c_int, [P, C.POINTER(DevStats)]),
        "gpuos_dev_alloc": (C.c_int, [P, C.c_uint64, C.POINTER(P)]),
        "gpuos_dev_free": (C.c_int, [P, P]),
        "gpuos_dev_copy": (C.c_int, [P, P, P, C.c_uint64, C.c_int]),
        "gpuos_dev_memset": (C.c_int, [P, P, C.c_int, C.c_uint64]),
        "gpuos_dev_last_error": (C.c_char_p, []),
        "gpuos_dev_launch_workers": (C.c_int, [P]),
        "gpuos_dev_run_batch": (C.c_int, [P, C.POINTER(AtomDesc), C.c_int32, C.POINTER(C.c_float)]),
        "gpuos_dev_host_alloc": (C.c_int, [P, C.c_uint64, C.POINTER(P)]),
        "gpuos_dev_host_free": (C.c_int, [P, P]),
        "gpuos_dev_consumed": (C.c_int, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "gpuos_dev_conv_desc": (C.c_int, [P, P, P, P] + [C.c_int32] * 9 + [C.c_uint32, C.POINTER(P),
                                          C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                          C.POINTER(C.c_int32)]),
        "gpuos_dev_fill_bf16": (C.c_int, [P, P, C.c_uint64, C.c_uint64]),
        "gpuos_dev_gemv_pack": (C.c_int, [P, P, P, C.c_int64, C.c_int64]),
        "gpuos_dev_set_pair_fence": (C.c_int, [P, C.POINTER(C.c_uint64), C.c_uint32, C.c_int32]),
        "gpuos_dev_body_id": (C.c_int, [C.c_char_p, C.POINTER(C.c_uint32)]),
        "gpuos_dev_debug_dump": (C.c_int, [P, C.c_char_p, C.c_int32]),
        "gpuos_dev_gemv_desc": (C.c_int, [P, P, P, P, C.c_int64, C.c_int64, C.c_uint32, C.c_int32,
                                          C.POINTER(P), C.POINTER(C.c_int64)]),
        "gpuos_dev_gemm_desc": (C.c_int, [P, P, P, P, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                          C.c_uint32, C.POINTER(P), C.POINTER(C.c_int64),
                                          C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "gpuos_dev_gemm_desc_splitk": (C.c_int, [P, P, P, P, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                                 C.c_uint32, C.c_int32, C.POINTER(P), C.POINTER(C.c_int64),
                                                 C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "gpuos_session_open": (C.c_int, [C.c_char_p, C.POINTER(P)]),
        "gpuos_session_run": (C.c_int, [P, C.c_char_p, C.POINTER(C.c_void_p)]),
        "gpuos_session_close": (C.c_int, [P]),
        "gpuos_run_json": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
        "gpuos_free_text": (None, [C.c_void_p]),
        "gpuos_sim_last_error": (C.c_char_p, []),
        "gpuos_probe_dispatch": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
        "gpuos_plan_atoms": (C.c_int64, [C.c_int64] * 4 + [C.POINTER(C.c_int64), C.c_int64]),
        "gpuos_should_atomize": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_double]),
        "gpuos_filter_cap": (C.c_int, [C.c_int64, C.c_int32, C.c_int32]),
        "gpuos_fit_scaling": (C.c_int, [C.c_int64, C.c_int64, C.c_int32, C.POINTER(C.c_double),
                                        C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
        "gpuos_choose_tpcs": (C.c_int, [C.c_double, C.c_double, C.c_int32, C.c_int32,
                                        C.c_double, C.c_int32]),
        "gpuos_fit_scaling_plateau": (C.c_int, [C.c_int64, C.c_int32, C.c_int64, C.c_int64, C.c_int32,
                                                C.POINTER(C.c_double), C.POINTER(C.c_double),
                                                C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
        "gpuos_choose_tpcs_wave_floor": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_int32, C.c_int32,
                                                   C.c_double, C.c_int64, C.c_int32]),
        "gpuos_choose_measured": (C.c_int, [C.POINTER(C.c_int32), C.POINTER(C.c_double), C.c_int32, C.c_double,
                                            C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "gpuos_choose_tpcs_wave": (C.c_int, [C.c_double, C.c_double, C.c_int32, C.c_int32,
                                             C.c_double, C.c_int64, C.c_int32]),
        "gpuos_block_latency": (C.c_int64, [C.c_int64, C.c_double, C.c_int32]),
        "gpuos_reference_kernel_latency": (C.c_int64, [C.c_int64, C.c_int64, C.c_double,
                                                       C.c_int32, C.c_int32, C.c_int32]),
        "gpuos_select_frequency": (C.c_int32, [C.c_double, C.c_double]),
        "gpuos_predictor_replay": (C.c_int, [C.POINTER(C.c_int64), C.c_int32,
                                             C.POINTER(C.c_int64), C.c_int32,
                                             C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


# ------------------------------------------------------------ scenarios
class Session:
    """A scheduler session on one backend (gpuos_session_*)."""

    def __init__(self, request: dict[str, Any]):
        self._lib = library()
        self._h = C.c_void_p()
        rc = self._lib.gpuos_session_open(json.dumps(request).encode(), C.byref(self._h))
        if rc != 0:
            raise GpuosError(rc, self._lib.gpuos_sim_last_error().decode())

    def run(self, **overrides: Any) -> dict[str, Any]:
        out = C.c_void_p()
        rc = self._lib.gpuos_session_run(self._h, json.dumps(overrides).encode(), C.byref(out))
        if rc != 0:
            raise GpuosError(rc, self._lib.gpuos_sim_last_error().decode())
        try:
            return json.loads(C.string_at(out.value).decode())
        finally:
            self._lib.gpuos_free_text(out)

    def close(self) -> None:
        if self._h:
            self._lib.gpuos_session_close(self._h)
            self._h = C.c_void_p()

    def __del__(self) -> None:
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self) -> "Session":
        return self

    def __exit__(self, *exc: Any) -> None:
        self.close()


def probe_dispatch(**opts: Any) -> dict[str, Any]:
    """Live-path dispatcher overhead (gpuos_probe_dispatch)."""
    lib = library()
    out = C.c_void_p()
    rc = lib.gpuos_probe_dispatch(json.dumps(opts).encode(), C.byref(out))
    if rc != 0:
        raise GpuosError(rc, lib.gpuos_sim_last_error().decode())
    try:
        return json.loads(C.string_at(out.value).decode())
    finally:
        lib.gpuos_free_text(out)


def run(request: dict[str, Any]) -> dict[str, Any]:
    with Session(request) as s:
        return s.run()


# ------------------------------------------------------------ device seam
class Device:
    """Direct handle on the persistent dispatcher (gpuos_dev_*)."""

    def __init__(self, workers_per_sm: int = 2, logical_tpcs: int = 0, device: int = 0,
                 atom_slots: int = 0, idle_sleep_ns: int = 0, flags: int = 0):
        self._lib = library()
        cfg = DevConfig(device_ordinal=device, workers_per_sm=workers_per_sm,
                        logical_tpcs=logical_tpcs, atom_slots=atom_slots,
                        idle_sleep_ns=idle_sleep_ns, flags=flags)
        self._h = C.c_void_p()
        self._check(self._lib.gpuos_dev_open(C.byref(cfg), C.byref(self._h)))
        self.topology = DevTopology()
        self._check(self._lib.gpuos_dev_get_topology(self._h, C.byref(self.topology)))

    def _check(self, rc: int) -> int:
        if rc < 0:
            raise GpuosError(rc, self._lib.gpuos_dev_last_error().decode())
        return rc

    def start(self) -> None:
        self._check(self._lib.gpuos_dev_start(self._h))

    def launch_workers(self) -> None:
        self._check(self._lib.gpuos_dev_launch_workers(self._h))

    def consumed(self) -> tuple[int, int]:
        c, p = C.c_uint64(), C.c_uint64()
        self._check(self._lib.gpuos_dev_consumed(self._h, C.byref(c), C.byref(p)))
        return c.value, p.value

    def stop(self, drain: bool = True) -> float:
        ms = C.c_float()
        self._check(self._lib.gpuos_dev_stop(self._h, 1 if drain else 0, C.byref(ms)))
        return ms.value

    @staticmethod
    def desc(lo: int, hi: int, tpcs, priority: int, body: int, args, tag: int = 0,
             trace: int | None = None, parts: int = 1, after: int | None = None,
             chain_head: bool = False, no_early: bool = False, tenant: int = 0) -> AtomDesc:
        """One atom. `after`: atom id of a predecessor this atom is chained
        behind (armed on the device when the predecessor's last block ends);
        the predecessor must have been submitted with chain_head=True.
        `tenant`: 1 + the submitting tenant's id (0: none), see set_owner."""
        d = AtomDesc()
        d.tenant = tenant
        d.parts = parts
        d.lo, d.hi, d.priority, d.body, d.tag = lo, hi, priority, body, tag
        m = [0, 0]
        for t in tpcs:
            m[t >> 6] |= 1 << (t & 63)
        d.tpc_mask[0], d.tpc_mask[1] = m
        for i, a in enumerate(args):
            d.args[i] = int(a)
        d.trace = trace
        d.after = 0 if after is None else after + 1
        d.flags = (GPUOS_ATOM_CHAIN_HEAD if chain_head else 0) | (GPUOS_ATOM_NO_EARLY if no_early else 0)
        return d

    def run_batch(self, descs: list[AtomDesc]) -> float:
        """Stage `descs` and run the worker kernel alone; returns its ms."""
        arr = (AtomDesc * len(descs))(*descs)
        ms = C.c_float()
        self._check(self._lib.gpuos_dev_run_batch(self._h, arr, len(descs), C.byref(ms)))
        return ms.value

    def submit(self, lo: int, hi: int, tpcs, priority: int, body: int, args, tag: int = 0,
               trace: int | None = None, parts: int = 1, after: int | None = None,
               chain_head: bool = False, no_early: bool = False, tenant: int = 0) -> int:
        d = self.desc(lo, hi, tpcs, priority, body, args, tag, trace, parts, after, chain_head, no_early,
                      tenant)
        aid = C.c_uint32()
        self._check(self._lib.gpuos_dev_submit_atom(self._h, C.byref(d), C.byref(aid)))
        return aid.value

    def try_submit(self, *a, **k) -> int | None:
        try:
            return self.submit(*a, **k)
        except GpuosError as e:
            if e.code == GPUOS_E_FULL:
                return None
            raise

    def gemm_desc(self, a: int, b: int, c: int, m: int, n: int, k: int, ldc: int | None = None,
                  bf16_out: bool = False, k_splits: int = 1) -> tuple[int, int, int, int]:
        """Descriptor for GPUOS_BODY_GEMM_BF16 (C = A . B^T on tcgen05):
        returns (device pointer for args[0], grid blocks, tile_m, tile_n).
        k_splits > 1: split-K (gpuos_dev_gemm_desc_splitk)."""
        desc, blocks = C.c_void_p(), C.c_int64()
        tm, tn = C.c_int32(), C.c_int32()
        self._check(self._lib.gpuos_dev_gemm_desc_splitk(
            self._h, a, b, c, m, n, k, n if ldc is None else ldc,
            GPUOS_GEMM_OUT_BF16 if bf16_out else 0, k_splits, C.byref(desc), C.byref(blocks),
            C.byref(tm), C.byref(tn)))
        return desc.value, blocks.value, tm.value, tn.value

    def gemv_desc(self, w: int, x: int, y: int, n: int, k: int, bf16_out: bool = False,
                  k_splits: int = 1, packed: bool = False) -> tuple[int, int]:
        """Descriptor for GPUOS_BODY_GEMV_BF16 (y = W . x, decode GEMV):
        returns (device pointer for args[0], grid blocks). k_splits > 1
        splits K; the last block of each row tile reduces the partials.
        packed: `w` is a gemv_pack()ed copy of W."""
        desc, blocks = C.c_void_p(), C.c_int64()
        flags = (GPUOS_GEMV_OUT_BF16 if bf16_out else 0) | (GPUOS_GEMV_W_PACKED if packed else 0)
        self._check(self._lib.gpuos_dev_gemv_desc(self._h, w, x, y, n, k, flags,
                                                  k_splits, C.byref(desc), C.byref(blocks)))
        return desc.value, blocks.value

    @staticmethod
    def gemv_packed_bytes(n: int, k: int) -> int:
        return -(-n // 128) * -(-k // 64) * 128 * 64 * 2

    def gemv_pack(self, dst: int, src: int, n: int, k: int) -> None:
        """Row-major bf16 W [n, k] -> the GEMV's packed layout (each ring
        stage one contiguous 16 KiB range; gemv_packed_bytes(n, k))."""
        self._check(self._lib.gpuos_dev_gemv_pack(self._h, dst, src, n, k))

    def conv_desc(self, x: int, w: int, y: int, n: int, h: int, wd: int, c: int, k: int, r: int,
                  s: int, pad: int, stride: int, bf16_out: bool = False) -> tuple[int, int, int, int]:
        """Descriptor for GPUOS_BODY_CONV_BF16 (NHWC implicit-GEMM conv on
        tcgen05): returns (device pointer for args[0], grid blocks, P, Q)."""
        desc, blocks, p, q = C.c_void_p(), C.c_int64(), C.c_int32(), C.c_int32()
        self._check(self._lib.gpuos_dev_conv_desc(self._h, x, w, y, n, h, wd, c, k, r, s, pad, stride,
                                                  1 if bf16_out else 0, C.byref(desc),
                                                  C.byref(blocks), C.byref(p), C.byref(q)))
        return desc.value, blocks.value, p.value, q.value

    def free(self, ptr: int) -> None:
        self._check(self._lib.gpuos_dev_free(self._h, ptr))

    def pause(self, atom: int, paused: bool) -> None:
        self._check(self._lib.gpuos_dev_set_atom_paused(self._h, atom, 1 if paused else 0))

    def fence(self, tpc: int, min_priority: int) -> None:
        self._check(self._lib.gpuos_dev_set_tpc_fence(self._h, tpc, min_priority))

    def fence_mask(self, tpcs, min_priority: int) -> None:
        m = (C.c_uint64 * 2)()
        for t in tpcs:
            m[t >> 6] |= 1 << (t & 63)
        self._check(self._lib.gpuos_dev_set_fence_mask(self._h, m, min_priority))

    def set_owner(self, tpcs, owner: int, min_priority: int) -> None:
        """TPC-ownership table: `owner` (1 + tenant id) starts its atoms on
        these TPCs at any priority, other atoms need >= min_priority."""
        m = (C.c_uint64 * 2)()
        for t in tpcs:
            m[t >> 6] |= 1 << (t & 63)
        self._check(self._lib.gpuos_dev_set_tpc_owner(self._h, m, owner, min_priority))

    def set_pair_fence(self, tpcs, pair_slots: int, min_priority: int) -> None:
        """Pair fence: only the TPCs' worker pairs in `pair_slots` (bit i =
        slot i) refuse blocks below min_priority (0 lifts)."""
        m = (C.c_uint64 * 2)()
        for t in tpcs:
            m[t >> 6] |= 1 << (t & 63)
        self._check(self._lib.gpuos_dev_set_pair_fence(self._h, m, pair_slots, min_priority))

    def poll(self, max_n: int = 256) -> list[Completion]:
        buf = (Completion * max_n)()
        n = self._check(self._lib.gpuos_dev_poll(self._h, buf, max_n))
        return [buf[i] for i in range(n)]

    def in_flight(self) -> int:
        return self._lib.gpuos_dev_in_flight(self._h)

    def now_ns(self) -> int:
        return self._lib.gpuos_dev_now_ns(self._h)

    def stats(self) -> DevStats:
        s = DevStats()
        self._check(self._lib.gpuos_dev_get_stats(self._h, C.byref(s)))
        return s

    def close(self) -> None:
        if self._h:
            self._lib.gpuos_dev_close(self._h)
            self._h = C.c_void_p()

    def __del__(self) -> None:
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self) -> "Device":
        return self

    def __exit__(self, *exc: Any) -> None:
        self.close()


# ------------------------------------------------------------ policy functions
def plan_atoms(n: int, pred: int, atom: int, min_blocks: int) -> list[tuple[int, int]]:
    lib = library()
    cap = max(1, n)
    buf = (C.c_int64 * (2 * cap))()
    k = lib.gpuos_plan_atoms(n, pred, atom, min_blocks, buf, cap)
    if k < 0:
        raise GpuosError(k, lib.gpuos_sim_last_error().decode())
    return [(buf[2 * i], buf[2 * i + 1]) for i in range(k)]


def should_atomize(pred: int, n: int, atom: int, factor: float = 2.0) -> bool:
    return bool(library().gpuos_should_atomize(pred, n, atom, factor))


def filter_cap(n: int, occ: int, total: int) -> int:
    return library().gpuos_filter_cap(n, occ, total)


def fit_scaling(l1: int, lT: int, T: int) -> tuple[float, float, bool]:
    m, b, v = C.c_double(), C.c_double(), C.c_int32()
    rc = library().gpuos_fit_scaling(l1, lT, T, C.byref(m), C.byref(b), C.byref(v))
    if rc != 0:
        raise GpuosError(rc, library().gpuos_sim_last_error().decode())
    return m.value, b.value, bool(v.value)


def choose_tpcs(m: float, b: float, valid: bool, t_alloc: int, slip: float, cap: int) -> int:
    return library().gpuos_choose_tpcs(m, b, int(valid), t_alloc, slip, cap)


def choose_tpcs_wave(m: float, b: float, valid: bool, t_alloc: int, slip: float, blocks: int,
                     occ: int) -> int:
    return library().gpuos_choose_tpcs_wave(m, b, int(valid), t_alloc, slip, blocks, occ)


def fit_scaling_plateau(l1: int, t_mid: int, l_mid: int, lT: int, T: int) -> tuple[float, float, float, bool]:
    """B200 measured-curve fit: l(t) = max(m/t + b, floor) (policy.hpp)."""
    m, b, fl, v = C.c_double(), C.c_double(), C.c_double(), C.c_int32()
    rc = library().gpuos_fit_scaling_plateau(l1, t_mid, l_mid, lT, T, C.byref(m), C.byref(b), C.byref(fl),
                                             C.byref(v))
    if rc != 0:
        raise GpuosError(rc, library().gpuos_sim_last_error().decode())
    return m.value, b.value, fl.value, bool(v.value)


def choose_tpcs_wave_floor(m: float, b: float, floor: float, valid: bool, t_alloc: int, slip: float,
                           blocks: int, occ: int) -> int:
    return library().gpuos_choose_tpcs_wave_floor(m, b, floor, int(valid), t_alloc, slip, blocks, occ)


def choose_measured(samples: dict[int, float], slip: float) -> tuple[int, int]:
    """Measured-curve right-sizer step: (narrowest width within the slip, next
    width to probe or 0) from {width: mean latency ns}."""
    ts = sorted(samples)
    t_arr = (C.c_int32 * max(1, len(ts)))(*ts)
    l_arr = (C.c_double * max(1, len(ts)))(*[float(samples[t]) for t in ts])
    ok, probe = C.c_int32(), C.c_int32()
    rc = library().gpuos_choose_measured(t_arr, l_arr, len(ts), slip, C.byref(ok), C.byref(probe))
    if rc != 0:
        raise GpuosError(rc, library().gpuos_sim_last_error().decode())
    return ok.value, probe.value


def block_latency(d0: int, s: float, f: int) -> int:
    return library().gpuos_block_latency(d0, s, f)


def reference_kernel_latency(blocks: int, d0: int, s: float, occ: int, t: int, f: int) -> int:
    return library().gpuos_reference_kernel_latency(blocks, d0, s, occ, t, f)


def select_frequency(S: float, slip: float) -> int:
    return library().gpuos_select_frequency(S, slip)


def predictor_replay(records, queries) -> list[tuple[int, int]]:
    lib = library()
    rec = (C.c_int64 * max(1, 4 * len(records)))(*[v for r in records for v in r])
    qry = (C.c_int64 * max(1, 3 * len(queries)))(*[v for q in queries for v in q])
    lat = (C.c_int64 * max(1, len(queries)))()
    conf = (C.c_int32 * max(1, len(queries)))()
    rc = lib.gpuos_predictor_replay(rec, len(records), qry, len(queries), lat, conf)
    if rc != 0:
        raise GpuosError(rc, lib.gpuos_sim_last_error().decode())
    return [(lat[i], conf[i]) for i in range(len(queries))]
