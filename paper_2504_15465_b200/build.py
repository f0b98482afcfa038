"""In-tree build of the B200 TPC dispatcher library and tools.

Outputs (git-ignored, travel to the GPU box with the gpurun snapshot):
  paper_2504_15465_b200/lib/libgpuos_b200.so   C ABI: include/gpuos_dev.h,
                                               include/gpuos_sim.h, plus the
                                               gpuos:: C++ API (include/gpuos)
  paper_2504_15465_b200/lib/libgpuos_host.a    host-only gpuos:: library
  paper_2504_15465_b200/bin/gpuos_replay       replay-backend log/report tool
  paper_2504_15465_b200/bin/topo_probe         topology probe (GPU)

CUDA code is compiled for sm_100a only
(-gencode arch=compute_100a,code=sm_100a, -lineinfo). Rebuilds are
incremental on source / header mtimes.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(PKG, "build", "obj")
LIB = os.path.join(PKG, "lib")
BIN = os.path.join(PKG, "bin")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", shutil.which("g++") or "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

_JSON_CANDIDATES = [
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann",
]


def json_include() -> str:
    """Directory holding nlohmann/json's single header `json.hpp` (v3.11.3 in
    this image, shipped inside cudnn_frontend)."""
    for d in _JSON_CANDIDATES:
        if os.path.exists(os.path.join(d, "json.hpp")):
            return d
    hits = glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "**",
                                  "nlohmann", "json.hpp"), recursive=True)
    if hits:
        return os.path.dirname(hits[0])
    raise RuntimeError("nlohmann json.hpp not found")


def _headers() -> list[str]:
    return (glob.glob(os.path.join(INCLUDE, "**", "*.h*"), recursive=True)
            + glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
            + glob.glob(os.path.join(CSRC, "**", "*.hpp"), recursive=True))


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)


def host_flags() -> list[str]:
    return ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-I" + INCLUDE,
            "-I" + json_include()]


def cuda_flags() -> list[str]:
    return ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC",
                   "-I" + INCLUDE, "-I" + os.path.join(CSRC, "device")]


def build(verbose: bool = False) -> dict[str, str]:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB, exist_ok=True)
    os.makedirs(BIN, exist_ok=True)
    headers = _headers()
    jobs = []
    host_objs, dev_objs = [], []
    for src in sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp"))):
        obj = os.path.join(OBJ, "host_" + os.path.basename(src)[:-4] + ".o")
        host_objs.append(obj)
        if _stale(obj, [src] + headers):
            jobs.append([CXX] + host_flags() + ["-c", src, "-o", obj])
    for src in sorted(glob.glob(os.path.join(CSRC, "device", "*.cu"))):
        obj = os.path.join(OBJ, "dev_" + os.path.basename(src)[:-3] + ".o")
        dev_objs.append(obj)
        if _stale(obj, [src] + headers):
            jobs.append([NVCC] + cuda_flags() + ["-c", src, "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for f in [ex.submit(_run, j) for j in jobs]:
            f.result()

    out = {}
    so = os.path.join(LIB, "libgpuos_b200.so")
    if _stale(so, host_objs + dev_objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", so] + dev_objs + host_objs
             + ["-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"])
    out["lib"] = so

    host_only = [o for o in host_objs if "b200_device" not in o and "sim_capi" not in o]
    ar = os.path.join(LIB, "libgpuos_host.a")
    if _stale(ar, host_only):
        if os.path.exists(ar):
            os.remove(ar)
        _run(["ar", "rcs", ar] + host_only)
    out["host_lib"] = ar

    tools = {
        "gpuos_replay": ([CXX] + host_flags(), os.path.join(CSRC, "tools", "gpuos_replay.cpp"), [ar]),
    }
    for name, (cc, src, libs) in tools.items():
        exe = os.path.join(BIN, name)
        if _stale(exe, [src] + libs + headers):
            _run(cc + [src] + libs + ["-o", exe])
        out[name] = exe
    for name in ("topo_probe", "racecheck_alloc_probe"):
        probe = os.path.join(BIN, name)
        psrc = os.path.join(CSRC, "tools", name + ".cu")
        if _stale(probe, [psrc]):
            _run([NVCC] + ARCH + ["-O2", "-lineinfo", "-std=c++17", psrc, "-o", probe])
        out[name] = probe
    if verbose:
        for k, v in out.items():
            print(f"{k}: {v}")
    return out


if __name__ == "__main__":
    build(verbose=True)
