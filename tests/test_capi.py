"""The C-ABI library loads on CPU and exports every function the headers in
include/ declare; error codes follow the reference CLI (2 config, 3
invariant). No device calls here."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"\b(gpuos_\w+)\s*\(", text)))


@pytest.mark.parametrize("header", ["gpuos_dev.h", "gpuos_sim.h"])
def test_library_exports_every_declared_symbol(api, header):
    lib = ctypes.CDLL(api.LIB_PATH)
    names = declared(header)
    assert names
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    listed = set(api.DEV_SYMBOLS + api.SIM_SYMBOLS)
    assert set(names) <= listed


def test_session_error_codes(api):
    with pytest.raises(api.GpuosError) as e:
        api.run({"scenario": {"preset": "nope"}, "backend": "replay"})
    assert e.value.code == 2
    with pytest.raises(api.GpuosError) as e:
        api.run({"scenario": {"preset": "fig7"}, "backend": "warp-drive"})
    assert e.value.code == 2
    with pytest.raises(api.GpuosError) as e:
        api.run({"scenario": {"preset": "fig7"}, "backend": "replay", "set": {"bogus": 1}})
    assert e.value.code == 2


def test_device_open_fails_loudly_without_gpu(api):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(api.GpuosError) as e:
        api.Device()
    assert e.value.code in (-2, -4)


def test_b200_backend_fails_loudly_without_gpu(api):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(api.GpuosError) as e:
        api.run({"scenario": {"preset": "fig7"}, "backend": "b200", "horizon_ms": 10})
    assert e.value.code in (2, 3)


def test_replay_session_reuse_is_deterministic(api):
    with api.Session({"scenario": {"preset": "inf-train"}, "backend": "replay", "horizon_ms": 500}) as s:
        a = s.run(log=True)
        b = s.run(log=True)
    assert a["log"] == b["log"] and a["report"] == b["report"]


def test_time_scaled_scenario_scales_latencies(api):
    base = api.run({"scenario": {"preset": "fig7"}, "backend": "replay", "horizon_ms": 1000})
    fast = api.run({"scenario": {"preset": "fig7"}, "backend": "replay", "horizon_ms": 1000,
                    "time_scale": 10.0})
    hp0 = base["report"]["apps"][0]
    hp1 = fast["report"]["apps"][0]
    assert fast["horizon_ns"] == base["horizon_ns"] // 10
    assert hp1["completed"] == hp0["completed"]
    assert abs(hp1["p99_ns"] * 10 - hp0["p99_ns"]) <= 0.02 * hp0["p99_ns"]


def test_ctypes_structs_match_the_header(api, tmp_path):
    """The Python mirror of every gpuos_dev.h struct has the C layout."""
    import subprocess

    structs = {"gpuos_dev_config": api.DevConfig, "gpuos_dev_topology": api.DevTopology,
               "gpuos_atom_desc": api.AtomDesc, "gpuos_completion": api.Completion,
               "gpuos_dev_stats": api.DevStats}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "gpuos_dev.h"', "int main(void) {"]
    for c_name, py in structs.items():
        lines.append(f'printf("{c_name} size %zu\\n", sizeof({c_name}));')
        for f in py._fields_:
            lines.append(f'printf("{c_name} {f[0]} %zu\\n", offsetof({c_name}, {f[0]}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    for line in filter(None, got):
        c_name, field, value = line.split()
        py = structs[c_name]
        want = ctypes.sizeof(py) if field == "size" else getattr(py, field).offset
        assert int(value) == want, (c_name, field, value, want)


def test_tenant_body_table(api):
    """The built-in tenant bodies are registered by name (host table, no GPU)."""
    names = ("attn_decode_bf16", "grid_probe", "rmsnorm_bf16", "silu_mul_bf16")  # sorted
    assert [api.body_id(n) for n in names] == [api.GPUOS_BODY_USER0 + i for i in range(len(names))]
    with pytest.raises(api.GpuosError) as e:
        api.body_id("missing")
    assert e.value.code == -2


def test_body_table_generation(tmp_path):
    """build.generate_body_table: GPUOS_USER_BODY(name) declarations of the
    body sources get ids in sorted-name order; duplicates are an error."""
    from paper_2504_15465_b200 import build

    a = tmp_path / "a.cu"
    a.write_text("GPUOS_USER_BODY(zeta) {}\nGPUOS_USER_BODY( alpha ) {}\n")
    b = tmp_path / "b.cu"
    b.write_text("// GPUOS_USER_BODY(not_at_line_start) is a comment\nGPUOS_USER_BODY(mid) {}\n")
    text = open(build.generate_body_table([str(a), str(b)], str(tmp_path))).read()
    assert "case 0: alpha(b, a);" in text and "case 1: mid(b, a);" in text and "case 2: zeta(b, a);" in text
    assert "not_at_line_start" not in text.split("kNames")[1]
    b.write_text("GPUOS_USER_BODY(alpha) {}\n")
    with pytest.raises(RuntimeError):
        build.generate_body_table([str(a), str(b)], str(tmp_path))
