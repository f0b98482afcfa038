"""Power telemetry on the B200 backend (NVML, loaded at run time): the GPU's
energy counter over a live run replaces the reference's modelled energy
(device.cpp:221-242). Clock locking (B200Options::dvfs_actuate) is not
exercised: this pool's operator manages clocks."""
from __future__ import annotations

import ctypes

import pytest

pytestmark = pytest.mark.gpu


class Sample(ctypes.Structure):
    _fields_ = [("energy_mj", ctypes.c_uint64), ("clock_event_reasons", ctypes.c_uint64),
                ("sm_mhz", ctypes.c_uint32), ("mem_mhz", ctypes.c_uint32),
                ("power_mw", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


def test_power_sample_reads_energy_and_clocks(api, cuda_device):
    lib = ctypes.CDLL(api.LIB_PATH)
    s = Sample()
    assert lib.gpuos_power_sample(0, ctypes.byref(s)) == 0
    assert s.energy_mj > 0 and s.sm_mhz > 0 and s.power_mw > 0


def test_live_run_reports_measured_energy(api, cuda_device):
    from paper_2504_15465_b200 import workloads

    cfg = workloads.fig7_b200(10.0, 2000.0)
    r = api.run({"scenario": {"config": cfg}, "backend": "b200", "device": "b200"})
    b = r["b200"]
    secs = b["run_wall_ns"] * 1e-9
    # a busy B200 draws between ~100 W and its 1 kW board limit
    assert 50.0 * secs < b["energy_j"] < 1200.0 * secs, (b["energy_j"], secs)
    assert b["sm_mhz_end"] > 0
    # the reference report's energy field now carries the measured value
    assert float(r["report"]["energy_joules"]) == pytest.approx(b["energy_j"], rel=1e-6)
