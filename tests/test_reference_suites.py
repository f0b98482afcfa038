"""The reference's OWN test suites, compiled unchanged against the B200
library's gpuos:: API (drop-in check): the eight doctest unit suites
(proj/tests/test_*.cpp, via the oracle/shim doctest stand-in) and the ten
SPEC acceptance criteria (proj/tests/acceptance.cpp). Needs the reference
sources, so it runs in the build container."""
from __future__ import annotations

import os
import subprocess

import pytest

from conftest import REFERENCE, ROOT

UNIT = ["test_atomizer", "test_device", "test_predictor", "test_rightsizer", "test_power",
        "test_metrics", "test_workload", "test_scheduler"]


def compile_against_library(built, src, out, shim=False):
    from paper_2504_15465_b200 import build as b

    cmd = ["g++", "-std=c++20", "-O2", "-w", "-I" + os.path.join(ROOT, "include"),
           "-I" + b.json_include()]
    if shim:
        cmd.append("-I" + os.path.join(ROOT, "oracle", "shim"))
    cmd += [src, built["host_lib"], "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.fixture(scope="module")
def reference_tests():
    if not os.path.isdir(os.path.join(REFERENCE, "tests")):
        pytest.skip("reference sources absent")
    return os.path.join(REFERENCE, "tests")


@pytest.mark.parametrize("suite", UNIT)
def test_reference_unit_suite(built, reference_tests, tmp_path, suite):
    exe = str(tmp_path / suite)
    compile_against_library(built, os.path.join(reference_tests, suite + ".cpp"), exe, shim=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_reference_acceptance(built, reference_tests, tmp_path):
    exe = str(tmp_path / "acceptance")
    compile_against_library(built, os.path.join(reference_tests, "acceptance.cpp"), exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=280)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") == 10, r.stdout
