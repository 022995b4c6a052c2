"""CPU: the C-ABI library loads, exports every symbol include/csattn_b200.h
declares, and its host-only helpers behave like the reference
(retrieval.cpp:10-38, metrics.cpp:32-38, synthetic.cpp:18-74)."""
import ctypes as C
import math
import os
import subprocess

import numpy as np
import pytest

import paper_2604_08584_b200 as cs
from paper_2604_08584_b200 import _abi
from tests.conftest import HAS_GPU  # noqa: E402


def test_library_exports_every_declared_symbol():
    lib = _abi.load()
    declared = _abi.header_symbols()
    assert len(declared) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        assert hasattr(lib, s)
    assert set(declared) == set(_abi.SIGNATURES), "ctypes signatures out of sync with header"


def test_library_is_sm100a_only_and_self_contained():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _abi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    nm = subprocess.run(["nm", "-D", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "csref_" not in nm and "ora_" not in nm  # never links the checkers


def test_keep_count_and_schedule_known_answers():
    assert cs.keep_count(0.05, 10) == 1
    assert cs.keep_count(0.05, 8192) == 410
    assert cs.keep_count(1.0, 77) == 77
    assert cs.keep_count(0.5, 3) == 2
    with pytest.raises(cs.ParameterError):
        cs.keep_count(0.0, 10)
    with pytest.raises(cs.ParameterError):
        cs.keep_count(1.5, 10)
    assert cs.parse_schedule("0.05-step-1") == (0.05, 1)
    assert cs.parse_schedule("0.15-step-4") == (0.15, 4)
    assert cs.parse_schedule("0.20-step-8") == (0.20, 8)
    for bad in ["0.05", "-step-4", "0.05-step-", "x-step-1", "0.05-step-2x", "0.0-step-1",
                "1.5-step-1", "0.05-step-0"]:
        with pytest.raises(cs.ParameterError):
            cs.parse_schedule(bad)


def test_h2d_bytes_closed_form():  # test_harness.cpp closed forms
    assert cs.h2d_bytes(0.05, 1000, 64, 2, 1) == pytest.approx(2 * 0.05 * 1000 * 64 * 2)
    assert cs.h2d_bytes(0.15, 8192, 64, 2, 4) == pytest.approx(2 * 0.15 * 8192 * 64 * 2 / 4)
    with pytest.raises(cs.ParameterError):
        cs.h2d_bytes(0.0, 10, 64, 2, 1)


def test_uniform_layout():
    assert cs.uniform_widths(128, 8) == [16] * 8
    assert cs.uniform_widths(10, 3) == [4, 3, 3]
    with pytest.raises(cs.ParameterError):
        cs.uniform_widths(4, 5)


def test_synthetic_deterministic_and_prefix_stable():
    a = cs.make_synthetic(cs.SyntheticSpec(rows=64, dim=32, seed=7))
    b = cs.make_synthetic(cs.SyntheticSpec(rows=128, dim=32, seed=7))
    for x, y in zip(a, b):
        assert np.array_equal(x, y[:64])
    assert np.isfinite(a[0]).all()


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU failure mode")
def test_context_without_gpu_fails_loudly():
    with pytest.raises(cs.CudaError):
        cs.Context(0)
