"""CPU: the C ABI library loads, exports every symbol include/wsvd_b200.h
declares, runs its host-only entry points, and fails loudly (never falls
back to the CPU) when no sm_100 device is visible."""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from paper_2604_02570_b200 import _native as N
from paper_2604_02570_b200.errors import ConfigError, CudaError, ShapeError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "wsvd_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(wsvd_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (wsvd_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    # and the ctypes table covers them all
    assert set(syms) <= set(N.SIGNATURES)
    N.lib()


def test_abi_version_and_errors():
    L = N.lib()
    assert L.wsvd_abi_version() == 1
    with pytest.raises(ConfigError):
        N.call("wsvd_device_count", None)
    with pytest.raises(ConfigError):
        N.call("wsvd_layer_create", None, None, None)


@pytest.mark.skipif(N.device_count() > 0, reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_a_device():
    desc = N.LayerDesc(16, 4, 2, 0, N.BF16, 0, 0)
    ranks = np.full((2, 3), 2, dtype=np.int32)
    h = C.c_void_p()
    with pytest.raises(CudaError, match="no sm_100"):
        N.call("wsvd_layer_create", C.byref(desc), ranks.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(h))
    from paper_2604_02570_b200 import decode as D
    from tests.helpers import to_factors
    f = to_factors(O.random_layer(O.Rng(1), 16, 4, [[2, 2, 2]] * 2))
    with pytest.raises(CudaError):
        D.LatentCache(f)


@pytest.mark.parametrize("bits", [8, 4])
def test_host_weight_quantizer_matches_oracle_and_reference(bits):
    for seed in range(3):
        w = O.Rng(700 + seed).normal_matrix(64, 11, 0.05 * (seed + 1))
        w[:, 5] = 0.0
        q = np.zeros(w.shape, dtype=np.int8)
        s = np.zeros(w.shape[1])
        clip = C.c_double()
        N.call("wsvd_quantize_weight", w.ctypes.data_as(C.POINTER(C.c_double)), 64, 11, bits,
               q.ctypes.data_as(C.POINTER(C.c_int8)), s.ctypes.data_as(C.POINTER(C.c_double)),
               C.byref(clip))
        oq, os_, oclip = O.quantize_weight(w, bits)
        assert (q == oq).all() and (s == os_).all() and clip.value == oclip
    with pytest.raises(ConfigError):
        N.call("wsvd_quantize_weight", w.ctypes.data_as(C.POINTER(C.c_double)), 64, 11, 6,
               q.ctypes.data_as(C.POINTER(C.c_int8)), s.ctypes.data_as(C.POINTER(C.c_double)), None)
    with pytest.raises(ShapeError):
        N.call("wsvd_quantize_weight", w.ctypes.data_as(C.POINTER(C.c_double)), 0, 11, 8,
               q.ctypes.data_as(C.POINTER(C.c_int8)), s.ctypes.data_as(C.POINTER(C.c_double)), None)


def test_build_entry_point_compiles_for_sm100a():
    # every kernel object carries sm_100a SASS (checked without a GPU)
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
