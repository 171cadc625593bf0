"""The C++ drop-in inside the reference's own build.

oracle/Makefile (target ``dropin``) compiles every reference source except
src/decode.cpp from /root/reference/proj/src -- matrix, rng, factorize,
toymodel, pipeline, ... unmodified -- twice: once with the reference's
decode.hpp + decode.cpp (``pipeline_ref``, CPU fp64) and once with this repo's
include/wsvd/decode.hpp ahead on the include path and
paper_2604_02570_b200/csrc/host_decode.cpp in decode.cpp's place, linked to
libwsvd_b200.so (``pipeline_gpu``).  The driver tests/cpp/dropin_pipeline.cpp
replays acceptance criterion 3 (tests/acceptance_main.cpp:212-274: ragged
ranks, every tiling; full-rank factors vs the dense flash / eager baselines),
the shared-latent baseline (decode.cpp:321-432) and pipe::decode_factored /
decode_dense over a 2-layer toy model (pipeline.cpp:304-375).

Traffic tallies and error classes must be identical; values within 1e-4
relative (the drop-in stores factors and caches in fp32 by default and
accumulates in fp32; the reference is fp64 -- north_star allows 1e-3)."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROP = os.path.join(ROOT, "oracle", "_ref", "dropin")
TOL = 1e-4


def _build():
    subprocess.run(["make", "-s", "-f", os.path.join(ROOT, "oracle", "Makefile"), "dropin"], check=True)
    for exe in ("pipeline_ref", "pipeline_gpu", "test_decode_api"):
        if not os.path.exists(os.path.join(DROP, exe)):
            pytest.skip(f"{exe} not built (needs /root/reference at build time)")


def _records(path):
    out = {}
    with open(path) as fh:
        lines = fh.read().split("\n")
    i = 0
    while i < len(lines) and lines[i]:
        name, r, c = lines[i].split()
        n = int(r) * int(c)
        vals = np.array([float.fromhex(v) for v in lines[i + 1:i + 1 + n]])
        out[name] = vals.reshape(int(r), int(c))
        i += 1 + n
    return out


def test_dropin_binaries_link():
    """CPU: both builds link (the drop-in header compiles the reference's
    pipeline.cpp), and the reference build runs."""
    _build()
    out = os.path.join(DROP, "ref_records.txt")
    r = subprocess.run([os.path.join(DROP, "pipeline_ref"), out], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rec = _records(out)
    assert "factored/out" in rec and "c3/31/tile1" in rec and rec["errors/flags"].all()


@pytest.mark.gpu
def test_dropin_matches_reference_build(tmp_path):
    _build()
    ref_out, gpu_out = str(tmp_path / "ref.txt"), str(tmp_path / "gpu.txt")
    for exe, out in (("pipeline_ref", ref_out), ("pipeline_gpu", gpu_out)):
        r = subprocess.run([os.path.join(DROP, exe), out], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, f"{exe}: {r.stderr[-2000:]}"
    ref, gpu = _records(ref_out), _records(gpu_out)
    assert ref.keys() == gpu.keys()
    worst = {}
    for name, a in ref.items():
        b = gpu[name]
        assert a.shape == b.shape, name
        if name.endswith("counter") or name.startswith("errors/"):
            assert np.array_equal(a, b), f"{name}: tallies differ\n{a}\n{b}"
            continue
        err = float(np.abs(a - b).max() / max(np.abs(a).max(), 1e-300))
        worst[name.split("/")[0]] = max(worst.get(name.split("/")[0], 0.0), err)
        assert err <= TOL, f"{name}: rel err {err:.2e}"
    print("worst relative error per group:", {k: f"{v:.1e}" for k, v in worst.items()})


@pytest.mark.gpu
def test_cpp_api_reference_decode_tests():
    """tests/cpp/test_decode_api.cpp -- the reference's decode unit tests
    (tests/test_decode.cpp) through the drop-in, checked against the oracle."""
    _build()
    r = subprocess.run([os.path.join(DROP, "test_decode_api")], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
    assert "0 failures" in r.stdout
