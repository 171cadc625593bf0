"""GPU: the C++ drop-in (include/wsvd/decode.hpp) replaying the reference's
decode unit tests (tests/cpp/test_decode_api.cpp), linked against the
in-tree libwsvd_b200.so and the oracle."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2604_02570_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "test_decode_api.cpp")


def build_test(out_dir: str) -> str:
    exe = os.path.join(out_dir, "test_decode_api")
    subprocess.run(["make", "-s", "-f", os.path.join(ROOT, "oracle", "Makefile")], check=True)
    cmd = ["g++", "-std=c++20", "-O1", f"-I{os.path.join(ROOT, 'include')}", "-I/usr/local/cuda/include", SRC,
           "-o", exe, f"-L{PKG}", "-lwsvd_b200", f"-Wl,-rpath,{PKG}",
           os.path.join(ROOT, "oracle", "liboracle.so"), f"-Wl,-rpath,{os.path.join(ROOT, 'oracle')}"]
    subprocess.run(cmd, check=True)
    return exe


def test_cpp_api_compiles(tmp_path):
    # CPU-side: the drop-in headers compile and link (no device needed)
    build_test(str(tmp_path))


@pytest.mark.gpu
def test_cpp_api_reference_decode_tests(tmp_path):
    exe = build_test(str(tmp_path))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
    assert "0 failures" in r.stdout
