"""The checkpoint reader (csrc/checkpoint.cpp through the C ABI) against the
reference's checkpoint format (src/checkpoint.cpp:168-333, matrix.cpp:251-284):
a fixture written by the reference's own ckpt::save (oracle/ckpt_tool.cpp,
tests/golden/ckpt_e64/) is read back bit-exactly -- checked against an
independent numpy parse of the files and, where the reference tree is
present, against the reference's own ckpt::load.  Host-only: no GPU."""
from __future__ import annotations

import json
import os
import shutil
import subprocess

import numpy as np
import pytest

from paper_2604_02570_b200.checkpoint import Checkpoint
from paper_2604_02570_b200.errors import IoError, ShapeError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = os.path.join(ROOT, "tests", "golden", "ckpt_e64")
TOOL = os.path.join(ROOT, "oracle", "_ref", "ckpt_tool")


def np_matrix(path):
    raw = open(path, "rb").read()
    assert raw[:8] == b"WSVDMAT1"
    r, c = np.frombuffer(raw[8:24], dtype="<u8")
    return np.frombuffer(raw[24:], dtype="<f8").reshape(int(r), int(c))


def np_int_matrix(path):
    raw = open(path, "rb").read()
    assert raw[:8] == b"WSVDI8T1"
    r, c = np.frombuffer(raw[8:24], dtype="<u8")
    return np.frombuffer(raw[24:24 + int(r) * int(c)], dtype=np.int8).reshape(int(r), int(c))


def test_info():
    ck = Checkpoint(FIX)
    assert (ck.embed_dim, ck.head_dim, ck.n_heads, ck.n_layers) == (64, 16, 4, 2)
    assert ck.weight_bits == 8 and ck.activation_bits == 8
    assert ck.has_factors and ck.has_quantized


def test_reader_matches_independent_parse():
    ck = Checkpoint(FIX)
    man = json.load(open(os.path.join(FIX, "manifest.json")))
    for e in man["factors"]:
        a, b = ck.head(e["layer"], e["head"], "qkv".index(e["role"]))
        assert a.shape == (64, e["rank"]) and b.shape == (e["rank"], 16)
        assert np.array_equal(a, np_matrix(os.path.join(FIX, e["a"])))
        assert np.array_equal(b, np_matrix(os.path.join(FIX, e["b"])))
    for e in man["quantized"]:
        aq, as_, bq, bs = ck.head_quantized(e["layer"], e["head"], "qkv".index(e["role"]))
        assert np.array_equal(aq, np_int_matrix(os.path.join(FIX, e["a"]["values"])))
        assert np.array_equal(bq, np_int_matrix(os.path.join(FIX, e["b"]["values"])))
        assert np.array_equal(as_, np_matrix(os.path.join(FIX, e["a"]["scales"]))[0])
        assert np.array_equal(bs, np_matrix(os.path.join(FIX, e["b"]["scales"]))[0])
        assert np.abs(aq).max() <= 127
    for li in range(2):
        assert np.array_equal(ck.weight(f"layer{li}.w_o"), np_matrix(os.path.join(FIX, f"layer{li}.w_o.wsvd")))


@pytest.mark.skipif(not os.path.exists(TOOL), reason="reference ckpt_tool not built (no /root/reference)")
@pytest.mark.parametrize("layer,head,role", [(0, 0, "q"), (0, 3, "k"), (1, 1, "v"), (1, 2, "q")])
def test_reader_matches_reference_loader(layer, head, role):
    out = subprocess.run([TOOL, "dump", FIX, str(layer), str(head), role], capture_output=True, text=True,
                         check=True).stdout.splitlines()
    rec = {}
    for ln in out:
        tok = ln.split()
        rec[tok[0]] = tok[1:]
    ck = Checkpoint(FIX)
    ri = "qkv".index(role)
    a, b = ck.head(layer, head, ri)
    aq, as_, bq, bs = ck.head_quantized(layer, head, ri)
    assert int(rec["rank"][0]) == a.shape[1]

    def mat(tag):
        r, c = int(rec[tag][0]), int(rec[tag][1])
        return np.array([float(v) for v in rec[tag][2:]]).reshape(r, c)
    assert np.array_equal(a, mat("a")) and np.array_equal(b, mat("b"))
    assert np.array_equal(aq, mat("qa").astype(np.int8)) and np.array_equal(bq, mat("qb").astype(np.int8))
    assert np.array_equal(as_, np.array([float(v) for v in rec["qa_scales"][1:]]))
    assert np.array_equal(bs, np.array([float(v) for v in rec["qb_scales"][1:]]))
    assert np.array_equal(ck.weight(f"layer{layer}.w_o"), mat("w_o"))


def test_errors_map_to_reference_classes(tmp_path):
    with pytest.raises(IoError):
        Checkpoint(str(tmp_path / "missing"))
    bad = tmp_path / "bad"
    shutil.copytree(FIX, bad)
    (bad / "manifest.json").write_text('{"schema": "wsvd-checkpoint-v1", "model": {')
    with pytest.raises(IoError):
        Checkpoint(str(bad))
    (bad / "manifest.json").write_text(json.dumps({"schema": "other"}))
    with pytest.raises(IoError):
        Checkpoint(str(bad))
    ck = Checkpoint(FIX)
    with pytest.raises(ShapeError):
        ck.head(0, 9, 0)
    trunc = tmp_path / "trunc"
    shutil.copytree(FIX, trunc)
    f = trunc / "layer0.q.h0.a.wsvd"
    f.write_bytes(f.read_bytes()[:100])
    with pytest.raises(IoError):
        Checkpoint(str(trunc)).head(0, 0, 0)
