"""CPU: pin the oracle (oracle/wsvd_oracle.c) to the reference.

Two anchors, per the parity contract: (1) the reference itself compiled from
/root/reference (oracle/_ref/libwsvdref.so, built by oracle/Makefile) when it
is present, bit-exact; (2) the committed golden vectors in tests/golden/
(generated from the reference by tests/golden/make_golden.py), bit-exact,
available everywhere.  Then the reference's own decode unit tests
(tests/test_decode.cpp) are replayed on the oracle."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz"))
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")


def oracle_fill(lay, toks):
    L = toks.shape[0]
    ck = np.zeros((lay.nh, L, lay.rmax))
    cv = np.zeros_like(ck)
    c = O.OrcCounter()
    q = None
    for t in range(L):
        q = O.append_token(lay, ck, cv, t, toks[t], c)
    return ck, cv, q, c


def counter21(c):
    return np.array(list(c.loads) + list(c.stores) + list(c.flops), dtype=np.uint64)


# ------------------------------------------------------------ golden ------
def test_rng_matches_golden():
    r = O.Rng(42)
    assert (np.array([r.next_u64() for _ in range(64)], dtype=np.uint64) == GOLD["rng_u64_seed42"]).all()
    n = O.Rng.stream(7, 5).normal_matrix(1, 65, 0.5).ravel()
    assert (n == GOLD["rng_normal_seed7_stream5_std05"]).all()
    r = O.Rng(9)
    assert [r.index(11) for _ in range(32)] == list(GOLD["rng_index_seed9_bound11"])


@pytest.mark.parametrize("case,tile", [("bench", 32), ("ragged", 5)])
def test_decode_matches_golden(case, tile):
    lay = O.Layer(GOLD[f"{case}_A"], GOLD[f"{case}_B"], GOLD[f"{case}_ranks"])
    toks = GOLD[f"{case}_tokens"]
    ck, cv, q, ca = oracle_fill(lay, toks)
    assert (ck == GOLD[f"{case}_ck"]).all() and (cv == GOLD[f"{case}_cv"]).all()
    assert (q == GOLD[f"{case}_q"]).all()
    assert (counter21(ca) == GOLD[f"{case}_append_counter"]).all()
    cd = O.OrcCounter()
    out = O.fused_decode_step(lay, ck, cv, toks.shape[0], q, tile, cd)
    assert (out == GOLD[f"{case}_out"]).all()
    assert (counter21(cd) == GOLD[f"{case}_decode_counter"]).all()


def test_bench_layer_draw_order_matches_golden():
    lay = O.bench_layer(64, 16, 4, 8, seed=0)
    assert (lay.A == GOLD["bench_A"]).all() and (lay.B == GOLD["bench_B"]).all()


@pytest.mark.parametrize("bits", [8, 4])
def test_weight_quantizer_matches_golden(bits):
    q, s, clip = O.quantize_weight(GOLD["qw_w"], bits)
    assert (q == GOLD[f"qw{bits}_q"]).all()
    assert (s == GOLD[f"qw{bits}_s"]).all()
    assert clip == float(GOLD[f"qw{bits}_clip"])
    assert s[3] == 1.0 and (q[:, 3] == 0).all()  # zero column -> scale 1 (quant.cpp:55)


def test_activation_quantizer_matches_golden():
    q, s = O.quantize_activation_f64(GOLD["qa_x"], 8)
    assert (q == GOLD["qa_q"]).all() and (s == GOLD["qa_s"]).all()
    assert s[2] == 1.0  # zero row -> scale 1 (quant.cpp:142)


def test_fwht_matches_reference_hadamard():
    h = GOLD["hadamard16"]
    x = O.Rng(5).normal_matrix(1, 16).ravel().astype(np.float32)
    got = O.rotate_token(x)
    ref = x.astype(np.float64) @ h.T  # x_hat = x . S1^T
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max()


# ------------------------------------------------- live reference (_ref) --
@needs_ref
@pytest.mark.parametrize("seed", range(6))
def test_oracle_bit_exact_with_reference(seed):
    R = O.ref()
    rng = O.Rng(2000 + seed)
    E = 16 << (seed % 3)
    nh = 2 if seed % 2 == 0 else 4
    H = E // nh
    L = 5 + (seed * 7) % 36
    ranks = [[1 + rng.index(H), 1 + rng.index(H), 1 + rng.index(H)] for _ in range(nh)]
    lay = O.random_layer(rng, E, H, ranks)
    toks = rng.normal_matrix(L, E)
    ck, cv, q, ca = oracle_fill(lay, toks)
    for tile in (1, 7, 16, L):
        cd = O.OrcCounter()
        out = O.fused_decode_step(lay, ck, cv, L, q, tile, cd)
        rck, rcv = np.zeros_like(ck), np.zeros_like(cv)
        rq, rout = np.zeros_like(q), np.zeros_like(out)
        a21 = np.zeros(21, dtype=np.uint64)
        d21 = np.zeros(21, dtype=np.uint64)
        lay.c()
        rc = R.ref_append_then_decode(E, H, nh, lay.rmax, lay.ranks.ctypes.data_as(O._ip),
                                      lay.A.ctypes.data_as(O._dp), lay.B.ctypes.data_as(O._dp), L,
                                      toks.ctypes.data_as(O._dp), tile, rck.ctypes.data_as(O._dp),
                                      rcv.ctypes.data_as(O._dp), rq.ctypes.data_as(O._dp),
                                      rout.ctypes.data_as(O._dp), a21.ctypes.data_as(O._u64p),
                                      d21.ctypes.data_as(O._u64p))
        assert rc == 0
        assert (rck == ck).all() and (rcv == cv).all() and (rq == q).all() and (rout == out).all()
        assert (a21 == counter21(ca)).all() and (d21 == counter21(cd)).all()


@needs_ref
@pytest.mark.parametrize("bits", [8, 4])
def test_quantizer_bit_exact_with_reference(bits):
    R = O.ref()
    for seed in range(4):
        w = O.Rng(90 + seed).normal_matrix(40, 9, 0.2 + seed)
        q, s, clip = O.quantize_weight(w, bits)
        rq = np.zeros_like(q)
        rs = np.zeros_like(s)
        rclip = R.ref_quantize_weight(w.ctypes.data_as(O._dp), 40, 9, bits, rq.ctypes.data_as(O._i8p),
                                      rs.ctypes.data_as(O._dp))
        assert (q == rq).all() and (s == rs).all() and clip == rclip


# ------------------------------ reference decode tests replayed (oracle) --
def test_online_softmax_and_merge_properties():
    # test_decode.cpp:100-177
    import ctypes as C
    rng = O.Rng(302)
    width = 4
    values = rng.normal_matrix(18, width)
    scores = [3.0 * rng.normal() for _ in range(18)]

    def state(lo, hi):
        buf = np.zeros(width)
        st = O.lib()
        s = _Softmax(buf)
        for j in range(lo, hi):
            st.orc_softmax_observe(C.byref(s.c), C.c_double(scores[j]),
                                   values[j].ctypes.data_as(O._dp))
        return s

    a, b, c = state(0, 5), state(5, 11), state(11, 18)
    left = _merge(_merge(_copy(a), b), c)
    right = _merge(_copy(a), _merge(_copy(b), c))
    swapped = _merge(_merge(_copy(c), a), b)
    ref = left.acc / left.c.denom
    assert np.allclose(right.acc / right.c.denom, ref, rtol=1e-12)
    assert np.allclose(swapped.acc / swapped.c.denom, ref, rtol=1e-12)
    full = state(0, 18)
    mx = max(scores)
    w = np.exp(np.array(scores) - mx)
    assert np.allclose(full.acc / full.c.denom, (w @ values) / w.sum(), rtol=1e-12)
    assert full.c.max_score == mx


class _Softmax:
    def __init__(self, buf):
        import ctypes as C

        class S(C.Structure):
            _fields_ = [("max_score", C.c_double), ("denom", C.c_double), ("acc", O._dp),
                        ("w", C.c_size_t), ("empty", C.c_int)]
        self.acc = buf
        self.c = S(0.0, 0.0, buf.ctypes.data_as(O._dp), buf.size, 1)


def _copy(s):
    t = _Softmax(s.acc.copy())
    t.c.max_score, t.c.denom, t.c.empty = s.c.max_score, s.c.denom, s.c.empty
    return t


def _merge(s, o):
    import ctypes as C
    O.lib().orc_softmax_merge(C.byref(s.c), C.byref(o.c))
    return s


@pytest.mark.parametrize("cfg,seed", [((16, 4, 2, 13), 310), ((32, 8, 4, 9), 311),
                                      ((24, 4, 3, 31), 312), ((32, 8, 2, 1), 313)])
def test_fused_matches_reconstruct_then_attend(cfg, seed):
    E, H, nh, L = cfg
    rng = O.Rng(seed)
    ranks = [[1 + rng.index(H), 1 + rng.index(H), 1 + rng.index(H)] for _ in range(nh)]
    lay = O.random_layer(rng, E, H, ranks)
    ck, cv, q, _ = oracle_fill(lay, rng.normal_matrix(L, E))
    out = O.fused_decode_step(lay, ck, cv, L, q, 5)
    assert np.abs(out - O.reconstruct_then_attend(lay, ck, cv, L, q)).max() <= 1e-9


def test_tile_invariance_and_counters():
    rng = O.Rng(320)
    L = 29
    lay = O.random_layer(rng, 32, 8, [[3, 3, 3]] * 4)
    ck, cv, q, _ = oracle_fill(lay, rng.normal_matrix(L, 32))
    c0 = O.OrcCounter()
    ref = O.fused_decode_step(lay, ck, cv, L, q, L, c0)
    for tile in (1, 7, 16, L, L + 5):
        c = O.OrcCounter()
        assert np.abs(O.fused_decode_step(lay, ck, cv, L, q, tile, c) - ref).max() <= 1e-10
        assert (counter21(c) == counter21(c0)).all()
    assert O.traffic_match_fused(c0, L, 4, 8, 3)
    assert not O.traffic_match_fused(c0, L + 1, 4, 8, 3)


def test_errors_empty_cache_and_zero_tile():
    rng = O.Rng(360)
    lay = O.random_layer(rng, 16, 4, [[2, 2, 2]] * 2)
    ck = np.zeros((2, 4, 2))
    with pytest.raises(ValueError, match="ShapeError"):
        O.fused_decode_step(lay, ck, ck, 0, np.zeros((2, 4)), 4)
    with pytest.raises(ValueError, match="ConfigError"):
        O.fused_decode_step(lay, ck, ck, 2, np.zeros((2, 4)), 0)


def test_int_path_rules():
    # quant.cpp:34-37 and the composed int8 rules of SURVEY Appendix A
    assert O.lib().orc_qmax(8) == 127 and O.lib().orc_qmax(4) == 7
    v = np.array([0.5, -1.5, 2.5, 127.0], dtype=np.float32)
    q, s = O.quant_token(v)
    assert s == np.float32(1.0) and list(q) == [1, -2, 3, 127]  # ties away from zero
    q, s = O.quant_token(np.zeros(8, dtype=np.float32))
    assert s == 1.0 and (q == 0).all()
    q, h = O.quant_cache_row(np.array([0.0, 254.0, -127.0], dtype=np.float32))
    assert O.f16_to_f32(h) == 2.0 and list(q) == [0, 127, -64]
    q, h = O.quant_cache_row(np.zeros(4, dtype=np.float32))
    assert h == 0x3C00 and (q == 0).all()
    packed = np.array([0x8F, 0x71], dtype=np.uint8)  # (-1, -8), (1, 7)
    out = np.zeros(4, dtype=np.int8)
    import ctypes as C
    O.lib().orc_unpack_int4(packed.ctypes.data_as(C.POINTER(C.c_uint8)), 4, out.ctypes.data_as(O._i8p))
    assert list(out) == [-1, -8, 1, 7]


def test_oracle_decode_factored_device_storage_close_to_reference():
    """the oracle's decode_factored: its device-storage variant stays within a
    few bf16 ulps of the plain fp64 composition (the bf16 storage is the only
    difference) -- a CPU-side sanity check of the restatement"""
    from paper_2604_02570_b200.stack import toy_ffn_weights  # noqa: F401 (numpy only)
    rng = O.Rng(1)
    E, nh, H, r, F = 256, 2, 128, 32, 512
    lbs = [O.random_layer(rng, E, H, [[r, r, r]] * nh).map(O.bf16_round) for _ in range(2)]
    wos = [O.bf16_round(rng.normal_matrix(nh * H, E, 1 / np.sqrt(E))) for _ in range(2)]
    ffn = [toy_ffn_weights(E, F, i) for i in range(2)]
    xs = O.bf16_round(rng.normal_matrix(4, E))
    a = O.decode_factored(lbs, wos, ffn, xs)
    b = O.decode_factored(lbs, wos, ffn, xs, device_storage=True, rpad=32)
    assert np.abs(a - b).max() <= 2 ** -6 * np.abs(a).max()
