"""Generates tests/golden/reference_vectors.npz from the REFERENCE itself
(oracle/_ref/libwsvdref.so, compiled from /root/reference/proj/src by
oracle/Makefile) so the oracle can be pinned on machines where the reference
tree does not exist.  Run here (where /root/reference exists):

    make -f oracle/Makefile && python tests/golden/make_golden.py

Every array is produced by a reference API call (see oracle/ref_shim.cpp):
decode::append_token / fused_decode_step, quant::quantize_weight /
quantize_activation, hadamard, and Rng streams.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.npz")


def ref_append_decode(lay, toks, tile):
    R = O.ref()
    nh, rmax, H, E = lay.nh, lay.rmax, lay.H, lay.E
    L = toks.shape[0]
    ck = np.zeros((nh, L, rmax))
    cv = np.zeros((nh, L, rmax))
    q = np.zeros((nh, H))
    out = np.zeros((nh, H))
    a21 = np.zeros(21, dtype=np.uint64)
    d21 = np.zeros(21, dtype=np.uint64)
    lay.c()
    rc = R.ref_append_then_decode(E, H, nh, rmax, lay.ranks.ctypes.data_as(O._ip),
                                  lay.A.ctypes.data_as(O._dp), lay.B.ctypes.data_as(O._dp), L,
                                  np.ascontiguousarray(toks).ctypes.data_as(O._dp), tile,
                                  ck.ctypes.data_as(O._dp), cv.ctypes.data_as(O._dp),
                                  q.ctypes.data_as(O._dp), out.ctypes.data_as(O._dp),
                                  a21.ctypes.data_as(O._u64p), d21.ctypes.data_as(O._u64p))
    assert rc == 0, R.ref_last_error()
    return ck, cv, q, out, a21, d21


def main():
    R = O.ref()
    g = {}
    # decode-bench recipe (wsvd_main.cpp:360-397) at a toy shape
    lay = O.bench_layer(64, 16, 4, 8, seed=0)
    toks = O.Rng.stream(0, 1000).normal_matrix(40, 64)
    ck, cv, q, out, a21, d21 = ref_append_decode(lay, toks, 32)
    g.update(bench_A=lay.A, bench_B=lay.B, bench_ranks=lay.ranks, bench_tokens=toks, bench_ck=ck,
             bench_cv=cv, bench_q=q, bench_out=out, bench_append_counter=a21,
             bench_decode_counter=d21)
    # ragged ranks (test_decode.cpp:179-204 style), tile 5
    rng = O.Rng(310)
    ranks = [[1 + rng.index(8), 1 + rng.index(8), 1 + rng.index(8)] for _ in range(3)]
    lay2 = O.random_layer(rng, 32, 8, ranks)
    toks2 = rng.normal_matrix(13, 32)
    ck, cv, q, out, a21, d21 = ref_append_decode(lay2, toks2, 5)
    g.update(ragged_A=lay2.A, ragged_B=lay2.B, ragged_ranks=lay2.ranks, ragged_tokens=toks2,
             ragged_ck=ck, ragged_cv=cv, ragged_q=q, ragged_out=out, ragged_append_counter=a21,
             ragged_decode_counter=d21)
    # quantizers (quant.cpp:99-150)
    w = O.Rng(81).normal_matrix(48, 12, 0.3)
    w[:, 3] = 0.0  # a zero column -> scale 1
    for bits in (8, 4):
        qv = np.zeros(w.shape, dtype=np.int8)
        s = np.zeros(w.shape[1])
        clip = R.ref_quantize_weight(w.ctypes.data_as(O._dp), 48, 12, bits, qv.ctypes.data_as(O._i8p),
                                     s.ctypes.data_as(O._dp))
        g[f"qw{bits}_q"], g[f"qw{bits}_s"], g[f"qw{bits}_clip"] = qv, s, np.float64(clip)
    g["qw_w"] = w
    x = O.Rng(82).normal_matrix(5, 24, 2.0)
    x[2, :] = 0.0
    qa = np.zeros(x.shape, dtype=np.int8)
    sa = np.zeros(5)
    R.ref_quantize_activation(x.ctypes.data_as(O._dp), 5, 24, 8, qa.ctypes.data_as(O._i8p),
                              sa.ctypes.data_as(O._dp))
    g.update(qa_x=x, qa_q=qa, qa_s=sa)
    # hadamard (linalg.cpp:219-243)
    h = np.zeros((16, 16))
    R.ref_hadamard(16, h.ctypes.data_as(O._dp))
    g["hadamard16"] = h
    # rng streams (rng.cpp)
    u = np.zeros(64, dtype=np.uint64)
    R.ref_rng_u64s(42, 64, u.ctypes.data_as(O._u64p))
    n = np.zeros(65)
    R.ref_rng_normals(7, 5, 1, 65, 0.5, n.ctypes.data_as(O._dp))
    idx = np.zeros(32, dtype=np.uint64)
    R.ref_rng_indices(9, 11, 32, idx.ctypes.data_as(O._u64p))
    g.update(rng_u64_seed42=u, rng_normal_seed7_stream5_std05=n, rng_index_seed9_bound11=idx)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
