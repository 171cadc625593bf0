"""Parity of the BENCHMARKED layer step at the exact BASELINE.json shapes
(configs 1-4), against the CPU oracle, at the north_star tolerance.

What runs on the device is exactly what bench.py times: one
``wsvd_layer_step_graph`` call (the fused persistent ``layer_step_kernel`` for
config 2; the multi-kernel step for the fp32 and integer configs) for every
sequence of a cache filled with ``L - 1`` synthetic latent rows
(``wsvd_cache_fill_synthetic``, the bench's prefill), with the decode-bench
factor recipe (``tools/wsvd_main.cpp:360-391``, ``oracle.bench_layer``).

The oracle then re-derives, for a sample of the sequences (all heads):

* the new token's latent row and query: ``decode::append_token``
  (``src/decode.cpp:127-153``) -- fp64 on the device-rounded factors for the
  float formats; the integer stages of SURVEY Appendix A (rotation, per-token
  int8, int32 accumulators, cache-row quantiser) for W8A8 / W4A8, whose
  cache rows must be bit-identical;
* the attention over the device's cache rows with that query:
  ``decode::fused_decode_step`` (``src/decode.cpp:155-206``), keeping the
  latent output v~ = acc / denom (``:198``);
* the O-projection ``heads_row . W_o`` (``src/pipeline.cpp:323-329``) as
  ``v~ . W'_o`` with ``W'_o = blockdiag(B_V) . W_o`` folded from the stored
  factor values and rounded to the device's bf16 storage -- the same product
  in real arithmetic; only where the weight rounding happens moves.

y must match within REL_TOL = 1e-3 (max |gpu - ref| / max |ref| per row).
"""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import REL_TOL, rel_err_rows, to_factors

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")
THREADS = os.cpu_count() or 4

CONFIGS = {
    # name: E, nh, H, r, B, L, cache, weights, sampled sequences
    "config1-7b-r32-b1-ctx2k-f32": (4096, 32, 128, 32, 1, 2048, "f32", "f32", [0]),
    "config2-7b-r32-b16-ctx4k-bf16": (4096, 32, 128, 32, 16, 4096, "bf16", "bf16", [0, 7, 15]),
    "config3-7b-r32-b32-ctx4k-w8a8-i8": (4096, 32, 128, 32, 32, 4096, "i8", "i8", [0, 31]),
    "config4-13b-r48-b64-ctx8k-w4a8-i8": (5120, 40, 128, 48, 64, 8192, "i8", "i4", [0, 63]),
}


def _rotate_rows(a, E):
    import scipy.linalg
    blk = int(O.lib().orc_rot_block(E))
    h = scipy.linalg.hadamard(blk) / math.sqrt(blk)
    out = np.empty_like(a)
    for b0 in range(0, E, blk):
        out[b0:b0 + blk] = h @ a[b0:b0 + blk]
    return out


def _quant_layer(lay, bits):
    """Q(S1 A), Q(B) per head and role (quant.cpp:344-352, S2 = I) and the
    dequantised B values the device folds from (int8 * float32(scale))."""
    quant, deq_b = [], np.zeros_like(lay.B)
    for h in range(lay.nh):
        roles = []
        for role in range(3):
            r = int(lay.ranks[h, role])
            aq, as_, _ = O.quantize_weight(_rotate_rows(lay.A[h, role, :, :r], lay.E), bits)
            bq, bs, _ = O.quantize_weight(lay.B[h, role, :r, :], bits)
            roles.append((aq, as_, bq, bs))
            deq_b[h, role, :r, :] = bq.astype(np.float64) * bs.astype(np.float32).astype(np.float64)
        quant.append(roles)
    return quant, deq_b


def _int_new_token(quant, x32, nh, r, R):
    """Appendix A.1-A.4 for one token: (c_Q, int8 K|V cache rows, fp16 scales, dequantised rows)."""
    xq, sx = O.quant_token(O.rotate_token(x32))
    cq = np.zeros((nh, r))
    rows = np.zeros((nh, 2, R), dtype=np.int8)
    hs = np.zeros((nh, 2), dtype=np.uint16)
    deq = np.zeros((nh, 2, R))
    for h in range(nh):
        for role in range(3):
            aq, as_, _, _ = quant[h][role]
            acc = O.int_gemv(xq, np.ascontiguousarray(aq.T))
            c = np.array([O.dequant_latent(acc[i], sx, np.float32(as_[i])) for i in range(r)], dtype=np.float32)
            if role == 0:
                cq[h] = c
                continue
            cpad = np.zeros(R, dtype=np.float32)
            cpad[:r] = c
            qv, s16 = O.quant_cache_row(cpad)
            rows[h, role - 1], hs[h, role - 1] = qv, s16
            deq[h, role - 1] = qv.astype(np.float64) * float(O.f16_to_f32(s16))
    return cq, rows, hs, deq


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_layer_step_at_baseline_shape(name):
    from paper_2604_02570_b200.layer import DecodeLayer
    E, nh, H, r, B, L, cache, weights, sample = CONFIGS[name]
    lay = O.bench_layer(E, H, nh, r)  # decode-bench recipe, seed 0
    rng = O.Rng.stream(0, 7)
    w_o = rng.normal_matrix(nh * H, E, 1.0 / math.sqrt(E))  # toymodel.cpp:81,90
    quant = None
    if weights in ("i8", "i4"):
        quant, deq_b = _quant_layer(lay, 8 if weights == "i8" else 4)
        ref_lay = O.Layer(lay.A, deq_b, lay.ranks)
    else:
        ref_lay = lay.map(O.bf16_round if weights == "bf16" else O.f32_round)
    layer = DecodeLayer(to_factors(lay), w_o, batch=B, capacity=L + 8, cache_dtype=cache,
                        weight_dtype=weights, oproj_dtype="bf16", quantized=quant)
    R = layer.rpad
    layer.fill_synthetic(L - 1, seed=11)
    dev = torch.device("cuda", 0)
    x = rng.normal_matrix(B, E)
    if weights == "bf16":
        x = O.bf16_round(x)  # config 2: bf16 activations
    x32 = x.astype(np.float32)
    y = torch.empty((B, E), device=dev)
    layer.step(torch.from_numpy(x32).to(dev), y)
    torch.cuda.synchronize()
    assert layer.length() == L
    y = y.cpu().numpy().astype(np.float64)

    nsamp = len(sample)
    ck = np.zeros((nsamp, nh, L, R))
    cv = np.zeros((nsamp, nh, L, R))
    q = np.zeros((nsamp, nh, H))
    for i, b in enumerate(sample):
        for h in range(nh):
            ck[i, h], cv[i, h] = layer.read_latents(b, h)
        if quant is None:
            # decode::append_token in fp64 on the stored factor values
            nk, nv = np.zeros((nh, 1, R)), np.zeros((nh, 1, R))
            q[i] = O.append_token(ref_lay, nk, nv, 0, O.f32_round(x32[b].astype(np.float64)))
            for part, new in ((ck, nk), (cv, nv)):
                got, want = part[i, :, L - 1], new[:, 0]
                tol = (2 ** -8 if cache == "bf16" else 2 ** -20) * np.abs(want).max()
                assert np.abs(got - want).max() <= tol, f"new latent row of sequence {b}"
        else:
            cq, rows, hs, deq = _int_new_token(quant, x32[b], nh, r, R)
            for h in range(nh):
                raw, sc = layer.read_raw(b, h)
                assert (raw[L - 1].view(np.int8) == rows[h].reshape(-1)).all(), f"int8 row b={b} h={h}"
                assert (sc[L - 1] == hs[h]).all(), f"fp16 scales b={b} h={h}"
                q[i, h] = cq[h] @ deq_b[h, 0, :r, :]
            assert np.array_equal(ck[i, :, L - 1], deq[:, 0]) and np.array_equal(cv[i, :, L - 1], deq[:, 1])
    out, lat = O.batched_decode_latent(ref_lay, ck, cv, L, q, 32, THREADS)
    wo_fold = O.fold_oproj(ref_lay, w_o, R, O.bf16_round)
    for i, b in enumerate(sample):
        y_ref = lat[i].reshape(-1) @ wo_fold
        err = rel_err_rows(y[b:b + 1], y_ref[None])
        assert err <= REL_TOL, f"{name}: y of sequence {b}: rel err {err:.2e}"


def test_chain_at_config2_shape():
    """The benchmarked 8-layer chain form at the config-2 shape, reduced to 3
    layers (E = 4096, 32 heads, B = 16, L = 4096: 11 projection items per CTA,
    7 of them parked in the attention ring and re-parked across layers during
    each layer's tail): every layer equals a single-layer step on the chain's
    own input bit for bit (cache rows and y), and the last layer's y is within
    the north_star 1e-3 of the oracle on its device input."""
    from paper_2604_02570_b200.layer import DecodeChain, DecodeLayer
    E, nh, H, r, B, L, n = 4096, 32, 128, 32, 16, 4096, 3
    rng = O.Rng.stream(0, 9)
    lays, wos, a, b = [], [], [], []
    for li in range(n):
        lay = O.bench_layer(E, H, nh, r, seed=li)
        wo = rng.normal_matrix(nh * H, E, 1.0 / math.sqrt(E))
        lays.append(lay)
        wos.append(wo)
        for dst in (a, b):
            d = DecodeLayer(to_factors(lay), wo, batch=B, capacity=L + 8, cache_dtype="bf16", weight_dtype="bf16")
            d.fill_synthetic(L - 1, seed=20 + li)
            dst.append(d)
    dev = torch.device("cuda", 0)
    x = torch.from_numpy(O.bf16_round(rng.normal_matrix(B, E)).astype(np.float32)).to(dev)
    ya = [torch.empty((B, E), device=dev) for _ in range(n)]
    yb = [torch.empty((B, E), device=dev) for _ in range(n)]
    chain = DecodeChain(a)
    assert chain.fused() and chain.launches_per_step() == 1
    chain.step(x, ya)
    for li in range(n):
        b[li].step(x if li == 0 else ya[li - 1], yb[li], graph=False)
    torch.cuda.synchronize()
    for li in range(n):
        assert torch.equal(ya[li], yb[li]), f"layer {li}"
    # the last layer against the oracle, sequences 0 and 15
    li = n - 1
    ref_lay = lays[li].map(O.bf16_round)
    xin = ya[li - 1].cpu().numpy().astype(np.float64)
    yl = ya[li].cpu().numpy().astype(np.float64)
    R = a[li].rpad
    sample = [0, B - 1]
    ck = np.zeros((len(sample), nh, L, R))
    cv = np.zeros((len(sample), nh, L, R))
    q = np.zeros((len(sample), nh, H))
    for i, s in enumerate(sample):
        for h in range(nh):
            ck[i, h], cv[i, h] = a[li].read_latents(s, h)
            kb, vb = b[li].read_latents(s, h)
            assert np.array_equal(ck[i, h], kb) and np.array_equal(cv[i, h], vb)
        nk, nv = np.zeros((nh, 1, R)), np.zeros((nh, 1, R))
        q[i] = O.append_token(ref_lay, nk, nv, 0, O.bf16_round(xin[s]))
    _, lat = O.batched_decode_latent(ref_lay, ck, cv, L, q, 32, THREADS)
    wo_fold = O.fold_oproj(ref_lay, wos[li], R, O.bf16_round)
    for i, s in enumerate(sample):
        y_ref = lat[i].reshape(-1) @ wo_fold
        err = rel_err_rows(yl[s:s + 1], y_ref[None])
        assert err <= REL_TOL, f"chain layer {li}, sequence {s}: rel err {err:.2e}"
