"""GPU parity of the composed integer path (W8A8 / W4A8 weights, INT8 latent
cache) against the oracle's restatement.

Bit-exact: the rotated+quantised tokens and their scales, the int32
projection accumulators, and the int8 cache rows with their fp16 scales.
Within the north_star tolerance (1e-3 relative per head row): the query
q_h and the attention outputs (fp32 arithmetic on dequantised values)."""
from __future__ import annotations

import math
import os
import subprocess
import sys

import numpy as np
import pytest
import scipy.linalg

from oracle import oracle as O
from tests.helpers import REL_TOL, rel_err_rows, to_factors

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
torch = pytest.importorskip("torch")


def rotate_rows(a, E):
    """S1 . a with S1 = blockdiag(H_blk / sqrt(blk)) (linalg.cpp:219-243; block H_128 for E = 5120)."""
    blk = int(O.lib().orc_rot_block(E))
    h = scipy.linalg.hadamard(blk) / math.sqrt(blk)
    out = np.empty_like(a)
    for b0 in range(0, E, blk):
        out[b0:b0 + blk] = h @ a[b0:b0 + blk]
    return out


def quant_layer(lay, bits):
    """QuantizedFactors-style int factors: Q(S1 A), Q(B) (quant.cpp:344-352, S2 = I)."""
    quant, deq_b = [], np.zeros_like(lay.B)
    for h in range(lay.nh):
        roles = []
        for role in range(3):
            r = int(lay.ranks[h, role])
            aq, as_, _ = O.quantize_weight(rotate_rows(lay.A[h, role, :, :r], lay.E), bits)
            bq, bs, _ = O.quantize_weight(lay.B[h, role, :r, :], bits)
            roles.append((aq, as_, bq, bs))
            deq_b[h, role, :r, :] = bq.astype(np.float64) * bs.astype(np.float32).astype(np.float64)
        quant.append(roles)
    return quant, deq_b


@pytest.mark.parametrize("E,nh,r,H,B,L,bits", [
    (512, 4, 32, 128, 3, 70, 8),     # W8A8, power-of-two S1
    (640, 2, 48, 128, 2, 40, 4),     # W4A8, block-Hadamard S1 (5 x H_128), rank 48
    (4096, 32, 32, 128, 4, 24, 8),   # config-3 shape (fewer sequences / tokens)
    (5120, 2, 48, 128, 2, 12, 4),    # config-4 width: block H_128 rotation in the fast quantiser
])
def test_int_path_bit_exact_and_attention_parity(E, nh, r, H, B, L, bits):
    from paper_2604_02570_b200.layer import DecodeLayer
    rng = O.Rng(900 + E + bits)
    lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
    quant, deq_b = quant_layer(lay, bits)
    f = to_factors(lay)
    wd = "i8" if bits == 8 else "i4"
    layer = DecodeLayer(f, None, batch=B, capacity=L + 8, cache_dtype="i8", weight_dtype=wd,
                        quantized=quant)
    R = layer.rpad
    dev = torch.device("cuda", 0)
    toks = rng.normal_matrix(L * B, E).reshape(L, B, E).astype(np.float32)
    q = torch.empty((B, nh, H), device=dev)
    for t in range(L):
        layer.append(torch.from_numpy(toks[t]).to(dev), q)
    torch.cuda.synchronize()

    # ---- the last token, re-derived by the oracle with the device's fp32 op order
    xq_dev = layer.debug_copy("xq").reshape(B, -1)
    sx_dev = layer.debug_copy("sx")
    acc_dev = layer.debug_copy("acc").reshape(B, nh * 3 * R)
    for b in range(B):
        xr = O.rotate_token(toks[-1, b])
        xq, sx = O.quant_token(xr)
        assert (xq_dev[b, :E] == xq).all() and (xq_dev[b, E:] == 0).all()
        assert sx_dev[b] == sx
        for h in range(nh):
            for role in range(3):
                aq, as_, _, _ = quant[h][role]
                acc = O.int_gemv(xq, np.ascontiguousarray(aq.T))
                got = acc_dev[b, (h * 3 + role) * R:(h * 3 + role) * R + r]
                assert (got == acc).all(), f"int32 accumulators differ (b={b} h={h} role={role})"

    # ---- int8 cache rows + fp16 scales, every token (oracle quantiser, Appendix A.4)
    lat_ref = np.zeros((B, nh, L, 2, R))  # dequantised oracle cache
    for b in range(B):
        for h in range(nh):
            rows, scales = layer.read_raw(b, h)
            rows = rows.view(np.int8)
            for t in range(L):
                xq, sx = O.quant_token(O.rotate_token(toks[t, b]))
                for part, role in ((0, 1), (1, 2)):
                    aq, as_, _, _ = quant[h][role]
                    acc = O.int_gemv(xq, np.ascontiguousarray(aq.T))
                    c = np.array([O.dequant_latent(acc[i], sx, np.float32(as_[i])) for i in range(r)]
                                 + [0.0] * (R - r), dtype=np.float32)
                    qv, hs = O.quant_cache_row(c)
                    assert (rows[t, part * R:(part + 1) * R] == qv).all(), f"cache row b={b} h={h} t={t}"
                    assert scales[t, part] == hs
                    lat_ref[b, h, t, part] = qv.astype(np.float64) * float(O.f16_to_f32(hs))

    # ---- query and attention within tolerance
    q_dev = q.cpu().numpy().astype(np.float64)
    out = torch.empty((B, nh, H), device=dev)
    layer.attend(q, out)
    torch.cuda.synchronize()
    out = out.cpu().numpy().astype(np.float64)
    deq = O.Layer(lay.A, deq_b, lay.ranks)
    for b in range(B):
        # q_h = c_Q . dequant(B_Q) from the exact dequantised latents
        xq, sx = O.quant_token(O.rotate_token(toks[-1, b]))
        q_ref = np.zeros((nh, H))
        for h in range(nh):
            aq, as_, _, _ = quant[h][0]
            acc = O.int_gemv(xq, np.ascontiguousarray(aq.T))
            cq = np.array([O.dequant_latent(acc[i], sx, np.float32(as_[i])) for i in range(r)], dtype=np.float64)
            q_ref[h] = cq @ deq_b[h, 0, :r, :]
        assert rel_err_rows(q_dev[b], q_ref) <= REL_TOL
        ck = np.ascontiguousarray(lat_ref[b, :, :, 0, :r])
        cv = np.ascontiguousarray(lat_ref[b, :, :, 1, :r])
        ref = O.fused_decode_step(deq, ck, cv, L, q_dev[b], 32)
        assert rel_err_rows(out[b], ref) <= REL_TOL


def test_layer_step_int8_matches_append_plus_attend():
    """The fused layer step (graph path: M_QK fold, split-KV, folded W_o) on
    an I8 layer equals append + fused_decode_step + O-projection."""
    from paper_2604_02570_b200.layer import DecodeLayer
    rng = O.Rng(77)
    E, nh, r, H, B, L = 512, 4, 32, 128, 2, 50
    lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
    quant, deq_b = quant_layer(lay, 8)
    f = to_factors(lay)
    w_o = O.bf16_round(rng.normal_matrix(nh * H, E, 1.0 / np.sqrt(E)))
    dev = torch.device("cuda", 0)
    toks = rng.normal_matrix(L * B, E).reshape(L, B, E).astype(np.float32)
    a = DecodeLayer(f, w_o, batch=B, capacity=L + 8, cache_dtype="i8", weight_dtype="i8", quantized=quant)
    b_ = DecodeLayer(f, w_o, batch=B, capacity=L + 8, cache_dtype="i8", weight_dtype="i8", quantized=quant)
    for t in range(L - 1):
        xt = torch.from_numpy(toks[t]).to(dev)
        a.append(xt)
        b_.append(xt)
    x = torch.from_numpy(toks[-1]).to(dev)
    y = torch.empty((B, E), device=dev)
    attn = torch.empty((B, nh, H), device=dev)
    a.step(x, y, attn_out=attn, graph=False)
    q = torch.empty((B, nh, H), device=dev)
    b_.append(x, q)
    out = torch.empty((B, nh, H), device=dev)
    b_.attend(q, out)
    torch.cuda.synchronize()
    assert rel_err_rows(attn.cpu().numpy(), out.cpu().numpy()) <= REL_TOL
    y_ref = out.cpu().numpy().reshape(B, -1).astype(np.float64) @ w_o
    assert np.abs(y.cpu().numpy() - y_ref).max() <= 1e-2 * np.abs(y_ref).max()


@pytest.mark.parametrize("r,L,chunk,variant", [
    (32, 2500, None, None),     # 1024-token stages (int8 P.V on the int8 tensor cores), ragged tail
    (32, 4100, "1024", None),   # one stage per chunk, a 4-token last chunk
    (32, 3000, None, "16"),     # the f16 P.V consumer on 1024-token stages
    (32, 2100, None, "32"),     # int8 P.V on 512-token stages
    (48, 1800, None, None),     # r = 48: half k-step scores, 512-token stages
    (16, 3000, None, None),
])
def test_int8_cache_attention_long_context(monkeypatch, r, L, chunk, variant):
    """INT8-cache attention over multi-stage contexts (the short-context cases
    above fit in one stage) against the oracle's fused_decode_step on the
    dequantised cache rows read back from the device."""
    if variant is not None and os.environ.get("WSVD_ATTN_VARIANT") != variant:
        # the variant switch is read once per process: run this case in a child
        env = dict(os.environ, WSVD_ATTN_VARIANT=variant)
        node = f"{__file__}::test_int8_cache_attention_long_context[{r}-{L}-{chunk}-{variant}]"
        res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", node],
                             env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
        assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
        return
    if chunk is not None:
        monkeypatch.setenv("WSVD_ATTN_CHUNK", chunk)
    from paper_2604_02570_b200.layer import DecodeLayer
    E, nh, H, B = 256, 4, 128, 2
    rng = O.Rng(4000 + r + L)
    lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
    quant, deq_b = quant_layer(lay, 8)
    layer = DecodeLayer(to_factors(lay), None, batch=B, capacity=L + 8, cache_dtype="i8", weight_dtype="i8",
                        quantized=quant)
    R = layer.rpad
    dev = torch.device("cuda", 0)
    layer.fill_synthetic(L - 1, seed=r + L)
    x = torch.from_numpy(rng.normal_matrix(B, E).astype(np.float32)).to(dev)
    q = torch.empty((B, nh, H), device=dev)
    layer.append(x, q)
    out = torch.empty((B, nh, H), device=dev)
    layer.attend(q, out)
    torch.cuda.synchronize()
    q_dev, out = q.cpu().numpy().astype(np.float64), out.cpu().numpy().astype(np.float64)
    deq = O.Layer(lay.A, deq_b, lay.ranks)
    for b in range(B):
        ck, cv = np.zeros((nh, L, r)), np.zeros((nh, L, r))
        for h in range(nh):
            rows, scales = layer.read_raw(b, h)
            rows = rows.view(np.int8).astype(np.float64)
            sk = np.array([O.f16_to_f32(s) for s in scales[:, 0]], dtype=np.float64)
            sv = np.array([O.f16_to_f32(s) for s in scales[:, 1]], dtype=np.float64)
            ck[h] = rows[:, :r] * sk[:, None]
            cv[h] = rows[:, R:R + r] * sv[:, None]
        ref = O.fused_decode_step(deq, ck, cv, L, q_dev[b], 32)
        assert rel_err_rows(out[b], ref) <= REL_TOL, f"b={b}"


@pytest.mark.parametrize("cache,B,nh,L,r", [
    ("i8", 37, 4, 300, 32), ("f32", 37, 4, 300, 32),   # 148 pairs = one per CTA: one chunk, helper-warp merge
    ("f32", 1, 32, 300, 32), ("i8", 1, 32, 300, 32),   # 32 pairs: 4-CTA clusters, chunks merged through DSMEM
    ("f32", 1, 32, 40, 32),                            # ... with two empty trailing chunks
    ("i8", 2, 8, 500, 48),                             # 16 pairs: 8-CTA clusters, r = 48
    ("f32", 3, 16, 257, 16),                           # 48 pairs: 2-CTA clusters, r = 16
])
def test_layer_step_in_kernel_merge(cache, B, nh, L, r):
    """The layer step's attention merges its split-KV partials inside the
    kernel -- one chunk per pair (helper warp), or one cluster of CTAs per pair
    (DSMEM) -- with no combine launch: the layer step's y must equal append +
    attend (combine kernel, full-rank output) followed by the O-projection."""
    from paper_2604_02570_b200.layer import DecodeLayer
    rng = O.Rng(91 + B + L)
    E, H = 512, 128
    lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
    f = to_factors(lay)
    w_o = O.bf16_round(rng.normal_matrix(nh * H, E, 1.0 / np.sqrt(nh * H)))
    kw = dict(batch=B, capacity=L + 8, cache_dtype=cache)
    if cache == "i8":
        quant, _ = quant_layer(lay, 8)
        kw.update(weight_dtype="i8", quantized=quant)
    else:
        kw.update(weight_dtype="f32")
    a = DecodeLayer(f, w_o, **kw)
    b_ = DecodeLayer(f, w_o, **kw)
    dev = torch.device("cuda", 0)
    toks = rng.normal_matrix(L * B, E).reshape(L, B, E).astype(np.float32)
    pre = torch.from_numpy(toks[:L - 1]).to(dev)
    a.prefill(pre)
    b_.prefill(pre)
    x = torch.from_numpy(toks[-1]).to(dev)
    y = torch.empty((B, E), device=dev)
    a.step(x, y, graph=False)
    q = torch.empty((B, nh, H), device=dev)
    b_.append(x, q)
    out = torch.empty((B, nh, H), device=dev)
    b_.attend(q, out)
    torch.cuda.synchronize()
    y_ref = out.cpu().numpy().reshape(B, -1).astype(np.float64) @ w_o
    assert np.abs(y.cpu().numpy() - y_ref).max() <= 1e-2 * np.abs(y_ref).max()


@pytest.mark.parametrize("r,L", [(32, 1500), (48, 300), (96, 260)])
def test_int8_attention_score_accumulators_bit_exact(r, L):
    """the int8 attention scores every cached row against
    the absorbed query split into int8 hi / lo parts (attn.cu consume_imma_i8 at
    r = 32, consume_mma_i8 above); the oracle restates the split
    (orc_i8_query_split) and the int32 accumulators must agree exactly for
    every row of every (sequence, head)."""
    from paper_2604_02570_b200.layer import DecodeLayer
    rng = O.Rng(7700 + r)
    E, nh, H, B = 512, 4, 128, 2
    lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
    quant, _ = quant_layer(lay, 8)
    layer = DecodeLayer(to_factors(lay), None, batch=B, capacity=L + 8, cache_dtype="i8", weight_dtype="i8",
                        quantized=quant)
    R = layer.rpad
    dev = torch.device("cuda", 0)
    layer.prefill(torch.from_numpy(rng.normal_matrix(L * B, E).reshape(L, B, E).astype(np.float32)).to(dev))
    q = torch.from_numpy(rng.normal_matrix(B * nh, H).reshape(B, nh, H).astype(np.float32)).to(dev)
    out = torch.empty((B, nh, H), device=dev)
    layer.set_debug(1)
    layer.attend(q, out)
    torch.cuda.synchronize()
    qt = layer.debug_copy("qt").reshape(B, nh, R)
    acc = layer.debug_copy("scores").reshape(B, nh, -1, 2)
    for b in range(B):
        for h in range(nh):
            rows, _ = layer.read_raw(b, h)
            ref = O.i8_scores(qt[b, h], rows.view(np.int8), R)
            assert np.array_equal(acc[b, h, :L], ref), f"int32 score accumulators differ (b={b} h={h})"
