"""GPU parity of the explicit key-reconstruction attention on tcgen05 tensor
cores (attn_tc.cu, WSVD_ATTN_EXPLICIT_TC) against the CPU oracle.

The reference rebuilds every key, key_j = C_K[j] . B_K (src/decode.cpp:188),
and attends with the raw query; the explicit mode runs exactly that contraction
on tcgen05 (C_K tile x B_K^T tile -> TMEM) and must give the oracle's result
on the rows the device stores, within the north_star tolerance (1e-3 max
relative error per head row), for every stage shape (partial 128-token tiles,
partial stages, split-KV chunks)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_2604_02570_b200.errors import ConfigError
from tests.helpers import REL_TOL, rel_err_rows, to_factors

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _layer(E, nh, H, r, B, cap, seed, cache_dtype="bf16", weight_dtype="bf16", w_o=False):
    from paper_2604_02570_b200.layer import DecodeLayer
    rng = O.Rng(seed)
    lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
    wo = O.bf16_round(rng.normal_matrix(nh * H, E, 1.0 / np.sqrt(E))) if w_o else None
    layer = DecodeLayer(to_factors(lay), wo, batch=B, capacity=cap, cache_dtype=cache_dtype,
                        weight_dtype=weight_dtype)
    return rng, lay, layer, wo


@pytest.mark.parametrize("L", [1, 7, 128, 129, 256, 300, 1100])
def test_explicit_tc_matches_oracle(L):
    E, nh, H, r, B = 256, 4, 128, 32, 3
    rng, lay, layer, _ = _layer(E, nh, H, r, B, L + 8, 7000 + L)
    layer.set_attention("explicit_tc")
    assert layer.attention == "explicit_tc"
    dev = torch.device("cuda", 0)
    toks = O.bf16_round(rng.normal_matrix(L * B, E)).reshape(L, B, E).astype(np.float32)
    layer.prefill(torch.from_numpy(toks).to(dev))
    q = rng.normal_matrix(B * nh, H).reshape(B, nh, H)
    qd = torch.from_numpy(q.astype(np.float32)).to(dev)
    out = torch.empty((B, nh, H), device=dev)
    layer.attend(qd, out)
    torch.cuda.synchronize()
    out = out.cpu().numpy().astype(np.float64)
    lb = lay.map(O.bf16_round)
    q32 = q.astype(np.float32).astype(np.float64)
    for b in range(B):
        ck = np.stack([layer.read_latents(b, h)[0] for h in range(nh)])
        cv = np.stack([layer.read_latents(b, h)[1] for h in range(nh)])
        ref = O.fused_decode_step(lb, np.ascontiguousarray(ck), np.ascontiguousarray(cv), L, q32[b], 32)
        assert rel_err_rows(out[b], ref) <= REL_TOL, f"b={b}"
    # the absorbed kernel on the same cache agrees too
    layer.set_attention("absorbed")
    out2 = torch.empty((B, nh, H), device=dev)
    layer.attend(qd, out2)
    torch.cuda.synchronize()
    assert rel_err_rows(out2.cpu().numpy().astype(np.float64), out) <= REL_TOL


def test_explicit_tc_split_kv_chunks(monkeypatch):
    """fixed 96-token chunks: many partial tiles and a merge over chunks"""
    monkeypatch.setenv("WSVD_ATTN_CHUNK", "96")
    E, nh, H, r, B, L = 128, 2, 128, 32, 2, 500
    rng, lay, layer, _ = _layer(E, nh, H, r, B, L + 8, 7100)
    layer.set_attention("explicit_tc")
    dev = torch.device("cuda", 0)
    toks = O.bf16_round(rng.normal_matrix(L * B, E)).reshape(L, B, E).astype(np.float32)
    layer.prefill(torch.from_numpy(toks).to(dev))
    q = rng.normal_matrix(B * nh, H).reshape(B, nh, H)
    out = torch.empty((B, nh, H), device=dev)
    layer.attend(torch.from_numpy(q.astype(np.float32)).to(dev), out)
    torch.cuda.synchronize()
    out = out.cpu().numpy().astype(np.float64)
    lb = lay.map(O.bf16_round)
    for b in range(B):
        ck = np.stack([layer.read_latents(b, h)[0] for h in range(nh)])
        cv = np.stack([layer.read_latents(b, h)[1] for h in range(nh)])
        ref = O.fused_decode_step(lb, ck, cv, L, q[b].astype(np.float32).astype(np.float64), 32)
        assert rel_err_rows(out[b], ref) <= REL_TOL


def test_explicit_tc_append_and_layer_step():
    """append_token's own q (pipeline.cpp:320-322) through the explicit kernel,
    and the whole layer step (append, explicit attention, O-projection) against
    the absorbed fused step on a twin cache"""
    E, nh, H, r, B, L = 512, 8, 128, 32, 4, 333
    rng, lay, tc, wo = _layer(E, nh, H, r, B, L + 8, 7200, w_o=True)
    _, _, ab, _ = _layer(E, nh, H, r, B, L + 8, 7200, w_o=True)
    tc.set_attention("explicit_tc")
    dev = torch.device("cuda", 0)
    toks = O.bf16_round(rng.normal_matrix((L + 1) * B, E)).reshape(L + 1, B, E).astype(np.float32)
    pre = torch.from_numpy(toks[:L]).to(dev)
    tc.prefill(pre)
    ab.prefill(pre)
    x = torch.from_numpy(toks[L]).to(dev)
    y_tc = torch.empty((B, E), device=dev)
    y_ab = torch.empty((B, E), device=dev)
    tc.step(x, y_tc)
    ab.step(x, y_ab)
    torch.cuda.synchronize()
    assert tc.length() == ab.length() == L + 1
    assert rel_err_rows(y_tc.cpu().numpy(), y_ab.cpu().numpy()) <= 1e-3
    # append + attention through the reference-shaped operators
    q = torch.empty((B, nh, H), device=dev)
    out = torch.empty((B, nh, H), device=dev)
    x2 = torch.from_numpy(O.bf16_round(rng.normal_matrix(B, E)).astype(np.float32)).to(dev)
    tc.append(x2, q)
    tc.attention_only(out)
    out_q = torch.empty((B, nh, H), device=dev)
    tc.attend(q, out_q)
    torch.cuda.synchronize()
    assert rel_err_rows(out.cpu().numpy(), out_q.cpu().numpy()) <= 1e-6


def test_explicit_tc_rejects_unsupported_caches():
    _, _, layer, _ = _layer(256, 2, 128, 32, 1, 16, 7300, cache_dtype="f32", weight_dtype="f32")
    with pytest.raises(ConfigError):
        layer.set_attention("explicit_tc")
    _, _, layer, _ = _layer(256, 2, 128, 16, 1, 16, 7301)
    with pytest.raises(ConfigError):
        layer.set_attention("explicit_tc")
