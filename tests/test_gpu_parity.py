"""GPU parity: the sm_100a path through the reference-shaped API (and the C
ABI underneath) against the CPU oracle on identical inputs.

The fp32 cases replay the reference's own decode tests
(tests/test_decode.cpp:179-365, acceptance_main.cpp:212-274) with the
north_star tolerance (max relative error 1e-3 per head row; the reference
itself uses 1e-9 in fp64).  The bf16 cases check config-2 storage: the oracle
runs in fp64 on exactly the values the device stores (bf16-rounded factors,
tokens and latent rows read back from the device)."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2604_02570_b200 import decode as D
from paper_2604_02570_b200.errors import ConfigError, ShapeError
from tests.helpers import REL_TOL, pad_latents, rel_err_rows, to_factors

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def oracle_fill(lay, toks):
    """append every token through the oracle; returns caches and last q."""
    L = toks.shape[0]
    ck = np.zeros((lay.nh, max(L, 1), lay.rmax))
    cv = np.zeros_like(ck)
    c = O.OrcCounter()
    q = None
    for t in range(L):
        q = O.append_token(lay, ck, cv, t, toks[t], c)
    return ck, cv, q, c


# test_decode.cpp:179-204 configs: (embed, head_dim, heads, len), ragged ranks
@pytest.mark.parametrize("cfg,seed", [((16, 4, 2, 13), 310), ((32, 8, 4, 9), 311),
                                      ((24, 4, 3, 31), 312), ((32, 8, 2, 1), 313)])
def test_fused_matches_reconstruct_then_attend(cfg, seed):
    E, H, nh, L = cfg
    rng = O.Rng(seed)
    ranks = [[1 + rng.index(H), 1 + rng.index(H), 1 + rng.index(H)] for _ in range(nh)]
    lay = O.random_layer(rng, E, H, ranks)
    f = to_factors(lay)
    toks = rng.normal_matrix(L, E)
    cache = D.LatentCache(f, capacity=64)
    q = None
    for t in range(L):
        q = D.append_token(cache, f, toks[t])
    out = D.fused_decode_step(cache, f, q, D.TileConfig(5), D.TrafficCounter())
    ck, cv, q_ref, _ = oracle_fill(lay, toks)
    ref = O.reconstruct_then_attend(lay, ck, cv, L, q_ref)
    assert rel_err_rows(q, q_ref) <= REL_TOL
    assert rel_err_rows(out, ref) <= REL_TOL
    # and on the oracle's own (fp64) q: attention alone
    out2 = D.fused_decode_step(cache, f, q_ref, D.TileConfig(5), D.TrafficCounter())
    assert rel_err_rows(out2, ref) <= REL_TOL


def test_tile_size_never_changes_output_and_counters():
    # test_decode.cpp:206-227
    rng = O.Rng(320)
    L = 29
    lay = O.random_layer(rng, 32, 8, [[3, 3, 3]] * 4)
    f = to_factors(lay)
    cache = D.LatentCache(f, capacity=64)
    toks = rng.normal_matrix(L, 32)
    for t in range(L):
        q = D.append_token(cache, f, toks[t])
    c0 = D.TrafficCounter()
    ref = D.fused_decode_step(cache, f, q, D.TileConfig(L), c0)
    for tile in (1, 7, 16, L, L + 5):
        c = D.TrafficCounter()
        out = D.fused_decode_step(cache, f, q, D.TileConfig(tile), c)
        assert np.abs(out - ref).max() <= 1e-6
        assert (c.raw == c0.raw).all()


def test_counters_match_reference_identities():
    # test_decode.cpp:229-292: exact integer tallies, ragged ranks
    rng = O.Rng(330)
    E, H, L = 24, 6, 17
    ranks = [[2, 3, 4], [5, 1, 2], [3, 6, 5]]
    lay = O.random_layer(rng, E, H, ranks)
    f = to_factors(lay)
    cache = D.LatentCache(f, capacity=32)
    ca = D.TrafficCounter()
    toks = rng.normal_matrix(L, E)
    for t in range(L):
        q = D.append_token(cache, f, toks[t], ca)
    cd = D.TrafficCounter()
    D.fused_decode_step(cache, f, q, D.TileConfig(4), cd)
    ck, cv, q_ref, oa = oracle_fill(lay, toks)
    od = O.OrcCounter()
    O.fused_decode_step(lay, ck, cv, L, q_ref, 4, od)
    assert list(ca.raw) == list(oa.loads) + list(oa.stores) + list(oa.flops)
    assert list(cd.raw) == list(od.loads) + list(od.stores) + list(od.flops)
    rep = D.traffic_report(D.Mode.Fused, D.TrafficCounter(), L, 3, H, 3, 0)
    assert not rep.match
    c1 = D.TrafficCounter()
    lay2 = O.random_layer(rng, 32, 8, [[3, 3, 3]] * 4)
    f2 = to_factors(lay2)
    cache2 = D.LatentCache(f2, capacity=32)
    for t in range(19):
        q2 = D.append_token(cache2, f2, rng.normal_matrix(1, 32)[0])
    D.fused_decode_step(cache2, f2, q2, D.TileConfig(4), c1)
    assert D.traffic_report(D.Mode.Fused, c1, 19, 4, 8, 3, 0).match


def test_cache_rows_are_projected_tokens():
    # test_decode.cpp:294-310 (fp32 device: within fp32 rounding of X.A)
    rng = O.Rng(332)
    lay = O.random_layer(rng, 16, 4, [[3, 3, 3]] * 2)
    f = to_factors(lay)
    cache = D.LatentCache(f, capacity=16)
    toks = rng.normal_matrix(5, 16)
    for t in range(5):
        D.append_token(cache, f, toks[t])
    assert cache.length() == 5
    for h in range(2):
        ek = toks @ lay.A[h, 1, :, :3]
        ev = toks @ lay.A[h, 2, :, :3]
        assert np.abs(cache.latent_k(h) - ek).max() <= 1e-5 * max(1, np.abs(ek).max())
        assert np.abs(cache.latent_v(h) - ev).max() <= 1e-5 * max(1, np.abs(ev).max())


def test_single_cached_token_yields_its_value_row():
    # test_decode.cpp:312-328
    rng = O.Rng(333)
    lay = O.random_layer(rng, 16, 4, [[2, 2, 2]] * 2)
    f = to_factors(lay)
    cache = D.LatentCache(f, capacity=8)
    x = rng.normal_matrix(1, 16)
    q = D.append_token(cache, f, x[0])
    out = D.fused_decode_step(cache, f, q, D.TileConfig(), D.TrafficCounter())
    for h in range(2):
        v = (x @ lay.A[h, 2, :, :2]) @ lay.B[h, 2, :2, :]
        assert np.abs(out[h] - v[0]).max() <= 1e-5 * np.abs(v).max()


def test_errors_are_rejected():
    # test_decode.cpp:523-558
    rng = O.Rng(360)
    lay = O.random_layer(rng, 16, 4, [[2, 2, 2]] * 2)
    f = to_factors(lay)
    cache = D.LatentCache(f, capacity=8)
    q = np.zeros((2, 4))
    with pytest.raises(ShapeError):
        D.fused_decode_step(cache, f, q, D.TileConfig(), D.TrafficCounter())
    for t in range(3):
        D.append_token(cache, f, rng.normal_matrix(1, 16)[0])
    with pytest.raises(ConfigError):
        D.fused_decode_step(cache, f, q, D.TileConfig(0), D.TrafficCounter())
    with pytest.raises(ShapeError):
        D.fused_decode_step(cache, f, np.zeros((2, 5)), D.TileConfig(), D.TrafficCounter())
    other = to_factors(O.random_layer(rng, 16, 4, [[2, 2, 2]] * 3))
    with pytest.raises(ShapeError):
        D.fused_decode_step(cache, other, q, D.TileConfig(), D.TrafficCounter())
    with pytest.raises(ShapeError):
        D.LatentCache(D.LayerFactors())
    with pytest.raises(ShapeError):
        D.append_token(cache, f, np.zeros(7))
    small = D.LatentCache(f, capacity=2)
    D.append_token(small, f, rng.normal_matrix(1, 16)[0])
    D.append_token(small, f, rng.normal_matrix(1, 16)[0])
    with pytest.raises(ShapeError):
        D.append_token(small, f, rng.normal_matrix(1, 16)[0])


def test_decode_with_other_factors_of_same_geometry():
    rng = O.Rng(361)
    lay = O.random_layer(rng, 32, 8, [[4, 4, 4]] * 2)
    lay2 = O.random_layer(rng, 32, 8, [[4, 4, 4]] * 2)
    f, f2 = to_factors(lay), to_factors(lay2)
    cache = D.LatentCache(f, capacity=16)
    toks = rng.normal_matrix(6, 32)
    for t in range(6):
        q = D.append_token(cache, f, toks[t])
    out = D.fused_decode_step(cache, f2, q, D.TileConfig(), D.TrafficCounter())
    ck, cv, _, _ = oracle_fill(lay, toks)
    ref = O.reconstruct_then_attend(lay2, ck, cv, 6, q)
    assert rel_err_rows(out, ref) <= REL_TOL


@pytest.mark.parametrize("length", [1, 127, 128, 129, 300, 1000])
@pytest.mark.parametrize("chunk", ["128", "512"])
def test_split_kv_lengths(monkeypatch, length, chunk):
    """Split-KV boundaries (SoftmaxState::merge, decode.cpp:59-75): lengths
    around the 128-token stage and the chunk size."""
    monkeypatch.setenv("WSVD_ATTN_CHUNK", chunk)
    rng = O.Rng(400 + length)
    E, H, nh, r, B = 64, 32, 3, 16, 2
    lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
    f = to_factors(lay)
    cache = D.LatentCache(f, batch=B, capacity=length + 8)
    lat_k = rng.normal_matrix(B * nh * length, r).reshape(B, nh, length, r)
    lat_v = rng.normal_matrix(B * nh * length, r).reshape(B, nh, length, r)
    for t in range(length):
        for h in range(nh):
            cache.push(h, lat_k[:, h, t], lat_v[:, h, t])
        cache.bump_length()
    q = rng.normal_matrix(B * nh, H).reshape(B, nh, H)
    out = D.fused_decode_step(cache, f, q, D.TileConfig(), D.TrafficCounter())
    lat_k32 = O.f32_round(lat_k)
    lat_v32 = O.f32_round(lat_v)
    for b in range(B):
        ref = O.fused_decode_step(lay, np.ascontiguousarray(lat_k32[b]), np.ascontiguousarray(lat_v32[b]),
                                  length, q[b], 32)
        assert rel_err_rows(out[b], ref) <= REL_TOL


# --------------------------------------------------------------- bf16 -----
def bf16_layer(lay):
    return lay.map(O.bf16_round)


@pytest.mark.parametrize("E,nh,r,H,B,L", [(256, 4, 32, 128, 3, 200), (4096, 32, 32, 128, 2, 96)])
def test_bf16_append_and_decode(E, nh, r, H, B, L):
    rng = O.Rng(500 + E)
    lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
    f = to_factors(lay)
    cache = D.LatentCache(f, batch=B, capacity=L + 4, cache_dtype="bf16", weight_dtype="bf16")
    toks = O.bf16_round(rng.normal_matrix(L * B, E)).reshape(L, B, E)
    q = None
    for t in range(L):
        q = D.append_token(cache, f, toks[t])
    out = D.fused_decode_step(cache, f, q, D.TileConfig(), D.TrafficCounter())
    lb = bf16_layer(lay)
    for b in range(B):
        # projection: oracle x.A on the same bf16 inputs vs device latents (bf16-rounded)
        ck_ref = np.zeros((nh, L, r))
        cv_ref = np.zeros((nh, L, r))
        q_ref = None
        for t in range(L):
            q_ref = O.append_token(lb, ck_ref, cv_ref, t, toks[t, b])
        assert rel_err_rows(q[b], q_ref) <= REL_TOL
        ck_dev = np.stack([cache.latent_k(h, b) for h in range(nh)])
        cv_dev = np.stack([cache.latent_v(h, b) for h in range(nh)])
        scale = np.abs(ck_ref).max()
        assert np.abs(ck_dev - ck_ref).max() <= 2 ** -7 * scale
        assert np.abs(cv_dev - cv_ref).max() <= 2 ** -7 * np.abs(cv_ref).max()
        # attention on exactly the stored rows
        ref = O.fused_decode_step(lb, np.ascontiguousarray(ck_dev), np.ascontiguousarray(cv_dev), L,
                                  q[b], 32)
        assert rel_err_rows(out[b], ref) <= REL_TOL
        # and against the unrounded-latent fp64 reference
        ref64 = O.fused_decode_step(lb, ck_ref, cv_ref, L, q_ref, 32)
        assert rel_err_rows(out[b], ref64) <= 2e-2


def test_prefill_large_matches_token_by_token_appends():
    """Prefill at the 7B width with 128-row GEMM chunks (8 K splits, many
    W-tiles per CTA, the 128-row consumer configuration) writes the same cache
    rows as one-token appends (16-row configuration)."""
    from paper_2604_02570_b200.layer import DecodeLayer
    from oracle import oracle as O
    from tests.helpers import to_factors
    rng = O.Rng(4242)
    E, nh, H, r, B, T = 4096, 32, 128, 32, 16, 16
    lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
    f = to_factors(lay)
    a = DecodeLayer(f, None, batch=B, capacity=T + 8, cache_dtype="bf16", weight_dtype="bf16")
    b = DecodeLayer(f, None, batch=B, capacity=T + 8, cache_dtype="bf16", weight_dtype="bf16")
    dev = torch.device("cuda", 0)
    toks = torch.from_numpy(rng.normal_matrix(T * B, E).reshape(T, B, E).astype(np.float32)).to(dev)
    a.prefill(toks)                 # 256 rows -> two 128-row GEMM chunks
    for t in range(T):
        b.append(toks[t])           # 16 rows each
    torch.cuda.synchronize()
    assert a.length() == b.length() == T
    for bb in (0, 7, 15):
        for h in (0, 13, 31):
            ka, va = a.read_latents(bb, h)
            kb, vb = b.read_latents(bb, h)
            assert np.abs(ka - kb).max() <= 1e-2 * np.abs(kb).max()
            assert np.abs(va - vb).max() <= 1e-2 * np.abs(vb).max()


def test_attend_two_chunk_shape_matches_oracle():
    """The operator-API attention (q -> full-rank head outputs) at a shape whose
    split-KV uses two chunks per (sequence, head) (512 pairs over the grid),
    merged by the combine kernel with the B_V up-projection."""
    from paper_2604_02570_b200.layer import DecodeLayer
    rng = O.Rng(777)
    E, nh, H, r, B, L = 1024, 32, 128, 32, 16, 300
    lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
    layer = DecodeLayer(to_factors(lay), None, batch=B, capacity=L + 4, cache_dtype="bf16", weight_dtype="bf16")
    dev = torch.device("cuda", 0)
    toks = O.bf16_round(rng.normal_matrix(L * B, E)).reshape(L, B, E)
    layer.prefill(torch.from_numpy(toks.astype(np.float32)).to(dev))
    q = torch.from_numpy(rng.normal_matrix(B * nh, H).reshape(B, nh, H).astype(np.float32)).to(dev)
    out = torch.empty((B, nh, H), device=dev)
    layer.attend(q, out)
    torch.cuda.synchronize()
    out = out.cpu().numpy().astype(np.float64)
    lb = lay.map(O.bf16_round)
    for b in (0, 7, 15):
        ck = np.stack([layer.read_latents(b, h)[0][:, :r] for h in range(nh)])
        cv = np.stack([layer.read_latents(b, h)[1][:, :r] for h in range(nh)])
        ref = O.fused_decode_step(lb, ck, cv, L, q[b].cpu().numpy().astype(np.float64), 32)
        assert rel_err_rows(out[b], ref) <= REL_TOL, f"b={b}"
