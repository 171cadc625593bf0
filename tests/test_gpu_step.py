"""GPU parity of the fused persistent layer-step kernel (step.cu) -- the whole
pipe::decode_factored layer body (src/pipeline.cpp:320-329: append_token,
fused_decode_step, heads_row . W_o) in one launch -- against the CPU oracle,
and of the host-buffer entry point (wsvd_layer_step_host: H2D, step, D2H
replayed as one CUDA graph) against the device-buffer step."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import REL_TOL, oracle_step_y, rel_err_rows, to_factors

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))


def _twin(E, nh, H, r, B, cap, seed, **kw):
    from paper_2604_02570_b200.layer import DecodeLayer
    rng = O.Rng(seed)
    lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
    wo = O.bf16_round(rng.normal_matrix(nh * H, E, 1.0 / np.sqrt(E)))
    mk = lambda: DecodeLayer(to_factors(lay), wo, batch=B, capacity=cap, cache_dtype="bf16",  # noqa: E731
                             weight_dtype="bf16", **kw)
    return rng, lay, wo, mk


@pytest.mark.parametrize("E,nh,B,L", [(512, 16, 1, 300), (512, 16, 5, 77), (1024, 16, 16, 600), (512, 16, 32, 130),
                                      # 512 (sequence, head) regions over 148 byte-balanced ranges:
                                      # segments split across CTAs, last-arriver merges
                                      (1024, 32, 16, 300), (1024, 32, 16, 33), (1024, 32, 16, 65),
                                      (1024, 32, 16, 2), (512, 16, 1, 3000)])
def test_fused_step_matches_oracle(E, nh, B, L):
    H, r = 128, 32
    rng, lay, wo, mk = _twin(E, nh, H, r, B, L + 8, 8000 + B)
    layer = mk()
    assert layer.launches_per_step() == 1, layer.step_kind()
    dev = torch.device("cuda", 0)
    toks = O.bf16_round(rng.normal_matrix(L * B, E)).reshape(L, B, E)
    layer.prefill(torch.from_numpy(toks[:-1].astype(np.float32)).to(dev))
    y = torch.empty((B, E), device=dev)
    layer.step(torch.from_numpy(toks[-1].astype(np.float32)).to(dev), y)
    torch.cuda.synchronize()
    assert layer.length() == L
    y = y.cpu().numpy().astype(np.float64)
    lb = lay.map(O.bf16_round)
    for b in range(B):
        ck = np.zeros((nh, L, r))
        cv = np.zeros((nh, L, r))
        q = None
        for t in range(L):
            q = O.append_token(lb, ck, cv, t, toks[t, b])
        dev_k = np.stack([layer.read_latents(b, h)[0] for h in range(nh)])
        dev_v = np.stack([layer.read_latents(b, h)[1] for h in range(nh)])
        # the step's own row was written by the fused kernel (bf16 of the fp32 latent)
        assert np.abs(dev_k[:, L - 1] - ck[:, L - 1]).max() <= 2 ** -7 * np.abs(ck[:, L - 1]).max()
        y_ref = oracle_step_y(lb, dev_k, dev_v, L, q, wo, layer.rpad)
        # hi + lo bf16 latent outputs feed the O-projection: north_star tolerance
        assert rel_err_rows(y[b:b + 1], y_ref[None]) <= REL_TOL, f"b={b}"


def test_fused_step_is_deterministic_and_matches_attention_path():
    """two twin caches stepped with the same tokens give bit-identical y; the
    attention output of the reference-API path agrees with the step's y"""
    E, nh, H, r, B, L = 512, 16, 128, 32, 4, 257
    rng, lay, wo, mk = _twin(E, nh, H, r, B, L + 8, 8100)
    a, b = mk(), mk()
    dev = torch.device("cuda", 0)
    toks = torch.from_numpy(O.bf16_round(rng.normal_matrix((L + 3) * B, E)).reshape(L + 3, B, E)
                            .astype(np.float32)).to(dev)
    a.prefill(toks[:L])
    b.prefill(toks[:L])
    for t in range(3):
        ya, yb = torch.empty((B, E), device=dev), torch.empty((B, E), device=dev)
        a.step(toks[L + t], ya)
        b.step(toks[L + t], yb)
        torch.cuda.synchronize()
        assert torch.equal(ya, yb)


@pytest.mark.parametrize("E,nh,B,L", [(512, 16, 16, 200),
                                      (1024, 32, 16, 200)])  # 2 chunks per pair: the CTA-pair path
def test_step_host_replays_match_device_step(E, nh, B, L):
    """wsvd_layer_step_host (pinned x / y moved by the kernel itself) -- every
    step bit-identical to the device-buffer step of a twin cache"""
    H, r = 128, 32
    rng, lay, wo, mk = _twin(E, nh, H, r, B, L + 16, 8200)
    dev_l, host_l = mk(), mk()
    dev = torch.device("cuda", 0)
    toks = O.bf16_round(rng.normal_matrix((L + 5) * B, E)).reshape(L + 5, B, E).astype(np.float32)
    pre = torch.from_numpy(toks[:L]).to(dev)
    dev_l.prefill(pre)
    host_l.prefill(pre)
    torch.cuda.synchronize()
    xh = torch.empty((B, E), dtype=torch.float32).pin_memory()
    yh = torch.empty((B, E), dtype=torch.float32).pin_memory()
    for t in range(5):
        xh.copy_(torch.from_numpy(toks[L + t]))
        host_l.step_host(xh, yh)
        yd = torch.empty((B, E), device=dev)
        dev_l.step(torch.from_numpy(toks[L + t]).to(dev), yd)
        torch.cuda.synchronize()
        assert torch.equal(yh, yd.cpu()), f"step {t}"
    assert host_l.length() == dev_l.length() == L + 5


def test_step_kind_reports_the_path():
    from paper_2604_02570_b200.layer import DecodeLayer
    rng = O.Rng(8300)
    lay = O.random_layer(rng, 256, 128, [[16, 16, 16]] * 2)
    wo = rng.normal_matrix(2 * 128, 256, 1.0 / 16)
    layer = DecodeLayer(to_factors(lay), wo, batch=2, capacity=16, cache_dtype="bf16", weight_dtype="bf16")
    assert layer.launches_per_step() > 1  # rank 16: multi-kernel path
    # (the fused kernel streams 512-wide K splits: E and nh*R multiples of 512)
    lay32 = O.random_layer(rng, 512, 128, [[32, 32, 32]] * 16)
    wo32 = rng.normal_matrix(16 * 128, 512, 1.0 / 16)
    layer32 = DecodeLayer(to_factors(lay32), wo32, batch=2, capacity=16, cache_dtype="bf16", weight_dtype="bf16")
    assert layer32.launches_per_step() == 1
    layer32.set_attention("explicit_tc")
    assert layer32.launches_per_step() > 1  # the explicit mode runs the multi-kernel step


@pytest.mark.parametrize("B,L", [(1, 1), (3, 2), (16, 33), (7, 257)])
def test_fused_step_short_caches_and_ragged_ranks(B, L):
    """the first tokens of a sequence (the step's own row is the only or almost
    the only one; decode.cpp:312-328 L = 1 case), odd batches, and ragged
    per-head ranks zero-padded to 32 (test_decode.cpp:190-194)"""
    from paper_2604_02570_b200.layer import DecodeLayer
    E, nh, H = 512, 16, 128
    rng = O.Rng(8400 + B * 1000 + L)
    ranks = [[32 - (h % 5), 32 - (h % 3), 17 + h] for h in range(nh)]
    lay = O.random_layer(rng, E, H, ranks)
    wo = O.bf16_round(rng.normal_matrix(nh * H, E, 1.0 / np.sqrt(E)))
    layer = DecodeLayer(to_factors(lay), wo, batch=B, capacity=L + 4, cache_dtype="bf16", weight_dtype="bf16")
    assert layer.launches_per_step() == 1
    dev = torch.device("cuda", 0)
    toks = O.bf16_round(rng.normal_matrix(L * B, E)).reshape(L, B, E)
    if L > 1:
        layer.prefill(torch.from_numpy(toks[:-1].astype(np.float32)).to(dev))
    y = torch.empty((B, E), device=dev)
    layer.step(torch.from_numpy(toks[-1].astype(np.float32)).to(dev), y)
    torch.cuda.synchronize()
    assert layer.length() == L and layer.sync_length() == L
    y = y.cpu().numpy().astype(np.float64)
    lb = lay.map(O.bf16_round)
    R = layer.rpad
    for b in range(B):
        ck = np.zeros((nh, L, lay.rmax))
        cv = np.zeros((nh, L, lay.rmax))
        q = None
        for t in range(L):
            q = O.append_token(lb, ck, cv, t, toks[t, b])
        dev_k = np.stack([layer.read_latents(b, h)[0][:, :lay.rmax] for h in range(nh)])
        dev_v = np.stack([layer.read_latents(b, h)[1][:, :lay.rmax] for h in range(nh)])
        for h in range(nh):  # zero-padded latent columns stay zero
            assert not layer.read_latents(b, h)[0][:, lay.ranks[h, 1]:R].any()
        y_ref = oracle_step_y(lb, dev_k, dev_v, L, q, wo, R)
        assert rel_err_rows(y[b:b + 1], y_ref[None]) <= REL_TOL, f"b={b}"


def test_cluster_pair_merge_matches_l2_merge():
    """The region a CTA pair shares meets through distributed shared memory;
    with WSVD_STEP_NOCLUSTER (child process: the switch is read once) every
    shared region merges through L2 instead.  Both merge the parts in range
    order with the same arithmetic: bit-identical y."""
    import os
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, sys
sys.path.insert(0, %r)
from oracle import oracle as O
from tests.helpers import to_factors
from paper_2604_02570_b200.layer import DecodeLayer
rng = O.Rng(8300)
E, nh, H, r, B, L = 1024, 32, 128, 32, 16, 400
lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
wo = O.bf16_round(rng.normal_matrix(nh * H, E, 1.0 / np.sqrt(E)))
layer = DecodeLayer(to_factors(lay), wo, batch=B, capacity=L + 8, cache_dtype="bf16", weight_dtype="bf16")
dev = torch.device("cuda", 0)
toks = torch.from_numpy(O.bf16_round(rng.normal_matrix((L + 2) * B, E)).reshape(L + 2, B, E).astype(np.float32)).to(dev)
layer.prefill(toks[:L])
ys = []
for t in range(2):
    y = torch.empty((B, E), device=dev)
    layer.step(toks[L + t], y)
    ys.append(y.cpu().numpy())
np.save(sys.argv[1], np.stack(ys))
""" % (ROOT,)
    outs = []
    for i, env_extra in enumerate(({}, {"WSVD_STEP_NOCLUSTER": "1"})):
        path = os.path.join(ROOT, "gpurun_out", f"pair_merge_{i}.npy")
        os.makedirs(os.path.dirname(path), exist_ok=True)
        res = subprocess.run([sys.executable, "-c", code, path], env=dict(os.environ, **env_extra),
                             capture_output=True, text=True, timeout=600, cwd=ROOT)
        assert res.returncode == 0, res.stderr[-3000:]
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.timeout(120)
def test_fused_steps_on_two_streams_do_not_overlap():
    """Two caches stepping on two non-blocking streams with no host sync in
    between: the fused step holds every SM at its barrier, so the library
    orders fused steps of different streams (capi.cu fused_serialize) --
    without that, two concurrent grids would each wait for SMs the other
    holds.  Results equal the same steps run one stream at a time."""
    E, nh, H, r, B, L = 1024, 32, 128, 32, 16, 300
    rng, lay, wo, mk = _twin(E, nh, H, r, B, L + 16, 8500)
    a, b, a2, b2 = mk(), mk(), mk(), mk()
    dev = torch.device("cuda", 0)
    toks = torch.from_numpy(O.bf16_round(rng.normal_matrix((L + 6) * B, E)).reshape(L + 6, B, E)
                            .astype(np.float32)).to(dev)
    for lay_ in (a, b, a2, b2):
        lay_.prefill(toks[:L])
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ya = [torch.empty((B, E), device=dev) for _ in range(6)]
    yb = [torch.empty((B, E), device=dev) for _ in range(6)]
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    for t in range(6):
        a.step(toks[L + t], ya[t], stream=s1)
        b.step(toks[L + t], yb[t], stream=s2)
    torch.cuda.synchronize()
    for t in range(6):
        ra, rb_ = torch.empty((B, E), device=dev), torch.empty((B, E), device=dev)
        a2.step(toks[L + t], ra)
        b2.step(toks[L + t], rb_)
        torch.cuda.synchronize()
        assert torch.equal(ya[t], ra) and torch.equal(yb[t], rb_), f"step {t}"


@pytest.mark.parametrize("E,nh,B,L", [(512, 8, 32, 700), (1024, 32, 8, 129), (512, 32, 16, 1030),
                                      (1536, 24, 12, 333), (512, 4, 29, 95), (1024, 16, 31, 2049)])
def test_fused_step_matches_multi_kernel_step(E, nh, B, L):
    """Assorted shapes (different split-KV chunk counts, cluster and non-cluster
    merges, parked-item counts, ragged batches): the fused step's y equals the
    multi-kernel step's (attn_out forces the operator path) up to fp32
    reassociation, and the caches agree row for row."""
    H, r = 128, 32
    rng, lay, wo, mk = _twin(E, nh, H, r, B, L + 4, 9000 + E + nh + B)
    a, b = mk(), mk()
    dev = torch.device("cuda", 0)
    toks = torch.from_numpy(O.bf16_round(rng.normal_matrix(L * B, E)).reshape(L, B, E).astype(np.float32)).to(dev)
    a.prefill(toks[:-1])
    b.prefill(toks[:-1])
    ya, yb = torch.empty((B, E), device=dev), torch.empty((B, E), device=dev)
    attn = torch.empty((B, nh, H), device=dev)
    a.step(toks[-1], ya)                  # fused persistent kernel
    b.step(toks[-1], yb, attn_out=attn)   # multi-kernel operator path
    torch.cuda.synchronize()
    assert a.length() == b.length() == L
    ya, yb = ya.cpu().numpy(), yb.cpu().numpy()
    assert np.abs(ya - yb).max() <= 1e-4 * np.abs(yb).max()  # both paths: hi + lo latents, fp32 sums
    for bb in (0, B - 1):
        for h in (0, nh - 1):
            ka, va = a.read_latents(bb, h)
            kb, vb = b.read_latents(bb, h)
            assert np.array_equal(ka, kb) and np.array_equal(va, vb)
