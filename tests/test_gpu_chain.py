"""GPU parity of the fused layer chain (wsvd_chain_step): the attention blocks
of pipe::decode_factored's layer loop (src/pipeline.cpp:318-336) run as ONE
persistent kernel, layer l + 1's token = layer l's output.

* against the single-layer steps: twin caches stepped layer by layer through
  wsvd_layer_step on the chain's own inputs append identical rows; y is
  bit-identical for the one-group chain (step.cu: the same arithmetic, only the
  launch boundaries and the weight loads move) and within 1e-5 for the
  two-group chain (step2.cu: its attention ranges split the rows differently);
* against the CPU oracle: every layer's y from the device token it was given
  (append_token + fused_decode_step + heads_row . W_o, decode.cpp:127-206,
  pipeline.cpp:323-329) within the north_star tolerance."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import REL_TOL, oracle_step_y, to_factors

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _build(n, E, nh, B, caps, seed):
    from paper_2604_02570_b200.layer import DecodeLayer
    H, r = 128, 32
    rng = O.Rng(seed)
    lays, wos = [], []
    for _ in range(n):
        lays.append(O.random_layer(rng, E, H, [[r, r, r]] * nh))
        wos.append(O.bf16_round(rng.normal_matrix(nh * H, E, 1.0 / np.sqrt(E))))

    def make():
        return [DecodeLayer(to_factors(lays[i]), wos[i], batch=B, capacity=caps[i], cache_dtype="bf16",
                            weight_dtype="bf16") for i in range(n)]
    return rng, lays, wos, make


def _prefill(layers, lens, rng, B, E, dev):
    for lay, L in zip(layers, lens):
        if L > 0:
            toks = O.bf16_round(rng.normal_matrix(L * B, E)).reshape(L, B, E)
            lay.prefill(torch.from_numpy(toks.astype(np.float32)).to(dev))


def _pipelined(B):
    """WSVD_CHAIN_PIPE=1 and 2 <= B <= 16: the chain runs as two batch groups
    half a layer apart (step2.cu, opt-in); otherwise as one group (step.cu)"""
    import os
    return 2 <= B <= 16 and os.environ.get("WSVD_CHAIN_PIPE", "0") == "1"


@pytest.mark.parametrize("E,nh,B,lens", [
    (512, 16, 5, [300, 77, 130]),        # ragged lengths: a range table per layer
    (1024, 32, 16, [257, 257, 257, 257]),  # CTA pairs (DSMEM merges) + L2 last-arriver merges
    (512, 16, 2, [40, 1, 0]),            # one sequence per group; a first token (empty cache)
    (512, 16, 20, [40, 1, 0]),           # one group, two token tiles
    (512, 16, 1, [3000, 2]),
])
def test_chain_equals_layer_steps(E, nh, B, lens):
    """every layer of the chain against wsvd_layer_step of a twin layer fed the
    chain's own input: the appended rows are identical; y is identical for the
    one-group chain (the same arithmetic) and within 1e-5 for the two-group
    chain (its attention ranges split the rows differently)"""
    from paper_2604_02570_b200.layer import DecodeChain
    n = len(lens)
    dev = torch.device("cuda", 0)
    caps = [L + 8 for L in lens]
    rng, lays, wos, make = _build(n, E, nh, B, caps, 9100 + B)
    a, b = make(), make()
    _prefill(a, lens, O.Rng(77), B, E, dev)
    _prefill(b, lens, O.Rng(77), B, E, dev)
    chain = DecodeChain(a)
    assert chain.fused() and chain.launches_per_step() == 1
    for step in range(2):
        x = torch.from_numpy(O.bf16_round(rng.normal_matrix(B, E)).astype(np.float32)).to(dev)
        ya = [torch.empty((B, E), device=dev) for _ in range(n)]
        yb = [torch.empty((B, E), device=dev) for _ in range(n)]
        chain.step(x, ya)
        for i in range(n):
            b[i].step(x if i == 0 else ya[i - 1], yb[i], graph=False)
        torch.cuda.synchronize()
        for i in range(n):
            if _pipelined(B):
                d = (ya[i] - yb[i]).abs().amax(dim=1) / yb[i].abs().amax(dim=1)
                assert float(d.max()) <= 1e-5, f"step {step} layer {i}: {float(d.max()):.2e}"
            else:
                assert torch.equal(ya[i], yb[i]), f"step {step} layer {i}: chain differs from the layer step"
            assert a[i].length() == b[i].length() == lens[i] + step + 1
    for i in range(n):
        for s in range(B):
            for h in range(0, nh, 5):
                ka, va = a[i].read_latents(s, h)
                kb, vb = b[i].read_latents(s, h)
                assert np.array_equal(ka, kb) and np.array_equal(va, vb)


def test_chain_is_deterministic():
    """twin chains stepped with the same tokens: bit-identical outputs"""
    from paper_2604_02570_b200.layer import DecodeChain
    E, nh, B, lens = 1024, 32, 16, [300, 300, 300]
    dev = torch.device("cuda", 0)
    rng, lays, wos, make = _build(3, E, nh, B, [L + 8 for L in lens], 9700)
    a, b = make(), make()
    _prefill(a, lens, O.Rng(4), B, E, dev)
    _prefill(b, lens, O.Rng(4), B, E, dev)
    ca, cb = DecodeChain(a), DecodeChain(b)
    for step in range(3):
        x = torch.from_numpy(O.bf16_round(rng.normal_matrix(B, E)).astype(np.float32)).to(dev)
        ya = [torch.empty((B, E), device=dev) for _ in range(3)]
        yb = [torch.empty((B, E), device=dev) for _ in range(3)]
        ca.step(x, ya)
        cb.step(x, yb)
        torch.cuda.synchronize()
        for i in range(3):
            assert torch.equal(ya[i], yb[i])


@pytest.mark.parametrize("E,nh,B,lens", [(512, 16, 4, [129, 300, 64]), (1024, 32, 16, [300, 300]),
                                         (512, 16, 3, [70, 1]), (512, 16, 24, [100, 90])])
def test_chain_matches_oracle(E, nh, B, lens):
    from paper_2604_02570_b200.layer import DecodeChain
    n = len(lens)
    dev = torch.device("cuda", 0)
    rng, lays, wos, make = _build(n, E, nh, B, [L + 8 for L in lens], 9300 + B)
    layers = make()
    _prefill(layers, lens, O.Rng(5), B, E, dev)
    chain = DecodeChain(layers)
    x = torch.from_numpy(O.bf16_round(rng.normal_matrix(B, E)).astype(np.float32)).to(dev)
    ys = [torch.empty((B, E), device=dev) for _ in range(n)]
    chain.step(x, ys)
    torch.cuda.synchronize()
    xs = [x.cpu().numpy().astype(np.float64)] + [t.cpu().numpy().astype(np.float64) for t in ys]
    r = 32
    for i in range(n):
        lb = lays[i].map(O.bf16_round)
        L = lens[i] + 1
        tok = O.bf16_round(xs[i])  # the kernel stages the token as bf16
        y = xs[i + 1]
        worst = 0.0
        for s in range(B):
            ck1, cv1 = np.zeros((nh, 1, r)), np.zeros((nh, 1, r))
            q = O.append_token(lb, ck1, cv1, 0, tok[s])
            dk = np.stack([layers[i].read_latents(s, h)[0] for h in range(nh)])
            dv = np.stack([layers[i].read_latents(s, h)[1] for h in range(nh)])
            # the own row: bf16 of the fp32 latent (append_token, decode.cpp:143-149)
            assert np.abs(dk[:, L - 1, :r] - ck1[:, 0]).max() <= 2 ** -7 * np.abs(ck1[:, 0]).max()
            assert np.abs(dv[:, L - 1, :r] - cv1[:, 0]).max() <= 2 ** -7 * np.abs(cv1[:, 0]).max()
            y_ref = oracle_step_y(lb, dk, dv, L, q, wos[i], layers[i].rpad)
            worst = max(worst, float(np.abs(y[s] - y_ref).max() / np.abs(y_ref).max()))
        assert worst <= REL_TOL, f"layer {i}: {worst:.2e}"


def test_chain_host_buffers_equal_device_chain():
    """wsvd_chain_step_host (pinned x / y; the one-group chain moves them with
    the kernel's own bus loads / stores, the two-group chain with the copy
    engine) equals the device-buffer chain bit for bit"""
    from paper_2604_02570_b200.layer import DecodeChain
    E, nh, B, lens = 1024, 32, 16, [200, 200, 200]
    dev = torch.device("cuda", 0)
    rng, lays, wos, make = _build(3, E, nh, B, [L + 8 for L in lens], 9500)
    a, b = make(), make()
    _prefill(a, lens, O.Rng(3), B, E, dev)
    _prefill(b, lens, O.Rng(3), B, E, dev)
    ca, cb = DecodeChain(a), DecodeChain(b)
    for step in range(3):
        xn = O.bf16_round(rng.normal_matrix(B, E)).astype(np.float32)
        xh = torch.from_numpy(xn).pin_memory()
        yh = torch.empty((B, E), dtype=torch.float32).pin_memory()
        ca.step_host(xh, yh)
        ys = [torch.empty((B, E), device=dev) for _ in range(3)]
        cb.step(torch.from_numpy(xn).to(dev), ys)
        torch.cuda.synchronize()
        assert torch.equal(yh, ys[-1].cpu()), f"step {step}"


def test_two_group_chain_in_subprocess():
    """the opt-in two-group chain (step2.cu, WSVD_CHAIN_PIPE=1, read once per
    process): this file's chain tests rerun in a subprocess with it enabled"""
    import os
    import subprocess
    import sys
    if os.environ.get("WSVD_CHAIN_PIPE") == "1":
        pytest.skip("already the two-group run")
    env = dict(os.environ, WSVD_CHAIN_PIPE="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", __file__, "-k", "not subprocess"],
                       env=env, capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_chain_and_layer_steps_interleave_on_the_same_caches():
    """chain launches and single-layer launches alternate on the same caches
    (each keeps its own control block: barrier counts, layer-step tags of the
    projection partials and of the chained tokens): the results equal a twin
    stepped layer by layer throughout, bit for bit"""
    import os
    if os.environ.get("WSVD_CHAIN_PIPE") == "1":
        pytest.skip("the two-group chain splits rows differently (1e-5, test_chain_equals_layer_steps)")
    from paper_2604_02570_b200.layer import DecodeChain
    E, nh, B, lens = 1024, 32, 16, [200, 201, 202]
    n = len(lens)
    dev = torch.device("cuda", 0)
    rng, lays, wos, make = _build(n, E, nh, B, [L + 12 for L in lens], 9300)
    a, b = make(), make()
    _prefill(a, lens, O.Rng(78), B, E, dev)
    _prefill(b, lens, O.Rng(78), B, E, dev)
    chain = DecodeChain(a)
    for step in range(6):
        x = torch.from_numpy(O.bf16_round(rng.normal_matrix(B, E)).astype(np.float32)).to(dev)
        ya = [torch.empty((B, E), device=dev) for _ in range(n)]
        yb = [torch.empty((B, E), device=dev) for _ in range(n)]
        if step % 3 == 1:  # this pass one launch per layer on the chain's caches
            for i in range(n):
                a[i].step(x if i == 0 else ya[i - 1], ya[i], graph=False)
        else:
            chain.step(x, ya)
        for i in range(n):
            b[i].step(x if i == 0 else yb[i - 1], yb[i], graph=False)
        torch.cuda.synchronize()
        for i in range(n):
            assert torch.equal(ya[i], yb[i]), f"step {step} layer {i}"


@pytest.mark.parametrize("env", ["WSVD_STEP_NOCLUSTER=1", "WSVD_STEP_NOXTAG=1", "WSVD_STEP_G1=1",
                                 "WSVD_STEP_G3=1", "WSVD_STEP_SHORTSEG=0"])
def test_chain_switches_in_subprocess(env):
    """the A/B switches of the fused step (read once per process): without CTA
    pairs (y through red.add, grid barrier 1 kept), untagged chained tokens
    (y flags), the grid barriers restored, short first segments in place --
    the chain still equals the single-layer steps bit for bit"""
    import os
    import subprocess
    import sys
    k, v = env.split("=")
    if os.environ.get(k) == v or os.environ.get("WSVD_CHAIN_PIPE") == "1":
        pytest.skip("already a switched run")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", __file__, "-k",
                        "test_chain_equals_layer_steps or interleave"],
                       env=dict(os.environ, **{k: v}), capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
