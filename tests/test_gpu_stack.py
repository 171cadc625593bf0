"""GPU tests of the layer stack (pipe::decode_factored, src/pipeline.cpp:304-339)
and the benchmark cache fill: the stack equals its layers run one after the
other with the reference's toy FFN, and a CUDA-graph replay of a stack step
equals the eager step (the caches advance on the device)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import to_factors

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _layers(n, E, nh, H, r, B, cap, seed):
    from paper_2604_02570_b200.layer import DecodeLayer
    rng = O.Rng(seed)
    out = []
    for li in range(n):
        lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
        wo = rng.normal_matrix(nh * H, E, 1.0 / np.sqrt(E))
        out.append((lay, wo, lambda lay=lay, wo=wo: DecodeLayer(to_factors(lay), wo, batch=B, capacity=cap,
                                                                 cache_dtype="bf16", weight_dtype="bf16")))
    return out


def test_fill_synthetic_sets_rows_and_length():
    from paper_2604_02570_b200.layer import DecodeLayer
    rng = O.Rng(9000)
    lay = O.random_layer(rng, 256, 128, [[32, 32, 32]] * 2)
    for dt in ("bf16", "f32", "i8"):
        layer = DecodeLayer(to_factors(lay), None, batch=3, capacity=100, cache_dtype=dt,
                            weight_dtype="bf16" if dt != "f32" else "f32")
        layer.fill_synthetic(77, seed=5)
        assert layer.length() == layer.sync_length() == 77
        ck, cv = layer.read_latents(2, 1)
        assert ck.shape == (77, 32) and np.isfinite(ck).all() and np.isfinite(cv).all()
        assert 0.7 < ck.std() < 1.3 and abs(ck.mean()) < 0.1  # N(0, 1) latents
        assert not np.array_equal(ck, cv)


def test_stack_equals_layers_in_sequence_and_graph_replay():
    from paper_2604_02570_b200.stack import DecodeStack
    E, nh, H, r, B, L, n = 512, 16, 128, 32, 40, 150, 3  # B > 32: the multi-kernel layer path
    specs = _layers(n, E, nh, H, r, B, L + 8, 9100)
    dev = torch.device("cuda", 0)
    a = [mk() for _, _, mk in specs]
    b = [mk() for _, _, mk in specs]
    for li in range(n):
        a[li].fill_synthetic(L, seed=li)
        b[li].fill_synthetic(L, seed=li)
    sa = DecodeStack(a, seed=3)
    x = torch.randn((B, E), device=dev)
    y = torch.empty((B, E), device=dev)
    sa.step(x, y)
    # the same body by hand
    cur = x
    o = torch.empty((B, E), device=dev)
    for li in range(n):
        b[li].step(cur, o, graph=False)
        nxt = torch.empty((B, E), device=dev)
        sa.ffns[li].forward(o, nxt)  # the same FFN objects (their weights)
        cur = nxt
    torch.cuda.synchronize()
    assert torch.equal(y, cur)
    # graph capture of the next step == the eager next step on the twin
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    x2 = torch.randn((B, E), device=dev)
    with torch.cuda.graph(g, stream=side):
        sa.step(x2, y)
    g.replay()
    sb = DecodeStack(b, seed=3)  # the same toy FFN weights (seeded)
    y2 = torch.empty((B, E), device=dev)
    sb.step(x2, y2)
    torch.cuda.synchronize()
    assert torch.equal(y, y2)
    for li in range(n):
        assert a[li].sync_length() == b[li].length() == L + 2


@pytest.mark.parametrize("E,nh,r,B", [(256, 2, 16, 2), (512, 16, 32, 4), (512, 16, 32, 40)])
def test_layer_step_commits_the_device_length(E, nh, r, B):
    """every step path (multi-kernel with fewer output tiles than SMs, fused,
    multi-kernel at B > 32) advances the device length once per step, so
    graph-replayed steps stay consistent with the host mirror"""
    from paper_2604_02570_b200.layer import DecodeLayer
    rng = O.Rng(9200 + E + B)
    lay = O.random_layer(rng, E, 128, [[r, r, r]] * nh)
    wo = rng.normal_matrix(nh * 128, E, 1.0 / np.sqrt(E))
    layer = DecodeLayer(to_factors(lay), wo, batch=B, capacity=64, cache_dtype="bf16", weight_dtype="bf16")
    layer.fill_synthetic(50, seed=1)
    dev = torch.device("cuda", 0)
    y = torch.empty((B, E), device=dev)
    for _ in range(3):
        layer.step(torch.randn((B, E), device=dev), y)
    torch.cuda.synchronize()
    assert layer.length() == 53
    assert layer.sync_length() == 53


@pytest.mark.parametrize("E,nh,B", [(256, 2, 3), (256, 2, 40), (512, 16, 3)])
def test_stack_matches_oracle_decode_factored(E, nh, B):
    """pipe::decode_factored (pipeline.cpp:304-339) on the device over T tokens
    from empty caches, checked layer by layer on the values the device chains:
    for every token and layer the oracle takes the layer's device input token
    (bf16 as staged) and the device's appended cache rows, runs append_token /
    fused_decode_step / v~ . W'_o (:320-329) and the toy FFN tanh(o . ff1) . ff2
    (:330-334, on the device's o), and both outputs agree within the
    north_star 1e-3.  E = 256: the multi-kernel layer path (B = 3 and B = 40);
    E = 512 with 16 heads, B = 3: the fused layer step."""
    from paper_2604_02570_b200.layer import DecodeLayer
    from paper_2604_02570_b200.stack import DecodeStack, toy_ffn_weights
    from tests.helpers import REL_TOL
    H, r, n, T = 128, 32, 3, 6
    F = 2 * E
    rng = O.Rng(9300 + B + E)
    lbs, wos, layers = [], [], []
    for li in range(n):
        lb = O.random_layer(rng, E, H, [[r, r, r]] * nh).map(O.bf16_round)
        wo = O.bf16_round(rng.normal_matrix(nh * H, E, 1.0 / np.sqrt(E)))
        lbs.append(lb)
        wos.append(wo)
        layers.append(DecodeLayer(to_factors(lb), wo, batch=B, capacity=T + 4, cache_dtype="bf16",
                                  weight_dtype="bf16"))
    ffn = [toy_ffn_weights(E, F, 40 + li) for li in range(n)]
    stack = DecodeStack(layers, ffn_dim=F, ffn_weights=ffn)
    dev = torch.device("cuda", 0)
    xs = O.bf16_round(rng.normal_matrix(T * B, E)).reshape(T, B, E)
    y = torch.empty((B, E), device=dev)
    recs = []
    for t in range(T):
        rec = []
        stack.step(torch.from_numpy(xs[t].astype(np.float32)).to(dev), y, record=rec)
        torch.cuda.synchronize()
        recs.append([[v.cpu().numpy().astype(np.float64) for v in lr] for lr in rec])
    rpad = layers[0].rpad
    folds = [O.fold_oproj(lb, wo, rpad, O.bf16_round) for lb, wo in zip(lbs, wos)]
    worst_o = worst_f = 0.0
    for b in (0, B - 1):
        rows = [(np.stack([layers[li].read_latents(b, h)[0] for h in range(nh)]),
                 np.stack([layers[li].read_latents(b, h)[1] for h in range(nh)])) for li in range(n)]
        for li in range(n):
            ck, cv = np.zeros((nh, T, r)), np.zeros((nh, T, r))
            for t in range(T):
                x_in, o_dev, out_dev = (v[b] for v in recs[t][li])
                q = O.append_token(lbs[li], ck, cv, t, O.bf16_round(x_in))
                ck[:, t], cv[:, t] = rows[li][0][:, t, :r], rows[li][1][:, t, :r]
                _, lat = O.batched_decode_latent(lbs[li], ck[None], cv[None], t + 1, q[None], 32, 1)
                lat_p = np.zeros((nh, rpad))
                lat_p[:, :r] = lat[0]
                o_ref = lat_p.reshape(-1) @ folds[li]
                worst_o = max(worst_o, float(np.abs(o_dev - o_ref).max() / np.abs(o_ref).max()))
                h = np.tanh(O.bf16_round(o_dev) @ ffn[li][0].astype(np.float64))
                out_ref = O.bf16_round(h) @ ffn[li][1].astype(np.float64)
                worst_f = max(worst_f, float(np.abs(out_dev - out_ref).max() / np.abs(out_ref).max()))
    assert worst_o <= REL_TOL, f"attention layer {worst_o:.2e}"
    assert worst_f <= REL_TOL, f"feed-forward {worst_f:.2e}"
