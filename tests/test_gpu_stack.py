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
        h = torch.tanh(o.to(torch.bfloat16) @ sa.ff1[li])
        cur = (h @ sa.ff2[li]).float()
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
    sb = DecodeStack(b, seed=3)
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
