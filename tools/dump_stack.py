import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle import oracle as O
from tests.helpers import to_factors
from paper_2604_02570_b200.layer import DecodeLayer
from paper_2604_02570_b200.stack import DecodeStack, toy_ffn_weights
for B in (3,):
    E, nh, H, r, F, n, T = 256, 2, 128, 32, 512, 3, 6
    rng = O.Rng(9300 + B)
    lbs, wos, layers = [], [], []
    for li in range(n):
        lb = O.random_layer(rng, E, H, [[r, r, r]] * nh).map(O.bf16_round)
        wo = O.bf16_round(rng.normal_matrix(nh * H, E, 1.0 / np.sqrt(E)))
        lbs.append(lb); wos.append(wo)
        layers.append(DecodeLayer(to_factors(lb), wo, batch=B, capacity=T + 4, cache_dtype="bf16", weight_dtype="bf16"))
    ffn = [toy_ffn_weights(E, F, 40 + li) for li in range(n)]
    stack = DecodeStack(layers, ffn_dim=F, ffn_weights=ffn)
    dev = torch.device("cuda", 0)
    xs = O.bf16_round(rng.normal_matrix(T * B, E)).reshape(T, B, E)
    ys = np.zeros((T, B, E))
    y = torch.empty((B, E), device=dev)
    for t in range(T):
        stack.step(torch.from_numpy(xs[t].astype(np.float32)).to(dev), y)
        torch.cuda.synchronize()
        ys[t] = y.cpu().numpy()
    lat = {li: [layers[li].read_latents(0, h) for h in range(nh)] for li in range(n)}
    np.savez("gpurun_out/stack_dump.npz", ys=ys, xs=xs, **{f"k{li}_{h}": lat[li][h][0] for li in range(n) for h in range(nh)},
             **{f"v{li}_{h}": lat[li][h][1] for li in range(n) for h in range(nh)})
print("ok")
