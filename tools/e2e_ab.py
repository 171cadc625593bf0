"""Wall time per host-buffer layer step (wsvd_layer_step_host) at the headline
shape: 5 trials x 200 steps, min and median -- for A/B runs of the host path
through environment switches (MODE=<label> names the line).

    MODE=zc WSVD_HOST_ZEROCOPY=1 python tools/e2e_ab.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_02570_b200.layer import DecodeLayer  # noqa: E402
cfg = bench.CONFIGS[bench.DEFAULT_CONFIG]
E, B, L = cfg["E"], cfg["B"], cfg["L"]
f, w_o = bench.synthetic_layer(cfg)
layer = DecodeLayer(f, w_o, batch=B, capacity=L + 1200, cache_dtype="bf16", weight_dtype="bf16")
layer.fill_synthetic(L - 1)
torch.cuda.synchronize()
xh = torch.randn((B, E)).pin_memory(); yh = torch.empty((B, E)).pin_memory()
xn, yn = xh.numpy(), yh.numpy()
for _ in range(10): layer.step_host(xn, yn)
res = []
for trial in range(5):
    t = time.perf_counter()
    for _ in range(200): layer.step_host(xn, yn)
    res.append((time.perf_counter() - t) / 200 * 1e6)
print(os.environ.get("MODE", ""), "min %.1f median %.1f" % (min(res), sorted(res)[2]))
