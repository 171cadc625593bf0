"""Wall-clock per host-buffer layer step (wsvd_layer_step_host), for A/B of the
host path (e.g. WSVD_HOST_ZEROCOPY=0)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_02570_b200.layer import DecodeLayer  # noqa: E402

cfg = bench.CONFIGS[bench.DEFAULT_CONFIG]
E, B, L = cfg["E"], cfg["B"], cfg["L"]
f, w_o = bench.synthetic_layer(cfg)
layer = DecodeLayer(f, w_o, batch=B, capacity=L + 600, cache_dtype="bf16", weight_dtype="bf16")
dev = torch.device("cuda", 0)
for t0 in range(0, L - 1, 256):
    layer.prefill(torch.randn((min(256, L - 1 - t0), B, E), device=dev))
torch.cuda.synchronize()
xh = torch.randn((B, E)).pin_memory()
yh = torch.empty((B, E)).pin_memory()
xn, yn = xh.numpy(), yh.numpy()
for _ in range(5):
    layer.step_host(xn, yn)
for trial in range(3):
    t = time.perf_counter()
    for _ in range(40):
        layer.step_host(xn, yn)
    print(f"step_host: {(time.perf_counter() - t) / 40 * 1e6:.1f} us/step")
y = torch.empty((B, E), device=dev)
x = torch.randn((B, E), device=dev)
t = time.perf_counter()
for _ in range(40):
    layer.step(x, y)
    torch.cuda.synchronize()
print(f"device step + sync: {(time.perf_counter() - t) / 40 * 1e6:.1f} us/step")
xd = torch.empty((B, E), device=dev)
for name, fn in (("H2D 256KB", lambda: xd.copy_(xh, non_blocking=True)),
                 ("D2H 256KB", lambda: yh.copy_(xd, non_blocking=True))):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(40):
        fn()
        torch.cuda.synchronize()
    print(f"{name} + sync: {(time.perf_counter() - t) / 40 * 1e6:.1f} us")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("H2D 256KB", lambda: xd.copy_(xh, non_blocking=True)),
                 ("D2H 256KB", lambda: yh.copy_(xd, non_blocking=True))):
    e0.record()
    for _ in range(40):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} device time: {e0.elapsed_time(e1) / 40 * 1e3:.1f} us")
t = time.perf_counter()
for _ in range(40):
    torch.cuda.synchronize()
print(f"empty sync: {(time.perf_counter() - t) / 40 * 1e6:.1f} us")
# device time of the zero-copy host step (events on the layer's stream around the call)
s = torch.cuda.current_stream()
e0.record(s)
for _ in range(40):
    layer.step_host(xn, yn)
e1.record(s)
torch.cuda.synchronize()
print(f"step_host device span: {e0.elapsed_time(e1) / 40 * 1e3:.1f} us/step")
# tiny kernel + sync wall: the launch / wake-up floor
t = time.perf_counter()
for _ in range(40):
    x.add_(0.0)
    torch.cuda.synchronize()
print(f"tiny kernel + sync: {(time.perf_counter() - t) / 40 * 1e6:.1f} us")
import ctypes  # noqa: E402
from paper_2604_02570_b200 import _native as N  # noqa: E402
t = time.perf_counter()
for _ in range(1000):
    N.lib().wsvd_last_error()
print(f"python->ctypes call: {(time.perf_counter() - t) / 1000 * 1e6:.2f} us")
