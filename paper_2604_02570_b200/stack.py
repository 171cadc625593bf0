"""A stack of WSVD decode layers: pipe::decode_factored on the device.

Reference (src/pipeline.cpp:304-339): for every token and layer,
    q    = append_token(caches[li], factors[li], cur)          (:320)
    attn = fused_decode_step(caches[li], factors[li], q, ...)  (:321-322)
    o    = concat_h(attn[h]) . W_o                             (:323-329)
    cur  = tanh(o . ff1) . ff2                                 (:330-334)
The reference's model has no residual or normalisation and a toy FFN of width
2E (toymodel.hpp:20-35); this stack keeps exactly that body.  Each layer is a
`DecodeLayer` (its own latent cache and factors; append + attention + the
B_V-folded O-projection run by the library's kernels), heads may be sharded
across GPUs (the O-projection partial sums meet in one NCCL all-reduce), and
the FFN is the library's `FeedForward` (wsvd_ffn_*: two tcgen05 GEMMs -- TMA
multicast operands, TMEM accumulators -- over K-chunk-major bf16 weights, the
tanh and bf16 rounding fused into the first GEMM's epilogue), replicated on
every GPU.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as N
from .errors import ShapeError


class FeedForward:
    """out = tanh(o . ff1) . ff2 on the device (pipeline.cpp:330-334).
    ff1 [E][F], ff2 [F][E] host arrays (stored as bf16)."""

    def __init__(self, ff1: np.ndarray, ff2: np.ndarray, device: int = 0):
        ff1 = np.ascontiguousarray(ff1, dtype=np.float32)
        ff2 = np.ascontiguousarray(ff2, dtype=np.float32)
        E, F = ff1.shape
        if ff2.shape != (F, E):
            raise ShapeError(f"ff2 must be [{F}][{E}], got {ff2.shape}")
        self.E, self.F, self.device = E, F, device
        h = C.c_void_p()
        N.call("wsvd_ffn_create", E, F, C.c_void_p(ff1.ctypes.data), C.c_void_p(ff2.ctypes.data), device,
               C.byref(h))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and N._lib is not None:
            N.lib().wsvd_ffn_destroy(self.h)
            self.h = None

    def forward(self, o, out, stream=None):
        """o, out: fp32 device tensors [rows][E] (out may alias o)."""
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        N.call("wsvd_ffn_forward", self.h, C.c_void_p(o.data_ptr()), int(o.shape[0]), C.c_void_p(out.data_ptr()),
               C.c_void_p(s.cuda_stream))


def toy_ffn_weights(E: int, F: int, seed: int):
    """ff1 ~ N(0, 1/E), ff2 ~ N(0, 1/F) (toymodel.cpp:81-95 initialisation
    scale), fp32, rounded to bf16 values (the device's storage)."""
    rng = np.random.default_rng(seed)
    ff1 = (rng.standard_normal((E, F), dtype=np.float32) / np.float32(math.sqrt(E)))
    ff2 = (rng.standard_normal((F, E), dtype=np.float32) / np.float32(math.sqrt(F)))
    for w in (ff1, ff2):  # round to nearest even bf16 in place
        u = w.view(np.uint32)
        u += np.uint32(0x7FFF) + ((u >> 16) & np.uint32(1))
        u &= np.uint32(0xFFFF0000)
    return ff1, ff2


class DecodeStack:
    def __init__(self, layers, ffn_dim: int | None = None, comm=None, seed: int = 0, ffn_weights=None):
        import torch
        self.torch = torch
        self.layers = list(layers)
        if not self.layers:
            raise ValueError("a stack needs at least one layer")
        l0 = self.layers[0]
        self.B, self.E = l0.batch, l0.embed_dim
        if l0.e_out != self.E:
            raise ValueError("stack layers must project back to the model width")
        self.F = ffn_dim or 2 * self.E
        self.comm = comm
        dev = torch.device("cuda", l0.device)
        # per layer (ff1, ff2): given, or the toy model's random init (generated
        # and uploaded one layer at a time; the host copies are not kept)
        self.ffn_weights = ffn_weights
        self.ffns = []
        for i in range(len(self.layers)):
            w1, w2 = ffn_weights[i] if ffn_weights else toy_ffn_weights(self.E, self.F, seed * 1000 + i)
            self.ffns.append(FeedForward(w1, w2, device=l0.device))
        self.o = torch.empty((self.B, self.E), device=dev, dtype=torch.float32)
        self.cur = torch.empty((self.B, self.E), device=dev, dtype=torch.float32)

    def ffn_bytes(self) -> int:
        return 2 * 2 * self.E * self.F * len(self.layers)  # bf16 ff1 + ff2 per layer

    def step(self, x, y, stream=None, record=None):
        """One token for every sequence through every layer: x, y [B][E] fp32.
        record (a list, tests): per layer (input token, O-projection output,
        FFN output) copies."""
        cur = x
        n = len(self.layers)
        for i, layer in enumerate(self.layers):
            if record is not None:
                record.append([cur.clone()])
            layer.step(cur, self.o, graph=False, stream=stream)
            if self.comm is not None:
                self.comm.allreduce_(self.o)
            dst = y if i == n - 1 else self.cur
            if record is not None:
                record[-1].append(self.o.clone())
            self.ffns[i].forward(self.o, dst, stream=stream)
            if record is not None:
                record[-1].append(dst.clone())
            cur = dst
        return y
