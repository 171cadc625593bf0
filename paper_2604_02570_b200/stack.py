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
the FFN is a replicated pair of bf16 cuBLAS GEMMs (a plain library GEMM: it is
not on the WSVD path).
"""
from __future__ import annotations

import math


class DecodeStack:
    def __init__(self, layers, ffn_dim: int | None = None, comm=None, seed: int = 0, dtype=None):
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
        dt = dtype or torch.bfloat16
        dev = torch.device("cuda", l0.device)
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        # ff1 ~ N(0, 1/E), ff2 ~ N(0, 1/F) (toymodel.cpp:81-95 initialisation scale)
        self.ff1 = [(torch.randn((self.E, self.F), generator=g, device=dev) / math.sqrt(self.E)).to(dt)
                    for _ in self.layers]
        self.ff2 = [(torch.randn((self.F, self.E), generator=g, device=dev) / math.sqrt(self.F)).to(dt)
                    for _ in self.layers]
        self.o = torch.empty((self.B, self.E), device=dev, dtype=torch.float32)
        self.o16 = torch.empty((self.B, self.E), device=dev, dtype=dt)
        self.h = torch.empty((self.B, self.F), device=dev, dtype=dt)
        self.cur16 = torch.empty((self.B, self.E), device=dev, dtype=dt)
        self.cur = torch.empty((self.B, self.E), device=dev, dtype=torch.float32)

    def ffn_bytes(self) -> int:
        return sum(w.numel() * w.element_size() for w in self.ff1 + self.ff2)

    def step(self, x, y, stream=None):
        """One token for every sequence through every layer: x, y [B][E] fp32."""
        torch = self.torch
        cur = x
        n = len(self.layers)
        for i, layer in enumerate(self.layers):
            layer.step(cur, self.o, graph=False, stream=stream)
            if self.comm is not None:
                self.comm.allreduce_(self.o)
            self.o16.copy_(self.o)
            torch.matmul(self.o16, self.ff1[i], out=self.h)
            torch.tanh_(self.h)
            torch.matmul(self.h, self.ff2[i], out=self.cur16)
            dst = y if i == n - 1 else self.cur
            dst.copy_(self.cur16)
            cur = dst
        return y
