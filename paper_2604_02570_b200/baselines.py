"""Comparison baseline of the paper's latency tables: a dense (full-rank) decode
layer over the FULL KV cache with Flash Decoding = PyTorch scaled-dot-product
attention ("For Flash Decoding, we adopt scaled dot-product
attention (SDPA)"; both Eager and Flash Decoding "operate on the full KV
cache").  It is the reference point of the speed-up the paper reports (> 1.8x
for WSVD-noQ), built from library kernels (cuBLAS GEMMs, the SDPA backend) on
purpose: it is a baseline, never the product path.

One step, per sequence: qkv = x . W_qkv (dense E x 3E), append k / v at the
cache tail, out = SDPA(q, K[:len], V[:len]), y = out . W_o -- the dense
counterpart of decode::append_token + fused_decode_step + heads_row . W_o
(src/decode.cpp:127-206, src/pipeline.cpp:320-329; the reference's own dense
path is decode::flash_decode_step, src/decode.cpp:250-303).
"""
from __future__ import annotations

import math


class DenseFlashDecodeLayer:
    def __init__(self, embed_dim: int, n_heads: int, head_dim: int, batch: int, capacity: int,
                 device=0, dtype=None, seed: int = 0):
        import torch
        self.torch = torch
        dt = dtype or torch.bfloat16
        self.E, self.nh, self.H, self.B = embed_dim, n_heads, head_dim, batch
        self.dev = torch.device("cuda", device)
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed)
        d = n_heads * head_dim
        self.w_qkv = (torch.randn((embed_dim, 3 * d), generator=g, device=self.dev) / math.sqrt(embed_dim)).to(dt)
        self.w_o = (torch.randn((d, embed_dim), generator=g, device=self.dev) / math.sqrt(d)).to(dt)
        # [B][nh][cap][H] full-rank caches (the bytes the latent cache replaces)
        self.k = torch.zeros((batch, n_heads, capacity, head_dim), device=self.dev, dtype=dt)
        self.v = torch.zeros_like(self.k)
        self.len = 0
        self.cap = capacity

    def fill(self, length: int, seed: int = 1):
        g = self.torch.Generator(device=self.dev)
        g.manual_seed(seed)
        self.k[:, :, :length].normal_(generator=g)
        self.v[:, :, :length].normal_(generator=g)
        self.len = length

    def kv_bytes(self, length: int) -> int:
        return 2 * self.B * self.nh * length * self.H * self.k.element_size()

    def step_fn(self, x, y, pos: int):
        """Returns a closure running one layer step for cache position `pos`
        (fixed: CUDA-graph capturable); x [B][E] bf16, y [B][E] bf16."""
        torch = self.torch
        F = torch.nn.functional
        B, nh, H = self.B, self.nh, self.H
        k_slot = self.k[:, :, pos:pos + 1]
        v_slot = self.v[:, :, pos:pos + 1]
        K = self.k[:, :, :pos + 1]
        V = self.v[:, :, :pos + 1]

        def run():
            qkv = x @ self.w_qkv                                   # [B][3 nh H]
            q, k, v = qkv.view(B, 3, nh, H).unbind(1)
            k_slot.copy_(k.view(B, nh, 1, H))
            v_slot.copy_(v.view(B, nh, 1, H))
            out = F.scaled_dot_product_attention(q.view(B, nh, 1, H), K, V)  # flash decoding
            torch.matmul(out.reshape(B, nh * H), self.w_o, out=y)
        return run


class SharedLatentLayer:
    """The paper's "W/o per-head" comparison (reference
    decode::shared_decode_step with materialize, src/decode.cpp:330-390): one
    shared latent of width R_s = n_heads * r per layer (the same cache bytes as
    the per-head latents), which every head reads in full; the naive schedule
    rebuilds every head's full keys and values (K = C_K . B_K, V = C_V . B_V,
    written back to memory) and then attends over them with SDPA.  Library
    kernels (cuBLAS, SDPA) on purpose: it is a baseline."""

    def __init__(self, embed_dim: int, n_heads: int, head_dim: int, shared_rank: int, batch: int,
                 capacity: int, device=0, dtype=None, seed: int = 0):
        import torch
        self.torch = torch
        dt = dtype or torch.bfloat16
        self.E, self.nh, self.H, self.R, self.B = embed_dim, n_heads, head_dim, shared_rank, batch
        self.dev = torch.device("cuda", device)
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed)
        d = n_heads * head_dim
        self.a_q = (torch.randn((embed_dim, d), generator=g, device=self.dev) / math.sqrt(embed_dim)).to(dt)
        self.a_kv = (torch.randn((embed_dim, 2 * shared_rank), generator=g, device=self.dev)
                     / math.sqrt(embed_dim)).to(dt)
        self.b_k = (torch.randn((shared_rank, d), generator=g, device=self.dev) / math.sqrt(shared_rank)).to(dt)
        self.b_v = (torch.randn((shared_rank, d), generator=g, device=self.dev) / math.sqrt(shared_rank)).to(dt)
        self.w_o = (torch.randn((d, embed_dim), generator=g, device=self.dev) / math.sqrt(d)).to(dt)
        self.ck = torch.zeros((batch, capacity, shared_rank), device=self.dev, dtype=dt)
        self.cv = torch.zeros_like(self.ck)
        self.cap = capacity

    def fill(self, length: int, seed: int = 1):
        g = self.torch.Generator(device=self.dev)
        g.manual_seed(seed)
        self.ck[:, :length].normal_(generator=g)
        self.cv[:, :length].normal_(generator=g)

    def latent_bytes(self, length: int) -> int:
        return self.B * length * 2 * self.R * self.ck.element_size()

    def step_fn(self, x, y, pos: int):
        torch = self.torch
        F = torch.nn.functional
        B, nh, H, R = self.B, self.nh, self.H, self.R
        CK, CV = self.ck[:, :pos + 1], self.cv[:, :pos + 1]

        def run():
            q = (x @ self.a_q).view(B, nh, 1, H)
            ckv = x @ self.a_kv
            self.ck[:, pos].copy_(ckv[:, :R])
            self.cv[:, pos].copy_(ckv[:, R:])
            # materialised keys and values of every head, [B][nh][L][H]
            K = (CK @ self.b_k).view(B, pos + 1, nh, H).transpose(1, 2).contiguous()
            V = (CV @ self.b_v).view(B, pos + 1, nh, H).transpose(1, 2).contiguous()
            out = F.scaled_dot_product_attention(q, K, V)
            torch.matmul(out.reshape(B, nh * H), self.w_o, out=y)
        return run
