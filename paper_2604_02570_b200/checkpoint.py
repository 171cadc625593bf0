"""Reader of the reference's checkpoint directories (wsvd::ckpt,
src/checkpoint.cpp:168-333) over the library's C++ reader
(csrc/checkpoint.cpp, include/wsvd_b200.h `wsvd_ckpt_*`), and the bridge to
device layers: real WSVD artefacts -- per-head SVD / fine-tuned factors or the
QAT export Q(S1 A S2^T), Q(S2 B) with per-column scales -- drive the kernels
instead of random-init factors.

    ck = Checkpoint("run/checkpoint")
    layer = ck.decode_layer(0, batch=16, capacity=8192, cache_dtype="i8", weight_dtype="i8")
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .decode import DeviceLayer, HeadFactors, HeadProjection, LayerFactors, Role

ROLES = ("q", "k", "v")


class Checkpoint:
    def __init__(self, path: str):
        self.path = str(path)
        self._p = self.path.encode()
        info = (C.c_int64 * 8)()
        N.call("wsvd_ckpt_info", self._p, info)
        (self.embed_dim, self.head_dim, self.n_heads, self.n_layers, self.weight_bits,
         self.activation_bits, has_f, has_q) = (int(v) for v in info)
        self.has_factors, self.has_quantized = bool(has_f), bool(has_q)

    def head(self, layer: int, head: int, role: int):
        """fp64 factors (a [E][rank], b [rank][H]) of factorize::HeadFactors."""
        r = C.c_int32()
        N.call("wsvd_ckpt_head", self._p, layer, head, role, C.byref(r), None, None)
        a = np.empty((self.embed_dim, r.value))
        b = np.empty((r.value, self.head_dim))
        N.call("wsvd_ckpt_head", self._p, layer, head, role, None,
               a.ctypes.data_as(C.POINTER(C.c_double)), b.ctypes.data_as(C.POINTER(C.c_double)))
        return a, b

    def head_quantized(self, layer: int, head: int, role: int):
        """quant::QuantizedFactors (quant.hpp:98-107): (a_q, a_scales, b_q, b_scales)."""
        r = C.c_int32()
        N.call("wsvd_ckpt_head_quantized", self._p, layer, head, role, C.byref(r), None, None, None, None)
        aq = np.empty((self.embed_dim, r.value), dtype=np.int8)
        bq = np.empty((r.value, self.head_dim), dtype=np.int8)
        as_ = np.empty(r.value)
        bs = np.empty(self.head_dim)
        N.call("wsvd_ckpt_head_quantized", self._p, layer, head, role, None,
               aq.ctypes.data_as(C.POINTER(C.c_int8)), as_.ctypes.data_as(C.POINTER(C.c_double)),
               bq.ctypes.data_as(C.POINTER(C.c_int8)), bs.ctypes.data_as(C.POINTER(C.c_double)))
        return aq, as_, bq, bs

    def weight(self, name: str) -> np.ndarray:
        rows, cols = C.c_int64(0), C.c_int64(0)
        N.call("wsvd_ckpt_weight", self._p, name.encode(), C.byref(rows), C.byref(cols), None)
        out = np.empty((rows.value, cols.value))
        N.call("wsvd_ckpt_weight", self._p, name.encode(), C.byref(rows), C.byref(cols),
               out.ctypes.data_as(C.POINTER(C.c_double)))
        return out

    def factors(self, layer: int, heads: tuple[int, int] | None = None, quantized: bool = False) -> LayerFactors:
        """decode::LayerFactors of (a head range of) one layer; with quantized the
        geometry comes from the quantised entries (their factors are rotated)."""
        h0, h1 = heads or (0, self.n_heads)
        hp = []
        for h in range(h0, h1):
            roles = []
            for role in range(3):
                if quantized:
                    aq, _, bq, _ = self.head_quantized(layer, h, role)
                    a, b = aq.astype(np.float64), bq.astype(np.float64)
                else:
                    a, b = self.head(layer, h, role)
                roles.append(HeadFactors(a=a, b=b, rank=a.shape[1], layer=layer, head=h, role=Role(role)))
            hp.append(HeadProjection(*roles))
        return LayerFactors(heads=hp, embed_dim=self.embed_dim, head_dim=self.head_dim)

    def decode_layer(self, layer: int, batch: int, capacity: int, cache_dtype: str = "bf16",
                     weight_dtype: str = "bf16", heads: tuple[int, int] | None = None,
                     oproj_dtype: str | None = "bf16", device: int = 0, **kw):
        """A DecodeLayer whose device factors (and W_o rows) the C++ loader
        built straight from the checkpoint files (wsvd_layer_load_checkpoint)."""
        from .layer import DecodeLayer
        h0, h1 = heads or (0, self.n_heads)
        quant = weight_dtype in ("i8", "i4")
        h = C.c_void_p()
        N.call("wsvd_layer_load_checkpoint", self._p, layer, h0, h1, N.DTYPES[weight_dtype],
               N.DTYPES[oproj_dtype] if oproj_dtype else -1, device, C.byref(h))
        f = self.factors(layer, (h0, h1), quantized=quant)
        dl = DeviceLayer.adopt(h, f, weight_dtype, device, e_out=self.embed_dim if oproj_dtype else None)
        return DecodeLayer(f, None, batch=batch, capacity=capacity, cache_dtype=cache_dtype,
                           weight_dtype=weight_dtype, device=device, device_layer=dl, **kw)
