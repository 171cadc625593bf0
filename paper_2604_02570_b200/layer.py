"""Batched, device-resident decode layer: the performance API used by the
benchmark and the multi-GPU path.

One object holds (a head shard of) one attention layer on one GPU: the
factored Q/K/V projections, the matching rows of W_o, and a latent cache for
``batch`` sequences.  ``step`` is pipe::decode_factored's per-token body for
one layer (pipeline.cpp:320-329): append the token, attend with its own
query, O-project -- launched as one CUDA graph (projection GEMM, append
epilogue, attention, O-proj GEMM, split reduction).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .decode import DeviceLayer, LayerFactors
from .errors import ConfigError, ShapeError


def _torch():
    import torch
    return torch


class DecodeLayer:
    def __init__(self, f: LayerFactors, w_o_rows: np.ndarray | None, batch: int, capacity: int,
                 cache_dtype: str = "bf16", weight_dtype: str = "bf16", oproj_dtype: str = "bf16",
                 device: int = 0, head_offset: int = 0, act_rotation: bool | None = None,
                 quantized=None, attention: str | None = None, device_layer=None):
        if cache_dtype not in ("f32", "bf16", "i8"):
            raise ConfigError(f"unknown cache dtype '{cache_dtype}'")
        self.device = device
        self.batch = batch
        if device_layer is not None:  # built by the library (e.g. from a checkpoint)
            self.layer = device_layer
        else:
            self.layer = DeviceLayer(f, weight_dtype, device, act_rotation=act_rotation,
                                     head_offset=head_offset, quantized=quantized)
        self.e_out = getattr(self.layer, "e_out", None)
        if w_o_rows is not None:
            self.layer.set_oproj(w_o_rows, oproj_dtype)
            self.e_out = self.layer.e_out
        h = C.c_void_p()
        N.call("wsvd_cache_create", self.layer.h, batch, capacity, N.DTYPES[cache_dtype],
               C.byref(h))
        self.h = h
        self.n_heads = self.layer.n_heads
        self.head_dim = self.layer.head_dim
        self.embed_dim = self.layer.embed_dim
        self.rpad = self.layer.rpad
        rb = C.c_int32()
        N.call("wsvd_cache_row_bytes", self.h, C.byref(rb))
        self.row_bytes = rb.value
        if attention is not None:
            self.set_attention(attention)

    ATTENTION = {"absorbed": 0, "explicit_tc": 1}

    def set_attention(self, mode: str):
        """'absorbed' (scores against qt = q . B_K^T) or 'explicit_tc' (the
        reference's key_j = C_K[j] . B_K rebuilt on tcgen05 tensor cores)."""
        if mode not in self.ATTENTION:
            raise ConfigError(f"unknown attention mode '{mode}'")
        N.call("wsvd_cache_set_attention_mode", self.h, self.ATTENTION[mode])

    @property
    def attention(self) -> str:
        m = C.c_int32()
        N.call("wsvd_cache_attention_mode", self.h, C.byref(m))
        return {v: k for k, v in self.ATTENTION.items()}[m.value]

    def __del__(self):
        if getattr(self, "h", None) and N._lib is not None:
            N.lib().wsvd_cache_destroy(self.h)
            self.h = None

    @staticmethod
    def _ptr(t):
        return C.c_void_p(t.data_ptr())

    @staticmethod
    def _stream(stream=None):
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream()
        return C.c_void_p(s.cuda_stream)

    def length(self) -> int:
        n = C.c_int32()
        N.call("wsvd_cache_length", self.h, C.byref(n))
        return n.value

    def reset(self):
        N.call("wsvd_cache_reset", self.h)

    def prefill(self, x, stream=None):
        """x: fp32 device tensor [T][batch][E] (token-major)."""
        if x.dim() != 3 or x.shape[1] != self.batch or x.shape[2] != self.embed_dim:
            raise ShapeError(f"prefill expects [T][{self.batch}][{self.embed_dim}], got {tuple(x.shape)}")
        N.call("wsvd_prefill", self.h, self._ptr(x), int(x.shape[0]), self._stream(stream))

    def append(self, x, q_out=None, stream=None):
        N.call("wsvd_append_token", self.h, self._ptr(x),
               self._ptr(q_out) if q_out is not None else None, self._stream(stream))

    def attend(self, q, out, tile_len: int = 32, stream=None):
        N.call("wsvd_fused_decode_step", self.h, self._ptr(q), tile_len, self._ptr(out),
               self._stream(stream))

    def attention_only(self, out, stream=None):
        """The attention kernel alone (absorbed query of the last append)."""
        N.call("wsvd_decode_attention", self.h, self._ptr(out), self._stream(stream))

    def step(self, x, y, attn_out=None, graph: bool = True, stream=None):
        """One layer step for every sequence: x [batch][E] -> y [batch][e_out]
        (this shard's partial O-projection)."""
        if self.e_out is None:
            raise ConfigError("layer built without W_o rows")
        if graph and attn_out is None:
            N.call("wsvd_layer_step_graph", self.h, self._ptr(x), self._ptr(y), self._stream(stream))
        else:
            N.call("wsvd_layer_step", self.h, self._ptr(x),
                   self._ptr(attn_out) if attn_out is not None else None, self._ptr(y),
                   self._stream(stream))

    def fill_synthetic(self, length: int, seed: int = 0, scale: float = 1.0):
        """Benchmark prefill: synthetic N(0, scale^2) latent rows, length rows."""
        N.call("wsvd_cache_fill_synthetic", self.h, int(length), int(seed), float(scale))

    def sync_length(self) -> int:
        """Host mirror of the length after steps replayed in a caller's graph."""
        n = C.c_int32()
        N.call("wsvd_cache_sync_length", self.h, C.byref(n))
        return n.value

    def _step_info(self):
        fused, launches = C.c_int32(0), C.c_int32(0)
        N.call("wsvd_cache_step_info", self.h, C.byref(fused), C.byref(launches))
        return bool(fused.value), int(launches.value)

    def launches_per_step(self) -> int:
        """Kernels one layer step launches (wsvd_cache_step_info)."""
        return self._step_info()[1]

    def step_kind(self) -> str:
        fused, n = self._step_info()
        return ("one persistent fused-step kernel per step (PDL launch)" if fused
                else f"{n} kernels per step, replayed as one CUDA graph")

    def step_host(self, x_host, y_host, stream=None):
        """Same through host buffers (pinned torch tensors or numpy arrays)."""
        def hp(t):
            if isinstance(t, np.ndarray):
                return C.c_void_p(t.ctypes.data)
            return C.c_void_p(t.data_ptr())
        N.call("wsvd_layer_step_host", self.h, hp(x_host), hp(y_host), self._stream(stream))

    def read_latents(self, seq: int, head: int):
        L, R = self.length(), self.rpad
        ck = np.zeros((L, R))
        cv = np.zeros((L, R))
        N.call("wsvd_cache_read_host", self.h, seq, head, ck.ctypes.data_as(C.POINTER(C.c_double)),
               cv.ctypes.data_as(C.POINTER(C.c_double)))
        return ck, cv

    def debug_copy(self, what: str) -> np.ndarray:
        """Internal buffers of the last append (see wsvd_cache_debug_copy)."""
        code = {"xq": 0, "sx": 1, "acc": 2, "qt": 3, "trace": 4, "scores": 5}[what]
        nbytes = C.c_int64(1 << 30)
        buf = np.empty(1 << 28, dtype=np.uint8)
        N.call("wsvd_cache_debug_copy", self.h, code, C.c_void_p(buf.ctypes.data), C.byref(nbytes))
        raw = buf[: nbytes.value].copy()
        if what == "xq":
            return raw.view(np.int8)
        if what == "trace":
            return raw.view(np.uint64).reshape(-1, 32)
        if what == "scores":
            return raw.view(np.int32)
        if what == "acc":
            return raw.view(np.int32 if self.layer.weight_dtype in ("i8", "i4") else np.float32)
        return raw.view(np.float32)

    def set_debug(self, flags: int):
        """Test hook (int8 caches): bit 0 records the int32 score accumulators
        of the following attention launches (debug_copy("scores"))."""
        N.call("wsvd_cache_set_debug", self.h, int(flags))

    def read_raw(self, seq: int, head: int):
        L = self.length()
        rows = np.zeros((L, self.row_bytes), dtype=np.uint8)
        scales = np.zeros((L, 2), dtype=np.uint16)
        N.call("wsvd_cache_read_raw", self.h, seq, head, C.c_void_p(rows.ctypes.data),
               C.c_void_p(scales.ctypes.data))
        return rows, scales


class DecodeChain:
    """The attention blocks of a decode stack chained on one GPU:
    pipe::decode_factored's layer loop (pipeline.cpp:318-336) with layer
    l + 1's token = layer l's output (no FFN between them).  ``step`` runs the
    whole chain as ONE persistent kernel when every layer takes the fused step
    (wsvd_chain_step); every layer appends to its own cache."""

    def __init__(self, layers):
        self.layers = list(layers)
        if not self.layers:
            raise ConfigError("a chain needs at least one layer")
        self._hs = (C.c_void_p * len(self.layers))(*[lay.h.value for lay in self.layers])
        l0 = self.layers[0]
        self.batch, self.embed_dim = l0.batch, l0.embed_dim

    def __len__(self):
        return len(self.layers)

    def fused(self) -> bool:
        return len(self.layers) <= 32 and all(lay._step_info()[0] for lay in self.layers)

    def launches_per_step(self) -> int:
        return 1 if self.fused() else sum(lay.launches_per_step() for lay in self.layers)

    def step(self, x, ys, stream=None):
        """x [batch][E] fp32 device tensor; ys: one [batch][E] fp32 device
        tensor per layer (layer l's output; the last is the chain's)."""
        if len(ys) != len(self.layers):
            raise ShapeError(f"{len(self.layers)} layers need {len(self.layers)} outputs, got {len(ys)}")
        yp = (C.c_void_p * len(ys))(*[t.data_ptr() for t in ys])
        N.call("wsvd_chain_step", self._hs, len(self.layers), DecodeLayer._ptr(x), yp,
               DecodeLayer._stream(stream))

    def step_host(self, x_host, y_host, stream=None):
        """Same through host buffers: x_host in, the last layer's y out."""
        def hp(t):
            if isinstance(t, np.ndarray):
                return C.c_void_p(t.ctypes.data)
            return C.c_void_p(t.data_ptr())
        N.call("wsvd_chain_step_host", self._hs, len(self.layers), hp(x_host), hp(y_host),
               DecodeLayer._stream(stream))
