"""Python mirror of the reference operator API ``wsvd::decode``
(/root/reference/proj/include/wsvd/decode.hpp), backed by the sm_100a kernels
through the C ABI (include/wsvd_b200.h).

Names, argument meaning and error behaviour follow the reference so that the
parity tests read like tests/test_decode.cpp:

    f = LayerFactors(heads=[HeadProjection(q, k, v), ...], embed_dim=E, head_dim=H)
    cache = LatentCache(f)                       # decode.hpp:83-96
    q = append_token(cache, f, x, counter)       # decode.cpp:127-153
    out = fused_decode_step(cache, f, q, TileConfig(32), counter)   # decode.cpp:155-206

Differences, all additive: the cache lives in device memory with a fixed
capacity; ``batch`` sequences advance together (x of shape (B, E) returns
(B, n_heads, H)); ``cache_dtype`` / ``weight_dtype`` select the storage
formats ("f32" keeps the reference's fp64 semantics up to fp32 rounding,
"bf16" is config 2, "i8"/"i4" the W8A8/W4A8 paths).  TrafficCounter is
filled from the reference's closed forms (decode.cpp:132-149, 176-203).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import ConfigError, NumericError, ShapeError


# --------------------------------------------------------------- counters --
class Stream(enum.IntEnum):
    """decode.hpp:16-24"""
    LatentK = 0
    LatentV = 1
    FullK = 2
    FullV = 3
    WeightsB = 4
    Query = 5
    Output = 6


kStreamCount = 7
_STREAM_NAMES = ["latent_k", "latent_v", "full_k", "full_v", "weights_b", "query", "output"]


def stream_name(s: Stream) -> str:
    return _STREAM_NAMES[int(s)]


@dataclass
class StreamTally:
    loads: int = 0
    stores: int = 0
    flops: int = 0


class TrafficCounter:
    """Monotone per-stream tallies (decode.hpp:35-49); storage is the C ABI's
    [loads(7) | stores(7) | flops(7)] uint64 block."""

    def __init__(self):
        self.raw = np.zeros(21, dtype=np.uint64)

    def add_loads(self, s: Stream, n: int):
        self.raw[int(s)] += np.uint64(n)

    def add_stores(self, s: Stream, n: int):
        self.raw[7 + int(s)] += np.uint64(n)

    def add_flops(self, s: Stream, n: int):
        self.raw[14 + int(s)] += np.uint64(n)

    def __getitem__(self, s: Stream) -> StreamTally:
        i = int(s)
        return StreamTally(int(self.raw[i]), int(self.raw[7 + i]), int(self.raw[14 + i]))

    def total_loads(self) -> int:
        return int(self.raw[:7].sum())

    def total_stores(self) -> int:
        return int(self.raw[7:14].sum())

    def _ptr(self):
        return self.raw.ctypes.data_as(C.POINTER(C.c_uint64))


@dataclass
class TileConfig:
    """decode.hpp:51-53 -- rows of cache per tile, >= 1.  The device streams
    128-token stages; tile_len only has to be valid (results are tile-free up
    to reassociation, as test_decode.cpp:206-227 pins for the reference)."""
    tile_len: int = 32


# ----------------------------------------------------------------- factors --
class Role(enum.IntEnum):
    """factorize.hpp:15"""
    Q = 0
    K = 1
    V = 2


@dataclass
class HeadFactors:
    """factorize.hpp:20-27: a (E x rank) and b (rank x head_dim)."""
    a: np.ndarray
    b: np.ndarray
    rank: int = 0
    layer: int = 0
    head: int = 0
    role: Role = Role.K

    def __post_init__(self):
        if not self.rank:
            self.rank = int(np.asarray(self.a).shape[1])


@dataclass
class HeadProjection:
    q: HeadFactors
    k: HeadFactors
    v: HeadFactors


@dataclass(eq=False)
class LayerFactors:
    """decode.hpp:76-79"""
    heads: list = field(default_factory=list)
    embed_dim: int = 0
    head_dim: int = 0

    def ranks(self) -> np.ndarray:
        return np.array([[p.q.rank, p.k.rank, p.v.rank] for p in self.heads], dtype=np.int32)


class DeviceLayer:
    """Device copy of (a head shard of) one layer's factors: wsvd_layer_t."""

    def __init__(self, f: LayerFactors, weight_dtype: str = "f32", device: int = 0,
                 act_rotation: bool | None = None, head_offset: int = 0, quantized=None):
        """quantized: optional per head, per role (q, k, v) tuples
        (a_q int8 E x r, a_scales r, b_q int8 r x H, b_scales H) -- already
        rotated factors as quant::QuantizedFactors holds them (quant.hpp:98-107);
        f then only supplies the geometry."""
        if not f.heads:
            raise ShapeError("latent cache over zero heads")
        if weight_dtype not in N.DTYPES:
            raise ConfigError(f"unknown weight dtype '{weight_dtype}'")
        wd = N.DTYPES[weight_dtype]
        if act_rotation is None:
            act_rotation = wd in (N.I8, N.I4)
        self.f = f
        self.weight_dtype = weight_dtype
        self.device = device
        self.n_heads = len(f.heads)
        self.embed_dim = f.embed_dim
        self.head_dim = f.head_dim
        self.ranks = f.ranks()
        desc = N.LayerDesc(f.embed_dim, f.head_dim, len(f.heads), head_offset, wd,
                           1 if act_rotation else 0, device)
        h = C.c_void_p()
        r = np.ascontiguousarray(self.ranks)
        N.call("wsvd_layer_create", C.byref(desc), r.ctypes.data_as(C.POINTER(C.c_int32)),
               C.byref(h))
        self.h = h
        for hi, p in enumerate(f.heads):
            for role, hf in enumerate((p.q, p.k, p.v)):
                if quantized is not None:
                    aq, as_, bq, bs = quantized[hi][role]
                    aq = np.ascontiguousarray(aq, dtype=np.int8)
                    bq = np.ascontiguousarray(bq, dtype=np.int8)
                    as_ = np.ascontiguousarray(as_, dtype=np.float64)
                    bs = np.ascontiguousarray(bs, dtype=np.float64)
                    N.call("wsvd_layer_set_head_quantized", self.h, hi, role,
                           aq.ctypes.data_as(C.POINTER(C.c_int8)),
                           as_.ctypes.data_as(C.POINTER(C.c_double)),
                           bq.ctypes.data_as(C.POINTER(C.c_int8)),
                           bs.ctypes.data_as(C.POINTER(C.c_double)))
                    continue
                a = np.ascontiguousarray(hf.a, dtype=np.float64)
                b = np.ascontiguousarray(hf.b, dtype=np.float64)
                if a.shape != (f.embed_dim, hf.rank) or b.shape != (hf.rank, f.head_dim):
                    raise ShapeError(f"head {hi} role {role}: factors {a.shape} x {b.shape} "
                                     f"disagree with E={f.embed_dim}, H={f.head_dim}, "
                                     f"rank={hf.rank}")
                N.call("wsvd_layer_set_head", self.h, hi, role,
                       a.ctypes.data_as(C.POINTER(C.c_double)),
                       b.ctypes.data_as(C.POINTER(C.c_double)))
        rp = C.c_int32()
        N.call("wsvd_layer_rank_pad", self.h, C.byref(rp))
        self.rpad = rp.value

    @classmethod
    def adopt(cls, handle, f: "LayerFactors", weight_dtype: str, device: int, e_out: int | None = None):
        """Wrap a wsvd_layer_t built by the library itself (e.g.
        wsvd_layer_load_checkpoint); f supplies the geometry."""
        self = cls.__new__(cls)
        self.f = f
        self.weight_dtype = weight_dtype
        self.device = device
        self.n_heads = len(f.heads)
        self.embed_dim = f.embed_dim
        self.head_dim = f.head_dim
        self.ranks = f.ranks()
        self.h = handle
        rp = C.c_int32()
        N.call("wsvd_layer_rank_pad", self.h, C.byref(rp))
        self.rpad = rp.value
        if e_out is not None:
            self.e_out = e_out
        return self

    def set_oproj(self, w_o_rows: np.ndarray, dtype: str = "bf16"):
        """pipeline.cpp:329: rows of W_o multiplying this layer's heads."""
        w = np.ascontiguousarray(w_o_rows, dtype=np.float64)
        if w.shape[0] != self.n_heads * self.head_dim:
            raise ShapeError(f"W_o rows {w.shape[0]} != n_heads*head_dim "
                             f"{self.n_heads * self.head_dim}")
        N.call("wsvd_layer_set_oproj", self.h, w.ctypes.data_as(C.POINTER(C.c_double)),
               w.shape[1], N.DTYPES[dtype])
        self.e_out = w.shape[1]

    def __del__(self):
        if getattr(self, "h", None) and N._lib is not None:
            N.lib().wsvd_layer_destroy(self.h)
            self.h = None


def _device_layer(f: LayerFactors, weight_dtype: str, device: int) -> DeviceLayer:
    """One upload per (factors object, dtype, device); call invalidate(f)
    after mutating a LayerFactors in place."""
    store = f.__dict__.setdefault("_wsvd_device", {})
    key = (weight_dtype, device)
    if key not in store:
        store[key] = DeviceLayer(f, weight_dtype, device)
    return store[key]


def invalidate(f: LayerFactors) -> None:
    f.__dict__.pop("_wsvd_device", None)


# ------------------------------------------------------------------- cache --
def _torch():
    import torch  # device buffers and streams are PyTorch plumbing
    return torch


class LatentCache:
    """decode.hpp:83-96: per-head latent rows x_t A_kh | x_t A_vh, on device."""

    def __init__(self, f: LayerFactors, batch: int = 1, capacity: int = 4096,
                 cache_dtype: str = "f32", weight_dtype: str = "f32", device: int = 0):
        if not f.heads:
            raise ShapeError("latent cache over zero heads")
        if cache_dtype not in ("f32", "bf16", "i8"):
            raise ConfigError(f"unknown cache dtype '{cache_dtype}'")
        self.f = f
        self.batch = batch
        self.capacity = capacity
        self.cache_dtype = cache_dtype
        self.weight_dtype = weight_dtype
        self.device = device
        self.layer = _device_layer(f, weight_dtype, device)
        h = C.c_void_p()
        N.call("wsvd_cache_create", self.layer.h, batch, capacity, N.DTYPES[cache_dtype],
               C.byref(h))
        self.h = h
        self._bound = self.layer
        self._staged: dict[int, tuple[np.ndarray, np.ndarray]] = {}

    def __del__(self):
        if getattr(self, "h", None) and N._lib is not None:
            N.lib().wsvd_cache_destroy(self.h)
            self.h = None

    def length(self) -> int:
        n = C.c_int32()
        N.call("wsvd_cache_length", self.h, C.byref(n))
        return n.value

    def n_heads(self) -> int:
        return self.layer.n_heads

    def _read(self, head: int, seq: int):
        L, R = self.length(), self.layer.rpad
        ck = np.zeros((L, R))
        cv = np.zeros((L, R))
        N.call("wsvd_cache_read_host", self.h, seq, head, ck.ctypes.data_as(C.POINTER(C.c_double)),
               cv.ctypes.data_as(C.POINTER(C.c_double)))
        return ck, cv

    def latent_k(self, head: int, seq: int = 0) -> np.ndarray:
        ck, _ = self._read(head, seq)
        return ck[:, : self.layer.ranks[head, 1]]

    def latent_v(self, head: int, seq: int = 0) -> np.ndarray:
        _, cv = self._read(head, seq)
        return cv[:, : self.layer.ranks[head, 2]]

    def push(self, head: int, ck, cv):
        """Stage one head's latent row; bump_length() commits all heads."""
        self._staged[head] = (np.asarray(ck, dtype=np.float64), np.asarray(cv, dtype=np.float64))

    def bump_length(self):
        nh, R = self.n_heads(), self.layer.rpad
        ck = np.zeros((self.batch, nh, R))
        cv = np.zeros((self.batch, nh, R))
        for h, (k, v) in self._staged.items():
            ck[:, h, : k.shape[-1]] = k
            cv[:, h, : v.shape[-1]] = v
        self._staged = {}
        N.call("wsvd_cache_push_host", self.h, ck.ctypes.data_as(C.POINTER(C.c_double)),
               cv.ctypes.data_as(C.POINTER(C.c_double)))

    def reset(self):
        N.call("wsvd_cache_reset", self.h)

    def _bind(self, f: LayerFactors):
        if f is self.f:
            target = self.layer
        else:
            if len(f.heads) != self.n_heads():
                raise ShapeError(f"cache holds {self.n_heads()} heads, factors {len(f.heads)}")
            target = _device_layer(f, self.weight_dtype, self.device)
        if target is not self._bound:
            N.call("wsvd_cache_bind_layer", self.h, target.h)
            self._bound = target


# --------------------------------------------------------------- operators --
def _stream():
    return C.c_void_p(_torch().cuda.current_stream().cuda_stream)


def append_token(cache: LatentCache, f: LayerFactors, x, counter: TrafficCounter | None = None):
    """decode.cpp:127-153.  x: (E,) -> q (n_heads, H); x: (B, E) -> (B, n_heads, H)."""
    torch = _torch()
    x = np.asarray(x, dtype=np.float64)
    single = x.ndim == 1
    x2 = x.reshape(1, -1) if single else x
    if x2.shape[-1] != f.embed_dim:
        raise ShapeError(f"token has {x2.shape[-1]} features, layer expects {f.embed_dim}")
    if x2.shape[0] != cache.batch:
        raise ShapeError(f"{x2.shape[0]} tokens for a cache of {cache.batch} sequences")
    if not np.isfinite(x2).all():
        raise NumericError("append_token: non-finite token")
    cache._bind(f)
    dev = torch.device("cuda", cache.device)
    xd = torch.from_numpy(x2.astype(np.float32)).to(dev)
    qd = torch.empty((cache.batch, cache.n_heads(), f.head_dim), dtype=torch.float32, device=dev)
    N.call("wsvd_append_token", cache.h, C.c_void_p(xd.data_ptr()), C.c_void_p(qd.data_ptr()),
           _stream())
    if counter is not None:
        N.call("wsvd_traffic_append", cache.h, counter._ptr())
    q = qd.cpu().numpy().astype(np.float64)
    return q[0] if single else q


def fused_decode_step(cache: LatentCache, f: LayerFactors, q_heads, tiles: TileConfig,
                      counter: TrafficCounter):
    """decode.cpp:155-206.  q_heads: (n_heads, H) or (B, n_heads, H)."""
    torch = _torch()
    if cache.length() == 0:
        raise ShapeError("decode step over an empty cache")
    if len(f.heads) != cache.n_heads():
        raise ShapeError(f"cache holds {cache.n_heads()} heads, factors {len(f.heads)}")
    q = np.asarray(q_heads, dtype=np.float64)
    single = q.ndim == 2
    q3 = q.reshape(1, *q.shape) if single else q
    if q3.shape[1:] != (len(f.heads), f.head_dim):
        raise ShapeError(f"query block must be {len(f.heads)}x{f.head_dim}, got "
                         f"{q3.shape[1]}x{q3.shape[2]}")
    if q3.shape[0] != cache.batch:
        raise ShapeError(f"{q3.shape[0]} query blocks for a cache of {cache.batch} sequences")
    if tiles.tile_len == 0:
        raise ConfigError("tile length must be >= 1")
    cache._bind(f)
    dev = torch.device("cuda", cache.device)
    qd = torch.from_numpy(q3.astype(np.float32)).to(dev)
    od = torch.empty_like(qd)
    N.call("wsvd_fused_decode_step", cache.h, C.c_void_p(qd.data_ptr()), int(tiles.tile_len),
           C.c_void_p(od.data_ptr()), _stream())
    N.call("wsvd_traffic_fused", cache.h, int(tiles.tile_len), counter._ptr())
    out = od.cpu().numpy().astype(np.float64)
    return out[0] if single else out


# ----------------------------------------------------------------- report --
class Mode(enum.IntEnum):
    """decode.hpp:172"""
    Fused = 0
    Eager = 1
    FlashFull = 2
    SharedLatent = 3


_MODE_NAMES = ["fused", "eager", "flash_full", "shared_latent"]


def mode_name(m: Mode) -> str:
    return _MODE_NAMES[int(m)]


def mode_from_name(name: str) -> Mode:
    if name not in _MODE_NAMES:
        raise ConfigError(f"unknown decode mode '{name}'")
    return Mode(_MODE_NAMES.index(name))


@dataclass
class TrafficReport:
    """decode.hpp:179-190"""
    mode: Mode = Mode.Fused
    seq_len: int = 0
    n_heads: int = 0
    analytic_gamma: int = 0
    analytic_eta: int = 0
    measured_cache_loads_per_head: int = 0
    measured_reconstruction_flops_per_head: int = 0
    match: bool = False
    bytes_loaded_fp64: float = 0.0
    bytes_loaded_fp16: float = 0.0


def traffic_report(mode: Mode, counter: TrafficCounter, seq_len: int, n_heads: int,
                   head_dim: int, rank_k: int, shared_rank: int) -> TrafficReport:
    """decode.cpp:452-487: closed-form gamma/eta against the measured tallies."""
    if n_heads == 0:
        raise ConfigError("traffic report over zero heads")
    rep = TrafficReport(mode=mode, seq_len=seq_len, n_heads=n_heads)
    if mode == Mode.Fused:
        rep.analytic_eta = seq_len * rank_k
        rep.analytic_gamma = seq_len * rank_k * head_dim
    elif mode == Mode.SharedLatent:
        rep.analytic_eta = seq_len * shared_rank
        rep.analytic_gamma = seq_len * shared_rank * head_dim
    else:
        rep.analytic_eta = seq_len * head_dim
        rep.analytic_gamma = 0
    latent = mode in (Mode.Fused, Mode.SharedLatent)
    st = counter[Stream.LatentK if latent else Stream.FullK]
    divisible = st.loads % n_heads == 0 and st.flops % n_heads == 0
    rep.measured_cache_loads_per_head = st.loads // n_heads if divisible else 0
    rep.measured_reconstruction_flops_per_head = st.flops // n_heads if divisible else 0
    rep.match = (divisible and rep.measured_cache_loads_per_head == rep.analytic_eta
                 and rep.measured_reconstruction_flops_per_head == rep.analytic_gamma)
    rep.bytes_loaded_fp64 = 8.0 * counter.total_loads()
    rep.bytes_loaded_fp16 = 2.0 * counter.total_loads()
    return rep
