"""ctypes bindings for the CPU oracle (liboracle.so) and the reference harness
(_ref/libwsvdref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py -- never by the product
package.  Layout conventions are documented in wsvd_oracle.h: factors are
padded A[nh][3][E][rmax], B[nh][3][rmax][H] with true ranks[nh][3]; one
sequence's cache is ck/cv[nh][cap][rmax].
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libwsvdref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_u64p = C.POINTER(C.c_uint64)
_i8p = C.POINTER(C.c_int8)
_fp = C.POINTER(C.c_float)
_sz = C.c_size_t

NSTREAMS = 7
STREAMS = ["latent_k", "latent_v", "full_k", "full_v", "weights_b", "query", "output"]


class OrcRng(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("mti", C.c_int), ("has_spare", C.c_int),
                ("spare", C.c_double)]


class OrcCounter(C.Structure):
    _fields_ = [("loads", C.c_uint64 * NSTREAMS), ("stores", C.c_uint64 * NSTREAMS),
                ("flops", C.c_uint64 * NSTREAMS)]

    def as_dict(self):
        return {s: (self.loads[i], self.stores[i], self.flops[i]) for i, s in enumerate(STREAMS)}


class OrcLayer(C.Structure):
    _fields_ = [("E", _sz), ("H", _sz), ("nh", _sz), ("rmax", _sz), ("ranks", _ip),
                ("A", _dp), ("B", _dp)]


def _ptr(a, t):
    return a.ctypes.data_as(t)


def build():
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")], check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.orc_rng_u64.restype = C.c_uint64
        L.orc_rng_normal.restype = C.c_double
        L.orc_rng_uniform.restype = C.c_double
        L.orc_rng_index.restype = C.c_uint64
        L.orc_rng_index.argtypes = [C.POINTER(OrcRng), C.c_uint64]
        L.orc_rng_seed.argtypes = [C.POINTER(OrcRng), C.c_uint64]
        L.orc_rng_stream.argtypes = [C.POINTER(OrcRng), C.c_uint64, C.c_uint64]
        L.orc_rng_normal_fill.argtypes = [C.POINTER(OrcRng), _dp, _sz, C.c_double]
        L.orc_append_token.argtypes = [C.POINTER(OrcLayer), _dp, _dp, _sz, _sz, _dp, _dp,
                                       C.POINTER(OrcCounter)]
        L.orc_fused_decode_step.argtypes = [C.POINTER(OrcLayer), _dp, _dp, _sz, _sz, _dp, _sz,
                                            _dp, C.POINTER(OrcCounter)]
        L.orc_reconstruct_then_attend.argtypes = [C.POINTER(OrcLayer), _dp, _dp, _sz, _sz, _dp,
                                                  _dp]
        L.orc_traffic_match_fused.argtypes = [C.POINTER(OrcCounter), C.c_uint64, C.c_uint64,
                                              C.c_uint64, C.c_uint64]
        L.orc_batched_append.argtypes = [C.POINTER(OrcLayer), _dp, _dp, _sz, _sz, _sz, _dp, _dp,
                                         C.c_int]
        L.orc_batched_decode.argtypes = [C.POINTER(OrcLayer), _dp, _dp, _sz, _sz, _sz, _dp, _sz,
                                         _dp, C.c_int]
        L.orc_batched_decode_latent.argtypes = [C.POINTER(OrcLayer), _dp, _dp, _sz, _sz, _sz, _dp,
                                                _sz, _dp, _dp, C.c_int]
        L.orc_bf16_bits.restype = C.c_uint16
        L.orc_bf16_bits.argtypes = [C.c_float]
        L.orc_f16_bits.restype = C.c_uint16
        L.orc_f16_bits.argtypes = [C.c_float]
        L.orc_f16_to_f32.restype = C.c_float
        L.orc_f16_to_f32.argtypes = [C.c_uint16]
        L.orc_quantize_weight.restype = C.c_double
        L.orc_quantize_weight.argtypes = [_dp, _sz, _sz, C.c_int, _i8p, _dp]
        L.orc_quantize_activation_f64.argtypes = [_dp, _sz, _sz, C.c_int, _i8p, _dp]
        L.orc_rotate_token_f32.argtypes = [_fp, _fp, _sz]
        L.orc_rot_block.restype = _sz
        L.orc_rot_block.argtypes = [_sz]
        L.orc_quant_token_f32.restype = C.c_float
        L.orc_quant_token_f32.argtypes = [_fp, _sz, _i8p]
        L.orc_int_gemv.argtypes = [_i8p, _i8p, _sz, _sz, _ip]
        L.orc_dequant_latent.restype = C.c_float
        L.orc_dequant_latent.argtypes = [C.c_int32, C.c_float, C.c_float]
        L.orc_quant_cache_row.restype = C.c_uint16
        L.orc_quant_cache_row.argtypes = [_fp, _sz, _i8p]
        L.orc_unpack_int4.argtypes = [C.POINTER(C.c_uint8), _sz, _i8p]
        L.orc_i8_scores.argtypes = [_fp, _sz, _i8p, _sz, _sz, _ip]
        _lib = L
    return _lib


def ref_available():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(REF_SO)
        R = C.CDLL(REF_SO)
        R.ref_last_error.restype = C.c_char_p
        R.ref_append_then_decode.argtypes = [_sz, _sz, _sz, _sz, _ip, _dp, _dp, _sz, _dp, _sz,
                                             _dp, _dp, _dp, _dp, _u64p, _u64p]
        R.ref_fused_decode.argtypes = [_sz, _sz, _sz, _sz, _ip, _dp, _dp, _sz, _dp, _dp, _dp,
                                       _sz, _dp, _u64p]
        R.ref_traffic_match_fused.argtypes = [_u64p, C.c_uint64, C.c_uint64, C.c_uint64,
                                              C.c_uint64]
        R.ref_rng_normals.argtypes = [C.c_uint64, C.c_uint64, C.c_int, _sz, C.c_double, _dp]
        R.ref_rng_u64s.argtypes = [C.c_uint64, _sz, _u64p]
        R.ref_rng_indices.argtypes = [C.c_uint64, C.c_uint64, _sz, _u64p]
        R.ref_quantize_weight.restype = C.c_double
        R.ref_quantize_weight.argtypes = [_dp, _sz, _sz, C.c_int, _i8p, _dp]
        R.ref_quantize_activation.argtypes = [_dp, _sz, _sz, C.c_int, _i8p, _dp]
        R.ref_hadamard.argtypes = [_sz, _dp]
        R.ref_baseline_create.restype = C.c_void_p
        R.ref_baseline_create.argtypes = [_sz, _sz, _sz, _sz, _sz, _sz, _sz, C.c_uint64, C.c_int]
        R.ref_baseline_step.restype = C.c_double
        R.ref_baseline_step.argtypes = [C.c_void_p, C.c_int]
        R.ref_baseline_destroy.argtypes = [C.c_void_p]
        _ref = R
    return _ref


# ----------------------------------------------------------------- rng ----

class Rng:
    """wsvd::Rng restated (rng.cpp) -- deterministic synthetic inputs."""

    def __init__(self, seed: int = 0, stream: int | None = None):
        self._s = OrcRng()
        if stream is None:
            lib().orc_rng_seed(C.byref(self._s), seed)
        else:
            lib().orc_rng_stream(C.byref(self._s), seed, stream)

    @classmethod
    def stream(cls, seed: int, stream_id: int) -> "Rng":
        return cls(seed, stream_id)

    def next_u64(self) -> int:
        return lib().orc_rng_u64(C.byref(self._s))

    def normal(self) -> float:
        return lib().orc_rng_normal(C.byref(self._s))

    def index(self, n: int) -> int:
        return lib().orc_rng_index(C.byref(self._s), n)

    def normal_matrix(self, rows: int, cols: int, stddev: float = 1.0) -> np.ndarray:
        out = np.empty((rows, cols), dtype=np.float64)
        lib().orc_rng_normal_fill(C.byref(self._s), _ptr(out, _dp), out.size, stddev)
        return out


# --------------------------------------------------------------- layer ----

@dataclass
class Layer:
    """Padded factors of one layer: A[nh,3,E,rmax], B[nh,3,rmax,H], ranks[nh,3]."""
    A: np.ndarray
    B: np.ndarray
    ranks: np.ndarray

    @property
    def nh(self):
        return self.A.shape[0]

    @property
    def E(self):
        return self.A.shape[2]

    @property
    def rmax(self):
        return self.A.shape[3]

    @property
    def H(self):
        return self.B.shape[3]

    def c(self) -> OrcLayer:
        self.A = np.ascontiguousarray(self.A, dtype=np.float64)
        self.B = np.ascontiguousarray(self.B, dtype=np.float64)
        self.ranks = np.ascontiguousarray(self.ranks, dtype=np.int32)
        return OrcLayer(self.E, self.H, self.nh, self.rmax, _ptr(self.ranks, _ip),
                        _ptr(self.A, _dp), _ptr(self.B, _dp))

    def map(self, fn) -> "Layer":
        """Apply a storage-format rounding to every factor value."""
        return Layer(fn(self.A), fn(self.B), self.ranks.copy())


def random_layer(rng: Rng, E: int, H: int, ranks, rmax: int | None = None) -> Layer:
    """tests/test_decode.cpp:25-46 random_layer draw order (per head: q, k, v;
    per role: a then b), padded to rmax."""
    ranks = np.asarray(ranks, dtype=np.int32).reshape(-1, 3)
    nh = ranks.shape[0]
    rmax = int(rmax or ranks.max())
    A = np.zeros((nh, 3, E, rmax))
    B = np.zeros((nh, 3, rmax, H))
    for h in range(nh):
        for role in range(3):
            r = int(ranks[h, role])
            A[h, role, :, :r] = rng.normal_matrix(E, r, 1.0 / np.sqrt(E))
            B[h, role, :r, :] = rng.normal_matrix(r, H, 1.0 / np.sqrt(r))
    return Layer(A, B, ranks)


def bench_layer(E: int, H: int, nh: int, r: int, seed: int = 0) -> Layer:
    """tools/wsvd_main.cpp:360-391 decode-bench draw order: Rng::stream(seed, 5),
    per head q.a q.b k.a k.b v.a v.b, A ~ N(0,1/E), B ~ N(0,1/r)."""
    rng = Rng.stream(seed, 5)
    A = np.zeros((nh, 3, E, r))
    B = np.zeros((nh, 3, r, H))
    for h in range(nh):
        for role in range(3):
            A[h, role] = rng.normal_matrix(E, r, 1.0 / np.sqrt(E))
            B[h, role] = rng.normal_matrix(r, H, 1.0 / np.sqrt(r))
    return Layer(A, B, np.full((nh, 3), r, dtype=np.int32))


# -------------------------------------------------------------- decode ----

def append_token(layer: Layer, ck, cv, pos: int, x, counter: OrcCounter | None = None):
    """decode::append_token for one sequence; ck/cv [nh,cap,rmax] updated in place."""
    q = np.zeros((layer.nh, layer.H))
    x = np.ascontiguousarray(x, dtype=np.float64)
    rc = lib().orc_append_token(C.byref(layer.c()), _ptr(ck, _dp), _ptr(cv, _dp), ck.shape[1],
                                pos, _ptr(x, _dp), _ptr(q, _dp),
                                C.byref(counter) if counter is not None else None)
    assert rc == 0
    return q


def fused_decode_step(layer: Layer, ck, cv, length: int, q, tile: int = 32,
                      counter: OrcCounter | None = None):
    out = np.zeros((layer.nh, layer.H))
    q = np.ascontiguousarray(q, dtype=np.float64)
    rc = lib().orc_fused_decode_step(C.byref(layer.c()), _ptr(ck, _dp), _ptr(cv, _dp),
                                     ck.shape[1], length, _ptr(q, _dp), tile, _ptr(out, _dp),
                                     C.byref(counter) if counter is not None else None)
    if rc == -1:
        raise ValueError("ShapeError: decode step over an empty cache")
    if rc == -2:
        raise ValueError("ConfigError: tile length must be >= 1")
    return out


def reconstruct_then_attend(layer: Layer, ck, cv, length: int, q):
    out = np.zeros((layer.nh, layer.H))
    q = np.ascontiguousarray(q, dtype=np.float64)
    lib().orc_reconstruct_then_attend(C.byref(layer.c()), _ptr(ck, _dp), _ptr(cv, _dp),
                                      ck.shape[1], length, _ptr(q, _dp), _ptr(out, _dp))
    return out


def batched_decode(layer: Layer, ck, cv, length: int, q, tile: int = 32, threads: int = 1):
    """ck/cv [B,nh,cap,rmax], q [B,nh,H] -> out [B,nh,H] (fp64 reference algorithm)."""
    Bn = ck.shape[0]
    out = np.zeros((Bn, layer.nh, layer.H))
    q = np.ascontiguousarray(q, dtype=np.float64)
    ck = np.ascontiguousarray(ck, dtype=np.float64)
    cv = np.ascontiguousarray(cv, dtype=np.float64)
    rc = lib().orc_batched_decode(C.byref(layer.c()), _ptr(ck, _dp), _ptr(cv, _dp), Bn,
                                  ck.shape[2], length, _ptr(q, _dp), tile, _ptr(out, _dp), threads)
    assert rc == 0
    return out


def batched_decode_latent(layer: Layer, ck, cv, length: int, q, tile: int = 32, threads: int = 1):
    """As batched_decode, also returning the latent outputs v~ = acc/denom
    (decode.cpp:198) [B,nh,rmax] -- what the folded O-projection multiplies."""
    Bn = ck.shape[0]
    out = np.zeros((Bn, layer.nh, layer.H))
    lat = np.zeros((Bn, layer.nh, layer.rmax))
    q = np.ascontiguousarray(q, dtype=np.float64)
    ck = np.ascontiguousarray(ck, dtype=np.float64)
    cv = np.ascontiguousarray(cv, dtype=np.float64)
    rc = lib().orc_batched_decode_latent(C.byref(layer.c()), _ptr(ck, _dp), _ptr(cv, _dp), Bn,
                                         ck.shape[2], length, _ptr(q, _dp), tile, _ptr(out, _dp),
                                         _ptr(lat, _dp), threads)
    assert rc == 0
    return out, lat


def fold_oproj(layer: Layer, w_o, rpad: int, storage=None):
    """W'_o = blockdiag_h(B_V,h) . W_o  ((nh*rpad) x e_out) from the factor
    values the device stores, as wsvd_layer_set_oproj folds it (fp64 sums),
    then the device's storage rounding (bf16_round for a bf16 O-projection).
    heads_row . W_o (pipeline.cpp:323-329) = v~ . W'_o exactly in real
    arithmetic: the fold only moves where the bf16 weight rounding happens."""
    nh, H = layer.nh, layer.H
    w_o = np.asarray(w_o, dtype=np.float64)
    fold = np.zeros((nh * rpad, w_o.shape[1]))
    for h in range(nh):
        rv = int(layer.ranks[h, 2])
        fold[h * rpad:h * rpad + rv] = layer.B[h, 2, :rv, :] @ w_o[h * H:(h + 1) * H]
    return storage(fold) if storage is not None else fold


def decode_factored(layers, w_os, ffn, xs, tile: int = 32, device_storage: bool = False, rpad: int | None = None,
                    device_rows=None):
    """pipe::decode_factored (reference src/pipeline.cpp:304-339) for one
    sequence: xs [T][E] tokens through len(layers) layers from empty caches.
    Per token and layer: append_token (:320), fused_decode_step (:321-322),
    heads_row . W_o (:323-329), cur = tanh(o . ff1) . ff2 (:330-334); the
    output row of token t is the last layer's cur (:336).  layers: Layer
    factors, w_os: W_o [nh*H][E] per layer, ffn: (ff1 [E][F], ff2 [F][E]) per
    layer.  Returns [T][E].

    device_storage=True keeps the arithmetic in fp64 but rounds the operands
    the device stores to bf16 where it stores them: the tokens entering each
    layer, the appended cache rows, the folded O-projection W'_o = B_V . W_o
    (heads_row . W_o = v~ . W'_o, fold_oproj) and the FFN GEMM inputs o and
    tanh(o . ff1).  The factors and FFN weights are taken as given (pass the
    bf16 values the device was given).  device_rows: per layer (K rows, V
    rows) [nh][T][>= rmax] read back from the device -- the appended rows the
    attention then runs over (a single bf16 rounding flip of a cache row is a
    2^-8 perturbation the softmax over a short context carries straight to
    the output; the layer tests compare on the device's rows the same way)."""
    xs = np.asarray(xs, dtype=np.float64)
    T, E = xs.shape
    caches = [(np.zeros((lay.nh, T, lay.rmax)), np.zeros((lay.nh, T, lay.rmax))) for lay in layers]
    folds = None
    if device_storage:
        rpad = rpad or max(lay.rmax for lay in layers)
        folds = [fold_oproj(lay, w, rpad, bf16_round) for lay, w in zip(layers, w_os)]
    out = np.zeros((T, E))
    for t in range(T):
        cur = xs[t]
        for li, lay in enumerate(layers):
            ck, cv = caches[li]
            q = append_token(lay, ck, cv, t, bf16_round(cur) if device_storage else cur)
            if device_storage:
                ck[:, t] = bf16_round(ck[:, t])
                cv[:, t] = bf16_round(cv[:, t])
            if device_rows is not None:
                ck[:, t] = device_rows[li][0][:, t, :lay.rmax]
                cv[:, t] = device_rows[li][1][:, t, :lay.rmax]
                _, lat = batched_decode_latent(lay, ck[None], cv[None], t + 1, q[None], tile, 1)
                lat_p = np.zeros((lay.nh, rpad))
                lat_p[:, :lay.rmax] = lat[0]
                o = lat_p.reshape(-1) @ folds[li]
            else:
                attn = fused_decode_step(lay, ck, cv, t + 1, q, tile)
                o = attn.reshape(-1) @ np.asarray(w_os[li], dtype=np.float64)
            ff1, ff2 = (np.asarray(w, dtype=np.float64) for w in ffn[li])
            h = np.tanh((bf16_round(o) if device_storage else o) @ ff1)
            cur = (bf16_round(h) if device_storage else h) @ ff2
        out[t] = cur
    return out


def batched_append(layer: Layer, ck, cv, pos: int, x, threads: int = 1):
    Bn = ck.shape[0]
    q = np.zeros((Bn, layer.nh, layer.H))
    x = np.ascontiguousarray(x, dtype=np.float64)
    rc = lib().orc_batched_append(C.byref(layer.c()), _ptr(ck, _dp), _ptr(cv, _dp), Bn,
                                  ck.shape[2], pos, _ptr(x, _dp), _ptr(q, _dp), threads)
    assert rc == 0
    return q


def traffic_match_fused(counter: OrcCounter, seq_len, n_heads, head_dim, rank_k) -> bool:
    return lib().orc_traffic_match_fused(C.byref(counter), seq_len, n_heads, head_dim,
                                         rank_k) == 1


# ----------------------------------------------------- storage formats ----

def bf16_round(a):
    """double -> f32 (RNE) -> bf16 (RNE), returned as float64 values."""
    f = np.asarray(a, dtype=np.float64).astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return (u.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def f32_round(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def quantize_weight(w, bits: int):
    w = np.ascontiguousarray(w, dtype=np.float64)
    q = np.zeros(w.shape, dtype=np.int8)
    s = np.zeros(w.shape[1])
    clip = lib().orc_quantize_weight(_ptr(w, _dp), w.shape[0], w.shape[1], bits, _ptr(q, _i8p),
                                     _ptr(s, _dp))
    return q, s, clip


def quantize_activation_f64(x, bits: int):
    x = np.ascontiguousarray(x, dtype=np.float64)
    q = np.zeros(x.shape, dtype=np.int8)
    s = np.zeros(x.shape[0])
    lib().orc_quantize_activation_f64(_ptr(x, _dp), x.shape[0], x.shape[1], bits, _ptr(q, _i8p),
                                      _ptr(s, _dp))
    return q, s


def rotate_token(x32):
    x32 = np.ascontiguousarray(x32, dtype=np.float32)
    out = np.empty_like(x32)
    lib().orc_rotate_token_f32(_ptr(x32, _fp), _ptr(out, _fp), x32.size)
    return out


def quant_token(v32):
    v32 = np.ascontiguousarray(v32, dtype=np.float32)
    q = np.zeros(v32.shape, dtype=np.int8)
    s = lib().orc_quant_token_f32(_ptr(v32, _fp), v32.size, _ptr(q, _i8p))
    return q, np.float32(s)


def int_gemv(xq, wq):
    xq = np.ascontiguousarray(xq, dtype=np.int8)
    wq = np.ascontiguousarray(wq, dtype=np.int8)
    acc = np.zeros(wq.shape[0], dtype=np.int32)
    lib().orc_int_gemv(_ptr(xq, _i8p), _ptr(wq, _i8p), xq.size, wq.shape[0], _ptr(acc, _ip))
    return acc


def dequant_latent(acc, sx, sw):
    return np.float32(lib().orc_dequant_latent(int(acc), float(sx), float(sw)))


def quant_cache_row(c32):
    c32 = np.ascontiguousarray(c32, dtype=np.float32)
    q = np.zeros(c32.shape, dtype=np.int8)
    h = lib().orc_quant_cache_row(_ptr(c32, _fp), c32.size, _ptr(q, _i8p))
    return q, np.uint16(h)


def f16_to_f32(h):
    return np.float32(lib().orc_f16_to_f32(int(h)))


def i8_scores(qt32, rows_i8, R):
    """int32 score accumulators (hi, lo) of every int8 cache row against the
    split absorbed query (orc_i8_scores; attn.cu's int8 consumers).
    qt32 [R] fp32, rows_i8 [L][ld] int8 -> [L][2] int32."""
    q = np.ascontiguousarray(qt32, dtype=np.float32)
    rows = np.ascontiguousarray(rows_i8, dtype=np.int8)
    acc = np.zeros((rows.shape[0], 2), dtype=np.int32)
    lib().orc_i8_scores(_ptr(q, _fp), R, _ptr(rows, _i8p), rows.shape[0], rows.shape[1], _ptr(acc, _ip))
    return acc
