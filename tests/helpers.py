"""Shared test helpers: convert between the oracle's padded layer layout and
the reference-API LayerFactors, and the parity metric."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O
from paper_2604_02570_b200.decode import HeadFactors, HeadProjection, LayerFactors, Role

# north_star: floating-point attention outputs within max relative error 1e-3
# (fp32 accumulate), measured per (sequence, head) row as max|gpu - ref| / max|ref|
# (SURVEY.md section 7 "Tolerance definition").
REL_TOL = 1e-3


def to_factors(lay: O.Layer) -> LayerFactors:
    heads = []
    for h in range(lay.nh):
        hf = []
        for role in range(3):
            r = int(lay.ranks[h, role])
            hf.append(HeadFactors(a=lay.A[h, role, :, :r].copy(), b=lay.B[h, role, :r, :].copy(),
                                  rank=r, head=h, role=Role(role)))
        heads.append(HeadProjection(*hf))
    return LayerFactors(heads=heads, embed_dim=lay.E, head_dim=lay.H)


def rel_err_rows(gpu: np.ndarray, ref: np.ndarray) -> float:
    """max over rows (last axis = H) of max|gpu-ref| / max|ref|."""
    g = gpu.reshape(-1, gpu.shape[-1])
    r = ref.reshape(-1, ref.shape[-1])
    num = np.abs(g - r).max(axis=1)
    den = np.maximum(np.abs(r).max(axis=1), 1e-30)
    return float((num / den).max())


def pad_latents(lat: np.ndarray, rmax: int) -> np.ndarray:
    out = np.zeros((lat.shape[0], rmax))
    out[:, : lat.shape[1]] = lat
    return out


def oracle_step_y(lb: O.Layer, ck, cv, length: int, q, w_o, rpad: int, tile: int = 32):
    """The oracle's O-projection output of one sequence's layer step:
    fused_decode_step (decode.cpp:155-206) over ck/cv [nh,L,rmax] with q
    [nh,H], keeping the latent output v~ (decode.cpp:198), times the folded
    W'_o = blockdiag(B_V) . W_o rounded to the device's bf16 storage
    (oracle.fold_oproj) -- heads_row . W_o of pipeline.cpp:323-329 with the
    weight rounding moved onto the stored product.  Returns y [e_out]."""
    ck = np.ascontiguousarray(ck, dtype=np.float64)[None]
    cv = np.ascontiguousarray(cv, dtype=np.float64)[None]
    _, lat = O.batched_decode_latent(lb, ck, cv, length, np.asarray(q)[None], tile, 1)
    lat_p = np.zeros((lb.nh, rpad))
    lat_p[:, :lb.rmax] = lat[0]
    return lat_p.reshape(-1) @ O.fold_oproj(lb, w_o, rpad, O.bf16_round)
