"""B200-native (sm_100a) WSVD per-head low-rank decode path.

Drop-in for the reference operator API wsvd::decode (see decode.py and the
C++ headers in include/wsvd/), built on the C ABI in include/wsvd_b200.h.
"""
from .decode import (HeadFactors, HeadProjection, LatentCache, LayerFactors, Mode, Role, Stream,
                     StreamTally, TileConfig, TrafficCounter, TrafficReport, append_token,
                     fused_decode_step, invalidate, mode_from_name, mode_name, stream_name,
                     traffic_report)
from .errors import ConfigError, CudaError, IoError, NumericError, ShapeError, WsvdError

__all__ = [
    "HeadFactors", "HeadProjection", "LatentCache", "LayerFactors", "Mode", "Role", "Stream",
    "StreamTally", "TileConfig", "TrafficCounter", "TrafficReport", "append_token",
    "fused_decode_step", "invalidate", "mode_from_name", "mode_name", "stream_name",
    "traffic_report", "ConfigError", "CudaError", "IoError", "NumericError", "ShapeError",
    "WsvdError",
]
