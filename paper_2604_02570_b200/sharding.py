"""Head sharding across GPUs.

GPU g of G owns heads [g*nh/G, (g+1)*nh/G): their A/B factors, their latent
cache and the W_o rows (nh/G * H) x E that multiply them.  The token x is
replicated.  Each rank's layer step produces the partial
y_g = concat_{h in g}(out_h) . W_o[rows_g]; one all-reduce (sum) over NVLink
completes y = sum_g y_g = concat_h(out_h) . W_o (pipeline.cpp:323-329).

The host logic here (ranges, slicing, the all-reduce call) is independent of
the device and is exercised with the gloo backend on CPU in tests/.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .decode import LayerFactors
from .errors import ConfigError


def head_range(n_heads: int, world: int, rank: int) -> tuple[int, int]:
    if world <= 0 or not 0 <= rank < world:
        raise ConfigError(f"rank {rank} outside world of {world}")
    if n_heads % world:
        raise ConfigError(f"{n_heads} heads do not shard evenly over {world} GPUs")
    per = n_heads // world
    return rank * per, (rank + 1) * per


def shard_factors(f: LayerFactors, world: int, rank: int) -> LayerFactors:
    h0, h1 = head_range(len(f.heads), world, rank)
    return LayerFactors(heads=f.heads[h0:h1], embed_dim=f.embed_dim, head_dim=f.head_dim)


def shard_oproj(w_o: np.ndarray, n_heads: int, head_dim: int, world: int, rank: int) -> np.ndarray:
    """Rows of W_o (n_heads*H x E_out) that multiply this rank's heads."""
    h0, h1 = head_range(n_heads, world, rank)
    return w_o[h0 * head_dim:h1 * head_dim]


def exchange_unique_id(rank: int, device: int = 0, group=None) -> np.ndarray:
    """Rank 0's NCCL unique id (from the native library) on every rank of an
    existing torch.distributed group (nccl: through device memory; gloo: host)."""
    import torch
    import torch.distributed as dist
    uid = np.zeros(128, dtype=np.uint8)
    if rank == 0:
        N.call("wsvd_nccl_unique_id", uid.ctypes.data_as(C.POINTER(C.c_uint8)))
    t = torch.from_numpy(uid.astype(np.int64))
    if dist.get_backend(group) == "nccl":
        t = t.cuda(device)
    dist.broadcast(t, src=0, group=group)
    return t.cpu().numpy().astype(np.uint8)


class NcclComm:
    """NCCL communicator owned by the native library (dlopen'd libnccl); the
    unique id travels over an existing torch.distributed group."""

    def __init__(self, world: int, rank: int, device: int, group=None):
        uid = exchange_unique_id(rank, device, group)
        h = C.c_void_p()
        N.call("wsvd_comm_create", uid.ctypes.data_as(C.POINTER(C.c_uint8)), world, rank, device,
               C.byref(h))
        self.h = h
        self.world, self.rank = world, rank

    def allreduce_(self, y, stream=None):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        N.call("wsvd_allreduce_sum_f32", self.h, C.c_void_p(y.data_ptr()), y.numel(),
               C.c_void_p(s.cuda_stream))

    def __del__(self):
        if getattr(self, "h", None) and N._lib is not None:
            N.lib().wsvd_comm_destroy(self.h)
            self.h = None
