"""GPU: the NCCL plumbing of the head-sharded layer on the one GPU a box
offers -- a world-size-1 communicator created through the C ABI (libnccl
dlopen'd at run time, id broadcast over torch.distributed), an all-reduce of
a layer-step output, and a sharded layer whose y equals the unsharded one."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import to_factors

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dist_world1():
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_nccl_comm_allreduce_world1(dist_world1):
    from paper_2604_02570_b200.sharding import NcclComm
    comm = NcclComm(1, 0, 0)
    y = torch.arange(4096, dtype=torch.float32, device="cuda")
    ref = y.clone()
    comm.allreduce_(y)
    torch.cuda.synchronize()
    assert torch.equal(y, ref)


def test_sharded_layer_sums_to_unsharded(dist_world1):
    """Two head shards on one device, their partial y summed by the same
    all-reduce path, equal the unsharded layer step."""
    from paper_2604_02570_b200.layer import DecodeLayer
    from paper_2604_02570_b200.sharding import NcclComm, shard_factors, shard_oproj
    rng = O.Rng(55)
    E, H, nh, r, B, L = 256, 128, 4, 32, 2, 60
    lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
    f = to_factors(lay)
    w_o = O.bf16_round(rng.normal_matrix(nh * H, E, 1.0 / np.sqrt(E)))
    dev = torch.device("cuda", 0)
    full = DecodeLayer(f, w_o, batch=B, capacity=L + 4, cache_dtype="bf16", weight_dtype="bf16")
    shards = [DecodeLayer(shard_factors(f, 2, g), shard_oproj(w_o, nh, H, 2, g), batch=B, capacity=L + 4,
                          cache_dtype="bf16", weight_dtype="bf16", head_offset=g * 2) for g in range(2)]
    toks = torch.from_numpy(O.bf16_round(rng.normal_matrix(L * B, E)).reshape(L, B, E).astype(np.float32)).to(dev)
    full.prefill(toks[:-1].contiguous())
    for s in shards:
        s.prefill(toks[:-1].contiguous())
    y_full = torch.empty((B, E), device=dev)
    full.step(toks[-1].contiguous(), y_full, graph=False)
    ys = [torch.empty((B, E), device=dev) for _ in shards]
    for s, y in zip(shards, ys):
        s.step(toks[-1].contiguous(), y, graph=False)
    comm = NcclComm(1, 0, 0)
    y_sum = ys[0] + ys[1]
    comm.allreduce_(y_sum)
    torch.cuda.synchronize()
    a, b = y_sum.cpu().numpy(), y_full.cpu().numpy()
    assert np.abs(a - b).max() <= 1e-4 * np.abs(b).max()
