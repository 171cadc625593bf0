"""CPU: host-side logic of the Python mirror (decode.py) and of head
sharding (sharding.py), including a world-size-2 gloo run of the sharded
O-projection all-reduce checked against the unsharded oracle."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2604_02570_b200 import decode as D
from paper_2604_02570_b200 import sharding as S
from paper_2604_02570_b200.errors import ConfigError, ShapeError
from tests.helpers import to_factors


def test_mode_and_stream_names_round_trip():
    # test_decode.cpp:657-668
    for m in D.Mode:
        assert D.mode_from_name(D.mode_name(m)) == m
    with pytest.raises(ConfigError):
        D.mode_from_name("turbo")
    assert D.stream_name(D.Stream.LatentK) == "latent_k"
    assert D.stream_name(D.Stream.FullV) == "full_v"
    assert D.stream_name(D.Stream.WeightsB) == "weights_b"
    assert D.stream_name(D.Stream.Query) == "query"
    assert D.stream_name(D.Stream.Output) == "output"


def test_traffic_counter_and_report_host_logic():
    # decode.cpp:452-487 closed forms against oracle counters
    rng = O.Rng(370)
    L, nh, hd, r = 19, 4, 8, 3
    lay = O.random_layer(rng, 32, hd, [[r, r, r]] * nh)
    ck = np.zeros((nh, L, r))
    cv = np.zeros_like(ck)
    q = None
    for t in range(L):
        q = O.append_token(lay, ck, cv, t, rng.normal_matrix(1, 32)[0])
    oc = O.OrcCounter()
    O.fused_decode_step(lay, ck, cv, L, q, 4, oc)
    c = D.TrafficCounter()
    for s in range(7):
        c.add_loads(D.Stream(s), oc.loads[s])
        c.add_stores(D.Stream(s), oc.stores[s])
        c.add_flops(D.Stream(s), oc.flops[s])
    rep = D.traffic_report(D.Mode.Fused, c, L, nh, hd, r, 0)
    assert rep.match
    assert rep.analytic_eta == L * r and rep.analytic_gamma == L * r * hd
    assert rep.measured_cache_loads_per_head == L * r
    assert rep.bytes_loaded_fp64 == 8.0 * c.total_loads()
    assert not D.traffic_report(D.Mode.Fused, c, L + 1, nh, hd, r, 0).match
    with pytest.raises(ConfigError):
        D.traffic_report(D.Mode.Fused, c, L, 0, hd, r, 0)
    flash = D.traffic_report(D.Mode.FlashFull, D.TrafficCounter(), L, nh, hd, 0, 0)
    assert flash.analytic_eta == L * hd and flash.analytic_gamma == 0


def test_head_ranges_and_slicing():
    assert S.head_range(32, 8, 3) == (12, 16)
    assert [S.head_range(40, 4, r) for r in range(4)] == [(0, 10), (10, 20), (20, 30), (30, 40)]
    with pytest.raises(ConfigError):
        S.head_range(40, 3, 0)
    with pytest.raises(ConfigError):
        S.head_range(32, 2, 2)
    f = to_factors(O.random_layer(O.Rng(3), 16, 4, [[2, 2, 2]] * 4))
    sh = S.shard_factors(f, 2, 1)
    assert len(sh.heads) == 2 and sh.heads[0] is f.heads[2]
    w_o = np.arange(16 * 5, dtype=np.float64).reshape(16, 5)
    assert (S.shard_oproj(w_o, 4, 4, 2, 1) == w_o[8:16]).all()


def _sharded_worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # identical synthetic layer on every rank (decode-bench recipe)
    E, H, nh, r, L = 32, 8, 4, 4, 11
    lay = O.bench_layer(E, H, nh, r, seed=3)
    w_o = O.Rng.stream(3, 77).normal_matrix(nh * H, E, 1.0 / np.sqrt(E))
    toks = O.Rng.stream(3, 1000).normal_matrix(L, E)
    h0, h1 = S.head_range(nh, world, rank)
    # this rank's heads only: its own latent caches, attention and O-proj rows
    shard = O.Layer(lay.A[h0:h1], lay.B[h0:h1], lay.ranks[h0:h1])
    ck = np.zeros((h1 - h0, L, r))
    cv = np.zeros_like(ck)
    q = None
    for t in range(L):
        q = O.append_token(shard, ck, cv, t, toks[t])
    out = O.fused_decode_step(shard, ck, cv, L, q, 4)
    y = torch.from_numpy(out.reshape(-1) @ S.shard_oproj(w_o, nh, H, world, rank))
    dist.all_reduce(y)  # the one collective of the layer
    if rank == 0:
        np.save(result_path, y.numpy())
    dist.destroy_process_group()


def test_head_sharded_oproj_allreduce_gloo(tmp_path):
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    path = str(tmp_path / "y.npy")
    mp.spawn(_sharded_worker, args=(2, port, path), nprocs=2, join=True)
    y = np.load(path)
    # unsharded reference on one process
    E, H, nh, r, L = 32, 8, 4, 4, 11
    lay = O.bench_layer(E, H, nh, r, seed=3)
    w_o = O.Rng.stream(3, 77).normal_matrix(nh * H, E, 1.0 / np.sqrt(E))
    toks = O.Rng.stream(3, 1000).normal_matrix(L, E)
    ck = np.zeros((nh, L, r))
    cv = np.zeros_like(ck)
    for t in range(L):
        q = O.append_token(lay, ck, cv, t, toks[t])
    y_ref = O.fused_decode_step(lay, ck, cv, L, q, 4).reshape(-1) @ w_o
    assert np.abs(y - y_ref).max() <= 1e-12 * np.abs(y_ref).max() * 10


def test_mirror_validates_before_touching_the_device():
    with pytest.raises(ShapeError):
        D.DeviceLayer(D.LayerFactors())
    with pytest.raises(ConfigError):
        D.DeviceLayer(to_factors(O.random_layer(O.Rng(1), 16, 4, [[2, 2, 2]])), weight_dtype="fp8")


def _uid_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = S.exchange_unique_id(rank)
    np.save(os.path.join(out_dir, f"uid{rank}.npy"), uid)
    dist.destroy_process_group()


def test_nccl_unique_id_exchange_gloo(tmp_path):
    """NcclComm's bootstrap on CPU: rank 0's NCCL unique id (the native
    library's wsvd_nccl_unique_id) reaches every rank of a world-size-2 gloo
    group unchanged; the communicator itself (wsvd_comm_create) needs GPUs
    (tests/test_gpu_nccl.py)"""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_uid_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    u0, u1 = np.load(tmp_path / "uid0.npy"), np.load(tmp_path / "uid1.npy")
    assert u0.shape == (128,) and u0.any() and np.array_equal(u0, u1)
