"""KV-head sharding: partition rules, a world-size-2 gloo
run of the shard -> compute -> all-gather path on CPU (the per-rank compute is
the oracle, standing in for the GPU kernel), and on the GPU the property that
sharded decoding is bit-identical to unsharded decoding."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import loki_oracle as O
from paper_2406_02542_b200 import sharding
from paper_2406_02542_b200.errors import ShapeError


def test_head_shard_partition():
    for Hq, Hkv, world in [(32, 32, 2), (32, 8, 4), (64, 8, 8), (32, 8, 8), (8, 8, 1)]:
        seen_kv, seen_q = [], []
        for r in range(world):
            s = sharding.head_shard(Hq, Hkv, world, r)
            assert s.kv_heads == Hkv // world and s.q_heads == Hq // world
            seen_kv += list(range(s.kv0, s.kv1))
            seen_q += list(range(s.q0, s.q1))
            G = Hq // Hkv
            assert all(h // G in range(s.kv0, s.kv1) for h in range(s.q0, s.q1))  # query heads follow their KV head
        assert seen_kv == list(range(Hkv)) and seen_q == list(range(Hq))
    with pytest.raises(ShapeError):
        sharding.head_shard(32, 8, 3, 0)
    with pytest.raises(ShapeError):
        sharding.head_shard(30, 8, 2, 0)
    with pytest.raises(ShapeError):
        sharding.head_shard(32, 8, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(seed=3):
    B, Hq, Hkv, D, S = 2, 8, 4, 32, 96
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((B, Hq, D)).astype(np.float32)
    K = rng.standard_normal((B, Hkv, S, D)).astype(np.float32)
    V = rng.standard_normal((B, Hkv, S, D)).astype(np.float32)
    return q, K, V, 8, 24  # d, k


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q, K, V, d, k = _case()
    B, Hq, D = q.shape
    sh = sharding.head_shard(Hq, K.shape[1], world, rank)
    qs = sharding.shard_heads(torch.from_numpy(q), sh, kv=False).numpy()
    Ks = sharding.shard_heads(torch.from_numpy(K), sh, kv=True).numpy()
    Vs = sharding.shard_heads(torch.from_numpy(V), sh, kv=True).numpy()
    y_local, _ = O.loki_decode_batched(qs, Ks, Vs, [K.shape[2]] * B, d, k=k)
    full = sharding.gather_heads(torch.from_numpy(np.ascontiguousarray(y_local)), world)
    if rank == 0:
        np.save(result_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_shard_and_gather_equals_unsharded(tmp_path):
    out = str(tmp_path / "y.npy")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    q, K, V, d, k = _case()
    y_ref, _ = O.loki_decode_batched(q, K, V, [K.shape[2]] * q.shape[0], d, k=k)
    np.testing.assert_array_equal(np.load(out), y_ref)


@pytest.mark.gpu
@pytest.mark.parametrize("halves", ["0", "2", None, "1"])
@pytest.mark.parametrize("B,Hq,Hkv", [(4, 16, 8), (8, 8, 8)])
def test_sharded_decode_bit_identical_on_gpu(monkeypatch, halves, B, Hq, Hkv):
    """Units are independent: decoding each KV-head shard separately gives the
    same bits as one unsharded launch (what an N-GPU run computes per rank).
    Opt-in tail halves (LOKI_PIPE_HALVES=1) split the parts of a set of tail
    units, which depends on the number of units: shards then agree to rounding."""
    import paper_2406_02542_b200 as L

    if halves is not None:
        monkeypatch.setenv("LOKI_TUNING", "1")
        monkeypatch.setenv("LOKI_PIPE_HALVES", halves)
    dev = torch.device("cuda", 0)
    D, S = 128, 4096
    g = torch.Generator(device=dev).manual_seed(11)
    K = torch.randn(B, Hkv, S, D, device=dev, generator=g).to(torch.bfloat16)
    V = torch.randn(B, Hkv, S, D, device=dev, generator=g).to(torch.bfloat16)
    q = torch.randn(B, Hq, D, device=dev, generator=g)
    cfg = L.LokiConfig(k_f=0.25, d_f=0.25)
    y_full = L.loki_decode(q, K, V, None, cfg=cfg)
    for world in (2, 4):
        parts = []
        for r in range(world):
            sh = sharding.head_shard(Hq, Hkv, world, r)
            parts.append(L.loki_decode(sharding.shard_heads(q, sh, kv=False).contiguous(),
                                       sharding.shard_heads(K, sh, kv=True), sharding.shard_heads(V, sh, kv=True),
                                       None, cfg=cfg))
        torch.cuda.synchronize()
        y_sh = torch.cat(parts, dim=1)
        if halves == "1":
            assert torch.allclose(y_sh, y_full, rtol=1e-5, atol=1e-6), world
        else:
            assert torch.equal(y_sh, y_full), world


def _gpu_worker(rank, world, port, backend, result_path):
    """One rank of a head-sharded decode: this rank's KV-head slice through the CUDA kernel (libloki_b200),
    then the layer's one exchange step (sharding.gather_heads).  NCCL ranks own one GPU each; gloo ranks
    share cuda:0 and exchange host copies (NCCL refuses two ranks on one device)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import paper_2406_02542_b200 as L

    dev = torch.device("cuda", rank if backend == "nccl" else 0)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    B, Hq, Hkv, D, S = 4, 16, 8, 128, 8192
    g = torch.Generator(device=dev).manual_seed(17)  # every rank draws the full problem, keeps its slice
    K = torch.randn(B, Hkv, S, D, device=dev, generator=g).to(torch.bfloat16)
    V = torch.randn(B, Hkv, S, D, device=dev, generator=g).to(torch.bfloat16)
    q = torch.randn(B, Hq, D, device=dev, generator=g)
    sh = sharding.head_shard(Hq, Hkv, world, rank)
    y = L.loki_decode(sharding.shard_heads(q, sh, kv=False).contiguous(), sharding.shard_heads(K, sh, kv=True),
                      sharding.shard_heads(V, sh, kv=True), None, k_f=0.25, d=32)
    full = sharding.gather_heads(y if backend == "nccl" else y.cpu(), world)
    if rank == 0:
        y_ref = L.loki_decode(q, K, V, None, k_f=0.25, d=32)
        torch.cuda.synchronize()
        np.save(result_path, np.stack([full.cpu().numpy(), y_ref.cpu().numpy()]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("backend", ["gloo", "nccl"])
def test_two_process_kernel_shard_and_gather_bit_identical(tmp_path, backend):
    """Two processes, each running its KV-head shard through the CUDA kernel, then the all-gather: the
    assembled [B, Hq, D] equals one unsharded launch bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if backend == "nccl" and torch.cuda.device_count() < 2:
        pytest.skip("NCCL needs one GPU per rank (fewer than 2 visible)")
    out = str(tmp_path / "y.npy")
    mp.start_processes(_gpu_worker, args=(2, _free_port(), backend, out), nprocs=2, join=True,
                       start_method="spawn")
    got, ref = np.load(out)
    np.testing.assert_array_equal(got, ref)
