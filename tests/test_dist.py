"""Multi-rank head sharding (paper_2602_03216_b200/dist.py) on CPU: gloo,
world_size 2, with the CPU oracle as the per-stage backend (test-only), so
the orchestration -- GQA-aligned head split, score all-gather in head order,
a single shared budget, local select/attend, output all-gather -- is checked
against the unsharded reference path bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import Oracle, RefRng, gqa_heads
from paper_2602_03216_b200.dist import Shard, ShardedSparseAttention
from paper_2602_03216_b200.ops import SparseMode, SparsePlan


class OracleBackend:
    """Stage-for-stage stand-in for CudaBackend on CPU tensors (test only)."""

    fused = False

    def __init__(self, plan, shard, L):
        self.port = Oracle("port")
        self.plan, self.shard, self.L = plan, shard, L
        self.k_keep = torch.zeros(1, dtype=torch.int32)

    def score(self, q, k, s_local):
        s_local.copy_(torch.from_numpy(self.port.score_tokens(q.numpy(), k.numpy(),
                                                              self.plan.last_q, self.plan.kernel)))

    def budget(self, s_full):
        forced = self.plan.forced_set(self.L)
        if self.plan.mode == SparseMode.kFixed:
            k = self.port.fixed_budget(self.L, self.plan.s_fixed, max(1, len(forced)))
        else:
            k = self.port.coverage_budget(self.port.aggregate_scores(s_full.numpy()), self.plan.tau,
                                          max(1, len(forced)))
        self.k_keep[0] = k
        return self.k_keep

    def select(self, s_local, k_keep):
        self.idx = self.port.select_tokens(s_local.numpy(), int(k_keep[0]),
                                           self.plan.forced_set(self.L))

    def gather(self, q, k, v, k_keep):
        self.qkv = (q.numpy(), k.numpy(), v.numpy())

    def attend(self, k_keep):
        self.o = self.port.token_sparse_attention(*self.qkv, self.idx)

    def scatter(self, out_local):
        out_local.copy_(torch.from_numpy(self.o))

    def dense(self, q, k, v, out_local):
        H, L = q.shape[0], q.shape[1]
        idx = np.tile(np.arange(L, dtype=np.int32), (H, 1))
        out_local.copy_(torch.from_numpy(
            self.port.token_sparse_attention(q.numpy(), k.numpy(), v.numpy(), idx)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASE = dict(H=8, Hkv=4, L=96, d=16, seed=77)


def run_rank(rank, world, port, plan_kw, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = CASE
    q, k, v = gqa_heads(RefRng(c["seed"]), c["H"], c["Hkv"], c["L"], c["d"])
    plan = SparsePlan(sparse_layers=[0], **plan_kw)
    shard = Shard(rank, world, c["H"], c["Hkv"])
    be = OracleBackend(plan, shard, c["L"])
    lay = ShardedSparseAttention(c["H"], c["Hkv"], c["L"], c["d"], torch.float32, plan,
                                 rank=rank, world=world, device=torch.device("cpu"), backend=be)
    out = lay.step(torch.from_numpy(q[shard.h0:shard.h1]), torch.from_numpy(k[shard.kv0:shard.kv1]),
                   torch.from_numpy(v[shard.kv0:shard.kv1]))
    assert lay.c2 == "nccl"  # gloo: the all-gather form of C2
    with pytest.raises(ValueError, match="c2='peer' needs CUDA devices"):
        ShardedSparseAttention(c["H"], c["Hkv"], c["L"], c["d"], torch.float32, plan, rank=rank,
                               world=world, device=torch.device("cpu"), backend=be, c2="peer")
    if rank == 0:
        np.savez(out_path, out=out.numpy(), k_keep=lay.k_keep, s=lay.s_full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("plan_kw", [dict(mode=SparseMode.kDynamic, tau=0.1),
                                     dict(mode=SparseMode.kDynamic, tau=0.6),
                                     dict(mode=SparseMode.kFixed, s_fixed=0.4)])
def test_two_rank_head_sharding_matches_unsharded(tmp_path, plan_kw):
    world = 2
    out_path = str(tmp_path / "r0.npz")
    mp.start_processes(run_rank, args=(world, free_port(), plan_kw, out_path), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(out_path)
    c = CASE
    port = Oracle("port")
    q, k, v = gqa_heads(RefRng(c["seed"]), c["H"], c["Hkv"], c["L"], c["d"])
    plan = SparsePlan(sparse_layers=[0], **plan_kw)
    s = port.score_tokens(q, k, plan.last_q, plan.kernel)
    forced = plan.forced_set(c["L"])
    if plan.mode == SparseMode.kFixed:
        kk = port.fixed_budget(c["L"], plan.s_fixed, 1)
    else:
        kk = port.coverage_budget(port.aggregate_scores(s), plan.tau, 1)
    idx = port.select_tokens(s, kk, forced)
    ref = port.token_sparse_attention(q, k, v, idx)
    assert int(got["k_keep"]) == kk
    assert np.array_equal(got["s"].view(np.uint32), s.view(np.uint32))   # head-ordered gather
    assert np.array_equal(got["out"].view(np.uint32), ref.view(np.uint32))


def test_c2_mode_is_validated():
    plan = SparsePlan(sparse_layers=[0])
    be = OracleBackend(plan, Shard(0, 1, 8, 4), 16)
    with pytest.raises(ValueError, match="c2 must be"):
        ShardedSparseAttention(8, 4, 16, 16, torch.float32, plan, device=torch.device("cpu"),
                               backend=be, c2="shmem")


def test_shard_geometry():
    s = Shard(1, 4, 32, 8)
    assert (s.h0, s.h1, s.kv0, s.kv1) == (8, 16, 2, 4)
    s = Shard(7, 8, 64, 8)  # 70B geometry: 8 Q + 1 KV head per GPU
    assert (s.h0, s.h1, s.kv0, s.kv1) == (56, 64, 7, 8)
    with pytest.raises(ValueError):
        Shard(0, 3, 32, 8)
