"""The head-sharded layer with the CUDA backend, world size 2 and 4 on ONE GPU
(all ranks on cuda:0; collectives over gloo, which moves CUDA tensors through
the host): the per-rank shard descriptors, the score exchange before the
shared budget and the output exchange must reproduce the single-process layer
bit for bit.  (The 8-GPU NCCL / peer-memory forms run the same orchestration;
only one GPU is available to these tests.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

def _rank(rank, world, port, out_path, tau, c, c2):
    if c2 == "auto-fail":  # the last rank's peer setup fails: every rank falls back together
        os.environ["TSA_TEST_PEER_FAIL_RANK"] = str(world - 1)
        c2 = "auto"
    if c2 == "auto-allocfail":  # rank 0's IPC allocation fails BEFORE the handle exchange
        os.environ["TSA_TEST_PEER_ALLOC_FAIL_RANK"] = "0"
        c2 = "auto"
    import paper_2602_03216_b200 as tsa
    from paper_2602_03216_b200 import workloads
    from paper_2602_03216_b200.dist import ShardedSparseAttention
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q, k, v = workloads.heavy_tailed_heads(c["H"], c["Hkv"], c["L"], 128, seed=c["seed"])
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=tau)
    lay = ShardedSparseAttention(c["H"], c["Hkv"], c["L"], 128, torch.bfloat16, plan, rank=rank,
                                 world=world, device=q.device, c2=c2)
    sh = lay.shard
    args = (q[sh.h0:sh.h1].contiguous(), k[sh.kv0:sh.kv1].contiguous(),
            v[sh.kv0:sh.kv1].contiguous())
    outs = []
    # repeated steps (barrier epochs, buffers rewritten in place) through every
    # entry: the one-call C form, the staged stage calls, the graph replay
    for run in ("c", "staged", "graph", "graph", "c"):
        if lay.c2 == "peer":
            lay.out_full.fill_(float("nan"))
            lay.s_full.fill_(float("nan"))
            torch.cuda.synchronize()
            dist.barrier()  # no rank refills after a peer's kernels started writing
        if run == "c":
            out = lay.step(*args)
        elif run == "staged":
            out = lay.step(*args, marks=lambda name: None)
        else:
            out = lay.step_graphed(*args)
        torch.cuda.synchronize()
        dist.barrier()
        outs.append(out.view(torch.int16).clone())
    assert all(torch.equal(outs[0], o) for o in outs)
    lay.check()
    if rank == 0:
        np.savez(out_path, out=out.view(torch.int16).cpu().numpy(), k_keep=lay.k_keep,
                 s=lay.s_full.cpu().numpy(), c2=lay.c2)
    dist.barrier()
    dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("c2", ["nccl", "peer", "auto-fail", "auto-allocfail"])
@pytest.mark.parametrize("world,H,Hkv,tau", [(2, 8, 2, 0.02), (2, 8, 2, 0.0), (4, 16, 4, 0.02)])
def test_multi_rank_cuda_sharding_matches_single_process(cuda, tmp_path, world, H, Hkv, tau, c2):
    """c2="nccl": the all-gathers (over gloo here); c2="peer": the score and
    output rows stored by the kernels into the other processes' IPC-mapped
    buffers, with device barriers -- the fused exchange across processes."""
    import paper_2602_03216_b200 as tsa
    from paper_2602_03216_b200 import workloads
    from paper_2602_03216_b200.dist import ShardedSparseAttention
    out_path = str(tmp_path / "r0.npz")
    c = dict(H=H, Hkv=Hkv, L=2500, seed=41)
    mp.start_processes(_rank, args=(world, _port(), out_path, tau, c, c2), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(out_path)
    q, k, v = workloads.heavy_tailed_heads(c["H"], c["Hkv"], c["L"], 128, seed=c["seed"])
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=tau)
    one = ShardedSparseAttention(c["H"], c["Hkv"], c["L"], 128, torch.bfloat16, plan,
                                 device=q.device)
    ref = one.step(q, k, v)
    torch.cuda.synchronize()
    assert str(got["c2"]) == ("nccl" if c2.startswith("auto-") else c2)
    assert int(got["k_keep"]) == one.k_keep
    assert np.array_equal(got["s"].view(np.uint32), one.s_full.cpu().numpy().view(np.uint32))
    assert np.array_equal(got["out"], ref.view(torch.int16).cpu().numpy())
