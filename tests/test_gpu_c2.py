"""The multi-GPU boundary fused into the producers (C2 over peer memory,
dist.py ``c2="peer"``): the zero-row pass and the attention epilogue store
every output row to each replica of the [H, L, d] output.  One GPU is
available to these tests, so the replicas are local buffers here and, in the
peer-buffer test, a world-size-1 group whose single buffer goes through the
same IPC allocation and device barrier the 8-GPU run uses (the cross-process
form runs in tests/test_gpu_dist.py with several ranks on one GPU)."""
import os
import subprocess
import sys
import textwrap
from pathlib import Path

import ctypes as C

import pytest
import torch

import paper_2602_03216_b200 as tsa

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _layer(L, seed, tau=0.02):
    from paper_2602_03216_b200 import workloads
    from paper_2602_03216_b200.dist import ShardedSparseAttention
    q, k, v = workloads.heavy_tailed_heads(8, 2, L, 128, seed=seed)
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=tau)
    lay = ShardedSparseAttention(8, 2, L, 128, torch.bfloat16, plan, device=q.device)
    return lay, q, k, v


@pytest.mark.parametrize("L,n_rep", [(3000, 3), (4096, 8), (700, 1)])
def test_replica_kernels_write_identical_rows(cuda, L, n_rep):
    from paper_2602_03216_b200 import _lib
    lay, q, k, v = _layer(L, seed=21)
    ref = lay.step(q, k, v).clone()  # single output: gather_zero + attend_indexed
    b = lay.backend
    outs = [torch.full_like(ref, float("nan")) for _ in range(n_rep)]
    arr = (C.c_void_p * _lib.TSA_MAX_REPLICAS)(*[o.data_ptr() for o in outs])
    b.gather_kv_zero_replicas(k, v, b.k_keep, arr, n_rep)
    b.attend_indexed_replicas(q, k, v, b.k_keep, arr, n_rep)
    torch.cuda.synchronize()
    assert lay.k_keep < L
    for o in outs:  # every row written (no NaN left), identical to the single-output path
        assert torch.equal(o.view(torch.int16), ref.view(torch.int16))


@pytest.mark.parametrize("scoring", [1, 2])  # REFERENCE-order and FAST (tensor-core) scoring
def test_score_replicas_write_identical_rows(cuda, scoring):
    from paper_2602_03216_b200 import _lib, workloads
    from paper_2602_03216_b200.dist import ShardedSparseAttention
    L = 2048
    q, k, v = workloads.heavy_tailed_heads(8, 2, L, 128, seed=8)
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.02)
    lay = ShardedSparseAttention(8, 2, L, 128, torch.bfloat16, plan, device=q.device,
                                 scoring=scoring)
    b = lay.backend
    ref = torch.empty((8, L), dtype=torch.float32, device=q.device)
    b.score(q, k, ref)
    # replicas of a [16, L] buffer, this "rank" owning rows 8..15 (offset bases)
    outs = [torch.full((16, L), float("nan"), device=q.device) for _ in range(3)]
    arr = (C.c_void_p * _lib.TSA_MAX_REPLICAS)(*[o.data_ptr() + 8 * L * 4 for o in outs])
    b.score_replicas(q, k, arr, 3)
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o[8:].view(torch.int32), ref.view(torch.int32))
        assert bool(torch.isnan(o[:8]).all())  # other ranks' rows untouched


def test_replica_count_is_validated(cuda):
    from paper_2602_03216_b200 import _lib
    lay, q, k, v = _layer(512, seed=3)
    lay.step(q, k, v)
    b = lay.backend
    arr = (C.c_void_p * _lib.TSA_MAX_REPLICAS)()
    for n in (0, _lib.TSA_MAX_REPLICAS + 1):
        with pytest.raises(_lib.InvalidArgument, match="n_outs"):
            b.attend_indexed_replicas(q, k, v, b.k_keep, arr, n)
    with pytest.raises(_lib.InvalidArgument, match="null output replica"):
        b.gather_kv_zero_replicas(k, v, b.k_keep, arr, 1)


SCRIPT = textwrap.dedent("""
    import os, sys, torch, torch.distributed as dist
    sys.path.insert(0, {root!r})
    import paper_2602_03216_b200 as tsa
    from paper_2602_03216_b200 import workloads
    from paper_2602_03216_b200.dist import ShardedSparseAttention
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", init_method="tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=dev)
    L = 3000
    q, k, v = workloads.heavy_tailed_heads(8, 2, L, 128, seed=5)
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.02)
    ref = ShardedSparseAttention(8, 2, L, 128, torch.bfloat16, plan, device=dev, c2="nccl")
    peer = ShardedSparseAttention(8, 2, L, 128, torch.bfloat16, plan, device=dev, c2="peer")
    assert peer.c2 == "peer", peer.c2
    a = ref.step(q, k, v).clone()
    same = lambda x, y: torch.equal(x.view(torch.int16), y.view(torch.int16))
    # the peer form: one C call (tsa_sparse_attention_layer_sharded), the staged
    # stage calls (marks) and the graph-replayed C call (device barrier epochs)
    for run in ("c", "staged", "graph", "graph", "c"):
        peer.out_full.fill_(float("nan"))
        peer.s_full.fill_(float("nan"))
        if run == "c":
            b = peer.step(q, k, v)
        elif run == "staged":
            b = peer.step(q, k, v, marks=lambda name: None)
        else:
            b = peer.step_graphed(q, k, v)
        torch.cuda.synchronize()
        assert same(a, b), run
        assert torch.equal(peer.s_full, ref.s_full) and peer.k_keep == ref.k_keep, run
    peer.check()  # no barrier timed out
    # a dense step in the peer form lands in the peer output buffer (staged and C)
    dense_ref, _ = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), tsa.SparsePlan())
    for marks in (None, lambda name: None):
        peer.out_full.fill_(float("nan"))
        b = peer.step(q, k, v, dense=True, marks=marks)
        torch.cuda.synchronize()
        assert same(dense_ref, b) and peer.k_keep == L
    # the NCCL form of the C entry on the process group's communicator (world 1)
    pg = dist.distributed_c10d._get_default_group()
    comm = int(pg._get_backend(dev)._comm_ptr())
    s_full = torch.full((8, L), float("nan"), device=dev)
    out_full = torch.full_like(q, float("nan"))
    ref.backend.layer_sharded(q, k, v, False, nccl_comm=comm, s_full=s_full, out_full=out_full)
    torch.cuda.synchronize()
    assert same(a, out_full) and torch.equal(s_full, ref.s_full)
    ref.backend.layer_sharded(q, k, v, True, nccl_comm=comm, s_full=s_full, out_full=out_full)
    torch.cuda.synchronize()
    assert same(dense_ref, out_full)
    dist.destroy_process_group()
    print("peer c2 ok", ref.k_keep)
""")


TIMEOUT_SCRIPT = textwrap.dedent("""
    import ctypes as C, os, sys, torch
    sys.path.insert(0, {root!r})
    from paper_2602_03216_b200 import _lib
    lib = _lib.load()
    world = 2
    sig = torch.zeros(2 * (world + 2), dtype=torch.int32, device="cuda")
    arr = (C.c_void_p * 8)(sig.data_ptr(), sig.data_ptr() + (world + 2) * 4)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    # rank 0 of 2 alone at the barrier: the peer never arrives
    _lib.check(lib.tsa_peer_barrier(arr, world, 0, 0, st))
    torch.cuda.synchronize()  # returns after TSA_PEER_TIMEOUT_S, no trap
    try:
        _lib.check(lib.tsa_peer_check(C.c_void_p(sig.data_ptr()), world, 1, st))
        print("no timeout reported")
    except _lib.CudaError as e:
        assert "did not reach barrier" in str(e), e
        x = torch.ones(4, device="cuda") * 2  # the context is still usable
        print("timeout ok", float(x.sum()))
""")


def test_peer_barrier_timeout_sets_a_flag_not_a_trap(cuda, tmp_path):
    """A peer that never arrives: the barrier returns after TSA_PEER_TIMEOUT_S
    with the timeout flag set (tsa_peer_check raises) and the CUDA context stays
    usable -- no __trap / sticky error (the 60 s trap)."""
    p = tmp_path / "timeout.py"
    p.write_text(TIMEOUT_SCRIPT.format(root=str(ROOT)))
    r = subprocess.run([sys.executable, str(p)], capture_output=True, text=True, timeout=120,
                       env={**os.environ, "TSA_PEER_TIMEOUT_S": "1"})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "timeout ok" in r.stdout


def test_peer_c2_ipc_buffers_world1(cuda, tmp_path):
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    p = tmp_path / "peer.py"
    p.write_text(SCRIPT.format(root=str(ROOT), port=port))
    r = subprocess.run([sys.executable, str(p)], capture_output=True, text=True, timeout=300,
                       env={**os.environ, "MASTER_ADDR": "127.0.0.1"})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "peer c2 ok" in r.stdout
