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
    for _ in range(2):
        peer.out_full.fill_(float("nan"))
        peer.s_full.fill_(float("nan"))
        b = peer.step(q, k, v)
        torch.cuda.synchronize()
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))
        assert torch.equal(peer.s_full, ref.s_full) and peer.k_keep == ref.k_keep
    dist.destroy_process_group()
    print("peer c2 ok", ref.k_keep)
""")


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
