"""Head-parallel Token Sparse Attention over G GPUs (one process per GPU).

The reference is single-process (SPEC.md:166-167 only notes heads "may be
processed in parallel").  The path shards by query heads, GQA-aligned: rank
g owns Q heads [g H/G, (g+1) H/G) and KV heads [g Hkv/G, (g+1) Hkv/G), so
score / select / gather / attend / scatter are local.  Two exchanges:

  C1  all-gather of the score rows s_h  ([H/G x L] f32 per rank) -- the layer
      budget sums every head (token_coverage.cpp:55-57), and summing the
      gathered rows in head order 0..H-1 reproduces the 1-GPU k_keep exactly;
  C2  all-gather of the head outputs    ([H/G x L x d] per rank) -- the head
      concat before W_O (model.cpp:197-200).

The exchanges have two forms (``c2`` selects; "auto" = peer when possible):

  ``c2="peer"``  both exchanges fused into the kernels that produce the rows:
                 the scores [H, L] and the output [H, L, d] are peer buffers
                 on every rank (``PeerBuffers``: tsa_ipc_alloc / tsa_ipc_open,
                 CUDA IPC mappings over NVLink); the pool pass of the scoring, the
                 zero-row pass and the attention epilogue store each row of
                 this rank's heads to every rank's buffer (tsa_*_replicas), so
                 the output exchange overlaps the attention tile by tile;
                 device-side barriers (tsa_peer_barrier) order the budget
                 after the scores and end the step (and one starts it, so no
                 rank overwrites a buffer a peer is still reading);
  ``c2="nccl"``  ``all_gather_into_tensor`` after the scoring and after the
                 attention through torch.distributed (the gloo
                 tests, the unfused f32 / d != 128 path, and the fallback when
                 peer mapping cannot be set up).

The per-stage compute is a pluggable backend: ``CudaBackend`` (the C ABI, the
product) or a test backend; the orchestration is shared.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import torch
import torch.distributed as dist

from . import _lib
from .ops import SparseMode, SparsePlan, _ptr, _stream


@dataclass
class Shard:
    rank: int
    world: int
    n_heads: int
    n_kv_heads: int

    def __post_init__(self):
        if self.n_kv_heads % self.world != 0:
            raise _lib.InvalidArgument(
                f"dist: {self.n_kv_heads} KV heads cannot be split over {self.world} ranks")
        g = self.n_heads // self.n_kv_heads
        self.kv_per = self.n_kv_heads // self.world
        self.h_per = self.kv_per * g
        self.h0, self.h1 = self.rank * self.h_per, (self.rank + 1) * self.h_per
        self.kv0, self.kv1 = self.rank * self.kv_per, (self.rank + 1) * self.kv_per


def forced_begin(plan: SparsePlan, L: int) -> int:
    fs = plan.forced_set(L)
    return fs[0]


class CudaBackend:
    """Stage calls into libtsa_b200.so on the current CUDA stream."""

    def __init__(self, H, Hkv, L, d, dtype_code, plan: SparsePlan, shard: Shard, device,
                 scoring: int = 0):
        self.shard, self.plan, self.device = shard, plan, device
        self.L, self.d = L, d
        common = dict(tau=plan.tau, s_fixed=plan.s_fixed, last_q=plan.last_q, kernel=plan.kernel,
                      forced_policy=int(plan.forced), scoring=scoring,
                      mode=int(plan.mode))
        # local heads as a self-contained layer (absolute head 0 = shard.h0)
        self.local = _lib.make_desc(shard.h_per, shard.kv_per, L, d, dtype_code, **common)
        # the budget reads all H score rows
        self.full = _lib.make_desc(H, Hkv, L, d, dtype_code, **common)
        # the whole layer with this rank's head range: tsa_sparse_attention_layer_sharded
        self.sharded = _lib.make_desc(H, Hkv, L, d, dtype_code, **common)
        self.sharded.head_begin, self.sharded.head_end = shard.h0, shard.h1
        self.sharded_dense = _lib.make_desc(H, Hkv, L, d, dtype_code,
                                            **dict(common, mode=int(SparseMode.kDense)))
        self.sharded_dense.head_begin, self.sharded_dense.head_end = shard.h0, shard.h1
        lib = _lib.load()
        n1 = C.c_size_t()
        _lib.check(lib.tsa_workspace_size(C.byref(self.local), C.byref(n1)))
        # the full-width workspace only serves the budget (headsum/status)
        self.ws = torch.zeros(max(n1.value, 256), dtype=torch.uint8, device=device)
        budget_bytes = 512 + (4 * L + 255) // 256 * 256  # see tsa_workspace_size docs
        self.ws_full = torch.zeros(budget_bytes, dtype=torch.uint8, device=device) \
            if shard.world > 1 else self.ws
        self.k_keep = torch.zeros(1, dtype=torch.int32, device=device)
        self.idx = torch.empty((shard.h_per, L), dtype=torch.int32, device=device)
        self.inv = torch.empty((shard.h_per, L), dtype=torch.int32, device=device)
        sz = (shard.h_per, L, d)
        dt = torch.bfloat16 if dtype_code == _lib.TSA_BF16 else torch.float32
        self.qc, self.kc, self.vc, self.oc = (torch.empty(sz, dtype=dt, device=device)
                                              for _ in range(4))
        fb = forced_begin(plan, L)
        self.forced = torch.arange(fb, L, dtype=torch.int32, device=device)
        self.lib = lib

    def score_replicas(self, q, k, s_outs, n_outs):
        _lib.check(self.lib.tsa_score_replicas(C.byref(self.local), _ptr(q), _ptr(k), s_outs,
                                               n_outs, _ptr(self.ws), _stream(self.device)))

    def score(self, q, k, s_local):
        _lib.check(self.lib.tsa_score(C.byref(self.local), _ptr(q), _ptr(k), _ptr(s_local),
                                      _ptr(self.ws), _stream(self.device)))

    def budget(self, s_full):
        _lib.check(self.lib.tsa_budget(C.byref(self.full), _ptr(s_full), _ptr(self.k_keep),
                                       _ptr(self.ws_full), _stream(self.device)))
        return self.k_keep

    def select(self, s_local, k_keep):
        _lib.check(self.lib.tsa_select(C.byref(self.local), _ptr(s_local), _ptr(k_keep),
                                       _ptr(self.forced), self.forced.numel(), _ptr(self.idx),
                                       _ptr(self.inv), _ptr(self.ws), _stream(self.device)))

    @property
    def fused(self) -> bool:
        return self.local.dtype == _lib.TSA_BF16 and self.local.d_head == 128

    def zero_unselected(self, out_local):
        _lib.check(self.lib.tsa_zero_unselected(C.byref(self.local), _ptr(self.inv),
                                                _ptr(out_local), _stream(self.device)))

    def gather_kv(self, k, v, k_keep):
        _lib.check(self.lib.tsa_gather(C.byref(self.local), None, _ptr(k), _ptr(v),
                                       _ptr(self.idx), _ptr(k_keep), None, _ptr(self.kc),
                                       _ptr(self.vc), _stream(self.device)))

    def gather_kv_zero(self, k, v, k_keep, out_local):
        _lib.check(self.lib.tsa_gather_zero(C.byref(self.local), _ptr(k), _ptr(v), _ptr(self.idx),
                                            _ptr(k_keep), _ptr(self.kc), _ptr(self.vc),
                                            _ptr(self.inv), _ptr(out_local), _stream(self.device)))

    def gather_kv_zero_replicas(self, k, v, k_keep, outs, n_outs):
        _lib.check(self.lib.tsa_gather_zero_replicas(
            C.byref(self.local), _ptr(k), _ptr(v), _ptr(self.idx), _ptr(k_keep), _ptr(self.kc),
            _ptr(self.vc), _ptr(self.inv), outs, n_outs, _stream(self.device)))

    def attend_indexed_replicas(self, q, k, v, k_keep, outs, n_outs):
        _lib.check(self.lib.tsa_attend_indexed_replicas(
            C.byref(self.local), _ptr(q), _ptr(k), _ptr(v), _ptr(self.kc), _ptr(self.vc),
            _ptr(self.idx), _ptr(k_keep), outs, n_outs, _stream(self.device)))

    def attend_indexed(self, q, k, v, k_keep, out_local):
        _lib.check(self.lib.tsa_attend_indexed(C.byref(self.local), _ptr(q), _ptr(k), _ptr(v),
                                               _ptr(self.kc),
                                               _ptr(self.vc), _ptr(self.idx), _ptr(k_keep),
                                               _ptr(out_local), _stream(self.device)))

    def gather(self, q, k, v, k_keep):
        _lib.check(self.lib.tsa_gather(C.byref(self.local), _ptr(q), _ptr(k), _ptr(v),
                                       _ptr(self.idx), _ptr(k_keep), _ptr(self.qc), _ptr(self.kc),
                                       _ptr(self.vc), _stream(self.device)))

    def attend(self, k_keep):
        _lib.check(self.lib.tsa_attend(C.byref(self.local), _ptr(self.qc), _ptr(self.kc),
                                       _ptr(self.vc), _ptr(k_keep), 1, _ptr(self.oc),
                                       _stream(self.device)))

    def scatter(self, out_local):
        _lib.check(self.lib.tsa_scatter(C.byref(self.local), _ptr(self.oc), _ptr(self.inv),
                                        _ptr(out_local), _stream(self.device)))

    def layer_sharded(self, q, k, v, dense, peer=None, nccl_comm=None, s_full=None,
                      out_full=None):
        """The whole sharded step in one C call (tsa_sparse_attention_layer_sharded)."""
        desc = self.sharded_dense if dense else self.sharded
        _lib.check(self.lib.tsa_sparse_attention_layer_sharded(
            C.byref(desc), _ptr(q), _ptr(k), _ptr(v), C.byref(peer) if peer is not None else None,
            C.c_void_p(nccl_comm) if nccl_comm else None, _ptr(s_full), _ptr(out_full),
            _ptr(self.k_keep), _ptr(self.ws), _stream(self.device)))

    def dense(self, q, k, v, out_local):
        _lib.check(self.lib.tsa_dense_attention(C.byref(self.local), _ptr(q), _ptr(k), _ptr(v),
                                                _ptr(out_local), _stream(self.device)))


class _CudaArray:
    """A raw device pointer as a torch tensor (__cuda_array_interface__; the
    memory stays owned by PeerBuffers)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


class TsaPeer(C.Structure):
    """struct tsa_peer (include/tsa_b200.h)."""
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32),
                ("scores", C.c_void_p * _lib.TSA_MAX_REPLICAS),
                ("out", C.c_void_p * _lib.TSA_MAX_REPLICAS),
                ("signals", (C.c_void_p * _lib.TSA_MAX_REPLICAS) * 3)]


class PeerBuffers:
    """Named device buffers every rank allocates with tsa_ipc_alloc and maps
    from every peer with tsa_ipc_open (handles exchanged through the process
    group), plus per-channel signal arrays for tsa_peer_barrier (int32 [world +
    2] per channel and rank: arrivals, the device epoch counter, the timeout
    flag).  ``ptrs[name]`` lists the buffer's base address on every rank, in
    rank order, as seen from this device.

    Setup is collective and failure-tolerant: a rank whose allocation or
    mapping fails still takes part in every exchange (with a failure marker),
    frees what it allocated or mapped, and every rank raises together -- the
    collectives never go out of step."""

    CHANNELS = 3

    def __init__(self, sizes: dict, rank: int, world: int, device):
        self.lib, self.rank, self.world, self.device = _lib.load(), rank, world, device
        if world > _lib.TSA_MAX_REPLICAS:
            raise RuntimeError(f"peer exchange: world {world} > {_lib.TSA_MAX_REPLICAS}")
        self._own, self._opened = [], []
        self.sig_stride = world + 2
        sizes = dict(sizes, _signals=self.CHANNELS * self.sig_stride * 4)
        err = None
        mine = {}
        with torch.cuda.device(device):
            try:
                for name, nbytes in sizes.items():
                    ptr, h = C.c_void_p(), (C.c_char * _lib.TSA_IPC_HANDLE_BYTES)()
                    _lib.check(self.lib.tsa_ipc_alloc(nbytes, C.byref(ptr), h))
                    self._own.append(ptr.value)
                    mine[name] = (ptr.value, bytes(h))
                if os.environ.get("TSA_TEST_PEER_ALLOC_FAIL_RANK") == str(rank):  # test hook
                    raise RuntimeError("injected peer allocation failure")
            except Exception as e:
                err = f"rank {rank}: {type(e).__name__}: {e}"
            every = [None] * world
            dev_index = torch.device(device).index if torch.device(device).index is not None \
                else torch.cuda.current_device()
            payload = {"err": err, "h": {k: v[1] for k, v in mine.items()} if not err else None,
                       "device": dev_index}
            if world > 1:
                dist.all_gather_object(every, payload)
            else:
                every = [payload]
            errs = [x["err"] for x in every if x["err"]]
            # direct peer access (NVLink / NVSwitch) to every other rank's device:
            # the kernels store into the peers' buffers
            self.peer_access = {}
            for r, x in enumerate(every):
                other = x["device"]
                ok = other == dev_index or torch.cuda.can_device_access_peer(dev_index, other)
                self.peer_access[r] = bool(ok)
                if not ok and not errs:
                    errs.append(f"rank {rank}: no peer access from cuda:{dev_index} to cuda:{other}")
            self.ptrs = {}
            if not errs:
                try:
                    for name in sizes:
                        row = []
                        for r in range(world):
                            if r == rank:
                                row.append(mine[name][0])
                                continue
                            ptr = C.c_void_p()
                            h = (C.c_char * _lib.TSA_IPC_HANDLE_BYTES).from_buffer_copy(
                                every[r]["h"][name])
                            _lib.check(self.lib.tsa_ipc_open(h, C.byref(ptr)))
                            self._opened.append(ptr.value)
                            row.append(ptr.value)
                        self.ptrs[name] = row
                except Exception as e:
                    errs.append(f"rank {rank}: {type(e).__name__}: {e}")
            if world > 1:  # the mapping outcome of every rank
                flag = [None] * world
                dist.all_gather_object(flag, errs[-1] if errs else None)
                errs = errs or [f for f in flag if f]
            if errs:
                self.close_mappings()
                if world > 1:
                    dist.barrier()  # every importer closed before any exporter frees
                self.free_own()
                raise RuntimeError("peer buffers: " + "; ".join(errs))
        base = self.ptrs["_signals"]
        self._sig = [(C.c_void_p * _lib.TSA_MAX_REPLICAS)(
            *[p + c * self.sig_stride * 4 for p in base]) for c in range(self.CHANNELS)]

    def tensor(self, name, shape, dtype):
        """This rank's buffer as a tensor (bf16 through an int16 view)."""
        ts = {torch.float32: "<f4", torch.bfloat16: "<i2", torch.int32: "<i4"}[dtype]
        t = torch.as_tensor(_CudaArray(self.ptrs[name][self.rank], shape, ts), device=self.device)
        return t.view(dtype) if dtype == torch.bfloat16 else t

    def barrier(self, channel: int, stream=None):
        """Device barrier on `channel` (epoch from the device counter: capturable)."""
        _lib.check(self.lib.tsa_peer_barrier(self._sig[channel], self.world, self.rank, 0,
                                             _stream(self.device)))

    def check(self):
        """Raises if a barrier of this rank timed out (synchronous)."""
        own = C.c_void_p(self.ptrs["_signals"][self.rank])
        _lib.check(self.lib.tsa_peer_check(own, self.world, self.CHANNELS, _stream(self.device)))

    def peer_struct(self, scores: str, out: str) -> TsaPeer:
        p = TsaPeer()
        p.world, p.rank = self.world, self.rank
        for r in range(self.world):
            p.scores[r] = self.ptrs[scores][r]
            p.out[r] = self.ptrs[out][r]
            for c in range(self.CHANNELS):
                p.signals[c][r] = self._sig[c][r]
        return p

    def close_mappings(self):
        """Unmap the peers' buffers (local; safe at any time after the last step)."""
        for p in self._opened:
            self.lib.tsa_ipc_close(C.c_void_p(p))
        self._opened = []

    def release(self):
        """Collective: every rank unmaps the peers' buffers, then frees its own
        (an exporter may only free after every importer has closed)."""
        torch.cuda.synchronize(self.device)
        self.close_mappings()
        if self.world > 1:
            dist.barrier()
        self.free_own()

    def free_own(self):
        for p in self._own:
            self.lib.tsa_ipc_free(C.c_void_p(p))
        self._own = []


class ShardedSparseAttention:
    """One attention layer's sparse branch (model.cpp:169-183), head-sharded.

    ``step(q_local, k_local, v_local)`` takes this rank's heads ([H/G, L, d]
    and [Hkv/G, L, d]) and returns the gathered output [H, L, d] (or the local
    [H/G, L, d] when ``gather_output`` is False).  ``marks`` (optional) is a
    callable(name) invoked between stages -- bench.py records CUDA events there.
    """

    def __init__(self, H, Hkv, L, d, dtype, plan: SparsePlan, rank=0, world=1, device=None,
                 backend=None, gather_output=True, scoring: int = 0, c2: str = "auto"):
        self.shard = Shard(rank, world, H, Hkv)
        self.H, self.Hkv, self.L, self.d = H, Hkv, L, d
        self.plan = plan
        self.device = device
        self.gather_output = gather_output
        dtype_code = _lib.TSA_BF16 if dtype == torch.bfloat16 else _lib.TSA_F32
        self.backend = backend or CudaBackend(H, Hkv, L, d, dtype_code, plan, self.shard, device,
                                              scoring=scoring)
        sh = self.shard
        self.s_local = torch.zeros((sh.h_per, L), dtype=torch.float32, device=device)
        self.s_full = self.s_local if world == 1 else torch.zeros((H, L), dtype=torch.float32,
                                                                  device=device)  # peer: mapped
        self.out_local = torch.empty((sh.h_per, L, d), dtype=dtype, device=device)
        self.c2 = "nccl"
        self._peer = None
        if c2 not in ("auto", "nccl", "peer"):
            raise _lib.InvalidArgument(f"dist: c2 must be auto, nccl or peer, got {c2!r}")
        want_peer = ((world > 1 or c2 == "peer") and gather_output and c2 != "nccl"
                     and getattr(self.backend, "fused", False)
                     and (world == 1 or dist.is_initialized())
                     and device is not None and torch.device(device).type == "cuda")
        if c2 == "peer" and not want_peer:
            raise _lib.InvalidArgument("dist: c2='peer' needs CUDA devices, a process group "
                                       "for world > 1, the gathered output and the fused "
                                       "bf16 / d = 128 path")
        if want_peer:
            err = None
            try:
                self._setup_peer(H, L, d, dtype, device)
                if os.environ.get("TSA_TEST_PEER_FAIL_RANK") == str(rank):  # test hook
                    raise RuntimeError("injected peer setup failure")
            except Exception as e:  # peer mapping unavailable: all-gathers instead
                if c2 == "peer" and world == 1:
                    raise
                err = f"{type(e).__name__}: {e}"
            if world > 1:  # every rank must take the same form of the exchange
                ok = torch.tensor([0 if err else 1], dtype=torch.int32)
                if dist.get_backend() == "nccl":
                    ok = ok.to(device)
                dist.all_reduce(ok, op=dist.ReduceOp.MIN)
                if not int(ok.item()) and not err:
                    err = "peer mapping failed on another rank"
            if err:  # every rank reaches this branch together (same collective sequence)
                if self._peer is not None:
                    torch.cuda.synchronize(device)
                    self._peer.close_mappings()
                if world > 1:
                    dist.barrier()
                if self._peer is not None:
                    self._peer.free_own()
                self.c2, self._peer = "nccl", None
                self.c2_error = err
                self.s_full = self.s_local if world == 1 else torch.zeros(
                    (H, L), dtype=torch.float32, device=device)  # not the freed peer buffer
                if c2 == "peer":
                    raise RuntimeError(f"dist: c2='peer' could not be set up: {err}")
            else:  # every rank mapped every peer: the device barrier works between them
                self._peer.barrier(0)
                torch.cuda.synchronize(device)
        if self.c2 != "peer":
            self.out_full = self.out_local if world == 1 or not gather_output else torch.empty(
                (H, L, d), dtype=dtype, device=device)
        # the unmarked step as one C call (tsa_sparse_attention_layer_sharded):
        # the peer form, or the NCCL form on the process group's communicator
        self._c_form, self._nccl_comm = None, None
        if isinstance(self.backend, CudaBackend) and gather_output:
            if self.c2 == "peer":
                self._c_form = "peer"
            elif world > 1 and dist.get_backend() == "nccl":
                try:
                    t = torch.zeros(1, device=device)
                    dist.all_reduce(t)  # the communicator exists from here on
                    pg = dist.distributed_c10d._get_default_group()
                    self._nccl_comm = int(pg._get_backend(torch.device("cuda", torch.device(
                        device).index))._comm_ptr())
                    self._c_form = "nccl" if self._nccl_comm else None
                except Exception:  # no raw communicator: the staged all-gathers
                    self._c_form = None

    def _setup_peer(self, H, L, d, dtype, device):
        sh = self.shard
        eb = 2 if dtype == torch.bfloat16 else 4
        self._peer = PeerBuffers({"out": H * L * d * eb, "s": H * L * 4}, sh.rank, sh.world,
                                 device)
        self.out_full = self._peer.tensor("out", (H, L, d), dtype)
        self.s_full = self._peer.tensor("s", (H, L), torch.float32)
        # the shard's descriptor numbers its heads from 0: its output rows start at
        # head h0 of every rank's [H, L, d] buffer, its score rows at row h0 of [H, L]
        out_off = sh.h0 * L * d * eb
        self._replicas = (C.c_void_p * _lib.TSA_MAX_REPLICAS)(
            *[p + out_off for p in self._peer.ptrs["out"]])
        self._peer_struct = self._peer.peer_struct("s", "out")
        off = sh.h0 * L * 4
        self._s_replicas = (C.c_void_p * _lib.TSA_MAX_REPLICAS)(
            *[p + off for p in self._peer.ptrs["s"]])
        self._n_replicas = sh.world
        self.c2 = "peer"

    def release(self):
        """Collective (all ranks together): frees the peer buffers.  Without it
        a dropped layer only unmaps the peers' buffers and keeps its own until
        the process exits -- freeing needs every importer closed first, and
        garbage collection does not run in step across ranks."""
        if self._peer is not None:
            self._peer.release()
            self._peer = None

    def __del__(self):
        peer = getattr(self, "_peer", None)
        if peer is not None:
            try:
                torch.cuda.synchronize(self.device)
                peer.close_mappings()
            except Exception:
                pass

    def _all_gather(self, dst, src):
        if self.shard.world == 1:
            return
        if dist.get_backend() == "nccl":
            dist.all_gather_into_tensor(dst, src)  # NVLink, rank-ordered = head-ordered
        else:  # gloo (CPU tests of the orchestration)
            parts = list(dst.chunk(self.shard.world, dim=0))
            dist.all_gather(parts, src.contiguous())

    def step_graphed(self, q, k, v, dense: bool = False):
        """``step`` replayed from a CUDA graph captured on the first call for
        these input buffers: the chain never waits on the host (k_keep stays
        on the device), so the launch sequence is fixed and one graph launch
        replaces ~8 host launches and their gaps.  The peer form of a sharded
        step is captured too (its barriers take their epochs from device
        counters, so every replay synchronises the ranks); the NCCL form runs
        eagerly."""
        if self.shard.world > 1 and self._c_form != "peer":
            return self.step(q, k, v, dense=dense)  # NCCL all-gathers run eagerly
        key = (q.data_ptr(), k.data_ptr(), v.data_ptr(), dense)
        graphs = self.__dict__.setdefault("_graphs", {})
        g = graphs.get(key)
        if g is None:
            side = torch.cuda.Stream(self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(side):  # warm once outside capture (attributes, maps)
                self.step(q, k, v, dense=dense)
            torch.cuda.current_stream(self.device).wait_stream(side)
            g = torch.cuda.CUDAGraph()
            n0 = _lib.load().tsa_kernel_launches()
            with torch.cuda.graph(g):
                self.step(q, k, v, dense=dense)
            # library kernels per replay (captured launches are counted at capture)
            g.tsa_kernels = _lib.load().tsa_kernel_launches() - n0
            graphs[key] = g
        g.replay()
        self.graph_kernels = g.tsa_kernels
        return self.out_full

    def _step_c(self, q, k, v, dense):
        b = self.backend
        if self._c_form == "peer":
            b.layer_sharded(q, k, v, dense, peer=self._peer_struct)
        else:
            b.layer_sharded(q, k, v, dense, nccl_comm=self._nccl_comm, s_full=self.s_full,
                            out_full=self.out_full)
        return self.out_full

    def check(self):
        """Raises if a peer barrier of this rank timed out (synchronous)."""
        if self._peer is not None:
            self._peer.check()

    def step(self, q, k, v, marks=None, dense: bool = False):
        dense = dense or self.plan.mode == SparseMode.kDense
        if marks is None and self._c_form is not None:
            return self._step_c(q, k, v, dense)
        # staged: one library call per stage (bench.py records events between them)
        mark = marks or (lambda name: None)
        b = self.backend
        if dense:
            mark("start")
            if self.c2 == "peer":
                self._peer.barrier(0)
            b.dense(q, k, v, self.out_local)
            mark("attend")
            if self.c2 == "peer" and self.shard.world == 1:
                self.out_full.copy_(self.out_local)  # the peer buffer is the output
            else:
                self._all_gather(self.out_full, self.out_local)
            if self.c2 == "peer":
                self._peer.barrier(1)
            mark("allgather_out")
            return self.out_full
        mark("start")
        if self.c2 == "peer":
            # no rank writes into a buffer a peer still reads; then the score
            # rows go to every rank's [H, L] buffer from the pool kernel
            self._peer.barrier(0)
            b.score_replicas(q, k, self._s_replicas, self._n_replicas)
            mark("score")
            self._peer.barrier(2)
            mark("c1_barrier")
            s_local = self.s_full[self.shard.h0:self.shard.h1]
        else:
            b.score(q, k, self.s_local)
            mark("score")
            self._all_gather(self.s_full, self.s_local)
            mark("allgather_scores")
            s_local = self.s_local
        k_keep = b.budget(self.s_full)
        mark("budget")
        b.select(s_local, k_keep)
        mark("select")
        if self.c2 == "peer":
            # C2 fused into the producers: zero rows and attention output rows
            # go to every rank's peer buffer over NVLink
            b.gather_kv_zero_replicas(k, v, k_keep, self._replicas, self._n_replicas)
            mark("gather_zero")
            b.attend_indexed_replicas(q, k, v, k_keep, self._replicas, self._n_replicas)
            mark("attend")
            self._peer.barrier(1)
            mark("c2_barrier")
            return self.out_full
        if getattr(b, "fused", False):
            # K/V compress + zero the dropped rows (one launch), then attend with
            # Q gathered by TMA gather4 and the output rows stored at their
            # original positions
            b.gather_kv_zero(k, v, k_keep, self.out_local)
            mark("gather_zero")
            b.attend_indexed(q, k, v, k_keep, self.out_local)
            mark("attend")
        else:
            b.gather(q, k, v, k_keep)
            mark("gather")
            b.attend(k_keep)
            mark("attend")
            b.scatter(self.out_local)
            mark("scatter")
        self._all_gather(self.out_full, self.out_local)
        mark("allgather_out")
        return self.out_full

    @property
    def k_keep(self) -> int:
        return int(self.backend.k_keep.item())
