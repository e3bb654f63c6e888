"""The operators are pure functions safe to call from several threads at once
(SPEC.md:90-91): per-stream scratch in the Python front end, per-thread host
pipelines and capture streams in the library, per-device kernel attributes.
Two threads, each on its own stream with its own inputs, run scoring, the
device layer (fresh and cached buffers: graph replay) and the host-tensor layer
concurrently; every result equals the serial run bit for bit."""
import threading

import pytest
import torch

import paper_2602_03216_b200 as tsa
from paper_2602_03216_b200 import workloads

pytestmark = pytest.mark.gpu


def _work(q, k, v, plan):
    h = tsa.HeadTensors(q, k, v)
    s = tsa.score_tokens(h, 64, 7).s.clone()
    out1, st = tsa.sparse_attention_layer(h, plan)
    out2 = torch.empty_like(q)
    for _ in range(3):  # cached scratch + graph replay
        tsa.sparse_attention_layer(h, plan, out=out2, stat=False)
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    hout = torch.empty(q.shape, dtype=q.dtype).pin_memory()
    tsa.sparse_attention_layer_host(hq, hk, hv, hout, plan, device=q.device, n_groups=2)
    torch.cuda.current_stream().synchronize()
    return s, out1.clone(), st.k_keep, out2.clone(), hout.clone()


def test_two_threads_two_streams_match_serial(cuda):
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.02)
    inputs = [workloads.heavy_tailed_heads(8, 2, 3000 + 500 * i, 128, seed=60 + i) for i in range(2)]
    serial = [_work(*x, plan) for x in inputs]
    torch.cuda.synchronize()
    results, errors = [None, None], []

    def run(i):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                for _ in range(3):
                    results[i] = _work(*inputs[i], plan)
        except Exception as e:  # surfaced below
            errors.append(e)

    ts = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    torch.cuda.synchronize()
    assert not errors, errors
    for got, ref in zip(results, serial):
        assert got[2] == ref[2]
        for a, b in zip(got[:2] + got[3:], ref[:2] + ref[3:]):
            assert torch.equal(a.view(torch.int16) if a.dtype == torch.bfloat16 else a,
                               b.view(torch.int16) if b.dtype == torch.bfloat16 else b)
