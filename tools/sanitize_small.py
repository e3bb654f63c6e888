"""Small end-to-end runs of every production path, for compute-sanitizer:
FAST bf16 layer (fused gather/attend), tau = 0 in-place, fixed mode, f32
reference-order layer, host-tensor pipeline (back-to-back, overlapping), dense, the
3xTF32 f32 attention, the exact budget total (chunk-monoid walk), the fused tcgen05
projections (2-CTA GEMM) and the row statistic / weight layout kernels."""
import math
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import workloads  # noqa: E402

for L in (1000, 1537):
    q, k, v = workloads.heavy_tailed_heads(8, 2, L, 128, seed=3)
    h = tsa.HeadTensors(q, k, v)
    for plan in (tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.02),
                 tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.0),
                 tsa.SparsePlan(mode=tsa.SparseMode.kFixed, sparse_layers=[0], s_fixed=0.5),
                 tsa.SparsePlan()):
        out, st = tsa.sparse_attention_layer(h, plan)
        hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
        hout = torch.empty(q.shape, dtype=q.dtype).pin_memory()
        tsa.sparse_attention_layer_host(hq, hk, hv, hout, plan, n_groups=2)
        tsa.sparse_attention_layer_host(hq, hk, hv, hout, plan)  # back to back, overlapping
    hf = tsa.HeadTensors(q.float(), k.float(), v.float())
    for pairs in ("0", "1"):  # the f32 attention, single-CTA and 2-CTA kernels
        os.environ["TSA_TF32_PAIRS"] = pairs
        tsa.sparse_attention_layer(hf, tsa.SparsePlan(mode=tsa.SparseMode.kDynamic,
                                                      sparse_layers=[0], tau=0.3))
    os.environ.pop("TSA_TF32_PAIRS")
    # exact total on adversarial values (ties, crossings) through aggregate_scores
    x = torch.linspace(-20, 5, 40000, device="cuda").exp()[None]
    tsa.aggregate_scores(tsa.HeadScores(x))
# the exact scorer's chain mode (>= 5 rows per row-sum CTA: the summing warp's float4
# reads of the e tile), ragged L
q, k, v = workloads.heavy_tailed_heads(32, 8, 1537, 128, seed=5)
tsa.score_tokens(tsa.HeadTensors(q, k, v), 64, 7)
# projections: QKV with norm / RoPE / split, W_o with residual, plain GEMM (ragged M)
L, D, H, Hkv = 300, 512, 4, 2
x = torch.randn((L, D), device="cuda").to(torch.bfloat16)
w = (torch.randn((D, (H + 2 * Hkv) * 128), device="cuda") / math.sqrt(D)).to(torch.bfloat16)
wo = (torch.randn((H * 128, D), device="cuda") / 16).to(torch.bfloat16)
table = tsa.rope_table(L, 128, 10000.0, "cuda")
heads = tsa.qkv_proj(x, tsa.prepare_weight(w, torch.ones(D, device="cuda")),
                     tsa.row_inv_rms(x, 1e-5), table, H, Hkv, 128)
tsa.out_proj_residual(heads.q.contiguous(), tsa.prepare_weight(wo), x)
tsa.gemm_bf16(x, tsa.prepare_weight(w))
torch.cuda.synchronize()
print("sanitize_small done")
