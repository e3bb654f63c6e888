"""Synthetic attention-layer inputs for the benchmark configurations.

BASELINE.json configs[] use random inputs of Llama-3 head geometry (there are
no checkpoints or datasets offline).  Two generators:

* ``uniform_heads``  -- i.i.d. uniform[-1, 1) (the reference's own inputs,
  random.hpp:36-44) on the device; k/L ~ 1 - tau for the scoring proxy.
* ``heavy_tailed_heads`` -- the "T" generator of SURVEY.md §8(d): per KV head
  a unit direction u_h; the trailing last_q query rows are sqrt(d) u_h plus
  noise, keys are a_t u_h plus noise with block-constant log-normal offsets
  a_t = sigma (sqrt(shared) z_shared + sqrt(1 - shared) z_head), so the
  proxy attention mass is heavy-tailed as in long-context prompts and the
  paper's tau levels produce the paper's sparsity.
  sigma is calibrated on the reference-order scoring (bench.py --calibrate).

Both are deterministic for a seed on a given device.
"""
from __future__ import annotations

import math

import torch

# Calibrated on the REFERENCE-order scoring at L=131072, Llama-3-8B geometry
# (bench.py --calibrate, see profiles/calibration.md): sigma 2.6 -> 2.8 moves tau=0.01
# from k/L 0.624 to 0.560; 2.75 targets the paper's 67.36% (k/L 0.571) and 54.44%.
DEFAULT_SIGMA = 2.75


def uniform_heads(H, Hkv, L, d, seed=0, dtype=torch.bfloat16, device="cuda"):
    g = torch.Generator(device=device).manual_seed(seed)
    mk = lambda n: (torch.rand((n, L, d), generator=g, device=device) * 2 - 1).to(dtype)
    return mk(H), mk(Hkv), mk(Hkv)


def heavy_tailed_heads(H, Hkv, L, d, sigma=DEFAULT_SIGMA, seed=0, dtype=torch.bfloat16,
                       device="cuda", last_q=64, block=32, shared=0.5, noise=0.1):
    g = torch.Generator(device=device).manual_seed(seed)
    u = torch.randn((Hkv, d), generator=g, device=device)
    u = u / u.norm(dim=-1, keepdim=True)
    nb = (L + block - 1) // block
    z_shared = torch.randn((1, nb), generator=g, device=device)
    z_head = torch.randn((Hkv, nb), generator=g, device=device)
    a = sigma * (math.sqrt(shared) * z_shared + math.sqrt(1.0 - shared) * z_head)
    a = a.repeat_interleave(block, dim=1)[:, :L]
    k = torch.empty((Hkv, L, d), dtype=dtype, device=device)
    v = torch.empty((Hkv, L, d), dtype=dtype, device=device)
    q = torch.empty((H, L, d), dtype=dtype, device=device)
    for j in range(Hkv):  # per head to bound the f32 temporaries
        k[j] = (a[j, :, None] * u[j][None, :]
                + noise * torch.randn((L, d), generator=g, device=device)).to(dtype)
        v[j] = (torch.rand((L, d), generator=g, device=device) * 2 - 1).to(dtype)
    group = H // Hkv
    lq = min(last_q, L)
    for h in range(H):
        qh = torch.rand((L, d), generator=g, device=device) * 2 - 1
        qh[L - lq:] = (math.sqrt(d) * u[h // group][None, :]
                       + noise * torch.randn((lq, d), generator=g, device=device))
        q[h] = qh.to(dtype)
    return q, k, v
