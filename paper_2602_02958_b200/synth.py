"""Synthetic clustered K/V planes, generated on the GPU.

Same family as the reference's generator (Q/datagen.py:44-161): tokens of a
plane fall into tight Gaussian clusters (sigma_within) around widely spread
means (sigma_between); every cluster amplifies its own subset of the
outlier channels 0, 16, ..., 112 by ``outlier_scale`` (10 for keys,
100 for values, |V| ~ 1e3).  Values are rounded to bf16, so
the bf16 device input and the float32 oracle input are the same numbers.
Not bit-identical to the reference's numpy stream (it cannot travel to the
GPU box); parity tests use the committed fixtures for that.
"""

from __future__ import annotations

import torch


def clustered_planes(n_planes: int, n_tokens: int, head_dim: int = 128, n_clusters: int = 256,
                     sigma_within: float = 0.125, sigma_between: float = 2.5,
                     outlier_scale: float = 10.0, seed: int = 0, device="cuda",
                     dtype=torch.bfloat16, planes_per_batch: int = 256) -> torch.Tensor:
    """[P, N, d] clustered planes (generated in batches to bound temporaries)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = torch.empty((n_planes, n_tokens, head_dim), dtype=dtype, device=device)
    ch = torch.arange(0, head_dim, 16, device=device)
    for p0 in range(0, n_planes, planes_per_batch):
        pb = min(planes_per_batch, n_planes - p0)
        means = torch.randn((pb, n_clusters, head_dim), generator=g, device=device) * sigma_between
        amp = torch.ones((pb, n_clusters, head_dim), device=device)
        mask = torch.rand((pb, n_clusters, ch.numel()), generator=g, device=device) < 0.5
        amp[:, :, ch] = torch.where(mask, torch.full_like(mask, outlier_scale, dtype=torch.float32),
                                    torch.ones_like(mask, dtype=torch.float32))
        asg = torch.randint(0, n_clusters, (pb, n_tokens), generator=g, device=device)
        idx = asg.unsqueeze(-1).expand(pb, n_tokens, head_dim)
        x = torch.gather(means, 1, idx)
        x += torch.randn((pb, n_tokens, head_dim), generator=g, device=device) * sigma_within
        x *= torch.gather(amp, 1, idx)
        out[p0:p0 + pb] = x.to(dtype)
    return out


def kv_cache_planes(n_layers: int, n_heads: int, n_tokens: int, head_dim: int = 128,
                    seed: int = 0, device="cuda") -> torch.Tensor:
    """[L*H*2, N, d] bf16: plane 2*(l*H+h) is K (outliers x10), +1 is V (x100)."""
    P = n_layers * n_heads
    k = clustered_planes(P, n_tokens, head_dim, outlier_scale=10.0, seed=2 * seed, device=device)
    v = clustered_planes(P, n_tokens, head_dim, outlier_scale=100.0, seed=2 * seed + 1,
                         device=device)
    return torch.stack([k, v], dim=1).reshape(2 * P, n_tokens, head_dim)
