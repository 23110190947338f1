"""Head / layer sharding over GPUs (one process per GPU, torch.distributed).

Every (layer, head, K|V) plane is compressed, decompressed and attended
independently, and stage seeds do not depend on the head (Q/prq.py:32-35),
so a rank can own any subset of heads with bit-identical results.  The hot
path has no collective; the only exchange is the final all-gather of each
rank's attention outputs (bf16, NCCL over NVLink on a B200 box; gloo in
the CPU tests).
"""

from __future__ import annotations

from typing import List, Optional, Tuple

import torch
import torch.distributed as dist


def head_range(n_heads: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block of heads owned by `rank` (sizes differ by at most 1)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, extra = divmod(n_heads, world)
    h0 = rank * base + min(rank, extra)
    return h0, h0 + base + (1 if rank < extra else 0)


def plane_pairs(n_layers: int, n_heads: int, world: int, rank: int) -> List[Tuple[int, int]]:
    """(layer, head) pairs owned by `rank` when heads do not divide evenly
    (e.g. Wan2.1: 30 x 12 = 360 pairs over 8 GPUs = 45 each)."""
    pairs = [(l, h) for l in range(n_layers) for h in range(n_heads)]
    lo, hi = head_range(len(pairs), world, rank)
    return pairs[lo:hi]


def kv_plane_index(layer: int, head: int, n_heads: int, kind: int) -> int:
    """Plane index of (layer, head, K=0|V=1) in the [L*H*2, N, d] cache layout."""
    return 2 * (layer * n_heads + head) + kind


def gather_heads(local: torch.Tensor, n_heads: int, group: Optional[dist.ProcessGroup] = None) -> torch.Tensor:
    """All-gather per-rank outputs [Nq, Hr, d] (rank r owns head_range(r)) into
    [Nq, H, d] on every rank."""
    world = dist.get_world_size(group)
    nq, _, d = local.shape
    sizes = [head_range(n_heads, world, r) for r in range(world)]
    hmax = max(h1 - h0 for h0, h1 in sizes)
    pad = torch.zeros((nq, hmax, d), dtype=local.dtype, device=local.device)
    pad[:, :local.shape[1]] = local
    buf = torch.empty((world, nq, hmax, d), dtype=local.dtype, device=local.device)
    if hasattr(dist, "all_gather_into_tensor") and local.is_cuda and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(buf, pad.contiguous(), group=group)
    elif local.element_size() == 2 and d % 2 == 0:
        # gloo has no 16-bit integer / bf16 all_gather: move the bits as int32 pairs
        b32 = buf.view(torch.int32)
        dist.all_gather(list(b32.unbind(0)), pad.contiguous().view(torch.int32), group=group)
    else:
        dist.all_gather(list(buf.unbind(0)), pad.contiguous(), group=group)
    out = torch.empty((nq, n_heads, d), dtype=local.dtype, device=local.device)
    for r, (h0, h1) in enumerate(sizes):
        out[:, h0:h1] = buf[r, :, : h1 - h0]
    return out


def attention_sharded(q: torch.Tensor, cache_local, k_cur: torch.Tensor, v_cur: torch.Tensor,
                      softmax_scale: Optional[float] = None,
                      group: Optional[dist.ProcessGroup] = None) -> torch.Tensor:
    """Attention for the heads this rank owns, then the output all-gather.

    q, k_cur, v_cur: [N, H, d] (replicated); cache_local: DeviceChunks with the
    2*Hr planes (K, V per owned head) of this rank."""
    from . import device as D

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    H = q.shape[1]
    h0, h1 = head_range(H, world, rank)
    sl = lambda t: t[:, h0:h1].contiguous()
    local = D.attention(sl(q), cache_local, sl(k_cur), sl(v_cur), softmax_scale)
    return gather_heads(local, H, group)
