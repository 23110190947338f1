"""Multi-process sharding logic on CPU (gloo, world size 2)."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_02958_b200.shard import gather_heads, head_range, kv_plane_index, plane_pairs


def test_head_range_partitions():
    for H in (1, 7, 12, 32):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                h0, h1 = head_range(H, world, r)
                seen.extend(range(h0, h1))
            assert seen == list(range(H))
    pairs = [p for r in range(8) for p in plane_pairs(30, 12, 8, r)]
    assert len(pairs) == 360 and len(set(pairs)) == 360
    assert all(len(plane_pairs(30, 12, 8, r)) == 45 for r in range(8))
    assert kv_plane_index(1, 2, 12, 1) == 2 * (12 + 2) + 1


def _worker(rank, world, port, H, ret, dtype=torch.float32):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.manual_seed(0)
    full = torch.randn(5, H, 16).to(dtype)           # what a 1-GPU run would produce
    h0, h1 = head_range(H, world, rank)
    local = full[:, h0:h1].clone()                   # this rank's heads
    out = gather_heads(local, H)
    ret[rank] = bool(torch.equal(out, full))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("H,dtype", [(4, torch.float32), (5, torch.float32), (5, torch.bfloat16)])
def test_gather_heads_gloo_world2(H, dtype):
    world = 2
    port = 29500 + H + (7 if dtype == torch.bfloat16 else 0) + os.getpid() % 1000
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, port, H, ret, dtype), nprocs=world, join=True)
    assert ret[0] and ret[1]
