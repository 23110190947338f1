"""Partitioned codec + head-sharded attention on 2 ranks (gloo) sharing one GPU.

SURVEY §8(e): every (layer, head, K|V) plane is independent and stage seeds do
not depend on the head (Q/prq.py:32-35,49), so a rank that owns a subset of
(layer, head) pairs (shard.plane_pairs) must produce byte-identical payload,
scales, centroids, assignments and reconstructions to the 1-rank run, and the
head-sharded attention gathered over the ranks must equal the 1-rank output.
The 2-rank bench (torchrun, gloo) must run its strong-scaling codec leg.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L, H, N, NQ, D_ = 2, 3, 640, 96, 128


def _cfg():
    from paper_2602_02958_b200.qvgcodec.types import QuantConfig

    return QuantConfig(bits=2, group_size=64, stages=2, centroids=16)


def _run_shard(pairs, dev):
    """compress + f32 dequantize of the planes of `pairs` (chunk 1, drifting streams)."""
    from paper_2602_02958_b200 import datagen as G
    from paper_2602_02958_b200 import device as D

    refs = [G.PlaneRef(l, h, v, 1) for (l, h) in pairs for v in (False, True)]
    xh = G.kv_cache_bf16(refs, H, N, drift=0.0125, workers=1)
    x = torch.from_numpy(np.ascontiguousarray(xh).view(np.int16)).to(dev).view(torch.bfloat16)
    dc = D.compress(x, _cfg(), chunk_index=1)
    rec = D.dequantize(dc, torch.float32)
    raw = lambda t: (t.view(torch.int16) if t.dtype == torch.bfloat16 else t).cpu().numpy()
    return {k: raw(getattr(dc, k)) for k in ("payload", "scales", "centroids", "assignments")} | {
        "rec": rec.cpu().numpy(), "x": x}


def _attention(dev, cache_x, h0, h1):
    """LongCat-style layer attention for heads [h0, h1): cache planes of layer 0."""
    from paper_2602_02958_b200 import device as D

    g = torch.Generator(device=dev)
    g.manual_seed(12345)
    q = torch.randn((NQ, H, D_), generator=g, device=dev).to(torch.bfloat16)
    kc = torch.randn((NQ, H, D_), generator=g, device=dev).to(torch.bfloat16)
    vc = torch.randn((NQ, H, D_), generator=g, device=dev).to(torch.bfloat16)
    cfg = _cfg()
    chunks = D.compress(cache_x.contiguous(), cfg, chunk_index=1)
    sl = lambda t: t[:, h0:h1].contiguous()
    return D.attention(sl(q), chunks, sl(kc), sl(vc))


def _worker(rank, world, port, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, ROOT)
    from paper_2602_02958_b200.shard import gather_heads, head_range, plane_pairs

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    pairs = plane_pairs(L, H, world, rank)
    r = _run_shard(pairs, dev)
    objs = [None] * world
    dist.all_gather_object(objs, {"pairs": pairs, **{k: v for k, v in r.items() if k != "x"}})
    # head-sharded attention over layer 0's planes (each rank generates its heads)
    h0, h1 = head_range(H, world, rank)
    lp = _run_shard([(0, h) for h in range(h0, h1)], dev)["x"]
    out = _attention(dev, lp, h0, h1).cpu()
    full = gather_heads(out, H)
    if rank == 0:
        ret["shards"] = objs
        ret["attn"] = full.view(torch.int16).numpy()
    dist.barrier()
    dist.destroy_process_group()


def test_partitioned_codec_and_sharded_attention_match_one_rank():
    sys.path.insert(0, ROOT)
    from paper_2602_02958_b200.shard import plane_pairs

    world = 2
    mgr = mp.Manager()
    ret = mgr.dict()
    port = 29700 + os.getpid() % 500
    mp.spawn(_worker, args=(world, port, ret), nprocs=world, join=True)
    dev = torch.device("cuda", 0)
    full_pairs = plane_pairs(L, H, 1, 0)
    full = _run_shard(full_pairs, dev)
    shards = ret["shards"]
    assert [p for s in shards for p in s["pairs"]] == full_pairs
    for k in ("payload", "scales", "centroids", "assignments", "rec"):
        got = np.concatenate([s[k] for s in shards])
        assert got.shape == full[k].shape, k
        assert np.array_equal(got.view(np.uint8), full[k].view(np.uint8)), f"{k} differs from the 1-rank run"
    one = _attention(dev, _run_shard([(0, h) for h in range(H)], dev)["x"], 0, H).cpu().view(torch.int16).numpy()
    assert np.array_equal(ret["attn"], one), "gathered head-sharded attention differs from the 1-rank run"


def test_bench_two_ranks_strong_scaling():
    env = dict(os.environ, QVG_BENCH_BACKEND="gloo", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29900 + os.getpid() % 90),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--workload", "config1_cpu_case", "--no-cpu-baseline", "--no-e2e", "--no-sweep",
           "--no-attention"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    line = [ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1]
    r = json.loads(line)
    assert r["n_gpus"] == 2 and r["scaling"] == "strong"
    assert r["config"]["planes"] == 24 and r["config"]["planes_per_rank"] == 12
    assert r["value"] > 0
