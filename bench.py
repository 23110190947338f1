"""Benchmark of the QVG KV-cache hot path on B200.

Headline metric (BASELINE.json): KV quant+dequant GB/s (% HBM roofline);
quantized-attn latency vs bf16; KV compression.

Workload (configs[1], C2): the Self-Forcing / Wan2.1-1.3B-shaped KV cache of a
10 s rollout -- 30 layers x 12 heads x {K, V} x 14 chunks of 4680 tokens
(3 latent frames x 1560 tokens) = 10 080 planes of 4680 x 128 bf16 (12.1 GB),
QVG b=2, B=64, S=2, K=64.  One step = quantize every plane (given its stage
metadata, computed once by the on-device k-means before timing) + dequantize
every plane to bf16, each one kernel launch over the rank's planes.  Inputs
live in HBM and are ~100x the L2, so no flush is needed.

Data: the reference generator's planes (Q/datagen.py gen_clustered_stream,
restated bit-identically in paper_2602_02958_b200/datagen.py), SURVEY §8(d)
parameters: drift 0.1*sigma_within for C2/C4, K planes x10 / V planes x100 on
the outlier channels, rounded to bf16 -- the bf16 device input and the CPU
reference input are the same numbers.

Multi-GPU (python -m torch.distributed.run ... bench.py --gpus N): the fixed
cache is partitioned by (layer, head) pairs (shard.plane_pairs: 360 pairs,
45 per GPU at N = 8); stage seeds do not depend on the head (Q/prq.py:32-35),
so every rank's planes are bit-identical to the 1-GPU run.  No collective on
the data path; value = all ranks' bytes / max-over-ranks time ("strong").

python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2602_02958_b200 import datagen as G  # noqa: E402
from paper_2602_02958_b200 import device as D  # noqa: E402
from paper_2602_02958_b200.qvgcodec.metrics import memory_breakdown  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import ChunkSpec, QuantConfig  # noqa: E402
from paper_2602_02958_b200.shard import plane_pairs  # noqa: E402

METRIC = "KV quant+dequant GB/s (% HBM roofline); quantized-attn latency vs bf16; KV compression"
SIGMA_WITHIN = 0.125
WORKLOADS = {
    # name: (layers, heads, chunks, tokens per chunk, drift, config)
    "self_forcing_10s": (30, 12, 14, 4680, 0.1 * SIGMA_WITHIN,
                         dict(bits=2, group_size=64, stages=2, centroids=64)),
    "config1_cpu_case": (1, 12, 1, 4680, 0.0, dict(bits=2, group_size=64, stages=2, centroids=64)),
}
DATA = ("reference generator (Q/datagen.py gen_clustered_stream restated bit-identically in "
        "paper_2602_02958_b200/datagen.py), bf16-rounded, SURVEY 8(d) parameters")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            m = json.load(fh)
        return float(m["hbm_gbs"]), float(m["bf16_tflops"]), float(m.get("bf16_tflops_sustained", 0)), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def plane_bytes(N, d, cfg: QuantConfig, out_bytes_per_elem=2):
    """Algorithmic bytes of one plane: bf16 side + payload +
    scales + assignments + centroid tables."""
    S, K = cfg.stages, cfg.centroids
    meta = (N * d * cfg.bits + 7) // 8 + N * d // cfg.group_size + S * N + S * K * d * 2
    return N * d * 2 + meta, N * d * out_bytes_per_elem + meta


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6 and parts[0].isdigit():
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [int(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": int(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


def rank_refs(workload, world, rank):
    """This rank's planes, chunk-major: per chunk its (layer, head) pairs x {K, V}."""
    L, H, C, N, drift, _ = WORKLOADS[workload]
    pairs = plane_pairs(L, H, world, rank)
    per_chunk = [[G.PlaneRef(l, h, v, c) for (l, h) in pairs for v in (False, True)] for c in range(C)]
    return per_chunk


def host_planes(refs, n_heads, n_tokens, drift):
    """[P, N, d] bf16 bit patterns (uint16) from the reference generator."""
    return G.kv_cache_bf16(refs, n_heads, n_tokens, drift=drift)


def to_device_bf16(u16, dev):
    return torch.from_numpy(np.ascontiguousarray(u16).view(np.int16)).to(dev).view(torch.bfloat16)


def build_cache(workload, world, rank, device):
    """Generate this rank's planes of every chunk on the host, compress each
    chunk on the device (chunk_index = chunk number, Q/prq.py:49)."""
    L, H, C, N, drift, cfgd = WORKLOADS[workload]
    cfg = QuantConfig(**cfgd)
    per_chunk = rank_refs(workload, world, rank)
    t0 = time.perf_counter()
    host = host_planes([r for ch in per_chunk for r in ch], H, N, drift)
    gen_s = time.perf_counter() - t0
    Pc = len(per_chunk[0])
    x = torch.empty((Pc * C, N, 128), dtype=torch.bfloat16, device=device)
    chunks, enc_ms = [], []
    for c in range(C):
        x[c * Pc:(c + 1) * Pc] = to_device_bf16(host[c * Pc:(c + 1) * Pc], device)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dc = D.compress(x[c * Pc:(c + 1) * Pc], cfg, chunk_index=c, check=(c == 0))
        torch.cuda.synchronize()
        enc_ms.append((time.perf_counter() - t0) * 1e3)
        chunks.append(dc)
    cat = lambda f: torch.cat([getattr(dc, f) for dc in chunks])
    dc = D.DeviceChunks(cfg, N, 128, cat("payload"), cat("scales"), cat("centroids"), cat("assignments"))
    del chunks
    torch.cuda.empty_cache()
    return cfg, host, x, dc, Pc, enc_ms, gen_s


def time_ms(fn, reps=5, warmup=2):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def allmax(vals, dev, world):
    if world == 1:
        return vals
    t = torch.tensor([float(v) for v in vals], device=dev, dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def bench_attention(dev, rank, world, H=32, nc=38400, nq=7800, d=128):
    """LongCat-Video-shaped layer (configs[2], C3): 32 heads, 38 400-token
    cache (QVG b2 S1 K256 B64, reference-generator planes, drift 0), current
    chunk of 7 800 tokens attending to cache + itself.  Quantized-cache
    attention vs the same kernel on the bf16 cache and vs torch SDPA
    (cuDNN/flash, library comparator).  Under torchrun the heads are sharded
    over the ranks (shard.head_range, no collective on the hot path) and the
    per-rank outputs are all-gathered (NCCL on the GPU box); latencies are
    the max over ranks."""
    from paper_2602_02958_b200.shard import gather_heads, head_range

    h0, h1 = head_range(H, world, rank)
    Hr = h1 - h0
    cfg = QuantConfig(bits=2, group_size=64, stages=1, centroids=256)
    refs = [G.PlaneRef(0, h, v, 0) for h in range(h0, h1) for v in (False, True)]
    planes = to_device_bf16(host_planes(refs, H, nc, 0.0), dev)            # this rank's K, V planes
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    chunks = D.compress(planes, cfg, chunk_index=0)
    torch.cuda.synchronize()
    enc_s = time.perf_counter() - t0
    # LongCat codec throughput (this rank's planes, same kernels as the C2 leg)
    qb, db = plane_bytes(nc, d, cfg)
    Pl = planes.shape[0]
    pay, scl = torch.empty_like(chunks.payload), torch.empty_like(chunks.scales)
    rec = torch.empty_like(planes)
    stw = torch.zeros(1, dtype=torch.int32, device=dev)
    ms_qz = time_ms(lambda: D.quantize(planes, cfg, chunks.centroids, chunks.assignments, payload=pay, scales=scl,
                                       check=False, status=stw), reps=10, warmup=3)
    ms_dq = time_ms(lambda: D.dequantize(chunks, out=rec, check=False, status=stw), reps=10, warmup=3)
    codec_ok = torch.equal(pay, chunks.payload) and torch.equal(scl, chunks.scales)
    del pay, scl, rec
    ms_qz, ms_dq = allmax([ms_qz, ms_dq], dev, world)
    hbm = peaks()[0]
    codec = {"planes": Pl * world, "tokens_per_plane": nc, "quantize_ms": round(ms_qz, 3),
             "quantize_GBps": round(Pl * world * qb / ms_qz / 1e6, 1),
             "dequantize_ms": round(ms_dq, 3), "dequantize_GBps": round(Pl * world * db / ms_dq / 1e6, 1),
             "quant_dequant_GBps": round(Pl * world * (qb + db) / (ms_qz + ms_dq) / 1e6, 1),
             "quant_dequant_frac": round(Pl * world * (qb + db) / (ms_qz + ms_dq) / 1e6 / hbm, 4),
             "requantize_matches_compress": bool(codec_ok),
             "note": "quantize given the compress output's centroids / assignments; input 5x larger than L2"}
    g = torch.Generator(device=dev)
    g.manual_seed(12345)
    q = torch.randn((nq, H, d), generator=g, device=dev).to(torch.bfloat16)
    kc = torch.randn((nq, H, d), generator=g, device=dev).to(torch.bfloat16)
    vc = torch.randn((nq, H, d), generator=g, device=dev).to(torch.bfloat16)
    ql, kl, vl = (t[:, h0:h1].contiguous() for t in (q, kc, vc))
    out = torch.empty((nq, Hr, d), dtype=torch.bfloat16, device=dev)
    # interleaved rounds (clocks drift under a long tensor-bound load), median of each
    tb, tq = [], []
    for _ in range(5):
        tb.append(time_ms(lambda: D.attention(ql, None, kl, vl, kv_bf16=planes, out=out, check=False), reps=3, warmup=1))
        tq.append(time_ms(lambda: D.attention(ql, chunks, kl, vl, out=out, check=False), reps=3, warmup=1))
    ms_b, ms_q = float(np.median(tb)), float(np.median(tq))
    # the in-tile decode kernel (fused=True: codes / scales / centroids read
    # inside the attention kernel, no bf16 workspace) at the layer shape and at
    # a small-query "step" shape (256 queries per head against the full cache)
    ms_f = time_ms(lambda: D.attention(ql, chunks, kl, vl, out=out, fused=True, check=False), reps=3, warmup=1)
    nq_s = 256
    qs_, ks_, vs_ = ql[:nq_s].contiguous(), kl[:nq_s].contiguous(), vl[:nq_s].contiguous()
    out_s = torch.empty((nq_s, Hr, d), dtype=torch.bfloat16, device=dev)
    step = {"query_tokens": nq_s, "cur_tokens": nq_s,
            "latency_ms_quantized": time_ms(lambda: D.attention(qs_, chunks, ks_, vs_, out=out_s, check=False), reps=10),
            "latency_ms_quantized_fused": time_ms(lambda: D.attention(qs_, chunks, ks_, vs_, out=out_s, fused=True,
                                                                      check=False), reps=10),
            "latency_ms_bf16_same_kernel": time_ms(lambda: D.attention(qs_, None, ks_, vs_, kv_bf16=planes, out=out_s,
                                                                       check=False), reps=10)}
    ms_f, step["latency_ms_quantized"], step["latency_ms_quantized_fused"], step["latency_ms_bf16_same_kernel"] = allmax(
        [ms_f, step["latency_ms_quantized"], step["latency_ms_quantized_fused"], step["latency_ms_bf16_same_kernel"]],
        dev, world)
    step = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in step.items()}
    ms_g = None
    if world > 1:
        D.attention(ql, chunks, kl, vl, out=out)
        ms_g = time_ms(lambda: gather_heads(out, H))
    # library comparator: SDPA on the materialised bf16 [cache ; current] (layout prep untimed)
    kall = torch.cat([planes[0::2].permute(1, 0, 2), kl], 0).permute(1, 0, 2)[None].contiguous()
    vall = torch.cat([planes[1::2].permute(1, 0, 2), vl], 0).permute(1, 0, 2)[None].contiguous()
    qq = ql.permute(1, 0, 2)[None].contiguous()
    try:
        ms_sdpa = time_ms(lambda: torch.nn.functional.scaled_dot_product_attention(qq, kall, vall))
    except Exception:
        ms_sdpa = None
    ms_q, ms_b, ms_sdpa_m, ms_gm = allmax([ms_q, ms_b, ms_sdpa or 0.0, ms_g or 0.0], dev, world)
    ms_sdpa = ms_sdpa_m or None
    flops = 4.0 * nq * (nc + nq) * d * H          # whole layer, all ranks
    _, tf_peak, tf_sus, kind = peaks()
    res = {
        "workload": "longcat_layer", "heads": H, "heads_per_rank": Hr, "n_gpus": world,
        "cache_tokens": nc, "query_tokens": nq, "cur_tokens": nq, "config": "b2 S1 K256 B64",
        "latency_ms_quantized": round(ms_q, 3), "latency_ms_bf16_same_kernel": round(ms_b, 3),
        "latency_ms_quantized_fused": round(ms_f, 3),
        "latency_ms_torch_sdpa_bf16": None if not ms_sdpa else round(ms_sdpa, 3),
        "ratio_quantized_vs_bf16": round(ms_q / ms_b, 4),
        "ratio_quantized_vs_sdpa": None if not ms_sdpa else round(ms_q / ms_sdpa, 4),
        "tflops_quantized": round(flops / ms_q / 1e9, 1), "tflops_bf16": round(flops / ms_b / 1e9, 1),
        "roofline": {"bound": "tensor", "achieved": round(flops / ms_q / 1e9 / world, 1), "peak": tf_peak,
                     "unit": "TFLOP/s per GPU", "frac": round(flops / ms_q / 1e9 / world / tf_peak, 4),
                     "peak_kind": kind},
        "encode_s": round(enc_s, 3),
        "kv_compression": round(memory_breakdown(cfg, ChunkSpec(nc, d)).ratio_vs_bf16, 3),
        "codec": codec,
        "step_shape": step,
    }
    if world > 1:
        backend = torch.distributed.get_backend()
        res[f"allgather_ms_{backend}"] = round(ms_gm, 3)
        res["latency_ms_quantized_plus_gather"] = round(ms_q + ms_gm, 3)
    return res


def bench_stage_sweep(dev, rank, world, H=24, N=4680, chunks=(0, 1)):
    """C4 (HY-WorldPlay 60 s long-horizon cache, configs[3]): PRQ stage sweep
    S = 0..4 x B in {16, 64} on streaming 4680-token chunks (12 latent frames,
    PAPER.md:462) of one layer's 24 heads x {K, V} (builder's choice: HY-World
    / HunyuanVideo-class 24 heads x 128; layers and the 120-chunk rollout
    repeat this per-chunk workload).  Per (S, B): stage_mse_curve's MSE
    (Q/prq.py:135-172, mean over planes), memory ratio, device encode time.
    Heads are sharded over the ranks; MSE sums are reduced over ranks."""
    from paper_2602_02958_b200.shard import head_range

    h0, h1 = head_range(H, world, rank)
    refs = [G.PlaneRef(0, h, v, c) for c in chunks for h in range(h0, h1) for v in (False, True)]
    host = host_planes(refs, H, N, 0.1 * SIGMA_WITHIN)
    x = to_device_bf16(host, dev)
    P = x.shape[0] // len(chunks)
    xf = x.double()
    out = []
    for B in (16, 64):
        for S in range(0, 5):
            cfg = QuantConfig(bits=2, group_size=B, stages=S, centroids=64)
            se, n, enc = 0.0, 0, 0.0
            for ci, c in enumerate(chunks):
                xs = x[ci * P:(ci + 1) * P]
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                dc = D.compress(xs, cfg, chunk_index=c)
                torch.cuda.synchronize()
                enc += (time.perf_counter() - t0) * 1e3
                rec = D.dequantize(dc, torch.float32)
                se += float(((xf[ci * P:(ci + 1) * P] - rec.double()) ** 2).sum())
                n += rec.numel()
            t = torch.tensor([se, n], device=dev, dtype=torch.float64)
            if world > 1:
                torch.distributed.all_reduce(t)
            enc_ms = allmax([enc / len(chunks)], dev, world)[0]
            out.append({"B": B, "S": S, "mse": float(t[0] / t[1]),
                        "ratio": round(memory_breakdown(cfg, ChunkSpec(N, 128)).ratio_vs_bf16, 3),
                        "encode_ms_per_chunk": round(enc_ms, 2)})
    return {"workload": "hy_worldplay_stage_sweep", "heads": H, "layers_sampled": 1,
            "chunks": list(chunks), "tokens_per_chunk": N, "planes_per_chunk": 2 * H, "bits": 2,
            "centroids": 64, "drift": 0.1 * SIGMA_WITHIN, "curve": out}


def cpu_sample_gbs(x_s, cent_s, asg_s, cfg, threads, min_seconds=10.0, max_seconds=30.0):
    """Oracle (CPU port) quantize+dequantize of a plane sample, repeated to ~10 s."""
    import oracle

    P, N, d = x_s.shape
    qb, db = plane_bytes(N, d, cfg)
    reps, t0 = 0, time.perf_counter()
    while True:
        pay, sc = oracle.quantize_given_metas_batch(x_s, cent_s, asg_s, cfg.bits, cfg.group_size,
                                                    threads)
        oracle.prq_decompress_batch(pay, sc, cent_s, asg_s, N, d, cfg.bits, cfg.group_size, threads)
        reps += 1
        el = time.perf_counter() - t0
        if el >= min_seconds or el * (reps + 1) / reps > max_seconds:
            break
    return P * (qb + db) * reps / el / 1e9, el, reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="self_forcing_10s", choices=list(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-attention", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, world, rank)
    # one process per GPU; QVG_BENCH_BACKEND=gloo + device wrap-around lets the
    # N>1 path be exercised on a single GPU (tests), the real run uses NCCL
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("QVG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    hbm_peak, _, _, peak_kind = peaks()

    cfg, host, x, dc, P_chunk, enc_ms, gen_s = build_cache(args.workload, world, rank, dev)
    P, N, d = x.shape
    qb, db = plane_bytes(N, d, cfg)
    L, H, C, _, drift, _ = WORKLOADS[args.workload]
    P_total = L * H * 2 * C
    step_bytes_total = P_total * (qb + db)
    payload = torch.empty_like(dc.payload)
    scales = torch.empty_like(dc.scales)
    out = torch.empty((P, N, d), dtype=torch.bfloat16, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    dq = D.DeviceChunks(cfg, N, d, payload, scales, dc.centroids, dc.assignments)

    def step(ev=None):
        if ev:
            ev[0].record()
        D.quantize(x, cfg, dc.centroids, dc.assignments, payload=payload, scales=scales,
                   check=False, status=status)
        if ev:
            ev[1].record()
        D.dequantize(dq, out=out, check=False, status=status)
        if ev:
            ev[2].record()

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    D.check_status(status)
    # the quantize of the timed loop rewrites the same bytes compress produced
    assert torch.equal(payload, dc.payload) and torch.equal(scales, dc.scales)

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        start.record()
        for i in range(args.steps):
            step(evs[i])
        stop.record()
        torch.cuda.synchronize()
    ms = start.elapsed_time(stop)
    q_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in evs]))
    dq_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in evs]))
    ms, q_ms, dq_ms = allmax([ms, q_ms, dq_ms], dev, world)
    if world > 1:
        torch.distributed.barrier()
    ms_step = ms / args.steps
    value = step_bytes_total / (ms_step * 1e-3) / 1e9

    # per-kernel rates of this rank's launches (max-over-ranks times, the
    # largest rank's bytes: the roofline of the kernel as launched)
    kernels = {
        "quantize": {"ms": q_ms, "bytes": P * qb, "GBps": P * qb / q_ms / 1e6},
        "dequantize": {"ms": dq_ms, "bytes": P * db, "GBps": P * db / dq_ms / 1e6},
    }
    dom = max(kernels, key=lambda k: kernels[k]["ms"])
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh).get(args.workload, {})
        traffic = tr.get(dom)
    except Exception:
        pass
    achieved = kernels[dom]["GBps"]
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": hbm_peak,
                "unit": "GB/s", "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                "peak_kind": peak_kind,
                "per_kernel_frac": {k: round(v["GBps"] / hbm_peak, 4) for k, v in kernels.items()}}

    # streaming warm start (SURVEY 8(f) row 1, Q/prq.py:61-71): chunk 1 of the
    # drifting streams encoded from chunk 0's float64 centroids of the same
    # (layer, head, K|V) streams -- k-means++ skipped
    warm = None
    if P >= 2 * P_chunk:
        c0 = D.compress(x[:P_chunk], cfg, chunk_index=0, keep_f64=True, check=False)
        wms = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            cw = D.compress(x[P_chunk:2 * P_chunk], cfg, chunk_index=1, warm_init=c0.centroids_f64, check=False)
            torch.cuda.synchronize()
            wms.append((time.perf_counter() - t0) * 1e3)
            del cw
        del c0
        warm = float(np.median(wms))
    enc_chunk = float(np.median(enc_ms[1:] or enc_ms))
    enc_chunk, warm_m = allmax([enc_chunk, warm or 0.0], dev, world)
    warm = warm_m if warm is not None else None
    planes_per_chunk_total = L * H * 2

    result = {
        "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": f"synthetic: {DATA}",
        "config": {"workload": args.workload, "planes": P_total, "planes_per_rank": P,
                   "tokens_per_plane": N, "head_dim": d, "bits": cfg.bits, "group_size": cfg.group_size,
                   "stages": cfg.stages, "centroids": cfg.centroids, "drift": drift,
                   "bytes_per_step": step_bytes_total,
                   "parallelism": f"(layer, head) pairs partitioned over {world} rank(s) (strong)",
                   "l2": "inputs 100x larger than L2; no flush needed"},
        "roofline": roofline, "kernels": kernels,
        "kv_compression": round(memory_breakdown(cfg, ChunkSpec(N, d)).ratio_vs_bf16, 3),
        "encode": {"tokens_per_s": round(planes_per_chunk_total * N / (enc_chunk / 1e3), 1),
                   "ms_per_chunk": round(enc_chunk, 2), "planes_per_chunk": planes_per_chunk_total,
                   "planes_per_chunk_per_rank": P_chunk,
                   "note": "full prq_compress (k-means++ / Lloyd / smoothing / quantize), one chunk",
                   "warm_ms_per_chunk": None if warm is None else round(warm, 2),
                   "warm_tokens_per_s": None if warm is None else round(planes_per_chunk_total * N / (warm / 1e3), 1),
                   "warm_note": "streaming warm start: the previous chunk's float64 centroids of the "
                                "same drifting streams as init",
                   "host_datagen_s": round(gen_s, 1)},
        "gpu_launches": 2 * args.steps,
        "clocks": clk.summary(),
    }
    if not args.no_e2e:
        result["e2e"] = run_e2e(cfg, x[:P_chunk], dc.select(slice(0, P_chunk)), dev, world,
                                planes_total=planes_per_chunk_total)
    if rank == 0 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        ns = max(threads, 8)
        idx = np.arange(ns) * (P // ns)
        xs = G.bf16_bits_to_f32(host[idx])
        cs = dc.centroids[torch.from_numpy(idx).to(dev)].float().cpu().numpy()
        asg = dc.assignments[torch.from_numpy(idx).to(dev)].cpu().numpy()
        gbs, el, reps = cpu_sample_gbs(xs, cs, asg, cfg, threads)
        result["cpu_baseline"] = {
            "value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": f"oracle quantize+dequantize of {ns} of the same planes x {reps} reps ({el:.1f} s), "
                      f"same byte accounting"}
    del host
    if not args.no_attention or not args.no_sweep:
        del x, out, dq, payload, scales, dc
        torch.cuda.empty_cache()
    if not args.no_attention:
        result["attention"] = bench_attention(dev, rank, world)
    if not args.no_sweep:
        result["stage_sweep"] = bench_stage_sweep(dev, rank, world)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_e2e(cfg, x, dc, dev, world, planes_total, n_chunks=8):
    """Same metric through the public API with HOST buffers: pinned H2D of the
    bf16 planes and their stage metadata, quantize, D2H of the compressed
    chunk (payload + scales), dequantize it, D2H of the decoded bf16 planes —
    all inside the timed region.  The planes go through in `n_chunks` slices
    on three CUDA streams, so one slice's device->host copies overlap other
    slices' host->device copies and kernels (PCIe is full duplex).  One chunk
    of the cache (its planes split over the ranks); value = the chunk's
    bytes / max-over-ranks time."""
    P, N, d = x.shape
    xh = x.cpu().pin_memory()
    comp = [dc.payload, dc.scales, dc.centroids, dc.assignments]
    comp_h = [t.cpu().pin_memory() for t in comp]
    comp_d = [torch.empty_like(t) for t in comp]
    out_h = torch.empty((P, N, d), dtype=torch.bfloat16).pin_memory()
    xd = torch.empty_like(x)
    out_d = torch.empty_like(x)
    st = torch.zeros(1, dtype=torch.int32, device=dev)

    qb, db = plane_bytes(N, d, cfg)
    h2d = xh.numel() * 2 + sum(t.numel() * t.element_size() for t in comp_h[2:])
    d2h = out_h.numel() * 2 + comp_h[0].numel() + comp_h[1].numel()
    bounds = [P * i // n_chunks for i in range(n_chunks + 1)]
    streams = [torch.cuda.Stream(dev) for _ in range(3)]
    main = torch.cuda.current_stream(dev)

    def step():
        for s in streams:
            s.wait_stream(main)
        for i in range(n_chunks):
            lo, hi = bounds[i], bounds[i + 1]
            if hi == lo:
                continue
            with torch.cuda.stream(streams[i % len(streams)]):
                xd[lo:hi].copy_(xh[lo:hi], non_blocking=True)
                for a, b in zip(comp_d[2:], comp_h[2:]):
                    a[lo:hi].copy_(b[lo:hi], non_blocking=True)     # stage metadata of the slice
                D.quantize(xd[lo:hi], cfg, comp_d[2][lo:hi], comp_d[3][lo:hi], payload=comp_d[0][lo:hi],
                           scales=comp_d[1][lo:hi], check=False, status=st)
                comp_h[0][lo:hi].copy_(comp_d[0][lo:hi], non_blocking=True)
                comp_h[1][lo:hi].copy_(comp_d[1][lo:hi], non_blocking=True)
                D.dequantize(D.DeviceChunks(cfg, N, d, comp_d[0][lo:hi], comp_d[1][lo:hi],
                                            comp_d[2][lo:hi], comp_d[3][lo:hi]),
                             out=out_d[lo:hi], check=False, status=st)
                out_h[lo:hi].copy_(out_d[lo:hi], non_blocking=True)
        for s in streams:
            main.wait_stream(s)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    # the host copies hold the right bytes: compressed chunk == compress's, and
    # the decoded planes == the device dequantize of the same chunk
    assert torch.equal(comp_h[0], dc.payload.cpu()) and torch.equal(comp_h[1], dc.scales.cpu())
    ref = D.dequantize(dc.select(slice(0, 2)), out_dtype=torch.bfloat16).cpu()
    assert torch.equal(out_h[:2], ref)
    reps = 5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = allmax([e0.elapsed_time(e1) / reps], dev, world)[0]
    return {"value": round(planes_total * (qb + db) / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": round(ms, 3), "planes": planes_total, "planes_per_rank": P,
            "path": "paper_2602_02958_b200.device.quantize/dequantize (C ABI) on pinned host buffers, "
                    "8 slices on 3 streams (copies overlap across slices)"}


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path (oracle C port of the
    numpy reference; the Python reference cannot travel to the box) timed on
    the host cores, same metric / unit / byte accounting, each step one
    bounded sample of the workload: quantize + dequantize of the first
    planes of chunk 0 of the SAME reference-generator planes the GPU arm
    compresses, with their stage metadata from the oracle's own k-means
    (identical to the GPU's, parity-tested)."""
    if rank != 0:
        return
    import oracle

    L, H, C, N, drift, cfgd = WORKLOADS[args.workload]
    cfg = QuantConfig(**cfgd)
    threads = len(os.sched_getaffinity(0))
    ns = max(threads, 8)
    refs = rank_refs(args.workload, 1, 0)[0][:ns]
    x = G.bf16_bits_to_f32(host_planes(refs, H, N, drift))
    draws = np.stack([oracle.pp_draws(cfg.seed, 0, cfg.stages, cfg.centroids)] * ns)
    _, _, cent, asg, _ = oracle.prq_compress_batch(x, cfg.bits, cfg.group_size, cfg.stages,
                                                   cfg.centroids, cfg.kmeans_max_iters, cfg.kmeans_tol,
                                                   draws, threads)
    qb, db = plane_bytes(N, 128, cfg)
    times = []
    for i in range(max(args.warmup, 3) + args.steps):
        t0 = time.perf_counter()
        pay, sc = oracle.quantize_given_metas_batch(x, cent, asg, cfg.bits, cfg.group_size, threads)
        oracle.prq_decompress_batch(pay, sc, cent, asg, N, 128, cfg.bits, cfg.group_size, threads)
        if i >= max(args.warmup, 3):
            times.append(time.perf_counter() - t0)
    sec = float(np.sum(times))
    value = ns * (qb + db) * len(times) / sec / 1e9
    res = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
           "steps": args.steps, "warmup": max(args.warmup, 3),
           "ms_per_step": round(sec / len(times) * 1e3, 3), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64/f32 (reference numerics)",
           "data": f"synthetic: {DATA} (the GPU arm's chunk-0 planes)", "impl": "reference",
           "config": {"workload": args.workload, "sample_planes": ns, "tokens_per_plane": N,
                      "head_dim": 128, "drift": drift, **cfgd},
           "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads,
                            "kind": "port",
                            "sample": f"{ns} planes quantize+dequantize per step (oracle C port)"},
           "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
