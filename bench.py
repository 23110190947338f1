"""Benchmark of the QVG KV-cache hot path on B200.

Headline metric (BASELINE.json): KV quant+dequant GB/s (% HBM roofline);
quantized-attn latency vs bf16; KV compression.

Workload (N=1, configs[1]): the Self-Forcing / Wan2.1-1.3B-shaped KV cache of
a 10 s rollout — 30 layers x 12 heads x {K, V} x 14 chunks of 4680 tokens
(3 latent frames x 1560 tokens) = 10 080 planes of 4680 x 128 bf16
(12.1 GB), QVG b=2, B=64, S=2, K=64.  One step = quantize every plane
(given its stage metadata, computed once by the on-device k-means before
timing) + dequantize every plane to bf16, each one kernel launch over the
whole cache.  Inputs live in HBM and are ~100x the L2, so no flush is
needed.  Synthetic clustered data (paper_2602_02958_b200/synth.py).

python bench.py [--gpus N --steps K --warmup W] [--impl reference]
Under torchrun each rank runs its own cache (weak scaling, no collective on
the data path); rank 0 prints one JSON line.
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

from paper_2602_02958_b200 import device as D  # noqa: E402
from paper_2602_02958_b200.qvgcodec.metrics import memory_breakdown  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import ChunkSpec, QuantConfig  # noqa: E402
from paper_2602_02958_b200.synth import kv_cache_planes  # noqa: E402

METRIC = "KV quant+dequant GB/s (% HBM roofline); quantized-attn latency vs bf16; KV compression"
WORKLOADS = {
    # name: (layers, heads, chunks, tokens per chunk, config)
    "self_forcing_10s": (30, 12, 14, 4680, dict(bits=2, group_size=64, stages=2, centroids=64)),
    "config1_cpu_case": (1, 12, 1, 4680, dict(bits=2, group_size=64, stages=2, centroids=64)),
}


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


def build_cache(workload, rank, device):
    L, H, C, N, cfgd = WORKLOADS[workload]
    cfg = QuantConfig(**cfgd)
    P_chunk = L * H * 2
    xs, chunks, enc_ms = [], [], []
    for c in range(C):
        x = kv_cache_planes(L, H, N, 128, seed=1000 * rank + c, device=device)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dc = D.compress(x, cfg, chunk_index=c, check=(c == 0))
        torch.cuda.synchronize()
        enc_ms.append((time.perf_counter() - t0) * 1e3)
        xs.append(x)
        chunks.append(dc)
    x = torch.cat(xs)
    del xs
    cat = lambda f: torch.cat([getattr(dc, f) for dc in chunks])
    dc = D.DeviceChunks(cfg, N, 128, cat("payload"), cat("scales"), cat("centroids"),
                        cat("assignments"))
    del chunks
    torch.cuda.empty_cache()
    return cfg, x, dc, P_chunk, enc_ms


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


def bench_attention(dev, rank, world=1, H=32, nc=38400, nq=7800, d=128):
    """LongCat-Video-shaped layer (configs[2]): 32 heads, ~38K-token cache
    (QVG b2 S1 K256 B64), current chunk of 7800 tokens attending to cache +
    itself.  Quantized-cache attention vs the same kernel on the bf16 cache
    and vs torch SDPA (cuDNN/flash, library comparator).  Under torchrun the
    heads are sharded over the ranks (shard.head_range, no collective on the
    hot path) and the per-rank outputs are all-gathered over NCCL; latencies
    are the max over ranks."""
    from paper_2602_02958_b200.shard import gather_heads, head_range

    h0, h1 = head_range(H, world, rank)
    Hr = h1 - h0
    cfg = QuantConfig(bits=2, group_size=64, stages=1, centroids=256)
    planes = kv_cache_planes(1, H, nc, d, seed=77, device=dev)[2 * h0:2 * h1].contiguous()  # this rank's K,V
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    chunks = D.compress(planes, cfg, chunk_index=0)
    torch.cuda.synchronize()
    enc_s = time.perf_counter() - t0
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
        tb.append(time_ms(lambda: D.attention(ql, None, kl, vl, kv_bf16=planes, out=out), reps=3, warmup=1))
        tq.append(time_ms(lambda: D.attention(ql, chunks, kl, vl, out=out), reps=3, warmup=1))
    ms_b, ms_q = float(np.median(tb)), float(np.median(tq))
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
    if world > 1:
        t = torch.tensor([ms_q, ms_b, ms_sdpa or 0.0, ms_g], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_q, ms_b, ms_sdpa, ms_g = (float(v) for v in t.tolist())
    flops = 4.0 * nq * (nc + nq) * d * H          # whole layer, all ranks
    _, tf_peak, tf_sus, kind = peaks()
    res = {
        "workload": "longcat_layer", "heads": H, "heads_per_rank": Hr, "n_gpus": world,
        "cache_tokens": nc, "query_tokens": nq, "cur_tokens": nq, "config": "b2 S1 K256 B64",
        "latency_ms_quantized": round(ms_q, 3), "latency_ms_bf16_same_kernel": round(ms_b, 3),
        "latency_ms_torch_sdpa_bf16": None if not ms_sdpa else round(ms_sdpa, 3),
        "ratio_quantized_vs_bf16": round(ms_q / ms_b, 4),
        "ratio_quantized_vs_sdpa": None if not ms_sdpa else round(ms_q / ms_sdpa, 4),
        "tflops_quantized": round(flops / ms_q / 1e9, 1), "tflops_bf16": round(flops / ms_b / 1e9, 1),
        "roofline": {"bound": "tensor", "achieved": round(flops / ms_q / 1e9 / world, 1), "peak": tf_peak,
                     "unit": "TFLOP/s per GPU", "frac": round(flops / ms_q / 1e9 / world / tf_peak, 4),
                     "peak_kind": kind},
        "encode_s": round(enc_s, 3),
        "kv_compression": round(memory_breakdown(cfg, ChunkSpec(nc, d)).ratio_vs_bf16, 3),
    }
    if ms_g is not None:
        res["allgather_ms_nccl"] = round(ms_g, 3)
        res["latency_ms_quantized_plus_gather"] = round(ms_q + ms_g, 3)
    return res


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

    cfg, x, dc, P_chunk, enc_ms = build_cache(args.workload, rank, dev)
    P, N, d = x.shape
    qb, db = plane_bytes(N, d, cfg)
    step_bytes = P * (qb + db)
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
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()
    q_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in evs]))
    dq_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in evs]))
    ms_step = ms / args.steps
    value = world * step_bytes / (ms_step * 1e-3) / 1e9

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

    # streaming warm start (SURVEY 8(f) row 1, Q/prq.py:61-71): chunk 1 encoded
    # from chunk 0's float64 centroids of the same planes -- k-means++ skipped
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

    result = {
        "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (clustered bf16 K/V planes, random-init; paper_2602_02958_b200/synth.py)",
        "config": {"workload": args.workload, "planes": P, "tokens_per_plane": N, "head_dim": d,
                   "bits": cfg.bits, "group_size": cfg.group_size, "stages": cfg.stages,
                   "centroids": cfg.centroids, "bytes_per_step": step_bytes,
                   "parallelism": f"planes-per-rank x{world} (weak)",
                   "l2": "inputs 100x larger than L2; no flush needed"},
        "roofline": roofline, "kernels": kernels,
        "kv_compression": round(memory_breakdown(cfg, ChunkSpec(N, d)).ratio_vs_bf16, 3),
        "encode": {"tokens_per_s": round(P_chunk * N / (np.median(enc_ms[1:] or enc_ms) / 1e3), 1),
                   "ms_per_chunk": round(float(np.median(enc_ms[1:] or enc_ms)), 2),
                   "planes_per_chunk": P_chunk,
                   "note": "full prq_compress (k-means++ / Lloyd / smoothing / quantize), one chunk",
                   "warm_ms_per_chunk": None if warm is None else round(warm, 2),
                   "warm_tokens_per_s": None if warm is None else round(P_chunk * N / (warm / 1e3), 1),
                   "warm_note": "streaming warm start: the previous chunk's float64 centroids as init"},
        "gpu_launches": 2 * args.steps,
        "clocks": clk.summary(),
    }
    if not args.no_e2e:
        result["e2e"] = run_e2e(cfg, x[:P_chunk], dc.select(slice(0, P_chunk)), dev, world)
    if rank == 0 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        ns = max(threads, 8)
        idx = torch.arange(ns) * (P // ns)
        xs = x[idx].float().cpu().numpy()
        cs = dc.centroids[idx].float().cpu().numpy()
        asg = dc.assignments[idx].cpu().numpy()
        gbs, el, reps = cpu_sample_gbs(xs, cs, asg, cfg, threads)
        result["cpu_baseline"] = {
            "value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": f"oracle quantize+dequantize of {ns} planes x {reps} reps ({el:.1f} s), "
                      f"same byte accounting"}
    if not args.no_attention:
        del x, out, dq, payload, scales, dc
        torch.cuda.empty_cache()
        result["attention"] = bench_attention(dev, rank, world)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_e2e(cfg, x, dc, dev, world, n_chunks=8):
    """Same metric through the public API with HOST buffers: pinned H2D of the
    bf16 planes and their stage metadata, quantize, D2H of the compressed
    chunk (payload + scales), dequantize it, D2H of the decoded bf16 planes —
    all inside the timed region.  The planes go through in `n_chunks` slices
    on three CUDA streams, so one slice's device->host copies overlap other
    slices' host->device copies and kernels (PCIe is full duplex)."""
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
    ms = e0.elapsed_time(e1) / reps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": round(world * P * (qb + db) / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": round(ms, 3), "planes": P,
            "path": "paper_2602_02958_b200.device.quantize/dequantize (C ABI) on pinned host buffers, "
                "8 slices on 3 streams (copies overlap across slices)"}


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path (oracle C port of the
    numpy reference; the Python reference cannot travel to the box) timed on
    the host cores, same metric / unit / byte accounting, each step one
    bounded sample of the workload (quantize + dequantize of sampled planes,
    stage metadata from the oracle's own k-means)."""
    if rank != 0:
        return
    import oracle

    L, H, C, N, cfgd = WORKLOADS[args.workload]
    cfg = QuantConfig(**cfgd)
    threads = len(os.sched_getaffinity(0))
    ns = max(threads, 8)
    rng = np.random.default_rng(0)
    # clustered planes on the host (same generator family as synth.py)
    means = rng.normal(0, 2.5, size=(ns, 256, 128))
    asg0 = rng.integers(0, 256, size=(ns, N))
    x = np.take_along_axis(means, asg0[:, :, None], 1) + rng.normal(0, 0.125, size=(ns, N, 128))
    x[:, :, ::16] *= np.where(np.arange(ns) % 2 == 0, 10.0, 100.0)[:, None, None]
    x = (x.astype(np.float32).view(np.uint32) & 0xFFFF0000).view(np.float32)
    draws = np.stack([oracle.pp_draws(0, 0, cfg.stages, cfg.centroids)] * ns)
    _, _, cent, asg, _ = oracle.prq_compress_batch(x, cfg.bits, cfg.group_size, cfg.stages,
                                                   cfg.centroids, 10, 1e-4, draws, threads)
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
           "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32 (reference numerics)",
           "data": "synthetic clustered planes (host)", "impl": "reference",
           "config": {"workload": args.workload, "sample_planes": ns, "tokens_per_plane": N,
                      "head_dim": 128, **cfgd},
           "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads,
                            "kind": "port",
                            "sample": f"{ns} planes quantize+dequantize per step (oracle C port)"},
           "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
