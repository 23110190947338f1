"""Time quantize / dequantize on the bench workload shape (A/B experiments).

The bench cache is 14 chunks of the reference generator's planes; for quick
A/B runs this tiles the first TC chunks (default 2) up to the full 10 080
planes -- same data statistics, ~1/7 of the host generation time."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2602_02958_b200 import device as D
dev = torch.device("cuda", 0)
wl = os.environ.get("WL", "self_forcing_10s")
tc = int(os.environ.get("TC", "2"))
L, H, C, N, drift, cfgd = bench.WORKLOADS[wl]
bench.WORKLOADS[wl] = (L, H, min(tc, C), N, drift, cfgd)
cfg, host, x0, dc0, P_chunk, enc_ms, _ = bench.build_cache(wl, 1, 0, dev)
del host
rep = (C + tc - 1) // tc
P = C * P_chunk
x = x0.repeat(rep, 1, 1)[:P].contiguous()
dc = D.DeviceChunks(cfg, N, 128, *(t.repeat(rep, *([1] * (t.dim() - 1)))[:P].contiguous()
                                   for t in (dc0.payload, dc0.scales, dc0.centroids, dc0.assignments)))
del x0, dc0
qb, db = bench.plane_bytes(N, 128, cfg)
payload = torch.empty_like(dc.payload); scales = torch.empty_like(dc.scales)
out = torch.empty((P, N, 128), dtype=torch.bfloat16, device=dev)
status = torch.zeros(1, dtype=torch.int32, device=dev)
dq = D.DeviceChunks(cfg, N, 128, dc.payload, dc.scales, dc.centroids, dc.assignments)
fq = lambda: D.quantize(x, cfg, dc.centroids, dc.assignments, payload=payload, scales=scales, check=False, status=status)
fd = lambda: D.dequantize(dq, out=out, check=False, status=status)
res = {}
for name, f, b in (("quantize", fq, qb), ("dequantize", fd, db)):
    ms = bench.time_ms(f, reps=10, warmup=3)
    res[name] = (round(ms, 3), round(P * b / ms / 1e6, 1))
ok = torch.equal(payload, dc.payload) and torch.equal(scales, dc.scales)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("QVG_")}, "res": res,
                  "quant_ok": ok, "enc_ms": enc_ms[-1], "planes": P}))
