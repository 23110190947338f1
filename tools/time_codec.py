"""Time quantize / dequantize on the bench workload (no checks; A/B experiments)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2602_02958_b200 import device as D
dev = torch.device("cuda", 0)
wl = os.environ.get("WL", "self_forcing_10s")
cfg, x, dc, P_chunk, enc_ms = bench.build_cache(wl, 0, dev)
P, N, d = x.shape
qb, db = bench.plane_bytes(N, d, cfg)
payload = torch.empty_like(dc.payload); scales = torch.empty_like(dc.scales)
out = torch.empty((P, N, d), dtype=torch.bfloat16, device=dev)
status = torch.zeros(1, dtype=torch.int32, device=dev)
dq = D.DeviceChunks(cfg, N, d, dc.payload, dc.scales, dc.centroids, dc.assignments)
fq = lambda: D.quantize(x, cfg, dc.centroids, dc.assignments, payload=payload, scales=scales, check=False, status=status)
fd = lambda: D.dequantize(dq, out=out, check=False, status=status)
res = {}
for name, f, b in (("quantize", fq, qb), ("dequantize", fd, db)):
    ms = bench.time_ms(f, reps=10, warmup=3)
    res[name] = (round(ms, 3), round(P * b / ms / 1e6, 1))
ok = torch.equal(payload, dc.payload) and torch.equal(scales, dc.scales)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("QVG_")}, "res": res, "quant_ok": ok, "enc_ms": enc_ms[-1]}))
