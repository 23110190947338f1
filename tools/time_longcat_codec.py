"""Time quantize / dequantize on the LongCat layer's 64 planes (b2 S1 K256 B64),
as in bench.bench_attention's codec block (A/B runs and ncu captures)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2602_02958_b200 import datagen as G
from paper_2602_02958_b200 import device as D
from paper_2602_02958_b200.qvgcodec.types import QuantConfig
dev = torch.device("cuda", 0)
H, nc, d = 32, 38400, 128
cfg = QuantConfig(bits=2, group_size=64, stages=1, centroids=256)
refs = [G.PlaneRef(0, h, v, 0) for h in range(H) for v in (False, True)]
planes = bench.to_device_bf16(bench.host_planes(refs, H, nc, 0.0), dev)
chunks = D.compress(planes, cfg, chunk_index=0)
qb, db = bench.plane_bytes(nc, d, cfg)
pay, scl = torch.empty_like(chunks.payload), torch.empty_like(chunks.scales)
rec = torch.empty_like(planes)
st = torch.zeros(1, dtype=torch.int32, device=dev)
fq = lambda: D.quantize(planes, cfg, chunks.centroids, chunks.assignments, payload=pay, scales=scl, check=False, status=st)
fd = lambda: D.dequantize(chunks, out=rec, check=False, status=st)
res = {}
for name, f, b in (("quantize", fq, qb), ("dequantize", fd, db)):
    ms = bench.time_ms(f, reps=10, warmup=3)
    res[name] = (round(ms, 4), round(64 * b / ms / 1e6, 1))
print(json.dumps({"res": res, "ok": torch.equal(pay, chunks.payload) and torch.equal(scl, chunks.scales)}))
