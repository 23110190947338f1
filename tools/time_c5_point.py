"""One C5 point (env N, K, BITS, S): quantize / dequantize of the reference
generator's planes given their compress metadata (ncu captures, A/B runs)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2602_02958_b200 import device as D
from paper_2602_02958_b200 import datagen as G
from paper_2602_02958_b200.qvgcodec.types import QuantConfig
dev = torch.device("cuda", 0)
N, K = int(os.environ.get("N", "65536")), int(os.environ.get("K", "16"))
bits, S = int(os.environ.get("BITS", "2")), int(os.environ.get("S", "1"))
P = max(2, (8 << 20) // N)
refs = [G.PlaneRef(0, h, v, 0) for h in range(P // 2) for v in (False, True)]
x = bench.to_device_bf16(G.kv_cache_bf16(refs, P // 2, N), dev)
cfg = QuantConfig(bits=bits, group_size=64, stages=S, centroids=K)
dc = D.compress(x, cfg, chunk_index=0)
qb, db = bench.plane_bytes(N, 128, cfg)
st = torch.zeros(1, dtype=torch.int32, device=dev)
pay, sc = torch.empty_like(dc.payload), torch.empty_like(dc.scales)
out = torch.empty_like(x)
fq = lambda: D.quantize(x, cfg, dc.centroids, dc.assignments, payload=pay, scales=sc, check=False, status=st)
fd = lambda: D.dequantize(dc, out=out, check=False, status=st)
res = {n: round(P * b / bench.time_ms(f, reps=10, warmup=3) / 1e6, 1) for n, f, b in (("q", fq, qb), ("d", fd, db))}
print(json.dumps({"N": N, "K": K, "bits": bits, "S": S, "GBps": res}))
