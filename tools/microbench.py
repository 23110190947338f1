"""BASELINE config 5 microbench (C5): tokens 4K..256K (7 points) x centroids
16..256 (5 points) x bits 2/4, d = 128, B = 64, S = 1, on the reference
generator's planes (drift 0, K/V outlier scales as SURVEY 8(d)).  For each
point: P planes so that P*N ~ 8M tokens,
full encode (k-means + PRQ) tokens/s, quantize and dequantize GB/s with the
same algorithmic byte accounting as bench.py (roofline fraction vs the
measured HBM copy peak).  Writes one JSON document to stdout."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_02958_b200 import device as D  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import QuantConfig  # noqa: E402
from paper_2602_02958_b200 import datagen as G  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    hbm, _, _, kind = bench.peaks()
    points = []
    Ns = [int(v) for v in os.environ.get("MB_N", "4096,8192,16384,32768,65536,131072,262144").split(",")]
    Ks = [int(v) for v in os.environ.get("MB_K", "16,32,64,128,256").split(",")]
    for N in Ns:
        P = max(2, (8 << 20) // N)
        refs = [G.PlaneRef(0, h, v, 0) for h in range(P // 2) for v in (False, True)]
        xh = G.kv_cache_bf16(refs, P // 2, N)
        x = bench.to_device_bf16(xh, dev)
        del xh
        for K in Ks:
            for bits in (2, 4):
                cfg = QuantConfig(bits=bits, group_size=64, stages=int(os.environ.get("MB_S", "1")), centroids=K)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                dc = D.compress(x, cfg, chunk_index=0)
                torch.cuda.synchronize()
                enc = time.perf_counter() - t0
                pay, sc = torch.empty_like(dc.payload), torch.empty_like(dc.scales)
                out = torch.empty_like(x)
                st = torch.zeros(1, dtype=torch.int32, device=dev)
                qb, db = bench.plane_bytes(N, 128, cfg)
                tq = bench.time_ms(lambda: D.quantize(x, cfg, dc.centroids, dc.assignments, payload=pay, scales=sc,
                                                      check=False, status=st), reps=10, warmup=3)
                td = bench.time_ms(lambda: D.dequantize(dc, out=out, check=False, status=st), reps=10, warmup=3)
                pt = {"N": N, "K": K, "bits": bits, "planes": P,
                      "encode_tokens_per_s": round(P * N / enc, 1),
                      "quantize_GBps": round(P * qb / tq / 1e6, 1), "dequantize_GBps": round(P * db / td / 1e6, 1),
                      "quant_dequant_GBps": round(P * (qb + db) / (tq + td) / 1e6, 1)}
                pt["hbm_frac"] = round(pt["quant_dequant_GBps"] / hbm, 4)
                points.append(pt)
                print(json.dumps(pt), file=sys.stderr, flush=True)
                del dc, pay, sc, out
                torch.cuda.empty_cache()
        del x
    print(json.dumps({"config": "BASELINE configs[4] microbench, d=128 B=64 S=1, reference-generator planes", "hbm_peak_GBps": hbm,
                      "peak_kind": kind, "points": points}))


if __name__ == "__main__":
    main()
