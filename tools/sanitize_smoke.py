"""One small invocation of every pipelined kernel, for compute-sanitizer
(racecheck / synccheck / memcheck) runs:
    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py
Shapes are small but take the same code paths as the bench: the persistent
ring quantize (>= 148 planes), the stream dequantize,
k-means++ / tensor-core assignment / Lloyd inside compress, attention (TMA,
tcgen05), container record pack/unpack."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_02958_b200 import datagen as G  # noqa: E402
from paper_2602_02958_b200 import device as D  # noqa: E402
from paper_2602_02958_b200.qvgcodec import container as C  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import QuantConfig  # noqa: E402

dev = torch.device("cuda", 0)
which = set((os.environ.get("SAN_ONLY") or "compress,codec,attention,container").split(","))


def planes(P, N, chunk=0):
    refs = [G.PlaneRef(0, h, v, chunk) for h in range(P // 2) for v in (False, True)]
    return torch.from_numpy(G.kv_cache_bf16(refs, P // 2, N, workers=8).view(np.int16)).to(dev).view(torch.bfloat16)


cfg = QuantConfig(bits=2, group_size=64, stages=2, centroids=16)
if "compress" in which:
    x = planes(4, 512)
    dc = D.compress(x, cfg, chunk_index=0)
    torch.cuda.synchronize()
    print("compress ok", flush=True)
if "codec_q" in which:
    # the persistent codec kernels on random stage metadata (no k-means: memcheck-sized)
    P, N = 152, 256
    x = planes(P, N)
    g = torch.Generator(device=dev).manual_seed(3)
    cent = (torch.randn((P, 2, 16, 128), generator=g, device=dev) * 2).to(torch.bfloat16)
    asg = torch.randint(0, 16, (P, 2, N), generator=g, device=dev, dtype=torch.uint8)
    pay, sc = D.quantize(x, cfg, cent, asg)
    out = D.dequantize(D.DeviceChunks(cfg, N, 128, pay, sc, cent, asg), torch.bfloat16)
    torch.cuda.synchronize()
    print("codec_q ok", flush=True)
if "codec" in which:
    x = planes(152, 256)                      # >= 148 planes: persistent kernels
    dc = D.compress(x, cfg, chunk_index=0)
    pay, sc = D.quantize(x, cfg, dc.centroids, dc.assignments)
    out = D.dequantize(dc, torch.bfloat16)
    torch.cuda.synchronize()
    assert torch.equal(pay, dc.payload) and torch.equal(sc, dc.scales)
    print("codec ok", flush=True)
if "attention" in which:
    H, nc, nq = 2, 512, 256
    x = planes(2 * H, nc)
    c1 = QuantConfig(bits=2, group_size=64, stages=1, centroids=16)
    dc = D.compress(x, c1, chunk_index=0)
    g = torch.Generator(device=dev).manual_seed(1)
    q, k, v = (torch.randn((nq, H, 128), generator=g, device=dev).to(torch.bfloat16) for _ in range(3))
    o = D.attention(q, dc, k, v)
    torch.cuda.synchronize()
    print("attention ok", flush=True)
if "container" in which:
    x = planes(4, 256)
    dc = D.compress(x, cfg, chunk_index=0)
    h = C.QvgcHeader.for_config(cfg, 128)
    recs = C.pack_records(dc, h, 0)
    back, ok = C.unpack_records(recs, h, 256)
    torch.cuda.synchronize()
    assert bool((ok == 1).all())
    print("container ok", flush=True)
