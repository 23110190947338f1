"""Re-run tests/test_gpu_random_configs.py::test_random_attention_vs_oracle
cases (seeds on the command line) and print the configuration and the errors
against the fp64 oracle on the f32 and on the bf16-rounded reconstruction,
plus the element-wise bound |O - O_ref| / (softmax |V|)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))   # repo root (this file: tests/)
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2602_02958_b200 import device as D  # noqa: E402
from paper_2602_02958_b200.qvgcodec.lowprec import round_to_bf16  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import QuantConfig  # noqa: E402
from paper_2602_02958_b200.synth import clustered_planes  # noqa: E402

oracle.build()


def softmax_abs(q, k, v, scale):
    """fp64 softmax(q k^T scale) |v| per head: the natural scale of the bf16-P error."""
    H = q.shape[1]
    out = np.zeros(q.shape)
    for h in range(H):
        s = q[:, h, :] @ k[h].T * scale
        s -= s.max(axis=1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(axis=1, keepdims=True)
        out[:, h, :] = p @ np.abs(v[h])
    return out


for seed in [int(a) for a in sys.argv[1:]]:
    rng = np.random.default_rng(9000 + seed)
    H, d = int(rng.integers(1, 4)), 128
    nq = int(rng.integers(1, 300))
    nc = int(rng.choice([0, int(rng.integers(1, 700))]))
    ncur = int(rng.integers(0 if nc else 1, 260))
    cfg = QuantConfig(bits=int(rng.choice([2, 4])), group_size=int(rng.choice([32, 64])),
                      stages=int(rng.integers(1, 3)), centroids=int(rng.choice([8, 16])))
    fused = bool(rng.integers(0, 2))
    scale = float(rng.choice([d ** -0.5, 0.3]))
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = (torch.randn((nq, H, d), generator=g, device="cuda") * 0.5).to(torch.bfloat16)
    kc = torch.randn((ncur, H, d), generator=g, device="cuda").to(torch.bfloat16)
    vc = torch.randn((ncur, H, d), generator=g, device="cuda").to(torch.bfloat16)
    planes = clustered_planes(2 * H, nc, d, n_clusters=8, outlier_scale=4.0, seed=seed)
    chunks = D.compress(planes, cfg)
    res = {}
    for fz in (False, True):
        out = D.attention(q, chunks, kc, vc, scale, fused=fz).float().cpu().numpy().astype(np.float64)
        deq = oracle.prq_decompress_batch(chunks.payload.cpu().numpy(), chunks.scales.cpu().numpy(),
                                          chunks.centroids.float().cpu().numpy(), chunks.assignments.cpu().numpy(),
                                          nc, d, cfg.bits, cfg.group_size, 8)
        for tag, dq in (("f32", deq), ("bf16", round_to_bf16(deq.astype(np.float32)).astype(np.float32))):
            kk, vv = dq[0::2], dq[1::2]
            ref = oracle.attention(q.float().cpu().numpy(), kk, vv, kc.float().cpu().numpy(),
                                   vc.float().cpu().numpy(), scale, 8)
            kall = np.concatenate([kk, kc.float().cpu().numpy().transpose(1, 0, 2)], axis=1)
            vall = np.concatenate([vv, vc.float().cpu().numpy().transpose(1, 0, 2)], axis=1)
            sab = softmax_abs(q.float().cpu().numpy().astype(np.float64), kall.astype(np.float64),
                              vall.astype(np.float64), scale)
            e = np.abs(out - ref)
            res[(fz, tag)] = (round(float(e.max() / np.abs(ref).max()), 5),
                              round(float(np.linalg.norm(out - ref) / np.linalg.norm(ref)), 5),
                              round(float((e / sab).max()), 5))
    print(dict(seed=seed, H=H, nq=nq, nc=nc, ncur=ncur, fused=fused, scale=round(scale, 4), cfg=cfg), flush=True)
    for k, v in res.items():
        print("   fused=%d vs %s: maxabs/max|O| %.5f  relL2 %.5f  max |err|/(softmax|V|) %.5f" % (k[0], k[1], *v))
