"""One prq_compress of a Self-Forcing chunk (720 planes) for an ncu launch list;
WARM=1 also encodes a second chunk from the first chunk's float64 centroids."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_02958_b200 import device as D  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import QuantConfig  # noqa: E402
from paper_2602_02958_b200.synth import kv_cache_planes  # noqa: E402

cfg = QuantConfig(bits=2, group_size=64, stages=2, centroids=64)
x = kv_cache_planes(30, 12, 4680, 128, seed=0, device="cuda")
c0 = D.compress(x, cfg, chunk_index=0, keep_f64=True)
if os.environ.get("WARM"):
    x1 = kv_cache_planes(30, 12, 4680, 128, seed=1, device="cuda")
    D.compress(x1, cfg, chunk_index=1, warm_init=c0.centroids_f64)
torch.cuda.synchronize()
print("ok")
