"""One prq_compress of a Self-Forcing chunk (720 planes) for an ncu launch list."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_02958_b200 import device as D  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import QuantConfig  # noqa: E402
from paper_2602_02958_b200.synth import kv_cache_planes  # noqa: E402

cfg = QuantConfig(bits=2, group_size=64, stages=2, centroids=64)
x = kv_cache_planes(30, 12, 4680, 128, seed=0, device="cuda")
D.compress(x, cfg, chunk_index=0)
torch.cuda.synchronize()
print("ok")
