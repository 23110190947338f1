"""Time the attention kernels on the LongCat-shaped layer (bench.bench_attention)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

r = bench.bench_attention(torch.device("cuda", 0), 0, 1)
r["env"] = {k: v for k, v in os.environ.items() if k.startswith("QVG_")}
print(json.dumps(r))
