"""paper_2602_02958_b200 — B200-native QVG KV-cache hot path.

* ``paper_2602_02958_b200.qvgcodec`` — drop-in mirror of the reference API
  (prq_compress / prq_decompress(_onepass) / quantize / k-means / ...).
* ``paper_2602_02958_b200.device``   — batched device API over P planes in HBM.
* ``paper_2602_02958_b200.shard``    — head/layer sharding over GPUs.
Compute: libqvg_b200.so (sm_100a kernels behind include/qvg.h).
"""

from . import qvgcodec  # noqa: F401

__version__ = "0.1.0"
