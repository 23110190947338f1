"""Drop-in mirror of the reference ``qvgcodec`` package's hot-path API.

Module paths follow the reference (``qvgcodec.prq``, ``.quant``,
``.smoothing``, ``.clustering``, ``.types``, ``.lowprec``, ``.metrics``,
``.errors``); the compute behind them is the sm_100a library.  Like the
reference, the package namespace re-exports the value types only.
"""

from .types import (ChunkSpec, CompressedChunk, KVPlane, MemoryBreakdown, QuantConfig, StageMeta,
                    validate_plane)

__all__ = ["ChunkSpec", "CompressedChunk", "KVPlane", "MemoryBreakdown", "QuantConfig",
           "StageMeta", "validate_plane"]

__version__ = "0.1.0"
