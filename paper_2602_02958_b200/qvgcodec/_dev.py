"""Host <-> device glue for the drop-in API (one call = one plane)."""

from __future__ import annotations

import numpy as np
import torch

from .. import _lib


def device() -> torch.device:
    _lib.load()                      # fail loudly without the native library
    if not torch.cuda.is_available():
        raise _lib.NativeLibraryError("a CUDA device is required (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def to_dev(a, dtype=None) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    if not a.flags.writeable:          # torch needs a writable buffer
        a = a.copy()
    t = torch.from_numpy(a)
    if dtype is not None:
        t = t.to(dtype)
    return t.to(device(), non_blocking=False).contiguous()


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()
