"""Loader for the reference-generated fixtures in tests/golden."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def bf16_bits_to_f32(u16):
    return (np.asarray(u16, np.uint16).astype(np.uint32) << 16).view(np.float32)


def load_plane(name):
    z = np.load(os.path.join(GOLDEN, f"plane_{name}.npz"))
    rec = {k: z[k] for k in z.files}
    rec["centroids_bf16"] = rec.pop("centroids")
    rec["x"] = bf16_bits_to_f32(rec["x_bf16"])
    for k in ("bits", "group_size", "stages", "centroids"):
        rec[k] = int(rec.pop("cfg_" + k))
    rec["chunk_index"] = int(rec["chunk_index"])
    return rec


def load_kat():
    z = np.load(os.path.join(GOLDEN, "kat.npz"))
    return {k: z[k] for k in z.files}
