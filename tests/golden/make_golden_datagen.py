"""Golden fixture for paper_2602_02958_b200/datagen.py, produced by running the
REFERENCE generator itself (Q/datagen.py gen_clustered_stream).

    python tests/golden/make_golden_datagen.py

Writes tests/golden/datagen.npz: one small drifting stream in full (float32
planes of 3 chunks) and SHA-256 digests of full-size planes at the bench
shapes (Self-Forcing 4680 tokens with drift, LongCat 38 400 tokens), so the
restatement is pinned at the sizes the benchmark generates.  The GPU box has
no /root/reference, so the outputs are committed."""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# (name, seed, n_chunks, n_tokens, n_clusters, drift, outlier_scale, chunks to digest)
DIGESTS = [
    ("sf_key_l0h0", 0, 3, 4680, 256, 0.0125, 10.0, (0, 2)),
    ("sf_val_l1h11", 2 * (1 * 12 + 11) + 1, 2, 4680, 256, 0.0125, 100.0, (1,)),
    ("sf_key_nodrift", 7, 2, 4680, 256, 0.0, 10.0, (1,)),
    ("longcat_val_h3", 2 * 3 + 1, 1, 38400, 256, 0.0, 100.0, (0,)),
]


def main():
    sys.path.insert(0, REF)
    from qvgcodec import datagen

    out = {}
    small = datagen.gen_clustered_stream(n_chunks=3, n_tokens=160, d=128, n_clusters=16,
                                         sigma_within=0.125, sigma_between=2.5, drift=0.05,
                                         outlier_channels=tuple(range(0, 128, 16)),
                                         outlier_scale=100.0, seed=5)
    out["small"] = np.stack([p.data for p in small]).astype(np.float32)
    names, digests = [], []
    for name, seed, nch, n, k, drift, osc, keep in DIGESTS:
        planes = datagen.gen_clustered_stream(n_chunks=nch, n_tokens=n, d=128, n_clusters=k,
                                              sigma_within=0.125, sigma_between=2.5, drift=drift,
                                              outlier_channels=tuple(range(0, 128, 16)),
                                              outlier_scale=osc, seed=seed)
        for c in keep:
            names.append(f"{name}/c{c}")
            digests.append(hashlib.sha256(np.ascontiguousarray(planes[c].data, np.float32).tobytes()).hexdigest())
    out["digest_names"] = np.array(names)
    out["digests"] = np.array(digests)
    np.savez_compressed(os.path.join(HERE, "datagen.npz"), **out)
    print("wrote datagen.npz:", len(names), "digests")


if __name__ == "__main__":
    main()
