"""Synthetic K/V planes, bit-identical to the reference generator.

The reference's synthetic input is ``gen_clustered_stream``
(Q/datagen.py:44-161): one numpy ``SeedSequence`` per (layer, head, K|V)
stream, a mean / outlier-channel generator on spawn key 0 and one generator
per chunk on spawn key ``chunk + 1`` (Q/datagen.py:69-70,86).
fixes the parameters and seeds (n_clusters 256, sigma_within 0.125,
sigma_between 2.5, outlier channels 0, 16, ..., 112 amplified x10 for keys
and x100 for values, seed = 2 * (layer * H + head) + {0: K, 1: V}) and the
bf16 rounding of the planes (Q/lowprec.py round_to_bf16), so the bf16
device input and the float32 reference input are the same numbers.

This module restates that algorithm chunk-addressably — chunk ``c`` of a
stream is produced without generating chunks ``0..c-1`` (only their cheap
drift steps are replayed, in order, so the float64 means evolve exactly as
the reference's) — and fills a host buffer with many planes in parallel
worker processes.  It is input generation for the benchmark and the parity
tests, not part of the codec; bit-identity with the reference is pinned by
``tests/golden/datagen.npz`` (written by the reference itself).
"""

from __future__ import annotations

import mmap
import multiprocessing as mp
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

OUTLIER_CHANNELS = tuple(range(0, 128, 16))


@dataclass(frozen=True)
class StreamParams:
    """gen_clustered_stream's knobs (Q/datagen.py:123-134)."""

    n_tokens: int
    d: int = 128
    n_clusters: int = 256
    sigma_within: float = 0.125
    sigma_between: float = 2.5
    drift: float = 0.0
    outlier_channels: tuple = OUTLIER_CHANNELS
    outlier_scale: float = 1.0


def _gen(seed: int, key: int) -> np.random.Generator:
    # root.spawn(1)[0] on its k-th call == SeedSequence(seed, spawn_key=(k,))
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(seed, spawn_key=(key,))))


def _stream_base(seed: int, p: StreamParams):
    """Initial means [n_clusters, d] f64 and the per-cluster amplification
    table (1.0, or outlier_scale on the cluster's own channel subset) drawn
    from the spawn-0 generator (Q/datagen.py:69-82)."""
    g = _gen(seed, 0)
    means = g.normal(0.0, p.sigma_between, size=(p.n_clusters, p.d))
    amp = np.ones((p.n_clusters, p.d))
    ch = np.asarray(sorted(set(int(c) for c in p.outlier_channels)), dtype=np.int64)
    if ch.size:
        for c in range(p.n_clusters):
            pick = g.random(ch.size) < 0.5
            if not pick.any():
                pick[int(g.random() * ch.size) % ch.size] = True
            amp[c, ch[pick]] = p.outlier_scale
    return means, amp


def _drift_step(g: np.random.Generator, p: StreamParams) -> np.ndarray:
    # the first draw of every chunk > 0, kept even without drift (Q/datagen.py:87-92)
    s = g.normal(0.0, 1.0, size=(p.n_clusters, p.d))
    return s / np.linalg.norm(s, axis=1, keepdims=True)


def stream_chunk(seed: int, chunk: int, p: StreamParams, base=None) -> np.ndarray:
    """Chunk ``chunk`` of stream ``seed`` as float32 [n_tokens, d] (not yet
    bf16-rounded), equal to gen_clustered_stream(...)[chunk].data."""
    if not (1 <= p.n_clusters <= p.n_tokens):
        raise ValueError("need 1 <= n_clusters <= n_tokens")
    means, amp = base if base is not None else _stream_base(seed, p)
    if p.drift > 0:
        for c in range(1, chunk + 1):                 # replay the drift in chunk order
            means = means + p.drift * _drift_step(_gen(seed, c + 1), p)
    g = _gen(seed, chunk + 1)
    if chunk > 0:
        g.normal(0.0, 1.0, size=(p.n_clusters, p.d))  # the chunk's step (applied above)
    extra = (g.random(p.n_tokens - p.n_clusters) * p.n_clusters).astype(np.int64)
    members = np.concatenate([np.arange(p.n_clusters), extra])[g.permutation(p.n_tokens)]
    rows = means[members] + g.normal(0.0, p.sigma_within, size=(p.n_tokens, p.d))
    for c in np.flatnonzero((amp != 1.0).any(axis=0)):  # x1.0 elsewhere is exact: skip it
        rows[:, c] *= amp[members, c]
    return rows.astype(np.float32)


def round_bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns (uint16), round to nearest even."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    return ((u + (np.uint32(0x7FFF) + ((u >> 16) & 1))) >> 16).astype(np.uint16)


def kv_params(n_tokens: int, value: bool, drift: float = 0.0, d: int = 128) -> StreamParams:
    """keys x10, values x100 on channels 0, 16, ..., 112."""
    return StreamParams(n_tokens=n_tokens, d=d, drift=drift,
                        outlier_scale=100.0 if value else 10.0)


def kv_seed(layer: int, head: int, n_heads: int, value: bool) -> int:
    return 2 * (layer * n_heads + head) + (1 if value else 0)


@dataclass(frozen=True)
class PlaneRef:
    """One plane of a K/V cache: (layer, head, K|V) stream at chunk ``chunk``."""

    layer: int
    head: int
    value: bool
    chunk: int


def cache_layout(n_layers: int, n_heads: int, chunks: Sequence[int]) -> list:
    """Plane order of a cache: chunk-major, then layer, head, K before V
    (plane 2 * (l * H + h) + {0, 1} within a chunk)."""
    return [PlaneRef(l, h, v, c) for c in chunks for l in range(n_layers) for h in range(n_heads)
            for v in (False, True)]


# --- parallel host fill --------------------------------------------------------

_JOB = {}


def _fill(idx):
    j = _JOB
    out = np.frombuffer(j["buf"], dtype=np.uint16).reshape(-1, j["n"], j["d"])
    bases = {}
    for i in idx:
        r = j["planes"][i]
        p = kv_params(j["n"], r.value, j["drift"], j["d"])
        s = kv_seed(r.layer, r.head, j["heads"], r.value)
        if s not in bases:
            bases[s] = _stream_base(s, p)
        out[i] = round_bf16_bits(stream_chunk(s, r.chunk, p, bases[s]))
    return len(idx)


def kv_cache_bf16(planes: Sequence[PlaneRef], n_heads: int, n_tokens: int, d: int = 128,
                  drift: float = 0.0, workers: Optional[int] = None) -> np.ndarray:
    """[len(planes), n_tokens, d] bf16 bit patterns (uint16) of the listed
    planes, generated by ``workers`` forked processes writing into one shared
    anonymous mapping (not /dev/shm).  The children run numpy only."""
    P = len(planes)
    nbytes = max(P * n_tokens * d * 2, 1)
    buf = mmap.mmap(-1, nbytes, flags=mmap.MAP_SHARED, prot=mmap.PROT_READ | mmap.PROT_WRITE)
    _JOB.update(buf=buf, planes=list(planes), n=n_tokens, d=d, heads=n_heads, drift=drift)
    workers = workers or len(os.sched_getaffinity(0))
    # one job per stream (all its chunks): the stream's base draws are made once
    by_stream = {}
    for i, r in enumerate(planes):
        by_stream.setdefault((r.layer, r.head, r.value), []).append(i)
    jobs = list(by_stream.values())
    try:
        if workers <= 1 or len(jobs) <= 1:
            for jb in jobs:
                _fill(jb)
        else:
            with mp.get_context("fork").Pool(workers) as pool:
                for _ in pool.imap_unordered(_fill, jobs):
                    pass
    finally:
        _JOB.clear()
    # a view over the mapping (the array keeps it alive): no copy of the cache
    return np.frombuffer(buf, dtype=np.uint16, count=P * n_tokens * d).reshape(P, n_tokens, d)


def bf16_bits_to_f32(u: np.ndarray) -> np.ndarray:
    return (np.asarray(u, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)
