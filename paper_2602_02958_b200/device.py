"""Batched device API: P planes resident in HBM, one C-ABI call per step.

This is the fast path the drop-in ``qvgcodec`` mirror is built on.  Every
function takes CUDA tensors, launches the sm_100a kernels of
libqvg_b200.so on the current torch stream, and returns CUDA tensors.  The
only host work is argument checking and drawing the k-means++ uniforms
(numpy's Philox, exactly the reference's generator, Q/clustering.py:32-33).

Layouts (plane-major, see include/qvg.h):
    x            [P, N, d]   bfloat16 or float32
    payload      [P, ceil(N*d*bits/8)] uint8
    scales       [P, N*d/B]  uint8 (E4M3 codes)
    centroids    [P, S, K, d] bfloat16 (the StageMeta centroids, bit-exact)
    assignments  [P, S, N]   uint8
"""

from __future__ import annotations

import ctypes
import hashlib
import struct
from dataclasses import dataclass
from typing import Optional, Sequence, Union

import numpy as np
import torch

from . import _lib
from .qvgcodec.types import QuantConfig

__all__ = [
    "DeviceChunks", "stage_seed", "pp_draws", "compress", "quantize", "dequantize",
    "kmeans_pp", "assign", "lloyd_step", "kmeans", "sa_smoothing", "add_back", "attention",
    "stage_mse_curve",
    "check_status",
]


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("device API expects CUDA tensors (no CPU fallback)")
        if t is not None and not t.is_contiguous():
            raise ValueError("device API expects contiguous tensors")


def _x_dtype(x: torch.Tensor) -> int:
    if x.dtype == torch.bfloat16:
        return _lib.DTYPE_BF16
    if x.dtype == torch.float32:
        return _lib.DTYPE_F32
    if x.dtype == torch.float64:
        return _lib.DTYPE_F64
    raise ValueError(f"unsupported input dtype {x.dtype}")


def check_status(status: torch.Tensor) -> None:
    """Synchronise on the status word and raise the mapped CodecError."""
    _lib.raise_for_status(int(status.item()))


# ---------------------------------------------------------------------------
# RNG (host): stage seeds + k-means++ uniforms (Q/prq.py:32-35,
# Q/clustering.py:32-33,40,58).  The draws do not depend on the data, so
# they are drawn up front and the whole seeding runs on the device.
# ---------------------------------------------------------------------------

def stage_seed(seed: int, chunk_index: int, stage: int) -> int:
    digest = hashlib.blake2b(struct.pack("<QQQ", seed, chunk_index, stage), digest_size=8).digest()
    return struct.unpack("<Q", digest)[0]


def pp_draws(config: QuantConfig, chunk_indices: Union[int, Sequence[int]], n_planes: int,
             device) -> torch.Tensor:
    """[P, S, K] float64 uniforms: rng.random() x K per stage per plane."""
    if isinstance(chunk_indices, int):
        chunk_indices = [chunk_indices] * n_planes
    if len(chunk_indices) != n_planes:
        raise ValueError("need one chunk index per plane")
    S, K = config.stages, config.centroids
    cache = {}
    out = np.empty((n_planes, S, K), np.float64)
    for p, c in enumerate(chunk_indices):
        if c not in cache:
            blk = np.empty((S, K), np.float64)
            for t in range(S):
                gen = np.random.Generator(np.random.Philox(stage_seed(config.seed, c, t + 1)))
                blk[t] = gen.random(K)
            cache[c] = blk
        out[p] = cache[c]
    return torch.from_numpy(out).to(device)


# ---------------------------------------------------------------------------
# codec
# ---------------------------------------------------------------------------

@dataclass
class DeviceChunks:
    """P compressed planes (one CompressedChunk each), resident on a GPU."""

    config: QuantConfig
    n_tokens: int
    head_dim: int
    payload: torch.Tensor
    scales: torch.Tensor
    centroids: torch.Tensor
    assignments: torch.Tensor
    centroids_f64: Optional[torch.Tensor] = None
    iters: Optional[torch.Tensor] = None

    @property
    def n_planes(self) -> int:
        return self.payload.shape[0]

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size()
                   for t in (self.payload, self.scales, self.centroids, self.assignments))

    def select(self, idx) -> "DeviceChunks":
        pick = lambda t: None if t is None else t[idx].contiguous()
        return DeviceChunks(self.config, self.n_tokens, self.head_dim, pick(self.payload),
                            pick(self.scales), pick(self.centroids), pick(self.assignments),
                            pick(self.centroids_f64), pick(self.iters))


def _alloc_chunks(config: QuantConfig, P: int, N: int, d: int, device, with_f64: bool,
                  with_iters: bool) -> DeviceChunks:
    S, K = config.stages, config.centroids
    kw = dict(device=device)
    return DeviceChunks(
        config, N, d,
        payload=torch.empty((P, (N * d * config.bits + 7) // 8), dtype=torch.uint8, **kw),
        scales=torch.empty((P, N * d // config.group_size), dtype=torch.uint8, **kw),
        centroids=torch.empty((P, S, K, d), dtype=torch.bfloat16, **kw),
        assignments=torch.empty((P, S, N), dtype=torch.uint8, **kw),
        centroids_f64=torch.empty((P, S, K, d), dtype=torch.float64, **kw) if with_f64 else None,
        iters=torch.empty((P, S), dtype=torch.int32, **kw) if with_iters else None,
    )


def compress(x: torch.Tensor, config: QuantConfig, chunk_index: Union[int, Sequence[int]] = 0,
             warm_init: Optional[torch.Tensor] = None, draws: Optional[torch.Tensor] = None,
             keep_f64: bool = False, check: bool = True,
             status: Optional[torch.Tensor] = None) -> DeviceChunks:
    """prq_compress (Q/prq.py:58-80) over P planes: x [P, N, d] -> DeviceChunks.

    warm_init: [P, S, K, d] float64 (Q/prq.py:61-71).  keep_f64 also returns
    the unrounded float64 centroids (the next chunk's warm start).
    """
    _require_cuda(x, warm_init, draws)
    if x.dim() != 3:
        raise ValueError("x must be [P, N, d]")
    P, N, d = x.shape
    dev = x.device
    S, K = config.stages, config.centroids
    out = _alloc_chunks(config, P, N, d, dev, keep_f64 or warm_init is not None, True)
    if S > 0 and warm_init is None and draws is None:
        draws = pp_draws(config, chunk_index, P, dev)
    elif draws is not None:
        draws = draws.to(torch.float64).contiguous()
        if tuple(draws.shape) != (P, S, K):
            raise ValueError("draws must be [P, S, K] float64")
    if warm_init is not None:
        warm_init = warm_init.to(torch.float64).contiguous()
        if tuple(warm_init.shape) != (P, S, K, d):
            raise ValueError("warm_init must be [P, S, K, d]")
    lib = _lib.load()
    cfg = _lib.cfg_ptr(config)
    ws = None
    if S > 0:
        wbytes = lib.qvg_compress_workspace_size(P, N, d, cfg)
        ws = torch.empty(wbytes, dtype=torch.uint8, device=dev)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(lib.qvg_compress(
        _ptr(x), _x_dtype(x), P, N, d, cfg, _ptr(draws), _ptr(warm_init), _ptr(out.payload),
        _ptr(out.scales), _ptr(out.centroids), _ptr(out.assignments), _ptr(out.centroids_f64),
        _ptr(out.iters), _ptr(st), _ptr(ws), 0 if ws is None else ws.numel(), _stream(dev)))
    if check:
        check_status(st)
    return out


def quantize(x: torch.Tensor, config: QuantConfig, centroids: Optional[torch.Tensor] = None,
             assignments: Optional[torch.Tensor] = None, payload: Optional[torch.Tensor] = None,
             scales: Optional[torch.Tensor] = None, check: bool = True,
             status: Optional[torch.Tensor] = None):
    """Quantize half of the codec given stage metadata -> (payload, scales)."""
    _require_cuda(x, centroids, assignments, payload, scales)
    P, N, d = x.shape
    dev = x.device
    if config.stages and (centroids is None or assignments is None):
        raise ValueError("stage metadata required when config.stages > 0")
    if payload is None:
        payload = torch.empty((P, (N * d * config.bits + 7) // 8), dtype=torch.uint8, device=dev)
    if scales is None:
        scales = torch.empty((P, N * d // config.group_size), dtype=torch.uint8, device=dev)
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _lib.load()
    _lib.check(lib.qvg_quantize(_ptr(x), _x_dtype(x), P, N, d, _lib.cfg_ptr(config),
                                _ptr(centroids), _ptr(assignments), _ptr(payload), _ptr(scales),
                                _ptr(st), _stream(dev)))
    if check:
        check_status(st)
    return payload, scales


def dequantize(chunks: DeviceChunks, out_dtype=torch.bfloat16, out: Optional[torch.Tensor] = None,
               check: bool = True, status: Optional[torch.Tensor] = None) -> torch.Tensor:
    """prq_decompress_onepass (Q/prq.py:113-132) over P planes -> [P, N, d]."""
    c = chunks
    _require_cuda(c.payload, c.scales, c.centroids, c.assignments, out)
    P, N, d = c.n_planes, c.n_tokens, c.head_dim
    dev = c.payload.device
    if out is None:
        out = torch.empty((P, N, d), dtype=out_dtype, device=dev)
    odt = _lib.DTYPE_BF16 if out.dtype == torch.bfloat16 else _lib.DTYPE_F32
    if out.dtype not in (torch.bfloat16, torch.float32):
        raise ValueError("out dtype must be bfloat16 or float32")
    st = status if status is not None else torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _lib.load()
    _lib.check(lib.qvg_dequantize(_ptr(c.payload), _ptr(c.scales), _ptr(c.centroids),
                                  _ptr(c.assignments), P, N, d, _lib.cfg_ptr(c.config), _ptr(out),
                                  odt, _ptr(st), _stream(dev)))
    if check:
        check_status(st)
    return out


def stage_mse_curve(x: torch.Tensor, config: QuantConfig, max_stages: int,
                    chunk_index: Union[int, Sequence[int]] = 0) -> torch.Tensor:
    """stage_mse_curve (Q/prq.py:135-172) over P planes -> float64 [P, max_stages + 1].

    Stage seeds depend only on (seed, chunk, stage), so one compress with
    ``max_stages`` stages yields every prefix chain; each prefix s is then
    quantized given its first s stages' metadata (the residual x - C_1[pi_1]
    - ... - C_s[pi_s] formed in the kernel), decoded to float32 and compared
    with x in float64.  The per-plane mean is torch's reduction, not numpy's
    pairwise order (the host mirror qvgcodec.prq.stage_mse_curve is the
    bit-exact one); the decoded planes themselves are bit-exact."""
    _require_cuda(x)
    P, N, d = x.shape
    full = compress(x, config.with_stages(max_stages), chunk_index=chunk_index) if max_stages else None
    x64 = x.to(torch.float64)
    curve = torch.empty((P, max_stages + 1), dtype=torch.float64, device=x.device)
    for s in range(max_stages + 1):
        cfg = config.with_stages(s)
        if s:
            cent = full.centroids[:, :s].contiguous()
            asg = full.assignments[:, :s].contiguous()
        else:
            cent = torch.empty((P, 0, config.centroids, d), dtype=torch.bfloat16, device=x.device)
            asg = torch.empty((P, 0, N), dtype=torch.uint8, device=x.device)
        pay, sc = quantize(x, cfg, cent, asg)
        rec = dequantize(DeviceChunks(cfg, N, d, pay, sc, cent, asg), torch.float32)
        curve[:, s] = ((x64 - rec.to(torch.float64)) ** 2).mean(dim=(1, 2))
    return curve


# ---------------------------------------------------------------------------
# clustering / smoothing (float64 rows [P, N, d])
# ---------------------------------------------------------------------------

def _f64(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.float64).contiguous()


def _km_ws(P, N, d, K, dev):
    n = _lib.load().qvg_kmeans_workspace_size(P, N, d, K)
    return torch.empty(max(n, 1), dtype=torch.uint8, device=dev)


def kmeans_pp(rows: torch.Tensor, k: int, draws: torch.Tensor) -> torch.Tensor:
    """kmeans_pp_init (Q/clustering.py:47-63): draws [P, K] -> centroids [P, K, d]."""
    rows = _f64(rows)
    _require_cuda(rows, draws)
    P, N, d = rows.shape
    cent = torch.empty((P, k, d), dtype=torch.float64, device=rows.device)
    ws = _km_ws(P, N, d, k, rows.device)
    _lib.check(_lib.load().qvg_kmeanspp(_ptr(rows), P, N, d, k, _ptr(_f64(draws)), _ptr(cent),
                                        _ptr(ws), ws.numel(), _stream(rows.device)))
    return cent


def assign(rows: torch.Tensor, centroids: torch.Tensor) -> torch.Tensor:
    """_assign (Q/clustering.py:66-71) -> int32 [P, N]."""
    rows, centroids = _f64(rows), _f64(centroids)
    _require_cuda(rows, centroids)
    P, N, d = rows.shape
    out = torch.empty((P, N), dtype=torch.int32, device=rows.device)
    _lib.check(_lib.load().qvg_assign(_ptr(rows), _ptr(centroids), P, N, d, centroids.shape[1],
                                      _ptr(out), _stream(rows.device)))
    return out


def lloyd_step(rows: torch.Tensor, centroids: torch.Tensor):
    """lloyd_step (Q/clustering.py:74-107) -> (new centroids, assign u8, objective f64 [P])."""
    rows = _f64(rows)
    cent = _f64(centroids).clone()
    _require_cuda(rows, cent)
    P, N, d = rows.shape
    K = cent.shape[1]
    asg = torch.empty((P, N), dtype=torch.uint8, device=rows.device)
    obj = torch.empty(P, dtype=torch.float64, device=rows.device)
    ws = _km_ws(P, N, d, K, rows.device)
    _lib.check(_lib.load().qvg_lloyd_step(_ptr(rows), _ptr(cent), P, N, d, K, _ptr(asg), _ptr(obj),
                                          _ptr(ws), ws.numel(), _stream(rows.device)))
    return cent, asg, obj


def kmeans(rows: torch.Tensor, k: int, max_iters: int = 10, tol: float = 1e-4,
           draws: Optional[torch.Tensor] = None, init: Optional[torch.Tensor] = None):
    """kmeans (Q/clustering.py:110-160) -> (centroids f64, assign u8, objective f64, iters i32)."""
    rows = _f64(rows)
    _require_cuda(rows, draws, init)
    P, N, d = rows.shape
    dev = rows.device
    cent = torch.empty((P, k, d), dtype=torch.float64, device=dev)
    asg = torch.empty((P, N), dtype=torch.uint8, device=dev)
    obj = torch.empty(P, dtype=torch.float64, device=dev)
    it = torch.empty(P, dtype=torch.int32, device=dev)
    ws = _km_ws(P, N, d, k, dev)
    _lib.check(_lib.load().qvg_kmeans(
        _ptr(rows), P, N, d, k, max_iters, float(tol),
        _ptr(None if draws is None else _f64(draws)), _ptr(None if init is None else _f64(init)),
        _ptr(cent), _ptr(asg), _ptr(obj), _ptr(it), _ptr(ws), ws.numel(), _stream(dev)))
    return cent, asg, obj, it


def sa_smoothing(x: torch.Tensor, k: int, draws: Optional[torch.Tensor] = None,
                 warm_init: Optional[torch.Tensor] = None, max_iters: int = 10,
                 tol: float = 1e-4):
    """sa_smoothing (Q/smoothing.py:23-41) -> (residual f64, centroids bf16 [P,K,d],
    assign u8 [P,N], centroids f64, iters)."""
    x = _f64(x)
    _require_cuda(x, draws, warm_init)
    P, N, d = x.shape
    dev = x.device
    res = torch.empty_like(x)
    cb = torch.empty((P, k, d), dtype=torch.bfloat16, device=dev)
    asg = torch.empty((P, N), dtype=torch.uint8, device=dev)
    c64 = torch.empty((P, k, d), dtype=torch.float64, device=dev)
    it = torch.empty(P, dtype=torch.int32, device=dev)
    lib = _lib.load()
    n = lib.qvg_sa_smoothing_workspace_size(P, N, d, k)
    ws = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    _lib.check(lib.qvg_sa_smoothing(
        _ptr(x), P, N, d, k, max_iters, float(tol),
        _ptr(None if draws is None else _f64(draws)),
        _ptr(None if warm_init is None else _f64(warm_init)), _ptr(res), _ptr(cb), _ptr(asg),
        _ptr(c64), _ptr(it), _ptr(ws), ws.numel(), _stream(dev)))
    return res, cb, asg, c64, it


def add_back(residual: torch.Tensor, centroids: torch.Tensor, assignments: torch.Tensor):
    """add_back (Q/smoothing.py:44-54): residual + C[pi] in float64."""
    residual = _f64(residual)
    centroids = centroids.to(torch.bfloat16).contiguous()
    assignments = assignments.to(torch.uint8).contiguous()
    _require_cuda(residual, centroids, assignments)
    P, N, d = residual.shape
    out = torch.empty_like(residual)
    _lib.check(_lib.load().qvg_add_back(_ptr(residual), _ptr(centroids), _ptr(assignments), P, N, d,
                                        centroids.shape[1], _ptr(out), _stream(residual.device)))
    return out


# ---------------------------------------------------------------------------
# attention over the quantized cache
# ---------------------------------------------------------------------------

def attention(q: torch.Tensor, cache: Optional[DeviceChunks], k_cur: torch.Tensor,
              v_cur: torch.Tensor, softmax_scale: Optional[float] = None,
              kv_bf16: Optional[torch.Tensor] = None,
              out: Optional[torch.Tensor] = None, fused: bool = False,
              workspace: Optional[torch.Tensor] = None, rope=None, check: bool = True) -> torch.Tensor:
    """O = softmax(q [Khat; k_cur]^T * scale) [Vhat; v_cur] per head.

    q [Nq, H, d] bf16; cache: 2H planes (plane 2h = K of head h, 2h+1 = V)
    or, for the bf16 comparator, kv_bf16 [2H, Nc, d]; k_cur/v_cur [Ncur, H, d].
    fused=True dequantizes the cache inside the attention kernel (no bf16
    staging buffer); the default reconstructs it to bf16 in a workspace with the
    HBM-bound decoder and runs the pipelined TMA/tcgen05 kernel.
    rope=(cos, sin, "rotate_half"|"interleaved") marks the cached keys as
    pre-RoPE: the reconstructed keys are rotated with cos/sin [n_cache, d/2]
    (float32, CUDA) before the attention; q and k_cur are post-RoPE.
    check: synchronise and raise NaNPattern / DimensionMismatch when the
    cache holds an E4M3 NaN-pattern scale or an assignment >= K (the codec
    status word, as dequantize does); check=False leaves the launch async.
    """
    _require_cuda(q, k_cur, v_cur, kv_bf16, out)
    for name, t in (("q", q), ("k_cur", k_cur), ("v_cur", v_cur), ("kv_bf16", kv_bf16), ("out", out)):
        if t is not None and t.dtype != torch.bfloat16:
            raise ValueError(f"{name} must be bfloat16, got {t.dtype}")
    if q.dim() != 3:
        raise ValueError("q must be [Nq, H, d]")
    nq, H, d = q.shape
    if k_cur.dim() != 3 or tuple(k_cur.shape[1:]) != (H, d) or tuple(v_cur.shape) != tuple(k_cur.shape):
        raise ValueError("k_cur / v_cur must be [Ncur, H, d] matching q")
    if out is not None and tuple(out.shape) != (nq, H, d):
        raise ValueError("out must be [Nq, H, d]")
    ncur = k_cur.shape[0]
    if cache is not None:
        if cache.n_planes != 2 * H:
            raise ValueError("cache must hold 2*H planes (K, V per head)")
        if cache.head_dim != d:
            raise ValueError(f"cache head_dim {cache.head_dim} != q head_dim {d}")
        nc, cfg = cache.n_tokens, cache.config
    elif kv_bf16 is not None:
        if kv_bf16.dim() != 3 or kv_bf16.shape[0] != 2 * H or kv_bf16.shape[2] != d:
            raise ValueError("kv_bf16 must be [2H, Nc, d]")
        nc, cfg = kv_bf16.shape[1], QuantConfig(stages=0)
    else:
        nc, cfg = 0, QuantConfig(stages=0)
    scale = float(softmax_scale) if softmax_scale is not None else d ** -0.5
    if out is None:
        out = torch.empty((nq, H, d), dtype=torch.bfloat16, device=q.device)
    lib = _lib.load()
    cp = _lib.cfg_ptr(cfg)
    n = lib.qvg_attention_workspace_size(nq, nc, ncur, H, d, cp)
    if fused or cache is None:
        ws, nbytes = None, 0
    else:
        ws = workspace if workspace is not None and workspace.numel() >= n else \
            torch.empty(max(n, 1), dtype=torch.uint8, device=q.device)
        nbytes = ws.numel()
    c = cache
    st = torch.zeros(1, dtype=torch.int32, device=q.device) if c is not None else None
    if rope is None:
        _lib.check(lib.qvg_attention(
            _ptr(q), _ptr(c.payload if c else None), _ptr(c.scales if c else None),
            _ptr(c.centroids if c else None), _ptr(c.assignments if c else None), _ptr(kv_bf16),
            _ptr(k_cur), _ptr(v_cur), nq, nc, ncur, H, d, cp, scale, _ptr(out), _ptr(ws), nbytes,
            _ptr(st), _stream(q.device)))
        if check and st is not None:
            check_status(st)
        return out
    cos_t, sin_t, mode = rope
    _require_cuda(cos_t, sin_t)
    if ws is None:
        ws = torch.empty(max(n, 1), dtype=torch.uint8, device=q.device)
        nbytes = ws.numel()
    _lib.check(lib.qvg_attention_rope(
        _ptr(q), _ptr(c.payload if c else None), _ptr(c.scales if c else None),
        _ptr(c.centroids if c else None), _ptr(c.assignments if c else None), _ptr(kv_bf16),
        _ptr(k_cur), _ptr(v_cur), nq, nc, ncur, H, d, cp, scale, _ptr(cos_t), _ptr(sin_t),
        {"rotate_half": 1, "interleaved": 2}[mode], _ptr(out), _ptr(ws), nbytes, _ptr(st), _stream(q.device)))
    if check and st is not None:
        check_status(st)
    return out


# ---------------------------------------------------------------------------
# baseline competitors (Q/baselines.py) on the device
# ---------------------------------------------------------------------------

def random_signs(d: int, seed: int) -> np.ndarray:
    """Seeded +-1 diagonal of the QuaRot rotation (Q/baselines.py:126-129):
    host Philox draws, data-independent, as the reference."""
    rng = np.random.Generator(np.random.Philox(seed))
    return np.where(rng.random(d) < 0.5, -1.0, 1.0).astype(np.float32)


def hadamard(x: torch.Tensor, signs: Union[np.ndarray, torch.Tensor], inverse: bool = False,
             out_dtype=torch.float32) -> torch.Tensor:
    """Rows of x [..., d] (f32/bf16) through the seeded Hadamard rotation:
    fwht(x * signs) / sqrt(d) (hadamard_transform, Q/baselines.py:148) or its
    inverse fwht(x) / sqrt(d) * signs (Q/baselines.py:159), float64
    butterflies in numpy's order, returned as float64 (the reference's value)
    or rounded to float32."""
    _require_cuda(x)
    d = x.shape[-1]
    s = torch.as_tensor(np.asarray(signs, dtype=np.float32) if not torch.is_tensor(signs) else signs,
                        dtype=torch.float32).to(x.device).contiguous()
    if s.numel() != d:
        from .qvgcodec.errors import DimensionMismatch
        raise DimensionMismatch("signs length != row length")
    out = torch.empty(x.shape, dtype=out_dtype, device=x.device)
    odt = _lib.DTYPE_F64 if out_dtype == torch.float64 else _lib.DTYPE_F32
    _lib.check(_lib.load().qvg_hadamard(_ptr(x), _x_dtype(x), x.numel() // d, d, _ptr(s),
                                        float(np.sqrt(d)), int(bool(inverse)), _ptr(out), odt,
                                        _stream(x.device)))
    return out


def token_transpose(x: torch.Tensor, group_size: int):
    """[P, N, d] -> ([P, d, N + pad] float32, pad): the KIVI key path's
    transposed plane with the final partial token group zero-padded
    (Q/baselines.py:60-73)."""
    _require_cuda(x)
    P, N, d = x.shape
    pad = (-N) % group_size
    out = torch.empty((P, d, N + pad), dtype=torch.float32, device=x.device)
    _lib.check(_lib.load().qvg_token_transpose(_ptr(x), _x_dtype(x), P, N, N + pad, d, 0, _ptr(out),
                                               _stream(x.device)))
    return out, pad


def token_untranspose(y: torch.Tensor, n_tokens: int) -> torch.Tensor:
    """[P, d, Np] float32 -> [P, n_tokens, d] float32 (Q/baselines.py:84-88)."""
    _require_cuda(y)
    P, d, Np = y.shape
    out = torch.empty((P, n_tokens, d), dtype=torch.float32, device=y.device)
    _lib.check(_lib.load().qvg_token_transpose(_ptr(y), _lib.DTYPE_F32, P, n_tokens, Np, d, 1, _ptr(out),
                                               _stream(y.device)))
    return out


def _rtn(bits: int, group_size: int) -> QuantConfig:
    return QuantConfig(bits=bits, group_size=group_size, stages=0, centroids=1)


def rtn_quantize(x: torch.Tensor, bits: int, group_size: int):
    """RTN (Q/baselines.py:24-27): the group quantizer with no smoothing."""
    return quantize(x, _rtn(bits, group_size))


def rtn_dequantize(payload: torch.Tensor, scales: torch.Tensor, n_tokens: int, head_dim: int, bits: int,
                   group_size: int, out_dtype=torch.float32) -> torch.Tensor:
    return dequantize(DeviceChunks(_rtn(bits, group_size), n_tokens, head_dim, payload, scales, None, None),
                      out_dtype)


def quarot_quantize(x: torch.Tensor, bits: int, group_size: int, seed: int):
    """QuaRot (Q/baselines.py:177-194): rotate every row, round to float32,
    then RTN.  Returns (payload, scales)."""
    rot = hadamard(x, random_signs(x.shape[-1], seed))
    return quantize(rot, _rtn(bits, group_size))


def quarot_dequantize(payload: torch.Tensor, scales: torch.Tensor, n_tokens: int, head_dim: int, bits: int,
                      group_size: int, seed: int) -> torch.Tensor:
    """Q/baselines.py:197-202: RTN decode, inverse rotation, float32."""
    rot = rtn_dequantize(payload, scales, n_tokens, head_dim, bits, group_size)
    return hadamard(rot, random_signs(head_dim, seed), inverse=True)


def token_axis_quantize(x: torch.Tensor, bits: int, group_size: int):
    """KIVI key path (Q/baselines.py:60-73): groups of consecutive tokens per
    channel.  Returns (payload, scales, pad)."""
    t, pad = token_transpose(x, group_size)
    pay, sc = quantize(t, _rtn(bits, group_size))
    return pay, sc, pad


def token_axis_dequantize(payload: torch.Tensor, scales: torch.Tensor, n_tokens: int, head_dim: int, bits: int,
                          group_size: int) -> torch.Tensor:
    pad = (-n_tokens) % group_size
    t = rtn_dequantize(payload, scales, head_dim, n_tokens + pad, bits, group_size)
    return token_untranspose(t, n_tokens)


# ---------------------------------------------------------------------------
# tracing: QVG_NVTX=1 wraps the device entry points in NVTX ranges (named as
# the reference functions they replace), visible in nsys / ncu --nvtx timelines
# ---------------------------------------------------------------------------
def _nvtx_wrap(name, fn):
    import functools

    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        torch.cuda.nvtx.range_push(name)
        try:
            return fn(*args, **kwargs)
        finally:
            torch.cuda.nvtx.range_pop()
    return wrapped


if __import__("os").environ.get("QVG_NVTX") == "1":
    for _n, _ref in (("compress", "prq_compress"), ("quantize", "quantize_matrix"),
                     ("dequantize", "prq_decompress_onepass"), ("attention", "qvg_attention"),
                     ("kmeans", "kmeans"), ("sa_smoothing", "sa_smoothing")):
        globals()[_n] = _nvtx_wrap(f"qvg.{_ref}", globals()[_n])

