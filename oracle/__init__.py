"""CPU ORACLE — test infrastructure only.

ctypes front end over ``libqvg_oracle.so`` (``qvg_oracle.c``), the plain-C
restatement of the reference codec's hot path.  Importable only from
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs, where it is the checker and never the thing
measured as the product.  Parity pins: ``tests/golden`` (fixtures written
by the reference itself) and ``tests/test_oracle_*.py``.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import struct
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libqvg_oracle.so")
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int
_D = ctypes.c_double


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "qvg_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "-B", "libqvg_oracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.qo_pairwise_sum.restype = _D
        L.qo_pairwise_sum.argtypes = [_P, _I64]
        L.qo_e4m3_decode.restype = _D
        L.qo_e4m3_decode.argtypes = [ctypes.c_uint8]
        L.qo_e4m3_encode.restype = ctypes.c_uint8
        L.qo_e4m3_encode.argtypes = [_D, _I32]
        L.qo_round_bf16.restype = ctypes.c_float
        L.qo_round_bf16.argtypes = [ctypes.c_float]
        L.qo_quantize_matrix.restype = _I32
        L.qo_quantize_matrix.argtypes = [_P, _I64, _I32, _I32, _I32, _P, _P]
        L.qo_dequantize_matrix.restype = None
        L.qo_dequantize_matrix.argtypes = [_P, _P, _I64, _I32, _I32, _I32, _P]
        L.qo_kmeans_pp.restype = _I32
        L.qo_kmeans_pp.argtypes = [_P, _I64, _I32, _I32, _P, _P, _P]
        L.qo_assign.restype = None
        L.qo_assign.argtypes = [_P, _I64, _I32, _P, _I32, _P]
        L.qo_lloyd_step.restype = _D
        L.qo_lloyd_step.argtypes = [_P, _I64, _I32, _P, _I32, _P]
        L.qo_kmeans.restype = _I32
        L.qo_kmeans.argtypes = [_P, _I64, _I32, _I32, _I32, _D, _P, _P, _P, _P, _P, _P]
        L.qo_prq_compress.restype = _I32
        L.qo_prq_compress.argtypes = [_P, _I64, _I32, _I32, _I32, _I32, _I32, _I32, _D, _P, _P,
                                      _P, _P, _P, _P, _P, _P]
        L.qo_prq_decompress.restype = None
        L.qo_prq_decompress.argtypes = [_P, _P, _P, _P, _I64, _I32, _I32, _I32, _I32, _I32, _P]
        L.qo_prq_compress_batch.restype = _I32
        L.qo_prq_compress_batch.argtypes = [_P, _I64, _I64, _I32, _I32, _I32, _I32, _I32, _I32,
                                            _D, _P, _P, _P, _P, _P, _P, _I32]
        L.qo_prq_decompress_batch.restype = None
        L.qo_prq_decompress_batch.argtypes = [_P, _P, _P, _P, _I64, _I64, _I32, _I32, _I32, _I32,
                                              _I32, _P, _I32]
        L.qo_quantize_given_metas_batch.restype = _I32
        L.qo_quantize_given_metas_batch.argtypes = [_P, _I64, _I64, _I32, _I32, _I32, _I32, _I32,
                                                    _P, _P, _P, _P, _I32]
        L.qo_attention.restype = None
        L.qo_attention.argtypes = [_P, _P, _P, _P, _P, _I64, _I64, _I64, _I32, _I32, _D, _P, _I32]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle error code {code}")
        self.code = code


# --- RNG restatement (Q/prq.py:32-35, Q/clustering.py:32-33,40,58) -------------

def stage_seed(seed: int, chunk_index: int, stage: int) -> int:
    h = hashlib.blake2b(struct.pack("<QQQ", seed, chunk_index, stage), digest_size=8)
    return struct.unpack("<Q", h.digest())[0]


def pp_draws(seed: int, chunk_index: int, stages: int, k: int) -> np.ndarray:
    """[stages][k] k-means++ draws: Generator(Philox(stage_seed)).random(), k per stage."""
    out = np.empty((stages, k), dtype=np.float64)
    for t in range(stages):
        out[t] = np.random.Generator(np.random.Philox(stage_seed(seed, chunk_index, t + 1))).random(k)
    return out


# --- thin wrappers -------------------------------------------------------------

def pairwise_sum(a) -> float:
    a = _c(a, np.float64).ravel()
    return lib().qo_pairwise_sum(_ptr(a), a.size)


def e4m3_encode(x: float, up: bool = True) -> int:
    return int(lib().qo_e4m3_encode(float(x), 1 if up else 0))


def e4m3_decode(b: int) -> float:
    return float(lib().qo_e4m3_decode(int(b)))


def round_bf16(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.float32)
    f = np.vectorize(lambda v: lib().qo_round_bf16(float(v)), otypes=[np.float32])
    return f(a)


def quantize_matrix(x, bits: int, group_size: int):
    x = _c(x, np.float64)
    n, d = x.shape
    payload = np.zeros((n * d * bits + 7) // 8, np.uint8)
    scales = np.zeros(n * d // group_size, np.uint8)
    rc = lib().qo_quantize_matrix(_ptr(x), n, d, bits, group_size, _ptr(payload), _ptr(scales))
    if rc:
        raise OracleError(rc)
    return payload, scales


def dequantize_matrix(payload, scales, n, d, bits, group_size) -> np.ndarray:
    payload = _c(payload, np.uint8)
    scales = _c(scales, np.uint8)
    out = np.empty((n, d), np.float32)
    lib().qo_dequantize_matrix(_ptr(payload), _ptr(scales), n, d, bits, group_size, _ptr(out))
    return out


def kmeans_pp(rows, k, draws):
    rows = _c(rows, np.float64)
    n, d = rows.shape
    draws = _c(draws, np.float64)
    cent = np.empty((k, d), np.float64)
    chosen = np.empty(k, np.int64)
    rc = lib().qo_kmeans_pp(_ptr(rows), n, d, k, _ptr(draws), _ptr(cent), _ptr(chosen))
    if rc:
        raise OracleError(rc)
    return cent, chosen


def assign(rows, cent) -> np.ndarray:
    rows = _c(rows, np.float64)
    cent = _c(cent, np.float64)
    out = np.empty(rows.shape[0], np.int32)
    lib().qo_assign(_ptr(rows), rows.shape[0], rows.shape[1], _ptr(cent), cent.shape[0], _ptr(out))
    return out


def lloyd_step(rows, cent):
    """Q/clustering.py:74-107 -> (new centroids, assignments int32, objective)."""
    rows = _c(rows, np.float64)
    cent = np.array(cent, dtype=np.float64, copy=True, order="C")
    asg = np.empty(rows.shape[0], np.int32)
    obj = lib().qo_lloyd_step(_ptr(rows), rows.shape[0], rows.shape[1], _ptr(cent), cent.shape[0], _ptr(asg))
    return cent, asg, obj


def kmeans(rows, k, max_iters, tol, draws=None, init=None):
    rows = _c(rows, np.float64)
    n, d = rows.shape
    cent = np.empty((k, d), np.float64)
    asg = np.empty(n, np.int32)
    obj = ctypes.c_double()
    it = ctypes.c_int32()
    rc = lib().qo_kmeans(_ptr(rows), n, d, k, max_iters, tol,
                         _ptr(None if draws is None else _c(draws, np.float64)),
                         _ptr(None if init is None else _c(init, np.float64)),
                         _ptr(cent), _ptr(asg), ctypes.byref(obj), ctypes.byref(it))
    if rc:
        raise OracleError(rc)
    return cent, asg, obj.value, it.value


def prq_compress(x, bits, group_size, stages, k, max_iters=10, tol=1e-4, draws=None, warm=None):
    """One plane.  Returns dict(payload, scales, centroids[S,K,d] f32 bf16-exact,
    assignments[S,N] u8, centroids_f64[S,K,d], iters[S])."""
    x = _c(x, np.float32)
    n, d = x.shape
    payload = np.zeros((n * d * bits + 7) // 8, np.uint8)
    scales = np.zeros(n * d // group_size, np.uint8)
    cent = np.zeros((stages, k, d), np.float32)
    asg = np.zeros((stages, n), np.uint8)
    c64 = np.zeros((stages, k, d), np.float64)
    iters = np.zeros(stages, np.int32)
    if draws is None and warm is None and stages:
        raise ValueError("need draws or warm")
    rc = lib().qo_prq_compress(_ptr(x), n, d, bits, group_size, stages, k, max_iters, tol,
                               _ptr(None if draws is None else _c(draws, np.float64)),
                               _ptr(None if warm is None else _c(warm, np.float64)),
                               _ptr(payload), _ptr(scales), _ptr(cent), _ptr(asg), _ptr(c64),
                               _ptr(iters))
    if rc:
        raise OracleError(rc)
    return dict(payload=payload, scales=scales, centroids=cent, assignments=asg,
                centroids_f64=c64, iters=iters)


def prq_decompress(payload, scales, centroids, assignments, n, d, bits, group_size) -> np.ndarray:
    centroids = _c(centroids, np.float32)
    assignments = _c(assignments, np.uint8)
    stages = centroids.shape[0] if centroids.ndim == 3 else 0
    k = centroids.shape[1] if stages else 1
    out = np.empty((n, d), np.float32)
    lib().qo_prq_decompress(_ptr(_c(payload, np.uint8)), _ptr(_c(scales, np.uint8)), _ptr(centroids),
                            _ptr(assignments), n, d, bits, group_size, stages, k, _ptr(out))
    return out


def prq_compress_batch(x, bits, group_size, stages, k, max_iters, tol, draws, n_threads):
    """x: [P,N,d] f32; draws: [P,S,K].  Device-layout outputs."""
    x = _c(x, np.float32)
    P, n, d = x.shape
    payload = np.zeros((P, (n * d * bits + 7) // 8), np.uint8)
    scales = np.zeros((P, n * d // group_size), np.uint8)
    cent = np.zeros((P, stages, k, d), np.float32)
    asg = np.zeros((P, stages, n), np.uint8)
    iters = np.zeros((P, stages), np.int32)
    rc = lib().qo_prq_compress_batch(_ptr(x), P, n, d, bits, group_size, stages, k, max_iters, tol,
                                     _ptr(_c(draws, np.float64)), _ptr(payload), _ptr(scales),
                                     _ptr(cent), _ptr(asg), _ptr(iters), n_threads)
    if rc:
        raise OracleError(rc)
    return payload, scales, cent, asg, iters


def prq_decompress_batch(payload, scales, cent, asg, n, d, bits, group_size, n_threads):
    P = payload.shape[0]
    stages, k = cent.shape[1], cent.shape[2]
    out = np.empty((P, n, d), np.float32)
    lib().qo_prq_decompress_batch(_ptr(_c(payload, np.uint8)), _ptr(_c(scales, np.uint8)),
                                  _ptr(_c(cent, np.float32)), _ptr(_c(asg, np.uint8)), P, n, d,
                                  bits, group_size, stages, k, _ptr(out), n_threads)
    return out


def quantize_given_metas_batch(x, cent, asg, bits, group_size, n_threads):
    x = _c(x, np.float32)
    P, n, d = x.shape
    stages = cent.shape[1]
    k = cent.shape[2] if stages else 1
    payload = np.zeros((P, (n * d * bits + 7) // 8), np.uint8)
    scales = np.zeros((P, n * d // group_size), np.uint8)
    rc = lib().qo_quantize_given_metas_batch(_ptr(x), P, n, d, bits, group_size, stages, k,
                                             _ptr(_c(cent, np.float32)), _ptr(_c(asg, np.uint8)),
                                             _ptr(payload), _ptr(scales), n_threads)
    if rc:
        raise OracleError(rc)
    return payload, scales


def attention(q, kc, vc, kn, vn, scale, n_threads=1) -> np.ndarray:
    """q [Nq,H,d]; kc/vc [H,Nc,d] (dequantized cache); kn/vn [Ncur,H,d]; fp64 out [Nq,H,d]."""
    q = _c(q, np.float32)
    nq, h, d = q.shape
    kc = _c(kc, np.float32)
    vc = _c(vc, np.float32)
    nc = kc.shape[1]
    kn = _c(kn, np.float32)
    vn = _c(vn, np.float32)
    ncur = kn.shape[0]
    out = np.empty((nq, h, d), np.float64)
    lib().qo_attention(_ptr(q), _ptr(kc), _ptr(vc), _ptr(kn), _ptr(vn), nq, nc, ncur, h, d,
                       float(scale), _ptr(out), n_threads)
    return out
