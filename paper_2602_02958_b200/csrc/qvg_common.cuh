// qvg_common.cuh — shared device helpers for the sm_100a QVG kernels.
//
// Numerics contract (restated from the reference, see oracle/qvg_oracle.c):
//  * E4M3 scales with "up" rounding and the 0x38 zero-group rule
//    (Q/lowprec.py:55-84, Q/quant.py:40-45);
//  * bf16 centroid rounding f64 -> f32 (RNE) -> bf16 (RNE bit trick)
//    (Q/smoothing.py:39, Q/lowprec.py:112-120);
//  * numpy pairwise summation for every ndarray.sum() on the k-means path.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "../../include/qvg.h"

namespace qvg {

constexpr int kMaxK = 256;

// ---- bf16 <-> f32 (bit level, exact) -----------------------------------
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ float bf16_to_f32(uint16_t h) { return __uint_as_float(uint32_t(h) << 16); }

// round_to_bf16 on a float32 (Q/lowprec.py:112-120): RNE, kept as bits.
__host__ __device__ __forceinline__ uint16_t f32_to_bf16_bits_rne(float f) {
#ifdef __CUDA_ARCH__
    uint32_t u = __float_as_uint(f);
#else
    uint32_t u;
    memcpy(&u, &f, 4);
#endif
    u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
    return uint16_t(u >> 16);
}

// ---- E4M3 (Q/lowprec.py:36-52, 87-92) -----------------------------------
// Exact value of a non-NaN E4M3 byte as float (all codes are f32-exact).
__device__ __forceinline__ float e4m3_to_f32(uint32_t b) {
    uint32_t e = (b >> 3) & 0xFu, m = b & 7u;
    float v = e ? __uint_as_float(((e + 120u) << 23) | (m << 20)) : float(m) * 0.001953125f;
    return (b & 0x80u) ? -v : v;
}

// fp8_e4m3_encode_array(x, "up") for one finite x >= 0 (Q/lowprec.py:55-84).
__device__ __forceinline__ uint32_t e4m3_encode_up(double x) {
    if (x > 448.0) x = 448.0;
    if (x == 0.0) return 0u;
    int e2;
    frexp(x, &e2);
    int e = e2 - 1;
    if (e < -6) e = -6;
    double k = ceil(ldexp(x, 3 - e));   // exact power-of-two scaling
    int ki = int(k);
    if (ki == 16) { e += 1; ki = 8; }
    if (e >= 8 && ki > 14) ki = 14;
    if (e > 8) e = 8;
    return ki >= 8 ? uint32_t(((e + 7) << 3) | (ki - 8)) : uint32_t(ki);
}

// ---- warp helpers ---------------------------------------------------------
__device__ __forceinline__ double shfl_xor_d(double v, int m, unsigned mask = 0xffffffffu) {
    return __shfl_xor_sync(mask, v, m);
}

// numpy pairwise_sum over n <= 128 values held 8 lanes wide: lane j (0..7)
// of an 8-lane group passes acc = v[j] + v[j+8] + ... (sequential, the
// r[j] accumulators of numpy's unrolled loop over floor(n/8)*8 elements);
// returns ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) in every lane of the group.
// IEEE addition is commutative, so the xor butterfly reproduces the tree.
__device__ __forceinline__ double pairwise8_tree(double acc) {
    acc += shfl_xor_d(acc, 1);
    acc += shfl_xor_d(acc, 2);
    acc += shfl_xor_d(acc, 4);
    return acc;
}

struct StatusFlag {
    int32_t *p;
    __device__ __forceinline__ void set(int bit) const { if (p) atomicOr(p, bit); }
};

}  // namespace qvg
