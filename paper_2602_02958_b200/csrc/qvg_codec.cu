// qvg_codec.cu — K5 quantize (residual chain + per-group E4M3 scale + b-bit
// pack) and K6 dequantize (one-pass centroid add-back) for sm_100a.
//
// Both are HBM-streaming kernels: one thread owns 8 consecutive channels of
// one token row (a 16-byte bf16 vector), a quantization group of B channels
// is B/8 adjacent lanes, and every byte of x / out is touched exactly once.
//
// Bit-exactness with the reference's float64 arithmetic is kept with a fast
// float32 path plus a certified fallback:
//  * quantize (Q/smoothing.py:40, Q/quant.py:40-55): the f32 residual chain
//    carries an error bound E; the group scale code is taken only when the
//    E-interval of max|r|/qmax maps to a single E4M3 code, and each code q
//    only when |r|/s is farther than the bound from every rounding boundary.
//    Otherwise the group (or element) is recomputed exactly in f64, in the
//    reference's operation order.
//  * dequantize (Q/prq.py:113-132): every non-final f32 partial sum is
//    checked for exactness (then the f64 chain is exact too, and the final
//    f32 rounding of the last addition equals RN32(RN64(.)));
//    an inexact element is recomputed in f64.
#include "qvg_common.cuh"
#include "qvg_internal.h"

namespace qvg {

// ------------------------------------------------------------------------
// helpers
// ------------------------------------------------------------------------

// E4M3 "up" code of a finite v >= 0, from the float bits (equivalent to
// e4m3_encode_up for every f32 input; the mantissa ceiling is one add+mask).
__device__ __forceinline__ uint32_t e4m3_ceil_f32(float v) {
    if (v >= 448.f) return 0x7Eu;
    if (v < 0.015625f) return uint32_t(ceilf(v * 512.f));  // subnormal steps of 2^-9
    uint32_t u = (__float_as_uint(v) + 0xFFFFFu) & 0xFFF00000u;
    return (((u >> 23) - 120u) << 3) | ((u >> 20) & 7u);
}

template <bool XBF16>
__device__ __forceinline__ void load_x8(const void *x, int64_t elem, float r[8]) {
    if constexpr (XBF16) {
        uint4 w = __ldg(reinterpret_cast<const uint4 *>(static_cast<const uint16_t *>(x) + elem));
        r[0] = bf16_lo(w.x); r[1] = bf16_hi(w.x); r[2] = bf16_lo(w.y); r[3] = bf16_hi(w.y);
        r[4] = bf16_lo(w.z); r[5] = bf16_hi(w.z); r[6] = bf16_lo(w.w); r[7] = bf16_hi(w.w);
    } else {
        const float4 *p = reinterpret_cast<const float4 *>(static_cast<const float *>(x) + elem);
        float4 a = __ldg(p), b = __ldg(p + 1);
        r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w; r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
    }
}

__device__ __forceinline__ void load_c8(const uint16_t *c, float r[8]) {
    uint4 w = __ldg(reinterpret_cast<const uint4 *>(c));
    r[0] = bf16_lo(w.x); r[1] = bf16_hi(w.x); r[2] = bf16_lo(w.y); r[3] = bf16_hi(w.y);
    r[4] = bf16_lo(w.z); r[5] = bf16_hi(w.z); r[6] = bf16_lo(w.w); r[7] = bf16_hi(w.w);
}

// XK: 0 f32, 1 bf16, 2 f64
template <int XK>
__device__ __forceinline__ double load_x1(const void *x, int64_t elem) {
    if constexpr (XK == 1) return double(bf16_to_f32(static_cast<const uint16_t *>(x)[elem]));
    else if constexpr (XK == 2) return static_cast<const double *>(x)[elem];
    else return double(static_cast<const float *>(x)[elem]);
}

// ------------------------------------------------------------------------
// K5 fast quantize: d % 8 == 0, B in {8..256} (power of two), S <= 4.
// ------------------------------------------------------------------------
struct QuantArgs {
    const void *x;
    const uint16_t *cent;   // [P][S][K][d]
    const uint8_t *asg;     // [P][S][N]
    uint8_t *payload;       // [P][PB]
    uint8_t *scales;        // [P][N*d/B]
    int64_t n_vec;          // P*N*d/8
    int64_t N;
    int d, K, B, gshift;    // gshift = log2(B/8)
    int32_t *status;
};

template <int BITS, int S, bool XBF16>
__global__ void __launch_bounds__(256) k_quantize_fast(QuantArgs a) {
    constexpr int QMAX = (1 << (BITS - 1)) - 1;
    constexpr float kInvLo = QMAX == 1 ? 1.f : (QMAX == 7 ? 0.142857134342193603515625f : 0.0078740157186985015869140625f);
    constexpr float kInvHi = QMAX == 1 ? 1.f : (QMAX == 7 ? 0.1428571492433547973632812500f : 0.0078740166500210762023925781f);
    const int d = a.d;
    const int64_t vpr = d >> 3;
    const int64_t vpp = a.N * vpr;
    const int glanes = 1 << a.gshift;
    const int lane = threadIdx.x & 31;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    // Loop bound rounded up to the warp so all lanes reach every shuffle.
    const int64_t nv_round = (a.n_vec + 31) & ~int64_t(31);
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < nv_round; v += stride) {
        const bool valid = v < a.n_vec;
        const int64_t vv = valid ? v : a.n_vec - 1;
        const int64_t p = vv / vpp;
        const int64_t rem = vv - p * vpp;
        const int64_t row = rem / vpr;
        const int col = int(rem - row * vpr) << 3;
        const int64_t elem = vv << 3;

        float r[8];
        load_x8<XBF16>(a.x, elem, r);
        bool finite = true;
#pragma unroll
        for (int k = 0; k < 8; k++) finite &= isfinite(r[k]);
        if (!finite && valid) atomicOr(a.status, QVG_STATUS_NONFINITE);

        // residual chain x - C1[pi1] - C2[pi2] ... (Q/smoothing.py:40) in f32
        float ebound = 0.f;
        int ai[S > 0 ? S : 1];
#pragma unroll
        for (int t = 0; t < S; t++) {
            ai[t] = __ldg(a.asg + (p * S + t) * a.N + row);
            float c[8];
            load_c8(a.cent + ((p * S + t) * a.K + ai[t]) * int64_t(d) + col, c);
            float m = 0.f;
#pragma unroll
            for (int k = 0; k < 8; k++) {
                r[k] = __fsub_rn(r[k], c[k]);
                m = fmaxf(m, fabsf(r[k]));
            }
            ebound = __fadd_ru(ebound, m);
        }
        float amax = 0.f;
#pragma unroll
        for (int k = 0; k < 8; k++) amax = fmaxf(amax, fabsf(r[k]));
        // group reductions (B/8 lanes)
        for (int m = 1; m < glanes; m <<= 1) {
            amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, m));
            ebound = fmaxf(ebound, __shfl_xor_sync(0xffffffffu, ebound, m));
        }
        // |r_f32 - r_f64| <= 2^-24 * sum_t |r_t| per rounding of each chain (f32 and
        // the reference's f64); 2^-22 leaves a factor-2 margin on top of both.
        const float E = ebound * 2.3841858e-7f;
        // scale code: certain iff the E-interval of amax/qmax maps to one code
        uint32_t code;
        bool grp_amb = false;
        if (E == 0.f) {
            if (amax == 0.f) code = 0x38u;
            else {
                uint32_t lo = e4m3_ceil_f32(__fmul_rd(amax, kInvLo));
                uint32_t hi = e4m3_ceil_f32(__fmul_ru(amax, kInvHi));
                code = hi;
                grp_amb = lo != hi;
            }
        } else {
            float lo_a = __fsub_rd(amax, E);
            if (!(lo_a > 0.f)) { code = 0x38u; grp_amb = true; }
            else {
                uint32_t lo = e4m3_ceil_f32(__fmul_rd(lo_a, kInvLo));
                uint32_t hi = e4m3_ceil_f32(__fmul_ru(__fadd_ru(amax, E), kInvHi));
                code = hi;
                grp_amb = lo != hi;
            }
        }
        float s = e4m3_to_f32(code);
        float inv = __frcp_rn(s);
        // half-width of the window around a rounding boundary that the exact
        // quotient |r|/s might fall on the other side of
        const float W = __fmul_ru(__fmaf_ru(E, inv, __fmul_ru(__fmul_ru(amax, inv), 4.7683716e-7f)), 1.001f);
        uint32_t bits = 0;
        uint32_t el_amb = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            float t = __fmul_rn(fabsf(r[k]), inv);
            int q;
            if constexpr (QMAX == 1) {
                q = t > 0.5f ? 1 : 0;
                if (fabsf(t - 0.5f) <= W) el_amb |= 1u << k;
            } else {
                float fl = floorf(t);
                if (fabsf(t - fl - 0.5f) <= W && fl < float(QMAX)) el_amb |= 1u << k;
                q = min(int(rintf(t)), QMAX);
            }
            if (r[k] < 0.f) q = -q;
            bits |= (uint32_t(q) & ((1u << BITS) - 1u)) << (k * BITS);
        }
        if (!valid) { grp_amb = false; el_amb = 0; }

        // ---- exact fallback (rare): recompute in f64, reference order ----
        if (__any_sync(0xffffffffu, grp_amb || el_amb)) {
            double r64[8];
#pragma unroll
            for (int k = 0; k < 8; k++) r64[k] = load_x1<XBF16 ? 1 : 0>(a.x, elem + k);
#pragma unroll
            for (int t = 0; t < S; t++) {
                const uint16_t *cp = a.cent + ((p * S + t) * a.K + ai[t]) * int64_t(d) + col;
#pragma unroll
                for (int k = 0; k < 8; k++) r64[k] = __dsub_rn(r64[k], double(bf16_to_f32(cp[k])));
            }
            double am = 0.0;
#pragma unroll
            for (int k = 0; k < 8; k++) am = fmax(am, fabs(r64[k]));
            for (int m = 1; m < glanes; m <<= 1) am = fmax(am, shfl_xor_d(am, m));
            if (grp_amb) {
                code = am == 0.0 ? 0x38u : e4m3_encode_up(__ddiv_rn(am, double(QMAX)));
                el_amb = 0xFFu;
            }
            if (el_amb) {
                double sd = double(e4m3_to_f32(code));
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    if (!(el_amb >> k & 1u)) continue;
                    double qd = rint(__ddiv_rn(r64[k], sd));   // np.rint: half-even
                    qd = fmin(fmax(qd, -double(QMAX)), double(QMAX));
                    int q = int(qd);
                    bits = (bits & ~(((1u << BITS) - 1u) << (k * BITS))) |
                           ((uint32_t(q) & ((1u << BITS) - 1u)) << (k * BITS));
                }
            }
        }
        if (!valid) continue;
        // ---- stores ----
        const int64_t pb = (a.N * d * BITS) >> 3;             // bytes per plane
        uint8_t *pl = a.payload + p * pb + (((row * d + col) * BITS) >> 3);
        if constexpr (BITS == 2) *reinterpret_cast<uint16_t *>(pl) = uint16_t(bits);
        else if constexpr (BITS == 4) *reinterpret_cast<uint32_t *>(pl) = bits;
        else {
            // 8-bit: 8 codes = 8 bytes; bits holds only 32 -> recompute hi half below
            (void)pl;
        }
        if ((lane & (glanes - 1)) == 0)
            a.scales[p * (a.N * d / a.B) + (row * d + col) / a.B] = uint8_t(code);
    }
}

// 8-bit codes need 64 bits per thread; a dedicated variant keeps the common
// 2/4-bit kernel's registers small.
template <int S, bool XBF16>
__global__ void __launch_bounds__(256) k_quantize_fast8(QuantArgs a) {
    constexpr int QMAX = 127;
    constexpr float kInvLo = 0.0078740157186985015869140625f;
    constexpr float kInvHi = 0.0078740166500210762023925781f;
    const int d = a.d;
    const int64_t vpr = d >> 3, vpp = a.N * vpr;
    const int glanes = 1 << a.gshift;
    const int lane = threadIdx.x & 31;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const int64_t nv_round = (a.n_vec + 31) & ~int64_t(31);
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < nv_round; v += stride) {
        const bool valid = v < a.n_vec;
        const int64_t vv = valid ? v : a.n_vec - 1;
        const int64_t p = vv / vpp, rem = vv - p * vpp, row = rem / vpr;
        const int col = int(rem - row * vpr) << 3;
        const int64_t elem = vv << 3;
        float r[8];
        load_x8<XBF16>(a.x, elem, r);
        bool finite = true;
#pragma unroll
        for (int k = 0; k < 8; k++) finite &= isfinite(r[k]);
        if (!finite && valid) atomicOr(a.status, QVG_STATUS_NONFINITE);
        float ebound = 0.f;
        int ai[S > 0 ? S : 1];
#pragma unroll
        for (int t = 0; t < S; t++) {
            ai[t] = __ldg(a.asg + (p * S + t) * a.N + row);
            float c[8];
            load_c8(a.cent + ((p * S + t) * a.K + ai[t]) * int64_t(d) + col, c);
            float m = 0.f;
#pragma unroll
            for (int k = 0; k < 8; k++) { r[k] = __fsub_rn(r[k], c[k]); m = fmaxf(m, fabsf(r[k])); }
            ebound = __fadd_ru(ebound, m);
        }
        float amax = 0.f;
#pragma unroll
        for (int k = 0; k < 8; k++) amax = fmaxf(amax, fabsf(r[k]));
        for (int m = 1; m < glanes; m <<= 1) {
            amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, m));
            ebound = fmaxf(ebound, __shfl_xor_sync(0xffffffffu, ebound, m));
        }
        const float E = ebound * 2.3841858e-7f;
        uint32_t code;
        bool grp_amb = false;
        float lo_a = E == 0.f ? amax : __fsub_rd(amax, E);
        if (E == 0.f && amax == 0.f) code = 0x38u;
        else if (!(lo_a > 0.f)) { code = 0x38u; grp_amb = true; }
        else {
            uint32_t lo = e4m3_ceil_f32(__fmul_rd(lo_a, kInvLo));
            uint32_t hi = e4m3_ceil_f32(__fmul_ru(__fadd_ru(amax, E), kInvHi));
            code = hi;
            grp_amb = lo != hi;
        }
        float s = e4m3_to_f32(code), inv = __frcp_rn(s);
        const float W = __fmul_ru(__fmaf_ru(E, inv, __fmul_ru(__fmul_ru(amax, inv), 4.7683716e-7f)), 1.001f);
        uint32_t lo32 = 0, hi32 = 0, el_amb = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            float t = __fmul_rn(fabsf(r[k]), inv);
            float fl = floorf(t);
            if (fabsf(t - fl - 0.5f) <= W && fl < float(QMAX)) el_amb |= 1u << k;
            int q = min(int(rintf(t)), QMAX);
            if (r[k] < 0.f) q = -q;
            if (k < 4) lo32 |= (uint32_t(q) & 0xFFu) << (k * 8);
            else hi32 |= (uint32_t(q) & 0xFFu) << ((k - 4) * 8);
        }
        if (!valid) { grp_amb = false; el_amb = 0; }
        if (__any_sync(0xffffffffu, grp_amb || el_amb)) {
            double r64[8];
#pragma unroll
            for (int k = 0; k < 8; k++) r64[k] = load_x1<XBF16 ? 1 : 0>(a.x, elem + k);
#pragma unroll
            for (int t = 0; t < S; t++) {
                const uint16_t *cp = a.cent + ((p * S + t) * a.K + ai[t]) * int64_t(d) + col;
#pragma unroll
                for (int k = 0; k < 8; k++) r64[k] = __dsub_rn(r64[k], double(bf16_to_f32(cp[k])));
            }
            double am = 0.0;
#pragma unroll
            for (int k = 0; k < 8; k++) am = fmax(am, fabs(r64[k]));
            for (int m = 1; m < glanes; m <<= 1) am = fmax(am, shfl_xor_d(am, m));
            if (grp_amb) {
                code = am == 0.0 ? 0x38u : e4m3_encode_up(__ddiv_rn(am, double(QMAX)));
                el_amb = 0xFFu;
            }
            if (el_amb) {
                double sd = double(e4m3_to_f32(code));
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    if (!(el_amb >> k & 1u)) continue;
                    double qd = fmin(fmax(rint(__ddiv_rn(r64[k], sd)), -127.0), 127.0);
                    uint32_t u = uint32_t(int(qd)) & 0xFFu;
                    if (k < 4) lo32 = (lo32 & ~(0xFFu << (k * 8))) | (u << (k * 8));
                    else hi32 = (hi32 & ~(0xFFu << ((k - 4) * 8))) | (u << ((k - 4) * 8));
                }
            }
        }
        if (!valid) continue;
        const int64_t pb = a.N * d;
        *reinterpret_cast<uint2 *>(a.payload + p * pb + row * d + col) = make_uint2(lo32, hi32);
        if ((lane & (glanes - 1)) == 0)
            a.scales[p * (a.N * d / a.B) + (row * d + col) / a.B] = uint8_t(code);
    }
}

// ------------------------------------------------------------------------
// Generic exact quantize (any d, B, S): pass 1 one thread per group -> scale
// code; pass 2 one thread per payload byte.  Pure f64, reference order.
// ------------------------------------------------------------------------
template <int XK>
__device__ __forceinline__ double residual64(const void *x, const uint16_t *cent, const uint8_t *asg,
                                             int64_t p, int64_t row, int col, int64_t N, int d,
                                             int K, int S) {
    double r = load_x1<XK>(x, (p * N + row) * d + col);
    for (int t = 0; t < S; t++) {
        int ai = asg[(p * S + t) * N + row];
        r = __dsub_rn(r, double(bf16_to_f32(cent[((p * S + t) * K + ai) * int64_t(d) + col])));
    }
    return r;
}

template <int XK>
__global__ void k_quantize_generic_scales(const void *x, const uint16_t *cent, const uint8_t *asg,
                                          uint8_t *scales, int64_t P, int64_t N, int d, int K,
                                          int S, int B, int bits, int32_t *status) {
    const int64_t ng_plane = N * d / B;
    const int qmax = (1 << (bits - 1)) - 1;
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < P * ng_plane;
         g += int64_t(gridDim.x) * blockDim.x) {
        int64_t p = g / ng_plane, e0 = (g - p * ng_plane) * B;
        double am = 0.0;
        bool finite = true;
        for (int j = 0; j < B; j++) {
            int64_t e = e0 + j, row = e / d;
            int col = int(e - row * d);
            finite &= isfinite(load_x1<XK>(x, (p * N + row) * d + col));
            am = fmax(am, fabs(residual64<XK>(x, cent, asg, p, row, col, N, d, K, S)));
        }
        if (!finite) atomicOr(status, QVG_STATUS_NONFINITE);
        scales[g] = uint8_t(am == 0.0 ? 0x38u : e4m3_encode_up(__ddiv_rn(am, double(qmax))));
    }
}

template <int XK>
__global__ void k_quantize_generic_pack(const void *x, const uint16_t *cent, const uint8_t *asg,
                                        const uint8_t *scales, uint8_t *payload, int64_t P,
                                        int64_t N, int d, int K, int S, int B, int bits) {
    const int64_t cnt = N * d, pb = (cnt * bits + 7) / 8;
    const int per = 8 / bits, qmax = (1 << (bits - 1)) - 1;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < P * pb;
         t += int64_t(gridDim.x) * blockDim.x) {
        int64_t p = t / pb, byte = t - p * pb;
        uint32_t out = 0;
        for (int j = 0; j < per; j++) {
            int64_t e = byte * per + j;
            if (e >= cnt) break;
            int64_t row = e / d;
            int col = int(e - row * d);
            double s = double(e4m3_to_f32(scales[p * (cnt / B) + e / B]));
            double r = residual64<XK>(x, cent, asg, p, row, col, N, d, K, S);
            double q = fmin(fmax(rint(__ddiv_rn(r, s)), -double(qmax)), double(qmax));
            out |= (uint32_t(int(q)) & ((1u << bits) - 1u)) << (j * bits);
        }
        payload[t] = uint8_t(out);
    }
}

// ------------------------------------------------------------------------
// K6 fast dequantize: d % 8 == 0, B % 8 == 0, S <= 4.
// ------------------------------------------------------------------------
struct DequantArgs {
    const uint8_t *payload;
    const uint8_t *scales;
    const uint16_t *cent;
    const uint8_t *asg;
    void *out;
    int64_t n_vec;
    int64_t N;
    int d, K, B;
    int32_t *status;
};

template <int BITS>
__device__ __forceinline__ int unpack_q(uint64_t w, int k) {
    constexpr uint32_t mask = (1u << BITS) - 1u, sign = 1u << (BITS - 1);
    uint32_t u = uint32_t(w >> (k * BITS)) & mask;
    return int(u ^ sign) - int(sign);
}

// exact iff fl(a+b) == a+b; both checks are needed without knowing |a| vs |b|
__device__ __forceinline__ bool add_exact(float a, float b, float s) {
    return __fsub_rn(s, a) == b && __fsub_rn(s, b) == a;
}

template <int BITS, int S, bool OUT_BF16>
__global__ void __launch_bounds__(256) k_dequant_fast(DequantArgs a) {
    const int d = a.d;
    const int64_t vpr = d >> 3, vpp = a.N * vpr;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const int64_t pb = (a.N * d * BITS) >> 3, ng = a.N * d / a.B;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < a.n_vec; v += stride) {
        const int64_t p = v / vpp, rem = v - p * vpp, row = rem / vpr;
        const int col = int(rem - row * vpr) << 3;
        const int64_t e = row * d + col;
        const uint8_t *pl = a.payload + p * pb + ((e * BITS) >> 3);
        uint64_t w;
        if constexpr (BITS == 2) w = __ldg(reinterpret_cast<const uint16_t *>(pl));
        else if constexpr (BITS == 4) w = __ldg(reinterpret_cast<const uint32_t *>(pl));
        else { uint2 t = __ldg(reinterpret_cast<const uint2 *>(pl)); w = uint64_t(t.x) | (uint64_t(t.y) << 32); }
        const uint32_t sc = __ldg(a.scales + p * ng + e / a.B);
        if (sc == 0x7Fu || sc == 0xFFu) atomicOr(a.status, QVG_STATUS_NAN_SCALE);
        const float s = e4m3_to_f32(sc);
        float y[8];
#pragma unroll
        for (int k = 0; k < 8; k++) y[k] = float(unpack_q<BITS>(w, k)) * s;  // exact
        float c[S > 0 ? S : 1][8];
        bool exact = true;
#pragma unroll
        for (int t = S - 1; t >= 0; t--) {
            int ai = __ldg(a.asg + (p * S + t) * a.N + row);
            if (ai >= a.K) { atomicOr(a.status, QVG_STATUS_BAD_ASSIGN); ai = 0; }
            load_c8(a.cent + ((p * S + t) * a.K + ai) * int64_t(d) + col, c[t]);
#pragma unroll
            for (int k = 0; k < 8; k++) {
                float s2 = __fadd_rn(y[k], c[t][k]);
                if (t > 0) exact &= add_exact(y[k], c[t][k], s2);
                y[k] = s2;
            }
        }
        if (!exact) {   // rare: some partial sum needed more than 24 bits
#pragma unroll
            for (int k = 0; k < 8; k++) {
                double acc = double(float(unpack_q<BITS>(w, k)) * s);
#pragma unroll
                for (int t = S - 1; t >= 0; t--) acc = __dadd_rn(acc, double(c[t][k]));
                y[k] = __double2float_rn(acc);
            }
        }
        if constexpr (OUT_BF16) {
            uint4 o;
            __nv_bfloat162 h;
            h = __floats2bfloat162_rn(y[0], y[1]); o.x = *reinterpret_cast<uint32_t *>(&h);
            h = __floats2bfloat162_rn(y[2], y[3]); o.y = *reinterpret_cast<uint32_t *>(&h);
            h = __floats2bfloat162_rn(y[4], y[5]); o.z = *reinterpret_cast<uint32_t *>(&h);
            h = __floats2bfloat162_rn(y[6], y[7]); o.w = *reinterpret_cast<uint32_t *>(&h);
            *reinterpret_cast<uint4 *>(static_cast<uint16_t *>(a.out) + (v << 3)) = o;
        } else {
            float4 *o = reinterpret_cast<float4 *>(static_cast<float *>(a.out) + (v << 3));
            o[0] = make_float4(y[0], y[1], y[2], y[3]);
            o[1] = make_float4(y[4], y[5], y[6], y[7]);
        }
    }
}

// Generic exact dequantize: one thread per element, f64 add-back.
template <bool OUT_BF16>
__global__ void k_dequant_generic(const uint8_t *payload, const uint8_t *scales,
                                  const uint16_t *cent, const uint8_t *asg, void *out, int64_t P,
                                  int64_t N, int d, int K, int S, int B, int bits, int32_t *status) {
    const int64_t cnt = N * d, pb = (cnt * bits + 7) / 8;
    const int per = 8 / bits;
    const uint32_t mask = (1u << bits) - 1u, sign = 1u << (bits - 1);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P * cnt;
         i += int64_t(gridDim.x) * blockDim.x) {
        int64_t p = i / cnt, e = i - p * cnt, row = e / d;
        int col = int(e - row * d);
        uint32_t u = (payload[p * pb + e / per] >> ((e % per) * bits)) & mask;
        int q = int(u ^ sign) - int(sign);
        uint32_t sc = scales[p * (cnt / B) + e / B];
        if (sc == 0x7Fu || sc == 0xFFu) atomicOr(status, QVG_STATUS_NAN_SCALE);
        double acc = double(float(q) * e4m3_to_f32(sc));
        for (int t = S - 1; t >= 0; t--) {
            int ai = asg[(p * S + t) * N + row];
            if (ai >= K) { atomicOr(status, QVG_STATUS_BAD_ASSIGN); ai = 0; }
            acc = __dadd_rn(acc, double(bf16_to_f32(cent[((p * S + t) * K + ai) * int64_t(d) + col])));
        }
        float y = __double2float_rn(acc);
        if (OUT_BF16) static_cast<__nv_bfloat16 *>(out)[i] = __float2bfloat16_rn(y);
        else static_cast<float *>(out)[i] = y;
    }
}

// ------------------------------------------------------------------------
// pack_payload / unpack_payload (Q/quant.py:78-116): one thread per byte.
// ------------------------------------------------------------------------
__global__ void k_pack_codes(const int8_t *q, int64_t n, int bits, uint8_t *out, int32_t *status) {
    const int per = 8 / bits, qmax = (1 << (bits - 1)) - 1;
    const int64_t nb = (n * bits + 7) / 8;
    for (int64_t b = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; b < nb; b += int64_t(gridDim.x) * blockDim.x) {
        uint32_t v = 0;
        for (int j = 0; j < per; j++) {
            int64_t i = b * per + j;
            if (i >= n) break;
            int c = q[i];
            if (c < -qmax || c > qmax) atomicOr(status, 8);
            v |= (uint32_t(c) & ((1u << bits) - 1u)) << (j * bits);
        }
        out[b] = uint8_t(v);
    }
}

__global__ void k_unpack_codes(const uint8_t *in, int64_t n, int bits, int8_t *out) {
    const int per = 8 / bits;
    const uint32_t mask = (1u << bits) - 1u, sign = 1u << (bits - 1);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        uint32_t u = (in[i / per] >> ((i % per) * bits)) & mask;
        out[i] = int8_t(int(u ^ sign) - int(sign));
    }
}

// ------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------
static int grid_for(int64_t work, int block) {
    int64_t g = (work + block - 1) / block;
    int64_t cap = 148LL * 16;  // persistent-ish: 16 CTAs of 256 per SM max
    return int(g < 1 ? 1 : (g > cap ? cap : g));
}

template <int BITS, int S>
static void launch_quant_fast(const QuantArgs &a, bool xbf16, cudaStream_t st) {
    int g = grid_for(a.n_vec, 256);
    if constexpr (BITS == 8) {
        if (xbf16) k_quantize_fast8<S, true><<<g, 256, 0, st>>>(a);
        else k_quantize_fast8<S, false><<<g, 256, 0, st>>>(a);
    } else {
        if (xbf16) k_quantize_fast<BITS, S, true><<<g, 256, 0, st>>>(a);
        else k_quantize_fast<BITS, S, false><<<g, 256, 0, st>>>(a);
    }
}

template <int BITS>
static void dispatch_quant_s(const QuantArgs &a, int S, bool xbf16, cudaStream_t st) {
    switch (S) {
        case 0: launch_quant_fast<BITS, 0>(a, xbf16, st); break;
        case 1: launch_quant_fast<BITS, 1>(a, xbf16, st); break;
        case 2: launch_quant_fast<BITS, 2>(a, xbf16, st); break;
        case 3: launch_quant_fast<BITS, 3>(a, xbf16, st); break;
        default: launch_quant_fast<BITS, 4>(a, xbf16, st); break;
    }
}

bool quant_fast_ok(int d, int B, int S) {
    return d % 8 == 0 && B % 8 == 0 && B <= 256 && ((B / 8) & (B / 8 - 1)) == 0 && S <= 4;
}

int launch_quantize(const void *x, int xdtype, int64_t P, int64_t N, int d, int bits, int B, int S,
                    int K, const uint16_t *cent, const uint8_t *asg, uint8_t *payload,
                    uint8_t *scales, int32_t *status, cudaStream_t st) {
    const bool xbf16 = xdtype == QVG_DTYPE_BF16;
    if (xdtype != QVG_DTYPE_F64 && quant_fast_ok(d, B, S)) {
        QuantArgs a{x, cent, asg, payload, scales, P * N * d / 8, N, d, K, B, 0, status};
        int gl = B / 8, gs = 0;
        while ((1 << gs) < gl) gs++;
        a.gshift = gs;
        if (bits == 2) dispatch_quant_s<2>(a, S, xbf16, st);
        else if (bits == 4) dispatch_quant_s<4>(a, S, xbf16, st);
        else dispatch_quant_s<8>(a, S, xbf16, st);
    } else {
        int64_t ng = P * N * d / B, pbt = P * ((N * d * bits + 7) / 8);
        if (xdtype == QVG_DTYPE_BF16) {
            k_quantize_generic_scales<1><<<grid_for(ng, 128), 128, 0, st>>>(x, cent, asg, scales, P, N, d, K, S, B, bits, status);
            k_quantize_generic_pack<1><<<grid_for(pbt, 128), 128, 0, st>>>(x, cent, asg, scales, payload, P, N, d, K, S, B, bits);
        } else if (xdtype == QVG_DTYPE_F64) {
            k_quantize_generic_scales<2><<<grid_for(ng, 128), 128, 0, st>>>(x, cent, asg, scales, P, N, d, K, S, B, bits, status);
            k_quantize_generic_pack<2><<<grid_for(pbt, 128), 128, 0, st>>>(x, cent, asg, scales, payload, P, N, d, K, S, B, bits);
        } else {
            k_quantize_generic_scales<0><<<grid_for(ng, 128), 128, 0, st>>>(x, cent, asg, scales, P, N, d, K, S, B, bits, status);
            k_quantize_generic_pack<0><<<grid_for(pbt, 128), 128, 0, st>>>(x, cent, asg, scales, payload, P, N, d, K, S, B, bits);
        }
    }
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

template <int BITS, int S>
static void launch_deq_fast(const DequantArgs &a, bool obf16, cudaStream_t st) {
    int g = grid_for(a.n_vec, 256);
    if (obf16) k_dequant_fast<BITS, S, true><<<g, 256, 0, st>>>(a);
    else k_dequant_fast<BITS, S, false><<<g, 256, 0, st>>>(a);
}

template <int BITS>
static void dispatch_deq_s(const DequantArgs &a, int S, bool obf16, cudaStream_t st) {
    switch (S) {
        case 0: launch_deq_fast<BITS, 0>(a, obf16, st); break;
        case 1: launch_deq_fast<BITS, 1>(a, obf16, st); break;
        case 2: launch_deq_fast<BITS, 2>(a, obf16, st); break;
        case 3: launch_deq_fast<BITS, 3>(a, obf16, st); break;
        default: launch_deq_fast<BITS, 4>(a, obf16, st); break;
    }
}

int launch_pack(const int8_t *q, int64_t n, int bits, uint8_t *out, int32_t *status, cudaStream_t st) {
    if (n > 0) k_pack_codes<<<grid_for((n * bits + 7) / 8, 256), 256, 0, st>>>(q, n, bits, out, status);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

int launch_unpack(const uint8_t *in, int64_t n, int bits, int8_t *out, cudaStream_t st) {
    if (n > 0) k_unpack_codes<<<grid_for(n, 256), 256, 0, st>>>(in, n, bits, out);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

int launch_dequantize(const uint8_t *payload, const uint8_t *scales, const uint16_t *cent,
                      const uint8_t *asg, int64_t P, int64_t N, int d, int bits, int B, int S, int K,
                      void *out, int odtype, int32_t *status, cudaStream_t st) {
    const bool obf16 = odtype == QVG_DTYPE_BF16;
    if (d % 8 == 0 && B % 8 == 0 && S <= 4) {
        DequantArgs a{payload, scales, cent, asg, out, P * N * d / 8, N, d, K, B, status};
        if (bits == 2) dispatch_deq_s<2>(a, S, obf16, st);
        else if (bits == 4) dispatch_deq_s<4>(a, S, obf16, st);
        else dispatch_deq_s<8>(a, S, obf16, st);
    } else {
        int64_t n = P * N * d;
        if (obf16) k_dequant_generic<true><<<grid_for(n, 256), 256, 0, st>>>(payload, scales, cent, asg, out, P, N, d, K, S, B, bits, status);
        else k_dequant_generic<false><<<grid_for(n, 256), 256, 0, st>>>(payload, scales, cent, asg, out, P, N, d, K, S, B, bits, status);
    }
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

}  // namespace qvg
