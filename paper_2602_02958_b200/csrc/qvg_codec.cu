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
#include <cstdlib>
#include <cstring>

#include "qvg_common.cuh"
#include "qvg_internal.h"
#include "qvg_codec_dev.cuh"

namespace qvg {


template <int BITS, int S, bool XBF16>
__global__ void __launch_bounds__(256) k_quantize_v3(QuantArgs a) {
    constexpr int QMAX = (1 << (BITS - 1)) - 1;
    constexpr uint64_t FMASK = (1u << BITS) - 1u;
    constexpr int SS = S > 0 ? S : 1;
    const uint32_t d = uint32_t(a.d), N = a.N;
    const int col = int(threadIdx.x & ((1u << a.lvpr) - 1u)) << 3;
    const uint32_t rslot = threadIdx.x >> a.lvpr;
    const int glanes = 1 << a.gshift;
    const int lane = threadIdx.x & 31;
    uint32_t stat = 0;
    for (uint32_t T = blockIdx.x; T < a.ta.n_tiles; T += gridDim.x) {
        const uint32_t p = a.ta.div_tpp.div(T);
        const uint32_t i0 = (T - p * a.ta.tpp) * a.ta.rows_per_pass * kUnroll;
        const uint64_t pN = uint64_t(p) * N;
        const uint8_t *xb = static_cast<const uint8_t *>(a.x) + pN * d * (XBF16 ? 2 : 4);
        const uint8_t *ap = a.asg + pN * S;
        const uint16_t *cp = a.cent + uint64_t(p) * S * a.K * d;
        float r[kUnroll][8];
        uint32_t ii[kUnroll];
        int ai[kUnroll][SS];
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
            const uint32_t i = i0 + u * a.ta.rows_per_pass + rslot;
            ii[u] = i < N ? i : N - 1;
            load_x8<XBF16>(xb, int64_t(ii[u] * d + col), r[u]);
#pragma unroll
            for (int t = 0; t < S; t++) ai[u][t] = __ldg(ap + t * N + ii[u]);
        }
        float eb[kUnroll], am[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
            bool fin = true;
#pragma unroll
            for (int k = 0; k < 8; k++) fin &= isfinite(r[u][k]);
            if (!fin) stat |= QVG_STATUS_NONFINITE;
            float e = 0.f;
#pragma unroll
            for (int t = 0; t < S; t++) {
                float c[8];
                load_c8(cp + (uint32_t(t * a.K + ai[u][t]) * d + col), c);
                float m = 0.f;
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    r[u][k] = __fsub_rn(r[u][k], c[k]);
                    m = fmaxf(m, fabsf(r[u][k]));
                }
                e = __fadd_ru(e, m);
            }
            float mx = 0.f;
#pragma unroll
            for (int k = 0; k < 8; k++) mx = fmaxf(mx, fabsf(r[u][k]));
            eb[u] = e;
            am[u] = mx;
        }
        for (int m = 1; m < glanes; m <<= 1) {
#pragma unroll
            for (int u = 0; u < kUnroll; u++) {
                am[u] = fmaxf(am[u], __shfl_xor_sync(0xffffffffu, am[u], m));
                eb[u] = fmaxf(eb[u], __shfl_xor_sync(0xffffffffu, eb[u], m));
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
            const bool valid = i0 + u * a.ta.rows_per_pass + rslot < N;
            // |r_f32 - r_ref| <= 2^-24 sum_t|r_t| (f32 chain) + 2^-53 (.) (the
            // reference's f64 chain) <= 2^-22 * sum_t max|r_t|: factor-2 margin
            const float E = __fmul_ru(eb[u], 2.38418579e-7f);
            uint32_t code;
            bool camb = false;
            if (am[u] == 0.f && E == 0.f) code = 0x38u;
            else {
                float lo = __fsub_rd(am[u], E), hi = __fadd_ru(am[u], E);
                if (lo > 0.f) code = scale_code<QMAX>(lo, hi, camb);
                else { code = 0x38u; camb = true; }
            }
            camb &= valid;
            auto exact_r = [&](int k) {   // the reference's f64 residual (rare path)
                return exact_residual<XBF16, S>(xb, cp, ii[u] * d + col + k, col + k, d, a.K,
                                                ai[u][0], ai[u][SS > 1 ? 1 : 0], ai[u][SS > 2 ? 2 : 0],
                                                ai[u][SS > 3 ? 3 : 0]);
            };
            // ---- exact scale (rare): max of the exact residual over the candidates
            if (__any_sync(0xffffffffu, camb)) {
                const float thr = __fsub_rd(am[u], __fmul_ru(E, 2.f));
                double a64 = 0.0;
                if (camb) {
#pragma unroll
                    for (int k = 0; k < 8; k++)
                        if (fabsf(r[u][k]) >= thr) a64 = fmax(a64, fabs(exact_r(k)));
                }
                for (int m = 1; m < glanes; m <<= 1) a64 = fmax(a64, shfl_xor_d(a64, m));
                if (camb) code = a64 == 0.0 ? 0x38u : e4m3_encode_up(__ddiv_rn(a64, double(QMAX)));
            }
            const float s = e4m3_to_f32(code);
            uint64_t bits = 0;
            uint32_t el_amb = 0;
            if constexpr (QMAX == 1) {
                // q != 0  <=>  RN64(|r|/s) > 0.5  <=>  |r| > s/2 for an f32-exact r
                const float wlo = __fsub_rd(0.5f * s, E), whi = __fadd_ru(0.5f * s, E);
                uint32_t b32 = 0;
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const float av = fabsf(r[u][k]);
                    const bool one = av > whi;
                    if (!one && !(av < wlo)) el_amb |= 1u << k;
                    const uint32_t f = one ? ((__float_as_uint(r[u][k]) >> 30) | 1u) : 0u;  // 1 or 3
                    b32 |= f << (2 * k);
                }
                bits = b32;
            } else {
                const float inv = __frcp_rn(s);
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const float av = fabsf(r[u][k]);
                    const float t = av * inv;
                    const float fl = floorf(t);
                    const float hb = (fl + 0.5f) * s;                    // exact
                    const float w = __fmaf_ru(hb, 2.38418579e-7f, E);
                    if (fl < float(QMAX) && av >= __fsub_rd(hb, w) && av <= __fadd_ru(hb, w)) el_amb |= 1u << k;
                    int q = min(int(rintf(fminf(t, float(QMAX + 1)))), QMAX);   // saturated scales: |r/s| >> QMAX
                    if (r[u][k] < 0.f) q = -q;
                    bits |= (uint64_t(uint32_t(q)) & FMASK) << (k * BITS);
                }
            }
            if (!valid) el_amb = 0;
            // ---- exact codes (rare): elements inside the error window of a boundary
            if (__any_sync(0xffffffffu, el_amb != 0)) {
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    if (!(el_amb >> k & 1u)) continue;
                    const uint32_t q = exact_code<QMAX>(exact_r(k), s);
                    bits = (bits & ~(FMASK << (k * BITS))) | ((uint64_t(q) & FMASK) << (k * BITS));
                }
            }
            if (!valid) continue;
            const uint32_t e0 = ii[u] * d + col;                               // element in plane
            uint8_t *pl = a.payload + uint64_t(p) * a.pb + ((e0 * BITS) >> 3);
            if constexpr (BITS == 2) *reinterpret_cast<uint16_t *>(pl) = uint16_t(bits);
            else if constexpr (BITS == 4) *reinterpret_cast<uint32_t *>(pl) = uint32_t(bits);
            else *reinterpret_cast<uint2 *>(pl) = make_uint2(uint32_t(bits), uint32_t(bits >> 32));
            if ((lane & (glanes - 1)) == 0) a.scales[uint64_t(p) * a.ng + (e0 >> a.lgB)] = uint8_t(code);
        }
    }
    stat = __reduce_or_sync(0xffffffffu, stat);
    if (stat && lane == 0) atomicOr(a.status, int(stat));
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
// K6 dequantize (fast path: d/8 and B powers of two, B % 8 == 0, S <= 4)
// ------------------------------------------------------------------------

// signed b-bit field k of w as an exact float: (u ^ sign) - sign via the
// 1.5*2^23 magic (used by the rare f64 path)
template <int BITS>
__device__ __forceinline__ float qfield(uint64_t w, int k) {
    constexpr uint32_t mask = (1u << BITS) - 1u, sign = 1u << (BITS - 1);
    const uint32_t u = uint32_t(w >> (k * BITS)) & mask;
    return __int_as_float(0x4B400000u | (u ^ sign)) - float(0xC00000u + sign);
}

// q*s for field k in one FFMA: with u' = u ^ sign placed at the top of the f32
// mantissa, f = 1 + u'/2^b and q = u' - 2^(b-1) = 2^b f - 3*2^(b-1), so
// q*s = fma(f, 2^b s, -3*2^(b-1) s).  Both products of s are exact (s has 4
// significant bits) and the fused result q*s is representable: exact.
template <int BITS>
__device__ __forceinline__ float qs_fma(uint64_t wx, int k, float s_hi, float s_off) {
    constexpr uint32_t mask = (1u << BITS) - 1u;
    uint32_t u;
    if (k * BITS <= 23 - BITS) u = (uint32_t(wx) << (23 - BITS - k * BITS)) & (mask << (23 - BITS));
    else u = uint32_t(wx >> (k * BITS - (23 - BITS))) & (mask << (23 - BITS));
    return __fmaf_rn(__uint_as_float(u | 0x3F800000u), s_hi, s_off);
}

// exact iff fl(x+y) == x+y; both checks are needed without knowing |x| vs |y|
__device__ __forceinline__ bool add_exact(float x, float y, float s) {
    return __fsub_rn(s, x) == y && __fsub_rn(s, y) == x;
}

// f64(q*s) + C_S[pi_S] + ... + C_1[pi_1] -> f32 for one channel, the
// reference's order (Q/prq.py:123-132); out of line, rare.
template <int BITS, int S>
__device__ __noinline__ float exact_addback1(float qs, const uint16_t *cp, uint32_t col, uint32_t d,
                                             int K, int a0, int a1, int a2, int a3) {
    const int ai[4] = {a0, a1, a2, a3};
    double acc = double(qs);
#pragma unroll
    for (int t = S - 1; t >= 0; t--)
        acc = __dadd_rn(acc, double(bf16_to_f32(cp[uint32_t(t * K + ai[t]) * d + col])));
    return __double2float_rn(acc);
}

template <int BITS, int S, bool OBF16>
__global__ void __launch_bounds__(256) k_dequant_v3(DequantArgs a) {
    constexpr int SS = S > 0 ? S : 1;
    const uint32_t d = uint32_t(a.d), N = a.N;
    const int col = int(threadIdx.x & ((1u << a.lvpr) - 1u)) << 3;
    const uint32_t rslot = threadIdx.x >> a.lvpr;
    uint32_t stat = 0;
    for (uint32_t T = blockIdx.x; T < a.ta.n_tiles; T += gridDim.x) {
        const uint32_t p = a.ta.div_tpp.div(T);
        const uint32_t i0 = (T - p * a.ta.tpp) * a.ta.rows_per_pass * kUnroll;
        const uint64_t pN = uint64_t(p) * N;
        const uint8_t *pp = a.payload + uint64_t(p) * a.pb;
        const uint8_t *sp = a.scales + uint64_t(p) * a.ng;
        const uint8_t *ap = a.asg + pN * S;
        const uint16_t *cp = a.cent + uint64_t(p) * S * a.K * d;
        uint64_t w[kUnroll];
        uint32_t sc[kUnroll], ii[kUnroll];
        int ai[kUnroll][SS];
        uint4 cw[kUnroll][SS];
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
            const uint32_t i = i0 + u * a.ta.rows_per_pass + rslot;
            ii[u] = i < N ? i : N - 1;
            const uint32_t e0 = ii[u] * d + col;
            const uint8_t *pl = pp + ((e0 * BITS) >> 3);
            if constexpr (BITS == 2) w[u] = __ldg(reinterpret_cast<const uint16_t *>(pl));
            else if constexpr (BITS == 4) w[u] = __ldg(reinterpret_cast<const uint32_t *>(pl));
            else { uint2 t = __ldg(reinterpret_cast<const uint2 *>(pl)); w[u] = uint64_t(t.x) | (uint64_t(t.y) << 32); }
            sc[u] = __ldg(sp + (e0 >> a.lgB));
#pragma unroll
            for (int t = 0; t < S; t++) {
                int at = __ldg(ap + t * N + ii[u]);
                if (at >= a.K) { stat |= QVG_STATUS_BAD_ASSIGN; at = 0; }
                ai[u][t] = at;
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; u++)
#pragma unroll
            for (int t = 0; t < S; t++)
                cw[u][t] = __ldg(reinterpret_cast<const uint4 *>(cp + uint32_t(t * a.K + ai[u][t]) * d + col));
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
            const bool valid = i0 + u * a.ta.rows_per_pass + rslot < N;
            if ((sc[u] & 0x7Fu) == 0x7Fu) stat |= QVG_STATUS_NAN_SCALE;
            const float s = e4m3_decode_fast(sc[u]);
            constexpr uint64_t SIGNS = (BITS == 2 ? 0xAAAAull : (BITS == 4 ? 0x88888888ull : 0x8080808080808080ull));
            const uint64_t wx = w[u] ^ SIGNS;
            const float s_hi = s * float(1 << BITS), s_off = s * (-1.5f * float(1 << BITS));
            float y[8];
#pragma unroll
            for (int k = 0; k < 8; k++) y[k] = qs_fma<BITS>(wx, k, s_hi, s_off);   // exact q*s
            uint32_t inexact = 0;
#pragma unroll
            for (int t = S - 1; t >= 0; t--) {                 // reversed(stages)
                const uint4 c4 = cw[u][t];
                const float c[8] = {bf16_lo(c4.x), bf16_hi(c4.x), bf16_lo(c4.y), bf16_hi(c4.y),
                                    bf16_lo(c4.z), bf16_hi(c4.z), bf16_lo(c4.w), bf16_hi(c4.w)};
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const float s2 = __fadd_rn(y[k], c[k]);
                    if (t > 0 && !add_exact(y[k], c[k], s2)) inexact |= 1u << k;  // non-final sums
                    y[k] = s2;
                }
            }
            if (inexact) {  // rare: a partial sum needed > 24 bits -> f64 chain
#pragma unroll
                for (int k = 0; k < 8; k++)
                    if (inexact >> k & 1u)
                        y[k] = exact_addback1<BITS, S>(qs_fma<BITS>(wx, k, s_hi, s_off), cp, col + k, d, a.K,
                                                       ai[u][0], ai[u][SS > 1 ? 1 : 0], ai[u][SS > 2 ? 2 : 0],
                                                       ai[u][SS > 3 ? 3 : 0]);
            }
            if (!valid) continue;
            const uint64_t o = (pN + ii[u]) * d + col;
            if constexpr (OBF16) {
                uint4 v;
                __nv_bfloat162 h;
                h = __floats2bfloat162_rn(y[0], y[1]); v.x = *reinterpret_cast<uint32_t *>(&h);
                h = __floats2bfloat162_rn(y[2], y[3]); v.y = *reinterpret_cast<uint32_t *>(&h);
                h = __floats2bfloat162_rn(y[4], y[5]); v.z = *reinterpret_cast<uint32_t *>(&h);
                h = __floats2bfloat162_rn(y[6], y[7]); v.w = *reinterpret_cast<uint32_t *>(&h);
                *reinterpret_cast<uint4 *>(static_cast<uint16_t *>(a.out) + o) = v;
            } else {
                float4 *op = reinterpret_cast<float4 *>(static_cast<float *>(a.out) + o);
                op[0] = make_float4(y[0], y[1], y[2], y[3]);
                op[1] = make_float4(y[4], y[5], y[6], y[7]);
            }
        }
    }
    stat = __reduce_or_sync(0xffffffffu, stat);
    if (stat && (threadIdx.x & 31) == 0) atomicOr(a.status, int(stat));
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
// v4 streaming kernels: 16 channels per thread-row (d % 16 == 0, B % 16 == 0),
// halving the per-row index/address/decode overhead of the 8-channel layout,
// with the per-element work written to split between the ALU and FMA pipes.
// ------------------------------------------------------------------------
template <int BITS, int S, bool OBF16>
__global__ void __launch_bounds__(256) k_dequant_v4(DequantArgs a) {
    constexpr int SS = S > 0 ? S : 1;
    constexpr uint32_t SIGNS = BITS == 2 ? 0xAAAAAAAAu : (BITS == 4 ? 0x88888888u : 0x80808080u);
    const uint32_t mhi = ((1u << BITS) - 1u) << (23 - BITS), one = 0x3F800000u;
    const uint32_t d = uint32_t(a.d), N = a.N;
    const int col = int(threadIdx.x & ((1u << a.lvpr) - 1u)) << 4;
    const uint32_t rslot = threadIdx.x >> a.lvpr;
    bool bad_scale = false, bad_asg = false;
    for (uint32_t T = blockIdx.x; T < a.ta.n_tiles; T += gridDim.x) {
        const uint32_t p = a.ta.div_tpp.div(T);
        const uint32_t i0 = (T - p * a.ta.tpp) * a.ta.rows_per_pass * kUnroll;
        const uint64_t pN = uint64_t(p) * N;
        const uint8_t *pp = a.payload + uint64_t(p) * a.pb;
        const uint8_t *sp = a.scales + uint64_t(p) * a.ng;
        const uint8_t *ap = a.asg + pN * S;
        const uint16_t *cp = a.cent + uint64_t(p) * S * a.K * d;
        Codes16<BITS> w[kUnroll];
        uint32_t sc[kUnroll], ii[kUnroll];
        int ai[kUnroll][SS];
        uint4 cw[kUnroll][SS][2];
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
            const uint32_t i = i0 + u * a.ta.rows_per_pass + rslot;
            ii[u] = i < N ? i : N - 1;
            const uint32_t e0 = ii[u] * d + col;
            w[u] = load_codes16<BITS>(pp + ((e0 * BITS) >> 3));
            sc[u] = __ldg(sp + (e0 >> a.lgB));
#pragma unroll
            for (int t = 0; t < S; t++) {
                int at = __ldg(ap + t * N + ii[u]);
                bad_asg |= at >= a.K;
                ai[u][t] = at < a.K ? at : 0;
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; u++)
#pragma unroll
            for (int t = 0; t < S; t++) {
                const uint4 *c4 = reinterpret_cast<const uint4 *>(cp + uint32_t(t * a.K + ai[u][t]) * d + col);
                cw[u][t][0] = __ldg(c4);
                cw[u][t][1] = __ldg(c4 + 1);
            }
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
            const bool valid = i0 + u * a.ta.rows_per_pass + rslot < N;
            bad_scale |= (sc[u] & 0x7Fu) == 0x7Fu;
            const float s = e4m3_decode_fast(sc[u]);
            Codes16<BITS> wx;
#pragma unroll
            for (int j = 0; j < Codes16<BITS>::NW; j++) wx.w[j] = w[u].w[j] ^ SIGNS;
            const float s_hi = s * float(1 << BITS), s_off = s * (-1.5f * float(1 << BITS));
            float y[16];
#pragma unroll
            for (int k = 0; k < 16; k++) y[k] = qs16<BITS>(wx, k, mhi, one, s_hi, s_off);   // exact
            bool inexact = false;
#pragma unroll
            for (int t = S - 1; t >= 0; t--) {                 // reversed(stages)
                float c[16];
                cvt16(cw[u][t][0], cw[u][t][1], c);
#pragma unroll
                for (int k = 0; k < 16; k++) {
                    const float s2 = __fadd_rn(y[k], c[k]);
                    if (t > 0) inexact |= (__fsub_rn(s2, y[k]) != c[k]) | (__fsub_rn(s2, c[k]) != y[k]);
                    y[k] = s2;
                }
            }
            if (inexact) {  // rare: a non-final partial sum needed > 24 bits -> f64 chain
#pragma unroll
                for (int k = 0; k < 16; k++)
                    y[k] = exact_addback1<BITS, S>(qs16<BITS>(wx, k, mhi, one, s_hi, s_off), cp, col + k, d,
                                                   a.K, ai[u][0], ai[u][SS > 1 ? 1 : 0],
                                                   ai[u][SS > 2 ? 2 : 0], ai[u][SS > 3 ? 3 : 0]);
            }
            if (!valid) continue;
            const uint64_t o = (pN + ii[u]) * d + col;
            if constexpr (OBF16) {
                uint32_t v[8];
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    __nv_bfloat162 h = __floats2bfloat162_rn(y[2 * j], y[2 * j + 1]);
                    v[j] = *reinterpret_cast<uint32_t *>(&h);
                }
                uint4 *op = reinterpret_cast<uint4 *>(static_cast<uint16_t *>(a.out) + o);
                op[0] = make_uint4(v[0], v[1], v[2], v[3]);
                op[1] = make_uint4(v[4], v[5], v[6], v[7]);
            } else {
                float4 *op = reinterpret_cast<float4 *>(static_cast<float *>(a.out) + o);
#pragma unroll
                for (int j = 0; j < 4; j++) op[j] = make_float4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]);
            }
        }
    }
    const uint32_t stat = (bad_scale ? QVG_STATUS_NAN_SCALE : 0u) | (bad_asg ? QVG_STATUS_BAD_ASSIGN : 0u);
    const uint32_t all = __reduce_or_sync(0xffffffffu, stat);
    if (all && (threadIdx.x & 31) == 0) atomicOr(a.status, int(all));
}

template <int BITS, int S, bool XBF16>
__global__ void __launch_bounds__(256) k_quantize_v4(QuantArgs a) {
    constexpr int QMAX = (1 << (BITS - 1)) - 1;
    constexpr int SS = S > 0 ? S : 1;
    const uint32_t d = uint32_t(a.d), N = a.N;
    const int col = int(threadIdx.x & ((1u << a.lvpr) - 1u)) << 4;
    const uint32_t rslot = threadIdx.x >> a.lvpr;
    const int glanes = 1 << a.gshift;     // B / 16 lanes per group
    const int lane = threadIdx.x & 31;
    bool nonfinite = false;
    for (uint32_t T = blockIdx.x; T < a.ta.n_tiles; T += gridDim.x) {
        const uint32_t p = a.ta.div_tpp.div(T);
        const uint32_t i0 = (T - p * a.ta.tpp) * a.ta.rows_per_pass * kUnroll;
        const uint64_t pN = uint64_t(p) * N;
        const uint8_t *xb = static_cast<const uint8_t *>(a.x) + pN * d * (XBF16 ? 2 : 4);
        const uint8_t *ap = a.asg + pN * S;
        const uint16_t *cp = a.cent + uint64_t(p) * S * a.K * d;
        float r[kUnroll][16];
        uint32_t ii[kUnroll];
        int ai[kUnroll][SS];
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
            const uint32_t i = i0 + u * a.ta.rows_per_pass + rslot;
            ii[u] = i < N ? i : N - 1;
            load_x16<XBF16>(xb, ii[u] * d + col, r[u]);
#pragma unroll
            for (int t = 0; t < S; t++) ai[u][t] = __ldg(ap + t * N + ii[u]);
        }
        float eb[kUnroll], am[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
#pragma unroll
            for (int k = 0; k < 16; k++) nonfinite |= !(fabsf(r[u][k]) <= 3.402823466e38f);
            float e = 0.f;
#pragma unroll
            for (int t = 0; t < S; t++) {
                const uint4 *c4 = reinterpret_cast<const uint4 *>(cp + uint32_t(t * a.K + ai[u][t]) * d + col);
                float c[16];
                cvt16(__ldg(c4), __ldg(c4 + 1), c);
#pragma unroll
                for (int k = 0; k < 16; k++) r[u][k] = __fsub_rn(r[u][k], c[k]);
                if (t < S - 1) {
                    float m = 0.f;
#pragma unroll
                    for (int k = 0; k < 16; k++) m = fmaxf(m, fabsf(r[u][k]));
                    e = __fadd_ru(e, m);
                }
            }
            float mx = 0.f;
#pragma unroll
            for (int k = 0; k < 16; k++) mx = fmaxf(mx, fabsf(r[u][k]));
            eb[u] = S > 0 ? __fadd_ru(e, mx) : 0.f;
            am[u] = mx;
        }
        for (int m = 1; m < glanes; m <<= 1) {
#pragma unroll
            for (int u = 0; u < kUnroll; u++) {
                am[u] = fmaxf(am[u], __shfl_xor_sync(0xffffffffu, am[u], m));
                eb[u] = fmaxf(eb[u], __shfl_xor_sync(0xffffffffu, eb[u], m));
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
            const bool valid = i0 + u * a.ta.rows_per_pass + rslot < N;
            // |r_f32 - r_ref| <= 2^-24 sum_t|r_t| (f32 chain) + 2^-53 (.) (the
            // reference's f64 chain) <= 2^-22 * sum_t max|r_t|: factor-2 margin
            const float E = __fmul_ru(eb[u], 2.38418579e-7f);
            uint32_t code;
            bool camb = false;
            if (am[u] == 0.f && E == 0.f) code = 0x38u;
            else {
                const float lo = __fsub_rd(am[u], E), hi = __fadd_ru(am[u], E);
                if (lo > 0.f) code = scale_code<QMAX>(lo, hi, camb);
                else { code = 0x38u; camb = true; }
            }
            camb &= valid;
            auto exact_r = [&](int k) {
                return exact_residual<XBF16, S>(xb, cp, ii[u] * d + col + k, col + k, d, a.K, ai[u][0],
                                                ai[u][SS > 1 ? 1 : 0], ai[u][SS > 2 ? 2 : 0],
                                                ai[u][SS > 3 ? 3 : 0]);
            };
            if (__any_sync(0xffffffffu, camb)) {          // exact scale (rare)
                // every element whose exact |r| could be the group max
                const float thr = __fsub_rd(am[u], __fmul_ru(E, 2.f));
                uint32_t cand = 0;
#pragma unroll
                for (int k = 0; k < 16; k++) cand |= (camb && fabsf(r[u][k]) >= thr) ? 1u << k : 0u;
                double a64 = 0.0;
                while (cand) {
                    const int k = __ffs(cand) - 1;
                    cand &= cand - 1;
                    a64 = fmax(a64, fabs(exact_r(k)));
                }
                for (int m = 1; m < glanes; m <<= 1) a64 = fmax(a64, shfl_xor_d(a64, m));
                if (camb) code = a64 == 0.0 ? 0x38u : e4m3_encode_up(__ddiv_rn(a64, double(QMAX)));
            }
            const float s = e4m3_decode_fast(code);
            uint32_t b32[BITS / 2];
#pragma unroll
            for (int j = 0; j < BITS / 2; j++) b32[j] = 0;
            bool amb = false;
            if constexpr (QMAX == 1) {
                // q != 0 <=> RN64(|r|/s) > 0.5 <=> |r| > s/2 (exact r); ambiguous iff
                // the exact r may lie on the other side: ||r~| - s/2| <= E.  The
                // difference is exact (Sterbenz) whenever it is that small, given
                // E < s/8; otherwise every element is rechecked.
                const float half = 0.5f * s;
                amb = !(E < 0.125f * s);
#pragma unroll
                for (int k = 0; k < 16; k++) {
                    const float av = fabsf(r[u][k]);
                    amb |= fabsf(av - half) <= E;
                    const uint32_t f = av > half ? ((__float_as_uint(r[u][k]) >> 30) | 1u) : 0u;   // 1 or 3
                    b32[0] |= f << (2 * k);
                }
            } else {
                const float inv = __frcp_rn(s);
#pragma unroll
                for (int k = 0; k < 16; k++) {
                    const float av = fabsf(r[u][k]);
                    const float t = av * inv;
                    const float fl = floorf(t);
                    const float hb = (fl + 0.5f) * s;                    // exact
                    const float w = __fmaf_ru(hb, 2.38418579e-7f, E);
                    amb |= fl < float(QMAX) && av >= __fsub_rd(hb, w) && av <= __fadd_ru(hb, w);
                    int q = min(int(rintf(fminf(t, float(QMAX + 1)))), QMAX);   // saturated scales: |r/s| >> QMAX
                    if (r[u][k] < 0.f) q = -q;
                    b32[(k * BITS) >> 5] |= (uint32_t(q) & ((1u << BITS) - 1u)) << ((k * BITS) & 31);
                }
            }
            amb &= valid;
            if (__any_sync(0xffffffffu, amb) && amb) {   // exact codes (rare)
                // re-derive which elements sit in an error window, then fix them
                uint32_t todo = 0;
                const bool all = !(E < 0.125f * s);
                const float inv = __frcp_rn(s);
#pragma unroll
                for (int k = 0; k < 16; k++) {
                    const float av = fabsf(r[u][k]);
                    bool in;
                    if constexpr (QMAX == 1) in = fabsf(av - 0.5f * s) <= E;
                    else {
                        const float fl = floorf(av * inv);
                        const float hb = (fl + 0.5f) * s;
                        const float w = __fmaf_ru(hb, 2.38418579e-7f, E);
                        in = fl < float(QMAX) && av >= __fsub_rd(hb, w) && av <= __fadd_ru(hb, w);
                    }
                    todo |= (all || in) ? 1u << k : 0u;
                }
                while (todo) {
                    const int k = __ffs(todo) - 1;
                    todo &= todo - 1;
                    const uint32_t q = exact_code<QMAX>(exact_r(k), s) & ((1u << BITS) - 1u);
                    const int sh = (k * BITS) & 31, wi = (k * BITS) >> 5;
#pragma unroll
                    for (int j = 0; j < BITS / 2; j++)
                        if (j == wi) b32[j] = (b32[j] & ~(((1u << BITS) - 1u) << sh)) | (q << sh);
                }
            }
            if (!valid) continue;
            const uint32_t e0 = ii[u] * d + col;
            uint8_t *pl = a.payload + uint64_t(p) * a.pb + ((e0 * BITS) >> 3);
            if constexpr (BITS == 2) *reinterpret_cast<uint32_t *>(pl) = b32[0];
            else if constexpr (BITS == 4) *reinterpret_cast<uint2 *>(pl) = make_uint2(b32[0], b32[1]);
            else *reinterpret_cast<uint4 *>(pl) = make_uint4(b32[0], b32[1], b32[2], b32[3]);
            if ((lane & (glanes - 1)) == 0) a.scales[uint64_t(p) * a.ng + (e0 >> a.lgB)] = uint8_t(code);
        }
    }
    const uint32_t all = __reduce_or_sync(0xffffffffu, nonfinite ? uint32_t(QVG_STATUS_NONFINITE) : 0u);
    if (all && lane == 0) atomicOr(a.status, int(all));
}

// ------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------
static int grid_for(int64_t work, int block) {
    int64_t g = (work + block - 1) / block;
    int64_t cap = 148LL * 16;
    return int(g < 1 ? 1 : (g > cap ? cap : g));
}

static int ilog2(int v) { int l = 0; while ((1 << l) < v) l++; return l; }

bool quant_fast_ok(int64_t P, int64_t N, int d, int B, int S) {
    const int vpr = d / 8;
    return d % 8 == 0 && (vpr & (vpr - 1)) == 0 && vpr <= 32 && B % 8 == 0 &&
           ((B / 8) & (B / 8 - 1)) == 0 && B / 8 <= vpr && S <= 4 && P * N < (int64_t(1) << 32) &&
           N * d < (int64_t(1) << 32);
}

static TileArgs make_tiles(int64_t P, int64_t N, int lvpr) {
    const uint32_t rpp = 256u >> lvpr;
    const uint32_t tpp = uint32_t((N + int64_t(rpp) * kUnroll - 1) / (int64_t(rpp) * kUnroll));
    return TileArgs{uint32_t(P * tpp), tpp, make_fastdiv(tpp), rpp};
}

static int tile_grid(const TileArgs &t) {
    // persistent: <= 148 SMs x 4 resident CTAs of 256 threads
    return int(t.n_tiles < 148u * 4u ? t.n_tiles : 148u * 4u);
}

// warp-specialised TMA ring kernels (qvg_stream.cu); return 0 when the
// configuration does not fit them (S = 0, N % 4 != 0, misaligned buffers, tables
// too large for shared memory) -- the tile kernels below take those
int launch_quantize_stream(const QuantArgs &a, int64_t P, int bits, int S, bool xbf16, cudaStream_t st);
int launch_dequantize_stream(const DequantArgs &a, int64_t P, int bits, int S, bool obf16, cudaStream_t st);
// 32-channel ring kernel (qvg_dring.cu): the default K6 where it fits
int launch_dequantize_ring32(const DequantArgs &a, int64_t P, int bits, int S, bool obf16, cudaStream_t st);

template <int BITS, int S>
static void launch_quant_fast(const QuantArgs &a, bool xbf16, cudaStream_t st) {
    if (S > 0 && a.v16 && launch_quantize_stream(a, a.P, BITS, S, xbf16, st)) return;
    const int g = tile_grid(a.ta);
    if (a.v16) {
        if (xbf16) k_quantize_v4<BITS, S, true><<<g, 256, 0, st>>>(a);
        else k_quantize_v4<BITS, S, false><<<g, 256, 0, st>>>(a);
        return;
    }
    if (xbf16) k_quantize_v3<BITS, S, true><<<g, 256, 0, st>>>(a);
    else k_quantize_v3<BITS, S, false><<<g, 256, 0, st>>>(a);
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

int launch_quantize(const void *x, int xdtype, int64_t P, int64_t N, int d, int bits, int B, int S,
                    int K, const uint16_t *cent, const uint8_t *asg, uint8_t *payload,
                    uint8_t *scales, int32_t *status, cudaStream_t st) {
    const bool xbf16 = xdtype == QVG_DTYPE_BF16;
    if (xdtype != QVG_DTYPE_F64 && quant_fast_ok(P, N, d, B, S)) {
        // 16 channels per thread when groups and rows split into 16-channel lanes
        const bool v16 = d % 16 == 0 && B % 16 == 0 && ((d / 16) & (d / 16 - 1)) == 0;
        const int lvpr = v16 ? ilog2(d / 16) : ilog2(d / 8);
        QuantArgs a{x, cent, asg, payload, scales, uint32_t(N), d, K, B, lvpr,
                    v16 ? ilog2(B / 16) : ilog2(B / 8), status,
                    uint32_t(N * d * bits / 8), uint32_t(N * d / B), uint32_t(ilog2(B)),
                    make_tiles(P, N, lvpr), v16 ? 1 : 0, uint32_t(P)};
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

int launch_pack(const int8_t *q, int64_t n, int bits, uint8_t *out, int32_t *status, cudaStream_t st) {
    if (n > 0) k_pack_codes<<<grid_for((n * bits + 7) / 8, 256), 256, 0, st>>>(q, n, bits, out, status);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

int launch_unpack(const uint8_t *in, int64_t n, int bits, int8_t *out, cudaStream_t st) {
    if (n > 0) k_unpack_codes<<<grid_for(n, 256), 256, 0, st>>>(in, n, bits, out);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

template <int BITS, int S>
static void launch_deq_fast(const DequantArgs &a, bool obf16, cudaStream_t st) {
    if (S > 0 && launch_dequantize_ring32(a, a.P, BITS, S, obf16, st)) return;
    if (S > 0 && a.v16 && launch_dequantize_stream(a, a.P, BITS, S, obf16, st)) return;
    const int g = tile_grid(a.ta);
    if (a.v16) {
        if (obf16) k_dequant_v4<BITS, S, true><<<g, 256, 0, st>>>(a);
        else k_dequant_v4<BITS, S, false><<<g, 256, 0, st>>>(a);
        return;
    }
    if (obf16) k_dequant_v3<BITS, S, true><<<g, 256, 0, st>>>(a);
    else k_dequant_v3<BITS, S, false><<<g, 256, 0, st>>>(a);
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

int launch_dequantize(const uint8_t *payload, const uint8_t *scales, const uint16_t *cent,
                      const uint8_t *asg, int64_t P, int64_t N, int d, int bits, int B, int S, int K,
                      void *out, int odtype, int32_t *status, cudaStream_t st) {
    const bool obf16 = odtype == QVG_DTYPE_BF16;
    const int vpr = d / 8;
    if (d % 8 == 0 && (vpr & (vpr - 1)) == 0 && vpr <= 32 && B % 8 == 0 && (B & (B - 1)) == 0 &&
        S <= 4 && P * N < (int64_t(1) << 32) && N * d < (int64_t(1) << 32)) {
        const bool v16 = d % 16 == 0 && B % 16 == 0 && ((d / 16) & (d / 16 - 1)) == 0;
        const int lvpr = v16 ? ilog2(d / 16) : ilog2(vpr);
        DequantArgs a{payload, scales, cent, asg, out, uint32_t(N), d, K, B, lvpr, status,
                      uint32_t(N * d * bits / 8), uint32_t(N * d / B), uint32_t(ilog2(B)),
                      make_tiles(P, N, lvpr), v16 ? 1 : 0, uint32_t(P)};
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
