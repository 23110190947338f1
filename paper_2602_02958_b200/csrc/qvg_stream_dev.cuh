// qvg_stream_dev.cuh — device helpers of the streaming codec kernels
// (qvg_stream.cu, qvg_wring.cu): padded f32 centroid tables + metadata,
// work schedule, out-of-line exact fallbacks.
#pragma once
#include <cstdlib>

#include "qvg_codec_dev.cuh"

namespace qvg {
namespace stream {

constexpr int kCW = 15;                    // consumer warps (+1 producer = 16 warps: 4 per SMSP, <= 128 regs)
constexpr int kThreads = 32 * (kCW + 1);   // + producer warp
constexpr int kU = 2;                      // rows per consumer thread per stage

struct Geo {
    uint32_t P, N, d, K;
    uint32_t R;            // rows per stage (= kCW * 32 / (d/16) * kU)
    uint32_t nst;          // ring stages
    uint32_t pitch;        // f32 table row pitch (floats)
    uint32_t tbytes;       // bf16 table bytes per plane (S*K*d*2)
    uint32_t nchunk;       // S*K*d/16
    uint32_t lchunk;       // log2(d/16)
    uint32_t ipp, rpi, n_items;
    uint32_t off_tab, off_meta, off_ring;   // smem byte offsets (staging at 0)
    uint32_t stage_bytes;  // bytes per ring stage
    uint32_t big_row;      // big-stream bytes per row (x row or packed code row)
    uint32_t small_row;    // scale bytes per row in the stage (K6), 0 for K5
    uint32_t off_small;    // offset of the small streams inside a stage
    uint32_t dbg;          // QVG_STREAM_DBG: 1 = consumers only drain the ring (measurement)
    uint32_t stg_global;   // 1: tables widened from global memory (no smem staging copy)
};

// padded f32 table: 16-channel block c of a row at float 16c + 4(c>>1), which
// puts the 8 blocks of a 128-channel row on 8 distinct bank quads
__host__ __device__ __forceinline__ uint32_t blk_off(uint32_t c) { return 16u * c + 4u * (c >> 1); }

template <int CW = kCW>
__device__ __forceinline__ void named_sync_consumers() {
    asm volatile("bar.sync 1, %0;" ::"n"(CW * 32) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s_cta(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ float max_nan(float a, float b) {
    float d;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}
__device__ __forceinline__ float min3_abs(float m, float a, float b) {
    float t, d;
    asm("min.f32 %0, %1, %2;" : "=f"(t) : "f"(fabsf(a)), "f"(fabsf(b)));
    asm("min.f32 %0, %1, %2;" : "=f"(d) : "f"(m), "f"(t));
    return d;
}
__device__ __forceinline__ float max3_abs(float m, float a, float b) {
    float t, d;
    asm("max.f32 %0, %1, %2;" : "=f"(t) : "f"(fabsf(a)), "f"(fabsf(b)));
    asm("max.f32 %0, %1, %2;" : "=f"(d) : "f"(m), "f"(t));
    return d;
}
__device__ __forceinline__ float max3_nan_abs(float m, float a, float b) {
    float t, d;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(t) : "f"(fabsf(a)), "f"(fabsf(b)));
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(m), "f"(t));
    return d;
}

// widen the staged bf16 tables [S*K][d] to the padded f32 layout + metadata
__device__ __forceinline__ void widen(const uint16_t *stg, float *tab, float2 *meta, const Geo &g,
                                      uint32_t nthr = kCW * 32) {
    const uint32_t cmask = (1u << g.lchunk) - 1u;
    for (uint32_t q = threadIdx.x; q < g.nchunk; q += nthr) {
        const uint4 *src = reinterpret_cast<const uint4 *>(stg + size_t(q) * 16);
        float c[16];
        cvt16(src[0], src[1], c);
        float mx = 0.f, mn = __int_as_float(0x7F800000);
#pragma unroll
        for (int k = 0; k < 16; k++) {
            const float a = fabsf(c[k]);
            mx = fmaxf(mx, a);
            mn = a > 0.f ? fminf(mn, a) : mn;
        }
        float4 *dst = reinterpret_cast<float4 *>(tab + size_t(q >> g.lchunk) * g.pitch + blk_off(q & cmask));
#pragma unroll
        for (int j = 0; j < 4; j++) dst[j] = make_float4(c[4 * j], c[4 * j + 1], c[4 * j + 2], c[4 * j + 3]);
        // 2^(e-7) = ulp of a bf16 with mn's exponent (0 if not a normal float:
        // certificates fail conservatively; +inf for an all-zero chunk)
        float unit;
        if (mn == __int_as_float(0x7F800000)) unit = mn;
        else {
            const uint32_t eb = __float_as_uint(mn) & 0x7F800000u;
            unit = eb > (7u << 23) ? __uint_as_float(eb - (7u << 23)) : 0.f;
        }
        meta[q] = make_float2(unit, mx);     // NaN/Inf in the chunk -> mx non-finite
    }
}

// ---- shared schedule: the CTA's contiguous items, each split into stages ----
struct Sched {
    uint32_t it, it1, p, r1, i0;
    __device__ __forceinline__ void init(const Geo &g) {
        it = uint32_t((uint64_t(blockIdx.x) * g.n_items) / gridDim.x);
        it1 = uint32_t((uint64_t(blockIdx.x + 1) * g.n_items) / gridDim.x);
        start(g);
    }
    __device__ __forceinline__ void start(const Geo &g) {
        if (it >= it1) return;
        p = it / g.ipp;
        i0 = (it - p * g.ipp) * g.rpi;
        r1 = min(g.N, i0 + g.rpi);
    }
    __device__ __forceinline__ bool valid() const { return it < it1; }
    __device__ __forceinline__ void next(const Geo &g) {
        i0 += g.R;
        if (i0 >= r1) { it++; start(g); }
    }
    // first plane after p that this CTA visits, or -1
    __device__ __forceinline__ int64_t next_plane(const Geo &g) const {
        return int64_t(p + 1) * g.ipp < int64_t(it1) ? int64_t(p + 1) : -1;
    }
};

struct Bars {
    uint64_t full[16], empty[16], tab;
};

// the reference's float64 add-back of one element (Q/prq.py:113-132)
template <int S>
__device__ __noinline__ float exact_addback(float qs, const float *tab, uint32_t pitch, uint32_t coff, int K,
                                            int a0, int a1, int a2, int a3) {
    const int ai[4] = {a0, a1, a2, a3};
    double acc = double(qs);
#pragma unroll
    for (int t = S - 1; t >= 0; t--) acc = __dadd_rn(acc, double(tab[uint32_t(t * K + ai[t]) * pitch + coff]));
    return __double2float_rn(acc);
}

// the reference's float64 residual x - C_1[pi_1] - ... (Q/smoothing.py:40)
template <int S>
__device__ __noinline__ double exact_residual_f(float x, const float *tab, uint32_t pitch, uint32_t coff, int K,
                                                int a0, int a1, int a2, int a3) {
    const int ai[4] = {a0, a1, a2, a3};
    double v = double(x);
#pragma unroll
    for (int t = 0; t < S; t++) v = __dsub_rn(v, double(tab[uint32_t(t * K + ai[t]) * pitch + coff]));
    return v;
}

template <int BITS>
__host__ __device__ constexpr uint32_t magic_sum() {
    uint32_t acc = 0;
    for (int k = 0; k < 32 / BITS; k++) acc += 0x4B400000u << (BITS * k);
    return acc;
}

struct Words4 {
    uint32_t w[4];
};

// the f32 residual row exactly as the fast path computes it (RN per stage)
template <int S, bool XBF16>
__device__ __forceinline__ void residual_row(const uint8_t *xrow, const float *tab, uint32_t pitch, uint32_t coff,
                                             int K, const int ai[4], float r[16]) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
        if constexpr (XBF16) r[k] = bf16_to_f32(reinterpret_cast<const uint16_t *>(xrow)[k]);
        else r[k] = reinterpret_cast<const float *>(xrow)[k];
    }
#pragma unroll
    for (int t = 0; t < S; t++) {
        const float *row = tab + uint32_t(t * K + ai[t]) * pitch + coff;
#pragma unroll
        for (int k = 0; k < 16; k++) r[k] = __fsub_rn(r[k], row[k]);
    }
}

template <int S>
__device__ __forceinline__ double exact_residual_row(float x, const float *tab, uint32_t pitch, uint32_t off,
                                                     int K, const int ai[4]) {
    double v = double(x);
#pragma unroll
    for (int t = 0; t < S; t++) v = __dsub_rn(v, double(tab[uint32_t(t * K + ai[t]) * pitch + off]));
    return v;
}

template <bool XBF16>
__device__ __forceinline__ float xat(const uint8_t *xrow, int k) {
    if constexpr (XBF16) return bf16_to_f32(reinterpret_cast<const uint16_t *>(xrow)[k]);
    else return reinterpret_cast<const float *>(xrow)[k];
}

// Bound on |r_f32 - r_ref| for a lane whose residual is not certified exact.
// The kernel forms r_t = RN32(r_{t-1} - C_t) (r_0 = x); each step's rounding
// error is at most u|r_t| (u = 2^-24, relative to the step's result), so
// r_S = x - sum C + sum_t e_t with |e_t| <= u' |r_t|, and |r_t| <= max|r_S| +
// sum_{tau > t} max|C_tau| (+ second order).  The reference's float64 chain
// has the same form with 2^-53.  Hence
//   |r_f32 - r_ref| <= 2^-23 (S max|r_S| + sum_{t >= 2} (t - 1) max|C_t|)
// (factor 2 over u' + u64' for the second-order terms), plus S * 2^-149 for
// steps whose result is subnormal.  The first stage's centroid never enters:
// its subtraction's error is relative to r_1 = x - C_1.  cwt = sum_t t max|C_t|
// over 0-based t (rounded up); all arithmetic rounds up.
__device__ __forceinline__ float err_bound(float S, float mx, float cwt) {
    return __fmaf_ru(__fmaf_ru(S, mx, cwt), 1.1920928955078125e-7f, S * 1.40129846e-45f);
}

// per-row threshold of the ambiguity window (see K5)
template <int QMAX>
__device__ __forceinline__ float window_thr(float sv, float inv, float E) {
    if constexpr (QMAX == 1) {
        // ||r| - s/2| <= W  =>  |r^2 - (s/2)^2| <= W (s + W), W = E + the 1/s rounding
        const float W = __fmaf_ru(0.5f * sv, 2.38418579e-7f, E);
        return __fmul_ru(__fmul_ru(W, __fadd_ru(sv, W)), 1.00000095367f);
    } else {
        // |t - rint(t)| >= 1/2 - delta, t = r/s
        const float delta = __fmaf_ru(__fmul_ru(E, inv), 1.0000002f, float(QMAX + 1) * 2.38418579e-7f);
        return __fsub_rd(0.5f, delta);
    }
}

// exact E4M3 scale of a group whose f32 amax interval straddles a code
// boundary: the exact |r| of every candidate element (those that could be
// the maximum), max over the group's lanes, encoded "up" (Q/quant.py:40-45).
// Called by every lane of the warp (shuffles); lanes with camb == false keep code.
template <int QMAX, int S, bool XBF16>
__device__ __noinline__ uint32_t fix_scale(const uint8_t *xrow, const float *tab, uint32_t pitch, uint32_t coff, int K,
                                           int a0, int a1, int a2, int a3, float am, float E, bool camb, int glanes,
                                           uint32_t code) {
    const int ai[4] = {a0, a1, a2, a3};
    float r[16];
    residual_row<S, XBF16>(xrow, tab, pitch, coff, K, ai, r);
    const float thr = __fsub_rd(am, __fmul_ru(E, 2.f));
    double a64 = 0.0;
    if (camb) {
#pragma unroll
        for (int k = 0; k < 16; k++)
            if (fabsf(r[k]) >= thr) a64 = fmax(a64, fabs(exact_residual_row<S>(xat<XBF16>(xrow, k), tab, pitch, coff + k, K, ai)));
    }
    for (int m = 1; m < glanes; m <<= 1) a64 = fmax(a64, shfl_xor_d(a64, m));
    if (camb) code = a64 == 0.0 ? 0x38u : e4m3_encode_up(__ddiv_rn(a64, double(QMAX)));
    return code;
}

// max over the masked elements of the reference's float64 |residual|
// (Q/smoothing.py:40) -- the exact group amax when its f32 interval straddles
// an E4M3 code boundary
template <int S, bool XBF16>
__device__ __noinline__ double exact_absmax(const uint8_t *xrow, const float *tab, uint32_t pitch, uint32_t coff,
                                            int K, int a0, int a1, int a2, int a3, uint32_t mask) {
    const int ai[4] = {a0, a1, a2, a3};
    double m = 0.0;
    while (mask) {
        const int k = __ffs(mask) - 1;
        mask &= mask - 1;
        m = fmax(m, fabs(exact_residual_row<S>(xat<XBF16>(xrow, k), tab, pitch, coff + k, K, ai)));
    }
    return m;
}

// exact codes of the elements in the ambiguity window (or all when `all`):
// with E == 0 the f32 residual is exact and q = clip(rint(r/s)) is decided by
// exact f32 compares against (n +- 1/2) s; otherwise by the float64 residual
// (Q/quant.py:48-55)
template <int BITS, int S, bool XBF16>
__device__ __noinline__ Words4 fix_codes(const uint8_t *xrow, const float *tab, uint32_t pitch, uint32_t coff, int K,
                                         int a0, int a1, int a2, int a3, float sv, float inv, float E, float thr,
                                         bool all, Words4 b32) {
    constexpr int QMAX = (1 << (BITS - 1)) - 1;
    constexpr float MAGIC = 12582912.f + float(1 << (BITS - 1));
    const int ai[4] = {a0, a1, a2, a3};
    float r[16];
    residual_row<S, XBF16>(xrow, tab, pitch, coff, K, ai, r);
#pragma unroll
    for (int k = 0; k < 16; k++) {
        bool in;
        if constexpr (QMAX == 1) {
            const float h = 0.5f * sv;
            in = fabsf(__fmaf_rn(r[k], r[k], -h * h)) <= thr;
        } else {
            const float y = __fmaf_rn(r[k], inv, MAGIC);
            const float qf = __fadd_rn(y, -MAGIC);
            in = fabsf(__fmaf_rn(r[k], inv, -qf)) >= thr;
        }
        in |= all || !(fabsf(r[k]) <= 3.402823466e38f);
        if (!in) continue;
        uint32_t qv;
        if (E == 0.f) {
            const float av = fabsf(r[k]);
            int nq = int(rintf(fminf(av * inv, float(QMAX + 1))));   // saturated scale: |r/s| >> QMAX
            const float up = (float(nq) + 0.5f) * sv, dn = (float(nq) - 0.5f) * sv;
            if (av > up || (av == up && (nq & 1))) nq++;
            else if (nq > 0 && (av < dn || (av == dn && (nq & 1)))) nq--;
            nq = min(nq, QMAX);
            qv = uint32_t(r[k] < 0.f ? -nq : nq) & ((1u << BITS) - 1u);
        } else {
            qv = exact_code<QMAX>(exact_residual_row<S>(xat<XBF16>(xrow, k), tab, pitch, coff + k, K, ai), sv) &
                 ((1u << BITS) - 1u);
        }
        const int sh = (k * BITS) & 31, wi = (k * BITS) >> 5;
        b32.w[wi] = (b32.w[wi] & ~(((1u << BITS) - 1u) << sh)) | (qv << sh);
    }
    return b32;
}

}  // namespace stream
}  // namespace qvg
