// qvg_codec_dev.cuh — device helpers shared by the K5/K6 kernels
// (qvg_codec.cu, qvg_stream.cu): E4M3 scale codes, bf16 widening, code
// fields, certified-exact fallbacks, mbarrier / bulk-copy wrappers.
#pragma once
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

// Branch-free exact E4M3 -> f32: the 7 magnitude bits placed at f32 bit 20
// read as 2^(e-127)(1+m/8) (or the denormal m*2^-129 when e == 0); scaling by
// 2^120 (exact) gives (8+m)*2^(e-10), resp. m*2^-9.
__device__ __forceinline__ float e4m3_decode_fast(uint32_t b) {
    const float mag = __uint_as_float((b & 0x7Fu) << 20) * 1.329227995784916e36f;   // 2^120
    return __uint_as_float(__float_as_uint(mag) | ((b & 0x80u) << 24));
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
// index helpers: n / N for the flattened [P*N] row space (< 2^32 rows) with a
// multiply-high (Granlund-Montgomery "round-up" variant, exact for all u32 n)
// ------------------------------------------------------------------------
struct FastDiv {
    uint32_t m, l;
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        return uint32_t((uint64_t(__umulhi(n, m)) + n) >> l);
    }
};

static inline FastDiv make_fastdiv(uint32_t d) {
    uint32_t l = 0;
    while ((uint64_t(1) << l) < d) l++;
    uint64_t m = ((uint64_t(1) << 32) * ((uint64_t(1) << l) - d)) / d + 1;
    return FastDiv{uint32_t(m), l};
}

// Tile mapping shared by K5/K6.  A tile is kUnroll*256/VPR consecutive rows
// of ONE plane (VPR = d/8 threads per row, each owning 8 channels), so the
// plane index is one division per tile and every in-plane offset is 32-bit.
// The tile loop is block-uniform, so every lane reaches every shuffle.
constexpr int kUnroll = 2;

struct TileArgs {
    uint32_t n_tiles, tpp;       // tiles in total / per plane
    FastDiv div_tpp;
    uint32_t rows_per_pass;      // 256 >> lvpr
};

// E4M3 code of RN64(A/QMAX) for every A in [lo, hi] (f32, lo > 0), or
// ambiguous.  Products QMAX * grid value are exact in f32 (<= 11 bits).
template <int QMAX>
__device__ __forceinline__ float grid_val(uint32_t code) { return e4m3_to_f32(code) * float(QMAX); }

// E4M3 "up" code without branches (v >= 0 finite, saturating at 448)
__device__ __forceinline__ uint32_t e4m3_ceil_f32_bf(float v) {
    const float vc = fminf(v, 448.f);
    const uint32_t sub = uint32_t(ceilf(vc * 512.f));                        // subnormal steps
    const uint32_t nrm = (((__float_as_uint(vc) + 0xFFFFFu) >> 20) - (120u << 3));
    return vc < 0.015625f ? sub : nrm;
}

template <int QMAX>
__device__ __forceinline__ uint32_t scale_code(float lo, float hi, bool &amb) {
    if constexpr (QMAX == 1) {
        // code(A) for A in [lo, hi] is certain iff ceil(lo) == ceil(hi)
        const uint32_t c = e4m3_ceil_f32_bf(hi);
        amb = c != e4m3_ceil_f32_bf(lo);
        return c;
    }
    uint32_t c = e4m3_ceil_f32(QMAX == 1 ? hi : __fmul_ru(hi, 1.0f / QMAX * 1.0000002f));
    if (QMAX > 1) {   // make c the exact ceil code of hi/QMAX
        while (c > 1 && hi <= grid_val<QMAX>(c - 1)) c--;
        while (c < 0x7Eu && hi > grid_val<QMAX>(c)) c++;
    }
    if (c == 0x7Eu) amb = !(lo > float(QMAX) * 416.f);        // saturating band (416, 448]
    else amb = c > 0 && !(lo > grid_val<QMAX>(c - 1));
    return c;
}


template <bool XBF16>
__device__ __forceinline__ float load_x1f(const void *x, uint64_t e) {
    if constexpr (XBF16) return bf16_to_f32(static_cast<const uint16_t *>(x)[e]);
    else return static_cast<const float *>(x)[e];
}

// Rare-path helpers, kept out of line so the compiler cannot hoist their
// address arithmetic into the streaming loop.
// The reference's float64 residual x - C_1[pi_1] - ... (Q/smoothing.py:40).
template <bool XBF16, int S>
__device__ __noinline__ double exact_residual(const uint8_t *xb, const uint16_t *cp, uint32_t e,
                                             uint32_t col, uint32_t d, int K, int a0, int a1,
                                             int a2, int a3) {
    double v = double(load_x1f<XBF16>(xb, e));
    const int ai[4] = {a0, a1, a2, a3};
#pragma unroll
    for (int t = 0; t < S; t++) v = __dsub_rn(v, double(bf16_to_f32(cp[uint32_t(t * K + ai[t]) * d + col])));
    return v;
}

// q = clip(rint(RN64(r / s))) (Q/quant.py:53-54)
template <int QMAX>
__device__ __noinline__ uint32_t exact_code(double r, float s) {
    const double qd = fmin(fmax(rint(__ddiv_rn(r, double(s))), -double(QMAX)), double(QMAX));
    return uint32_t(int(qd));
}

// ------------------------------------------------------------------------
// K5 quantize (fast path: d/8 a power of two <= 32, B/8 a power of two, S <= 4)
// ------------------------------------------------------------------------
struct QuantArgs {
    const void *x;
    const uint16_t *cent;   // [P][S][K][d]
    const uint8_t *asg;     // [P][S][N]
    uint8_t *payload;       // [P][PB]
    uint8_t *scales;        // [P][N*d/B]
    uint32_t N;
    int d, K, B, lvpr, gshift;
    int32_t *status;
    uint32_t pb, ng, lgB;   // payload bytes / scale bytes per plane, log2(B)
    TileArgs ta;
    int v16;                // 16 channels per thread (k_quantize_v4, the ring kernel)
    uint32_t P;
};

struct DequantArgs {
    const uint8_t *payload;
    const uint8_t *scales;
    const uint16_t *cent;
    const uint8_t *asg;
    void *out;
    uint32_t N;
    int d, K, B, lvpr;
    int32_t *status;
    uint32_t pb, ng, lgB;
    TileArgs ta;
    int v16;                // 16 channels per thread (k_dequant_v4, the ring kernel)
    uint32_t P;
};

__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));   // (a & b) | c
    return d;
}

template <int BITS>
struct Codes16 {                     // 16 b-bit fields
    static constexpr int NW = BITS / 2;
    uint32_t w[NW];
};

template <int BITS>
__device__ __forceinline__ Codes16<BITS> load_codes16(const uint8_t *p) {
    Codes16<BITS> c;
    if constexpr (BITS == 2) c.w[0] = __ldg(reinterpret_cast<const uint32_t *>(p));
    else if constexpr (BITS == 4) { uint2 v = __ldg(reinterpret_cast<const uint2 *>(p)); c.w[0] = v.x; c.w[1] = v.y; }
    else { uint4 v = __ldg(reinterpret_cast<const uint4 *>(p)); c.w[0] = v.x; c.w[1] = v.y; c.w[2] = v.z; c.w[3] = v.w; }
    return c;
}

// exact q*s of field k (see qs_fma): field moved to the top of the mantissa
// with one shift + one LOP3, then one FFMA
template <int BITS>
__device__ __forceinline__ float qs16(const Codes16<BITS> &wx, int k, uint32_t mhi, uint32_t one,
                                      float s_hi, float s_off) {
    constexpr int POS = 23 - BITS;
    const int bit = k * BITS, wi = bit >> 5, off = bit & 31;
    const uint32_t v = off <= POS ? (wx.w[wi] << (POS - off)) : (wx.w[wi] >> (off - POS));
    return __fmaf_rn(__uint_as_float(lop3_and_or(v, mhi, one)), s_hi, s_off);
}

__device__ __forceinline__ void cvt16(uint4 a, uint4 b, float c[16]) {
    c[0] = bf16_lo(a.x); c[1] = bf16_hi(a.x); c[2] = bf16_lo(a.y); c[3] = bf16_hi(a.y);
    c[4] = bf16_lo(a.z); c[5] = bf16_hi(a.z); c[6] = bf16_lo(a.w); c[7] = bf16_hi(a.w);
    c[8] = bf16_lo(b.x); c[9] = bf16_hi(b.x); c[10] = bf16_lo(b.y); c[11] = bf16_hi(b.y);
    c[12] = bf16_lo(b.z); c[13] = bf16_hi(b.z); c[14] = bf16_lo(b.w); c[15] = bf16_hi(b.w);
}

template <bool XBF16>
__device__ __forceinline__ void load_x16(const uint8_t *xb, uint32_t e, float r[16]) {
    if constexpr (XBF16) {
        const uint4 *p = reinterpret_cast<const uint4 *>(xb + uint64_t(e) * 2);
        cvt16(__ldg(p), __ldg(p + 1), r);
    } else {
        const float4 *p = reinterpret_cast<const float4 *>(xb + uint64_t(e) * 4);
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const float4 v = __ldg(p + j);
            r[4 * j] = v.x; r[4 * j + 1] = v.y; r[4 * j + 2] = v.z; r[4 * j + 3] = v.w;
        }
    }
}


__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}



// issue the bulk copy of plane p's centroid table into buffer b
__device__ __forceinline__ void stage_table(const uint16_t *cent, uint32_t p, uint32_t tbytes,
                                            uint16_t *buf, uint64_t *bar) {
    mbar_arrive_expect_tx(bar, tbytes);
    bulk_g2s(buf, reinterpret_cast<const uint8_t *>(cent) + uint64_t(p) * tbytes, tbytes, bar);
}


}  // namespace qvg
