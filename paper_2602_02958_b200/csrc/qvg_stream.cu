// qvg_stream.cu — K5 quantize / K6 dequantize as warp-specialised TMA
// streaming kernels (the "v7" fast path for the HBM-bound codec).
//
// One persistent CTA per SM = 16 consumer warps + 1 producer warp.
//  * The producer streams the row-major inputs of the CTA's work items
//    (plane, row range) through an NST-stage shared-memory ring: the big
//    stream (bf16/f32 K/V rows for K5, packed code rows for K6) with one
//    cp.async.bulk per stage, the small byte streams (assignments, scales)
//    with 4-byte cp.async, all completing on the stage's mbarrier.  Bytes in
//    flight per SM = the ring, independent of how many warps compute.
//  * The consumers widen each plane's bf16 centroid tables (staged by TMA one
//    plane ahead) ONCE to f32 in a padded, bank-conflict-free layout plus
//    per-(stage, centroid, 16-channel chunk) metadata {ulp of the smallest
//    non-zero |c|, max|c|}, then run the packed f32x2 element loop:
//      K5: r = x - C_1[pi_1] - ... (FADD2), amax by 3-input max, E4M3 "up"
//          scale with the certified error bound, codes from the magic-number
//          rounding fma(r, 1/s, 1.5*2^23 + 2^(b-1)) packed by integer
//          multiply-add, one reduction per row for the ambiguity test;
//      K6: q*s (FFMA2), + C_S[pi_S] ... + C_1[pi_1] (FADD2) with a per-row
//          exactness certificate for the non-final partial sums, bf16/f32 out.
//    Rows whose fast result is not certified are recomputed in float64 in
//    the reference's order (Q/smoothing.py:40, Q/quant.py:40-55,
//    Q/prq.py:113-132), so the outputs are bit-identical to the reference.
#include "qvg_stream_dev.cuh"

namespace qvg {
namespace stream {

// ============================================================================
// K5 quantize
// ============================================================================
template <int BITS, int S, bool XBF16, int CW, int QU>
__global__ void __launch_bounds__(32 * (CW + 1), 1) k_quantize_stream(QuantArgs a, Geo g) {
    constexpr int QMAX = (1 << (BITS - 1)) - 1;
    constexpr int SS = S > 0 ? S : 1;
    constexpr int FPW = 32 / BITS;
    constexpr uint32_t SIGNS = BITS == 2 ? 0xAAAAAAAAu : (BITS == 4 ? 0x88888888u : 0x80808080u);
    constexpr float MAGIC = 12582912.f + float(1 << (BITS - 1));   // 1.5*2^23 + bias
    constexpr uint32_t XB = XBF16 ? 2 : 4;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ Bars bars;
    uint16_t *const stg = reinterpret_cast<uint16_t *>(smem);
    float *const tab = reinterpret_cast<float *>(smem + g.off_tab);
    float2 *const meta = reinterpret_cast<float2 *>(smem + g.off_meta);
    uint8_t *const ring = smem + g.off_ring;
    __shared__ float rcp_tab[128];          // 1 / e4m3(code): rounded down for 2-bit (see the codes), else RN
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t d = g.d, N = g.N;

    if (threadIdx.x < 128)
        rcp_tab[threadIdx.x] = QMAX == 1 ? __frcp_rd(e4m3_decode_fast(threadIdx.x)) : __frcp_rn(e4m3_decode_fast(threadIdx.x));
    if (threadIdx.x == 0) {
        for (uint32_t k = 0; k < g.nst; k++) {
            mbar_init(&bars.full[k], 1 + 32);
            mbar_init(&bars.empty[k], CW);
        }
        mbar_init(&bars.tab, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    Sched sc;
    sc.init(g);

    if (warp == CW) {
        // ---------------- producer ----------------
        uint32_t s = 0, k = 0, ph = 0;                  // stage, slot, slot phase
        for (; sc.valid(); sc.next(g), s++, k = k + 1 == g.nst ? (ph ^= 1u, 0u) : k + 1) {
            if (s >= g.nst) mbar_wait(&bars.empty[k], ph ^ 1u);
            const uint32_t nr = min(g.R, sc.r1 - sc.i0);
            uint8_t *st = ring + k * g.stage_bytes;
            if (lane == 0) {
                mbar_arrive_expect_tx(&bars.full[k], nr * g.big_row);
                bulk_g2s_cta(st, static_cast<const uint8_t *>(a.x) + (uint64_t(sc.p) * N + sc.i0) * g.big_row,
                             nr * g.big_row, &bars.full[k]);
            }
            // assignments: S streams of nr bytes (nr % 4 == 0), 4 bytes per cp.async
            const uint32_t nw = nr >> 2;
#pragma unroll
            for (int t = 0; t < S; t++)
                for (uint32_t q = lane; q < nw; q += 32)
                    cp_async4(st + g.off_small + t * g.R + 4 * q,
                              a.asg + (uint64_t(sc.p) * S + t) * N + sc.i0 + 4 * q);
            cp_async_arrive_noinc(&bars.full[k]);
        }
        return;
    }

    // ---------------- consumers ----------------
    // Thread = 16 channels of QU rows per stage.  Per row:
    //  * r = x - C_1[pi_1] - ... - C_S[pi_S] in f32 (FADD2 over the padded f32
    //    tables), amax by 3-input |.| max;
    //  * a lane certificate: when x and the chosen centroid blocks are all
    //    multiples of a power of two `unit` and every partial sum stays below
    //    2^23 unit, the f32 chain is exact, i.e. r IS the reference's float64
    //    residual (Q/smoothing.py:40) and the lane's error bound is 0; else
    //    E_l = 2^-22 S (max|r_S| + sum_t max|c_t|) bounds |r_f32 - r_ref|;
    //  * the group's amax lies in [max_l(am_l - E_l), max_l(am_l + E_l)]: the
    //    E4M3 "up" code (Q/quant.py:40-45) is certain unless that interval
    //    straddles a code boundary -> exact f64 maxima of the candidates (rare);
    //  * codes = bits of fma(r, 1/s, 1.5*2^23 + 2^(b-1)) packed by an integer
    //    multiply-add tree.  2-bit certified lanes: with 1/s rounded DOWN and
    //    s/2 a multiple of `unit`, every |r| != s/2 is >= unit away from the
    //    rounding boundary and |r| == s/2 rounds to 0 (half-even), so the codes
    //    are exact with no further test.  Other lanes test an ambiguity window
    //    (E_l plus the 1/s rounding) and recompute flagged elements in float64
    //    (Q/quant.py:48-55).
    const uint32_t lvpr = g.lchunk;                 // log2(threads per row)
    const uint32_t c = threadIdx.x & ((1u << lvpr) - 1u);
    const uint32_t col = c << 4;
    const uint32_t coff = blk_off(c);
    const uint32_t rslot = threadIdx.x >> lvpr, rpp = (CW * 32) >> lvpr;
    const int glanes = 1 << a.gshift;
    const bool slead = (lane & uint32_t(glanes - 1)) == 0;
    const uint32_t pitch = g.pitch, KK = g.K, big_row = g.big_row;
    bool nonfinite = false;
    uint32_t cur = 0xFFFFFFFFu, jp = 0, k = 0, ph = 0;
    uint8_t *pay = a.payload, *scl = a.scales;
    if (S > 0 && !g.stg_global && threadIdx.x == 0 && sc.valid()) stage_table(a.cent, sc.p, g.tbytes, stg, &bars.tab);
    for (; sc.valid(); sc.next(g), k = k + 1 == g.nst ? (ph ^= 1u, 0u) : k + 1) {
        const uint32_t p = sc.p;
        if (p != cur) {
            if (S > 0) {
                named_sync_consumers<CW>();
                if (!g.stg_global) mbar_wait(&bars.tab, jp & 1u);
                widen(g.stg_global ? a.cent + size_t(p) * (g.tbytes / 2) : stg, tab, meta, g, CW * 32);
                named_sync_consumers<CW>();
                if (!g.stg_global && threadIdx.x == 0) {
                    const int64_t nx = sc.next_plane(g);
                    if (nx >= 0) {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        stage_table(a.cent, uint32_t(nx), g.tbytes, stg, &bars.tab);
                    }
                }
                jp++;
            }
            pay = a.payload + uint64_t(p) * a.pb;
            scl = a.scales + uint64_t(p) * a.ng;
            cur = p;
        }
        mbar_wait(&bars.full[k], ph);
        const uint8_t *st = ring + k * g.stage_bytes;
        const uint32_t nr = min(g.R, sc.r1 - sc.i0);
#pragma unroll 1
        for (int u = 0; u < QU; u++) {
            // ---- one row: residual, amax, lane certificate
            const uint32_t l = u * rpp + rslot;
            const bool valid = l < nr;
            const uint32_t lr = valid ? l : nr - 1;
            const uint8_t *xr = st + lr * big_row + col * XB;
            float2 r[8];
            float xmn = __int_as_float(0x7F800000);
            if constexpr (XBF16) {
                const uint4 w0 = *reinterpret_cast<const uint4 *>(xr);
                const uint4 w1 = *reinterpret_cast<const uint4 *>(xr + 16);
                cvt16(w0, w1, reinterpret_cast<float *>(r));
                if constexpr (S > 0) {
                    float m0 = xmn, m1 = xmn;
#pragma unroll
                    for (int q = 0; q < 8; q += 2) {
                        m0 = min3_abs(m0, r[q].x, r[q].y);
                        m1 = min3_abs(m1, r[q + 1].x, r[q + 1].y);
                    }
                    xmn = fminf(m0, m1);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const float4 v = *reinterpret_cast<const float4 *>(xr + 16 * j);
                    r[2 * j] = make_float2(v.x, v.y);
                    r[2 * j + 1] = make_float2(v.z, v.w);
                }
            }
            int ai[SS];
#pragma unroll
            for (int t = 0; t < S; t++) ai[t] = st[g.off_small + t * g.R + lr];
            float csum = 0.f, cunit = __int_as_float(0x7F800000), cwt = 0.f;
#pragma unroll
            for (int t = 0; t < S; t++) {
                const uint32_t row = uint32_t(t * int(KK) + ai[t]);
                const float *cr = tab + row * pitch + coff;
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const float4 cv = *reinterpret_cast<const float4 *>(cr + 4 * j);
                    r[2 * j] = __fadd2_rn(r[2 * j], make_float2(-cv.x, -cv.y));
                    r[2 * j + 1] = __fadd2_rn(r[2 * j + 1], make_float2(-cv.z, -cv.w));
                }
                const float2 m = meta[(row << lvpr) + c];
                csum = __fadd_ru(csum, m.y);
                if (t > 0) cwt = __fmaf_ru(float(t), m.y, cwt);
                cunit = fminf(cunit, m.x);
            }
            float m0 = 0.f, m1 = 0.f;
#pragma unroll
            for (int q = 0; q < 8; q += 2) {
                m0 = max3_nan_abs(m0, r[q].x, r[q].y);
                m1 = max3_nan_abs(m1, r[q + 1].x, r[q + 1].y);
            }
            const float mx = max_nan(m0, m1);
            nonfinite |= !(mx <= 3.402823466e38f) && valid;
            // certificate (bf16 x): |partials| <= max|x| + sum max|c| <= max|r_S| + 2 sum max|c|
            const uint32_t xe = __float_as_uint(xmn) & 0x7F800000u;
            const float un = fminf(xe > (7u << 23) ? __uint_as_float(xe - (7u << 23)) : 0.f, cunit);
            const bool cert = S == 0 || (XBF16 && __fmaf_ru(2.f, csum, mx) < un * 8388608.f);
            const float El = cert ? 0.f : err_bound(float(S), mx, cwt);
            // ---- the group's amax interval and its E4M3 "up" code
            float lo = __fsub_rd(mx, El), hi = __fadd_ru(mx, El);
            if (glanes == 4) {           // the three partners at once: one shuffle latency
                const float l1 = __shfl_xor_sync(0xffffffffu, lo, 1), l2 = __shfl_xor_sync(0xffffffffu, lo, 2),
                            l3 = __shfl_xor_sync(0xffffffffu, lo, 3);
                const float h1 = __shfl_xor_sync(0xffffffffu, hi, 1), h2 = __shfl_xor_sync(0xffffffffu, hi, 2),
                            h3 = __shfl_xor_sync(0xffffffffu, hi, 3);
                lo = fmaxf(fmaxf(lo, l1), fmaxf(l2, l3));
                hi = fmaxf(fmaxf(hi, h1), fmaxf(h2, h3));
            } else {
                for (int m = 1; m < glanes; m <<= 1) {
                    lo = fmaxf(lo, __shfl_xor_sync(0xffffffffu, lo, m));
                    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, m));
                }
            }
            bool cb = false;
            uint32_t code;
            if constexpr (QMAX == 1) {
                // normal E4M3 range: the ceiling code from the f32 bits (3 mantissa
                // bits kept, rounded up), its lower neighbour's value one step down
                const float hc = fminf(hi, 448.f);
                const uint32_t t = (__float_as_uint(hc) + 0xFFFFFu) & 0xFFF00000u;
                if (hc >= 0.015625f) {
                    code = (t >> 20) - (120u << 3);
                    cb = !(lo > __uint_as_float(t - 0x100000u));
                } else {
                    code = e4m3_ceil_f32_bf(hi);
                    cb = !(lo > e4m3_decode_fast(code - 1u));
                }
            } else {
                code = scale_code<QMAX>(lo > 0.f ? lo : hi, hi, cb);
            }
            const bool zero = hi == 0.f;                            // exact all-zero group
            if (zero || !(lo > 0.f)) code = 0x38u;
            const bool camb = valid && !zero && (cb || !(lo > 0.f));
            if (__any_sync(0xffffffffu, camb)) {                    // exact scale (rare)
                double a64 = 0.0;
                if (camb) {
                    // elements whose true |r| could reach the group's lower bound
                    const float thr = __fsub_rd(lo, El);
                    uint32_t cand = 0;
#pragma unroll
                    for (int q = 0; q < 8; q++)
                        cand |= (fabsf(r[q].x) >= thr ? 1u << (2 * q) : 0u) | (fabsf(r[q].y) >= thr ? 2u << (2 * q) : 0u);
                    if (cand)
                        a64 = exact_absmax<S, XBF16>(xr, tab, pitch, coff, int(KK), ai[0], ai[SS > 1 ? 1 : 0],
                                                     ai[SS > 2 ? 2 : 0], ai[SS > 3 ? 3 : 0], cand);
                }
                for (int m = 1; m < glanes; m <<= 1) a64 = fmax(a64, shfl_xor_d(a64, m));
                if (camb) code = a64 == 0.0 ? 0x38u : e4m3_encode_up(__ddiv_rn(a64, double(QMAX)));
            }
            // ---- codes
            const float sv = e4m3_decode_fast(code);
            const float inv = rcp_tab[code & 0x7Fu];
            const float2 inv2 = make_float2(inv, inv);
            if (__any_sync(0xffffffffu, code == 0x7Eu)) {
                // saturated scale (amax / QMAX > 448, e.g. outlier channels of a
                // coarse K): the reference clips, clip(rint(r / s), +-QMAX) ==
                // rint(clamp(r, +-QMAX s) / s), so the magic-number codes stay in
                // range and the lane needs no exact fallback for it
                const float lim = code == 0x7Eu ? float(QMAX) * sv : __int_as_float(0x7F800000);
#pragma unroll
                for (int q = 0; q < 8; q++)
                    r[q] = make_float2(fminf(fmaxf(r[q].x, -lim), lim), fminf(fmaxf(r[q].y, -lim), lim));
            }
            float2 yv[8];
#pragma unroll
            for (int q = 0; q < 8; q++) yv[q] = __ffma2_rn(r[q], inv2, make_float2(MAGIC, MAGIC));
            Words4 b32;
#pragma unroll
            for (int w = 0; w < BITS / 2; w++) {
                uint32_t v[FPW];
#pragma unroll
                for (int k2 = 0; k2 < FPW; k2++) {
                    const int e = w * FPW + k2;
                    v[k2] = __float_as_uint((e & 1) ? yv[e >> 1].y : yv[e >> 1].x);
                }
#pragma unroll
                for (int span = 1; span < FPW; span *= 2)
#pragma unroll
                    for (int k2 = 0; k2 < FPW; k2 += 2 * span) v[k2] += v[k2 + span] << (BITS * span);
                b32.w[w] = (v[0] - magic_sum<BITS>()) ^ SIGNS;
            }
            const bool allv = !(El < 0.125f * sv);
            const float thr = window_thr<QMAX>(sv, inv, El);
            bool amb;
            if constexpr (QMAX == 1) {
                // exact without a window: certified lane, s/2 a multiple of unit
                // (its lowest set bit >= 2^(exponent(s) - 4)), s/2 < 2^22 unit
                const float sexp = __uint_as_float(__float_as_uint(sv) & 0x7F800000u);
                const bool fast = cert && sexp * 0.0625f >= un && sv < un * 4194304.f;
                amb = false;
                if (__any_sync(0xffffffffu, !fast)) {
                    const float h = 0.5f * sv;
                    const float2 pa = make_float2(-h * h, -h * h);
                    float w0 = __int_as_float(0x7F800000), w1 = w0;
#pragma unroll
                    for (int q = 0; q < 8; q += 2) {
                        const float2 g0 = __ffma2_rn(r[q], r[q], pa);
                        const float2 g1 = __ffma2_rn(r[q + 1], r[q + 1], pa);
                        w0 = min3_abs(w0, g0.x, g0.y);
                        w1 = min3_abs(w1, g1.x, g1.y);
                    }
                    amb = !fast && (allv || fminf(w0, w1) <= thr);
                }
            } else {
                const float2 pa = make_float2(-MAGIC, -MAGIC);
                float w0 = 0.f, w1 = 0.f;
#pragma unroll
                for (int q = 0; q < 8; q += 2) {
                    const float2 q0 = __fadd2_rn(yv[q], pa), q1 = __fadd2_rn(yv[q + 1], pa);
                    const float2 d0 = __ffma2_rn(r[q], inv2, make_float2(-q0.x, -q0.y));
                    const float2 d1 = __ffma2_rn(r[q + 1], inv2, make_float2(-q1.x, -q1.y));
                    w0 = max3_abs(w0, d0.x, d0.y);
                    w1 = max3_abs(w1, d1.x, d1.y);
                }
                amb = allv || fmaxf(w0, w1) >= thr;
            }
            if (amb && valid)          // exact codes of the flagged elements (rare)
                b32 = fix_codes<BITS, S, XBF16>(xr, tab, pitch, coff, int(KK), ai[0], ai[SS > 1 ? 1 : 0],
                                                ai[SS > 2 ? 2 : 0], ai[SS > 3 ? 3 : 0], sv, inv, El, thr, allv, b32);
            if (valid) {
                const uint32_t e0 = (sc.i0 + lr) * d + col;
                uint8_t *plp = pay + ((e0 * BITS) >> 3);
                if constexpr (BITS == 2) *reinterpret_cast<uint32_t *>(plp) = b32.w[0];
                else if constexpr (BITS == 4) *reinterpret_cast<uint2 *>(plp) = make_uint2(b32.w[0], b32.w[1]);
                else *reinterpret_cast<uint4 *>(plp) = make_uint4(b32.w[0], b32.w[1], b32.w[2], b32.w[3]);
                if (slead) scl[e0 >> a.lgB] = uint8_t(code);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.empty[k]);
    }
    const uint32_t all = __reduce_or_sync(0xffffffffu, nonfinite ? uint32_t(QVG_STATUS_NONFINITE) : 0u);
    if (all && lane == 0) atomicOr(a.status, int(all));
}

// ============================================================================
// K5 quantize, 32 channels per thread (d = 128 / 256, groups of >= 32)
// ============================================================================
// Same pipeline and numerics as k_quantize_stream; a thread owns a 32-channel
// slice of a row, so the per-row work (certificate, group interval, scale code,
// window thresholds, stores) is amortised over twice the elements and a
// 64-channel group spans two lanes (one shuffle round).
// Bank-conflict-free table reads: slices are stored as 36 floats (8 blocks of
// 4 + {unit, max |c|} + 2 spare) and table rows padded to a multiple of 32
// floats, so the 4 slices of one table row sit on bank quads 0..3 (+ block).
// With d = 128 a quarter-warp holds two rows (rho = 0, 1) reading unrelated
// table rows; the rho = 1 row reads its slice's upper half first (blocks 4-7,
// then 0-3), which puts the two rows on disjoint quads.  Its registers hold
// the slice half-rotated, so x is loaded with the same rotation and the two
// halves of the packed codes are swapped back at the store.
// A stage is released to the producer as soon as its bytes are in registers
// (the rare exact paths re-read x from global memory), so the whole ring stays
// in flight.
__device__ __forceinline__ void widen32(const uint16_t *src, float *tab, const Geo &g, uint32_t nthr) {
    const uint32_t ns = g.d / 32, nslice = g.tbytes / 64;          // 32-channel slices of all tables
    for (uint32_t q = threadIdx.x; q < nslice; q += nthr) {
        const uint4 *sp = reinterpret_cast<const uint4 *>(src + size_t(q) * 32);
        float c[32];
        cvt16(sp[0], sp[1], c);
        cvt16(sp[2], sp[3], c + 16);
        float mx = 0.f, mn = __int_as_float(0x7F800000);
#pragma unroll
        for (int k = 0; k < 32; k++) {
            const float a = fabsf(c[k]);
            mx = max_nan(mx, a);
            mn = a > 0.f ? fminf(mn, a) : mn;
        }
        float *dst = tab + size_t(q / ns) * g.pitch + 36u * (q % ns);
#pragma unroll
        for (int j = 0; j < 8; j++)
            reinterpret_cast<float4 *>(dst)[j] = make_float4(c[4 * j], c[4 * j + 1], c[4 * j + 2], c[4 * j + 3]);
        float unit;
        if (mn == __int_as_float(0x7F800000)) unit = mn;
        else {
            const uint32_t eb = __float_as_uint(mn) & 0x7F800000u;
            unit = eb > (7u << 23) ? __uint_as_float(eb - (7u << 23)) : 0.f;
        }
        *reinterpret_cast<float2 *>(dst + 32) = make_float2(unit, mx);
    }
}

template <int BITS, int S, bool XBF16, int CW>
__global__ void __launch_bounds__(32 * (CW + 1), 1) k_quantize_ring32(QuantArgs a, Geo g) {
    constexpr int QMAX = (1 << (BITS - 1)) - 1;
    constexpr int SS = S > 0 ? S : 1;
    constexpr int FPW = 32 / BITS;
    constexpr uint32_t SIGNS = BITS == 2 ? 0xAAAAAAAAu : (BITS == 4 ? 0x88888888u : 0x80808080u);
    constexpr float MAGIC = 12582912.f + float(1 << (BITS - 1));
    constexpr uint32_t XB = XBF16 ? 2 : 4;
    constexpr int NWD = BITS;               // 32-bit code words per 32 fields
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ Bars bars;
    uint16_t *const stg = reinterpret_cast<uint16_t *>(smem);
    float *const tab = reinterpret_cast<float *>(smem + g.off_tab);
    uint8_t *const ring = smem + g.off_ring;
    __shared__ float rcp_tab[128];
    __shared__ uint32_t rcp_sink[CW * 32];  // release-ordering stores (see below), one word per thread
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t d = g.d, N = g.N;

    if (threadIdx.x < 128)
        rcp_tab[threadIdx.x] = QMAX == 1 ? __frcp_rd(e4m3_decode_fast(threadIdx.x)) : __frcp_rn(e4m3_decode_fast(threadIdx.x));
    if (threadIdx.x == 0) {
        for (uint32_t k = 0; k < g.nst; k++) {
            mbar_init(&bars.full[k], 1 + 32);
            mbar_init(&bars.empty[k], CW);
        }
        mbar_init(&bars.tab, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    Sched sc;
    sc.init(g);

    if (warp == CW) {
        // ---------------- producer ----------------
        uint32_t s = 0, k = 0, ph = 0;
        for (; sc.valid(); sc.next(g), s++, k = k + 1 == g.nst ? (ph ^= 1u, 0u) : k + 1) {
            if (s >= g.nst) mbar_wait(&bars.empty[k], ph ^ 1u);
            const uint32_t nr = min(g.R, sc.r1 - sc.i0);
            uint8_t *st = ring + k * g.stage_bytes;
            if (lane == 0) {
                mbar_arrive_expect_tx(&bars.full[k], nr * g.big_row);
                bulk_g2s_cta(st, static_cast<const uint8_t *>(a.x) + (uint64_t(sc.p) * N + sc.i0) * g.big_row,
                             nr * g.big_row, &bars.full[k]);
            }
            const uint32_t nw = nr >> 2;
#pragma unroll
            for (int t = 0; t < S; t++)
                for (uint32_t q = lane; q < nw; q += 32)
                    cp_async4(st + g.off_small + t * g.R + 4 * q,
                              a.asg + (uint64_t(sc.p) * S + t) * N + sc.i0 + 4 * q);
            cp_async_arrive_noinc(&bars.full[k]);
        }
        return;
    }

    // ---------------- consumers ----------------
    const uint32_t lt = g.lchunk;                       // log2(threads per row) = log2(d / 32)
    const uint32_t c = threadIdx.x & ((1u << lt) - 1u);
    const uint32_t rho = d == 128 ? (uint32_t(lane) >> 2) & 1u : 0u;
    const uint32_t rslot = threadIdx.x >> lt;
    const uint32_t soff = 36u * c;                      // this thread's slice in a table row
    const uint32_t hlo = 16u * rho, hhi = 16u * (rho ^ 1u);   // slot halves -> channel halves
    const int glanes = 1 << (a.gshift - 1);             // B / 32 lanes per group
    const bool slead = (uint32_t(lane) & uint32_t(glanes - 1)) == 0;
    const uint32_t pitch = g.pitch, KK = g.K, big_row = g.big_row;
    bool nonfinite = false;
    uint32_t cur = 0xFFFFFFFFu, jp = 0, k = 0, ph = 0;
    uint8_t *pay = a.payload, *scl = a.scales;
    if (!g.stg_global && threadIdx.x == 0 && sc.valid()) stage_table(a.cent, sc.p, g.tbytes, stg, &bars.tab);
    for (; sc.valid(); sc.next(g), k = k + 1 == g.nst ? (ph ^= 1u, 0u) : k + 1) {
        const uint32_t p = sc.p;
        if (p != cur) {
            named_sync_consumers<CW>();
            if (!g.stg_global) mbar_wait(&bars.tab, jp & 1u);
            widen32(g.stg_global ? a.cent + size_t(p) * (g.tbytes / 2) : stg, tab, g, CW * 32);
            named_sync_consumers<CW>();
            if (!g.stg_global && threadIdx.x == 0) {
                const int64_t nx = sc.next_plane(g);
                if (nx >= 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    stage_table(a.cent, uint32_t(nx), g.tbytes, stg, &bars.tab);
                }
            }
            jp++;
            pay = a.payload + uint64_t(p) * a.pb;
            scl = a.scales + uint64_t(p) * a.ng;
            cur = p;
        }
        mbar_wait(&bars.full[k], ph);
        if (g.dbg == 1) {                      // measurement: consumers only drain the ring
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars.empty[k]);
            continue;
        }
        const uint8_t *st = ring + k * g.stage_bytes;
        const uint32_t nr = min(g.R, sc.r1 - sc.i0);
        const uint32_t l = rslot;
        const bool valid = l < nr;
        const uint32_t lr = valid ? l : nr - 1;
        const uint8_t *xr = st + lr * big_row + 32u * c * XB;     // the slice's x in the ring slot
        float2 r[16];
        float xmn = __int_as_float(0x7F800000);
        {
            const uint8_t *xa = xr + hlo * XB, *xb = xr + hhi * XB;   // slot halves (rotated for rho = 1)
            if constexpr (XBF16) {
                cvt16(*reinterpret_cast<const uint4 *>(xa), *reinterpret_cast<const uint4 *>(xa + 16),
                      reinterpret_cast<float *>(r));
                cvt16(*reinterpret_cast<const uint4 *>(xb), *reinterpret_cast<const uint4 *>(xb + 16),
                      reinterpret_cast<float *>(r + 8));
                float m0 = xmn, m1 = xmn;
#pragma unroll
                for (int q = 0; q < 16; q += 2) {
                    m0 = min3_abs(m0, r[q].x, r[q].y);
                    m1 = min3_abs(m1, r[q + 1].x, r[q + 1].y);
                }
                xmn = fminf(m0, m1);
            } else {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const float4 v = *reinterpret_cast<const float4 *>(xa + 16 * j);
                    const float4 w = *reinterpret_cast<const float4 *>(xb + 16 * j);
                    r[2 * j] = make_float2(v.x, v.y);
                    r[2 * j + 1] = make_float2(v.z, v.w);
                    r[8 + 2 * j] = make_float2(w.x, w.y);
                    r[8 + 2 * j + 1] = make_float2(w.z, w.w);
                }
            }
        }
        int ai[SS];
#pragma unroll
        for (int t = 0; t < S; t++) ai[t] = st[g.off_small + t * g.R + lr];
        // the stage is released after the scale codes: the exact-scale path
        // below re-reads x from the ring slot (shared memory, not L2)
        // the rare exact paths re-read x from global memory (the slot may be refilled)
        const uint32_t xrow = sc.i0 + lr;
        auto xg = [&]() { return static_cast<const uint8_t *>(a.x) + (uint64_t(p) * N + xrow) * big_row + 32u * c * XB; };
        float csum = 0.f, cunit = __int_as_float(0x7F800000), cwt = 0.f;   // cwt = sum_t t max|C_t| (0-based t)
#pragma unroll
        for (int t = 0; t < S; t++) {
            const float *cr = tab + uint32_t(t * int(KK) + ai[t]) * pitch + soff;
            const float *ca = cr + hlo, *cb = cr + hhi;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const float4 u = *reinterpret_cast<const float4 *>(ca + 4 * j);
                r[2 * j] = __fadd2_rn(r[2 * j], make_float2(-u.x, -u.y));
                r[2 * j + 1] = __fadd2_rn(r[2 * j + 1], make_float2(-u.z, -u.w));
            }
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const float4 u = *reinterpret_cast<const float4 *>(cb + 4 * j);
                r[8 + 2 * j] = __fadd2_rn(r[8 + 2 * j], make_float2(-u.x, -u.y));
                r[8 + 2 * j + 1] = __fadd2_rn(r[8 + 2 * j + 1], make_float2(-u.z, -u.w));
            }
            const float2 m = *reinterpret_cast<const float2 *>(cr + 32);
            csum = __fadd_ru(csum, m.y);
            if (t > 0) cwt = __fmaf_ru(float(t), m.y, cwt);
            cunit = fminf(cunit, m.x);
        }
        float m0 = 0.f, m1 = 0.f;
#pragma unroll
        for (int q = 0; q < 16; q += 2) {
            m0 = max3_nan_abs(m0, r[q].x, r[q].y);
            m1 = max3_nan_abs(m1, r[q + 1].x, r[q + 1].y);
        }
        const float mx = max_nan(m0, m1);
        nonfinite |= !(mx <= 3.402823466e38f) && valid;
        const uint32_t xe = __float_as_uint(xmn) & 0x7F800000u;
        const float un = fminf(xe > (7u << 23) ? __uint_as_float(xe - (7u << 23)) : 0.f, cunit);
        const bool cert = XBF16 && __fmaf_ru(2.f, csum, mx) < un * 8388608.f;
        const float El = cert ? 0.f : err_bound(float(S), mx, cwt);
        float lo = __fsub_rd(mx, El), hi = __fadd_ru(mx, El);
        for (int m = 1; m < glanes; m <<= 1) {
            lo = fmaxf(lo, __shfl_xor_sync(0xffffffffu, lo, m));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, m));
        }
        bool cb = false;
        uint32_t code;
        if constexpr (QMAX == 1) {
            const float hc = fminf(hi, 448.f);
            const uint32_t t = (__float_as_uint(hc) + 0xFFFFFu) & 0xFFF00000u;
            if (hc >= 0.015625f) {
                code = (t >> 20) - (120u << 3);
                cb = !(lo > __uint_as_float(t - 0x100000u));
            } else {
                code = e4m3_ceil_f32_bf(hi);
                cb = !(lo > e4m3_decode_fast(code - 1u));
            }
        } else {
            code = scale_code<QMAX>(lo > 0.f ? lo : hi, hi, cb);
        }
        const bool zero = hi == 0.f;
        if (zero || !(lo > 0.f)) code = 0x38u;
        const bool camb = valid && !zero && (cb || !(lo > 0.f));
        if (__any_sync(0xffffffffu, camb)) {                    // exact scale (rare)
            double a64 = 0.0;
            if (camb) {
                const float thr = __fsub_rd(lo, El);
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    uint32_t cand = 0;
#pragma unroll
                    for (int q = 0; q < 8; q++)
                        cand |= (fabsf(r[8 * h + q].x) >= thr ? 1u << (2 * q) : 0u) |
                                (fabsf(r[8 * h + q].y) >= thr ? 2u << (2 * q) : 0u);
                    const uint32_t hc = h == 0 ? hlo : hhi;
                    if (cand)
                        a64 = fmax(a64, exact_absmax<S, XBF16>(xr + hc * XB, tab, pitch, soff + hc, int(KK), ai[0],
                                                               ai[SS > 1 ? 1 : 0], ai[SS > 2 ? 2 : 0],
                                                               ai[SS > 3 ? 3 : 0], cand));
                }
            }
            for (int m = 1; m < glanes; m <<= 1) a64 = fmax(a64, shfl_xor_d(a64, m));
            if (camb) code = a64 == 0.0 ? 0x38u : e4m3_encode_up(__ddiv_rn(a64, double(QMAX)));
        }
        // every shared-memory load of the stage must have landed before the
        // release (the producer's TMA may overwrite the stage right after it):
        // a store of a value depending on one register of each load (x, the
        // assignments, and through `code` the exact-scale re-reads) cannot
        // issue before those loads complete
        {
            uint32_t dep = code;
#pragma unroll
            for (int t = 0; t < S; t++) dep ^= uint32_t(ai[t]);
#pragma unroll
            for (int q = 0; q < 16; q += 2) dep ^= __float_as_uint(r[q].x);
            reinterpret_cast<volatile uint32_t *>(rcp_sink)[threadIdx.x] = dep;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.empty[k]);
        // ---- codes (slot order), fixed up per 16-field half, stored in channel order
        const float sv = e4m3_decode_fast(code);
        const float inv = rcp_tab[code & 0x7Fu];
        const float2 inv2 = make_float2(inv, inv);
        uint32_t w[NWD];
#pragma unroll
        for (int wd = 0; wd < NWD; wd++) {
            uint32_t v[FPW];
#pragma unroll
            for (int k2 = 0; k2 < FPW; k2++) {
                const int e = wd * FPW + k2;
                const float2 y = __ffma2_rn(r[e >> 1], inv2, make_float2(MAGIC, MAGIC));
                v[k2] = __float_as_uint((e & 1) ? y.y : y.x);
            }
#pragma unroll
            for (int span = 1; span < FPW; span *= 2)
#pragma unroll
                for (int k2 = 0; k2 < FPW; k2 += 2 * span) v[k2] += v[k2 + span] << (BITS * span);
            w[wd] = (v[0] - magic_sum<BITS>()) ^ SIGNS;
        }
        const bool allv = !(El < 0.125f * sv) || code == 0x7Eu;
        const float thr = window_thr<QMAX>(sv, inv, El);
        bool amb;
        if constexpr (QMAX == 1) {
            const float sexp = __uint_as_float(__float_as_uint(sv) & 0x7F800000u);
            const bool fast = cert && code != 0x7Eu && sexp * 0.0625f >= un && sv < un * 4194304.f;
            amb = false;
            if (__any_sync(0xffffffffu, !fast)) {
                const float h = 0.5f * sv;
                const float2 pa = make_float2(-h * h, -h * h);
                float w0 = __int_as_float(0x7F800000), w1 = w0;
#pragma unroll
                for (int q = 0; q < 16; q += 2) {
                    const float2 g0 = __ffma2_rn(r[q], r[q], pa);
                    const float2 g1 = __ffma2_rn(r[q + 1], r[q + 1], pa);
                    w0 = min3_abs(w0, g0.x, g0.y);
                    w1 = min3_abs(w1, g1.x, g1.y);
                }
                amb = !fast && (allv || fminf(w0, w1) <= thr);
            }
        } else {
            const float2 pa = make_float2(-MAGIC, -MAGIC);
            float w0 = 0.f, w1 = 0.f;
#pragma unroll
            for (int q = 0; q < 16; q += 2) {
                const float2 y0 = __ffma2_rn(r[q], inv2, make_float2(MAGIC, MAGIC));
                const float2 y1 = __ffma2_rn(r[q + 1], inv2, make_float2(MAGIC, MAGIC));
                const float2 q0 = __fadd2_rn(y0, pa), q1 = __fadd2_rn(y1, pa);
                const float2 d0 = __ffma2_rn(r[q], inv2, make_float2(-q0.x, -q0.y));
                const float2 d1 = __ffma2_rn(r[q + 1], inv2, make_float2(-q1.x, -q1.y));
                w0 = max3_abs(w0, d0.x, d0.y);
                w1 = max3_abs(w1, d1.x, d1.y);
            }
            amb = allv || fmaxf(w0, w1) >= thr;
        }
        if (amb && valid) {                                     // exact codes (rare), per half
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint32_t hc = h == 0 ? hlo : hhi;
                Words4 b;
#pragma unroll
                for (int wd = 0; wd < NWD / 2; wd++) b.w[wd] = w[h * (NWD / 2) + wd];
                b = fix_codes<BITS, S, XBF16>(xg() + hc * XB, tab, pitch, soff + hc, int(KK), ai[0],
                                              ai[SS > 1 ? 1 : 0], ai[SS > 2 ? 2 : 0], ai[SS > 3 ? 3 : 0], sv,
                                              inv, El, thr, allv, b);
#pragma unroll
                for (int wd = 0; wd < NWD / 2; wd++) w[h * (NWD / 2) + wd] = b.w[wd];
            }
        }
        if (valid) {
            // slot halves back to channel order (rho = 1 holds the upper half first)
            uint32_t o[NWD];
#pragma unroll
            for (int wd = 0; wd < NWD; wd++) {
                const int sw = (wd + NWD / 2) % NWD;
                o[wd] = rho ? w[sw] : w[wd];
            }
            const uint32_t e0 = (sc.i0 + lr) * d + 32u * c;
            uint8_t *plp = pay + ((e0 * BITS) >> 3);
            if constexpr (NWD == 2) *reinterpret_cast<uint2 *>(plp) = make_uint2(o[0], o[1]);
            else {
#pragma unroll
                for (int q4 = 0; q4 < NWD / 4; q4++)
                    reinterpret_cast<uint4 *>(plp)[q4] = make_uint4(o[4 * q4], o[4 * q4 + 1], o[4 * q4 + 2], o[4 * q4 + 3]);
            }
            if (slead) scl[e0 >> a.lgB] = uint8_t(code);
        }
    }
    const uint32_t all = __reduce_or_sync(0xffffffffu, nonfinite ? uint32_t(QVG_STATUS_NONFINITE) : 0u);
    if (all && lane == 0) atomicOr(a.status, int(all));
}

// ============================================================================
// K6 dequantize
// ============================================================================
template <int BITS, int S, bool OBF16>
__global__ void __launch_bounds__(kThreads, 1) k_dequant_stream(DequantArgs a, Geo g) {
    constexpr int SS = S > 0 ? S : 1;
    constexpr uint32_t SIGNS = BITS == 2 ? 0xAAAAAAAAu : (BITS == 4 ? 0x88888888u : 0x80808080u);
    constexpr int POS = 23 - BITS;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ Bars bars;
    uint16_t *const stg = reinterpret_cast<uint16_t *>(smem);
    float *const tab = reinterpret_cast<float *>(smem + g.off_tab);
    float2 *const meta = reinterpret_cast<float2 *>(smem + g.off_meta);
    uint8_t *const ring = smem + g.off_ring;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t d = g.d, N = g.N;

    if (threadIdx.x == 0) {
        for (uint32_t k = 0; k < g.nst; k++) {
            mbar_init(&bars.full[k], 1 + 32);
            mbar_init(&bars.empty[k], kCW);
        }
        mbar_init(&bars.tab, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    Sched sc;
    sc.init(g);

    if (warp == kCW) {
        // ---------------- producer ----------------
        uint32_t s = 0, k = 0, ph = 0;                  // stage, slot, slot phase
        for (; sc.valid(); sc.next(g), s++, k = k + 1 == g.nst ? (ph ^= 1u, 0u) : k + 1) {
            if (s >= g.nst) mbar_wait(&bars.empty[k], ph ^ 1u);
            const uint32_t nr = min(g.R, sc.r1 - sc.i0);
            uint8_t *st = ring + k * g.stage_bytes;
            if (lane == 0) {
                mbar_arrive_expect_tx(&bars.full[k], nr * g.big_row);
                bulk_g2s_cta(st, a.payload + uint64_t(sc.p) * a.pb + uint64_t(sc.i0) * g.big_row,
                             nr * g.big_row, &bars.full[k]);
            }
            // scales: nr * small_row bytes; assignments: S streams of nr bytes
            const uint32_t nws = (nr * g.small_row) >> 2;
            for (uint32_t q = lane; q < nws; q += 32)
                cp_async4(st + g.off_small + 4 * q,
                          a.scales + (uint64_t(sc.p) * N + sc.i0) * g.small_row + 4 * q);
            const uint32_t nw = nr >> 2;
            uint8_t *sa = st + g.off_small + g.R * g.small_row;
#pragma unroll
            for (int t = 0; t < S; t++)
                for (uint32_t q = lane; q < nw; q += 32)
                    cp_async4(sa + t * g.R + 4 * q, a.asg + (uint64_t(sc.p) * S + t) * N + sc.i0 + 4 * q);
            cp_async_arrive_noinc(&bars.full[k]);
        }
        return;
    }

    // ---------------- consumers ----------------
    const uint32_t lvpr = g.lchunk;
    const uint32_t c = threadIdx.x & ((1u << lvpr) - 1u);
    const uint32_t col = c << 4;
    const uint32_t coff = blk_off(c);
    const uint32_t rslot = threadIdx.x >> lvpr, rpp = (kCW * 32) >> lvpr;
    const uint32_t mhi = ((1u << BITS) - 1u) << POS, one = 0x3F800000u;
    bool bad_scale = false, bad_asg = false;
    uint32_t cur = 0xFFFFFFFFu, jp = 0, k = 0, ph = 0;
    if (S > 0 && !g.stg_global && threadIdx.x == 0 && sc.valid()) stage_table(a.cent, sc.p, g.tbytes, stg, &bars.tab);
    for (; sc.valid(); sc.next(g), k = k + 1 == g.nst ? (ph ^= 1u, 0u) : k + 1) {
        const uint32_t p = sc.p;
        if (S > 0 && p != cur) {
            named_sync_consumers();
            if (!g.stg_global) mbar_wait(&bars.tab, jp & 1u);
            widen(g.stg_global ? a.cent + size_t(p) * (g.tbytes / 2) : stg, tab, meta, g);
            named_sync_consumers();
            if (!g.stg_global && threadIdx.x == 0) {
                const int64_t nx = sc.next_plane(g);
                if (nx >= 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    stage_table(a.cent, uint32_t(nx), g.tbytes, stg, &bars.tab);
                }
            }
            jp++;
        }
        cur = p;
        mbar_wait(&bars.full[k], ph);
        const uint8_t *st = ring + k * g.stage_bytes;
        const uint8_t *sa = st + g.off_small + g.R * g.small_row;
        const uint32_t nr = min(g.R, sc.r1 - sc.i0);
        const uint64_t obase = (uint64_t(p) * N + sc.i0) * d + col;   // this stage's first output row
        Codes16<BITS> w[kU];
        uint32_t scb[kU], lr[kU];
        int ai[kU][SS];
#pragma unroll
        for (int u = 0; u < kU; u++) {
            const uint32_t l = u * rpp + rslot;
            lr[u] = l < nr ? l : nr - 1;
            const uint8_t *cr = st + lr[u] * g.big_row + ((col * BITS) >> 3);
            if constexpr (BITS == 2) w[u].w[0] = *reinterpret_cast<const uint32_t *>(cr);
            else if constexpr (BITS == 4) {
                const uint2 v = *reinterpret_cast<const uint2 *>(cr);
                w[u].w[0] = v.x; w[u].w[1] = v.y;
            } else {
                const uint4 v = *reinterpret_cast<const uint4 *>(cr);
                w[u].w[0] = v.x; w[u].w[1] = v.y; w[u].w[2] = v.z; w[u].w[3] = v.w;
            }
            scb[u] = st[g.off_small + lr[u] * g.small_row + (col >> a.lgB)];
#pragma unroll
            for (int t = 0; t < S; t++) {
                const int at = sa[t * g.R + lr[u]];
                bad_asg |= at >= int(g.K);
                ai[u][t] = at < int(g.K) ? at : 0;
            }
        }
#pragma unroll
        for (int u = 0; u < kU; u++) {
            const bool valid = u * rpp + rslot < nr;
            bad_scale |= (scb[u] & 0x7Fu) == 0x7Fu;
            const float sv = e4m3_decode_fast(scb[u]);
            Codes16<BITS> wx;
#pragma unroll
            for (int q = 0; q < Codes16<BITS>::NW; q++) wx.w[q] = w[u].w[q] ^ SIGNS;
            const float2 s_hi = make_float2(sv * float(1 << BITS), sv * float(1 << BITS));
            const float2 s_off = make_float2(sv * (-1.5f * float(1 << BITS)), sv * (-1.5f * float(1 << BITS)));
            float2 y[8];
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const int b0 = 2 * q * BITS, b1 = (2 * q + 1) * BITS;
                const uint32_t v0 = (b0 & 31) <= POS ? (wx.w[b0 >> 5] << (POS - (b0 & 31))) : (wx.w[b0 >> 5] >> ((b0 & 31) - POS));
                const uint32_t v1 = (b1 & 31) <= POS ? (wx.w[b1 >> 5] << (POS - (b1 & 31))) : (wx.w[b1 >> 5] >> ((b1 & 31) - POS));
                const float2 f = make_float2(__uint_as_float(lop3_and_or(v0, mhi, one)),
                                             __uint_as_float(lop3_and_or(v1, mhi, one)));
                y[q] = __ffma2_rn(f, s_hi, s_off);          // q*s, exact
            }
            // every non-final partial sum exact in f32 <= all terms multiples of
            // `unit` and sum of magnitudes < 2^24 unit
            // (a row whose codes are all zero has q*s == 0: only the centroid terms count)
            bool cert = true, swap01 = false;
            if constexpr (S >= 2) {
                uint32_t anyq = 0;
#pragma unroll
                for (int q = 0; q < Codes16<BITS>::NW; q++) anyq |= w[u].w[q];
                const float unit_s = anyq ? fmaxf(__uint_as_float((__float_as_uint(sv) & 0x7F800000u) - (3u << 23)), 0.001953125f)
                                          : __int_as_float(0x7F800000);
                const float bound_s = anyq ? sv * float(1 << (BITS - 1)) : 0.f;
                float unit = unit_s, bound = bound_s;
#pragma unroll
                for (int t = 1; t < S; t++) {
                    const float2 m = meta[(uint32_t(t * int(g.K) + ai[u][t]) << lvpr) + c];
                    unit = fminf(unit, m.x);
                    bound = __fadd_ru(bound, m.y);
                }
                cert = S == 2 && !anyq ? true : bound < unit * 16777216.f;
                if constexpr (S == 2) {
                    // the other order: q*s + C_1 exact in f32, C_2 added last = ONE
                    // rounding of the exact three-term sum.  That is the reference's
                    // RN32 of its float64 chain when that chain is exact too (all terms
                    // multiples of the common unit, magnitudes < 2^53 units); it
                    // certifies rows whose stage-2 centroid block has tiny entries
                    if (!cert) {
                        const float2 m0 = meta[(uint32_t(ai[u][0]) << lvpr) + c];
                        swap01 = __fadd_ru(bound_s, m0.y) < fminf(unit_s, m0.x) * 16777216.f &&
                                 __fadd_ru(bound, m0.y) < fminf(unit, m0.x) * 9007199254740992.f;
                        cert = swap01;
                    }
                }
            }
            if constexpr (S == 2) {
                const float *ra = tab + uint32_t(int(g.K) + ai[u][1]) * g.pitch + coff;
                const float *rb = tab + uint32_t(ai[u][0]) * g.pitch + coff;
                const float *first = swap01 ? rb : ra, *last = swap01 ? ra : rb;
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const float4 cv = *reinterpret_cast<const float4 *>(first + 4 * j);
                    y[2 * j] = __fadd2_rn(y[2 * j], make_float2(cv.x, cv.y));
                    y[2 * j + 1] = __fadd2_rn(y[2 * j + 1], make_float2(cv.z, cv.w));
                }
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const float4 cv = *reinterpret_cast<const float4 *>(last + 4 * j);
                    y[2 * j] = __fadd2_rn(y[2 * j], make_float2(cv.x, cv.y));
                    y[2 * j + 1] = __fadd2_rn(y[2 * j + 1], make_float2(cv.z, cv.w));
                }
            } else {
#pragma unroll
                for (int t = S - 1; t >= 0; t--) {             // reversed(stages)
                    const float *row = tab + uint32_t(t * int(g.K) + ai[u][t]) * g.pitch + coff;
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        const float4 cv = *reinterpret_cast<const float4 *>(row + 4 * j);
                        y[2 * j] = __fadd2_rn(y[2 * j], make_float2(cv.x, cv.y));
                        y[2 * j + 1] = __fadd2_rn(y[2 * j + 1], make_float2(cv.z, cv.w));
                    }
                }
            }
            if constexpr (S >= 2) {
                if (!cert) {
                    // per element: each non-final partial sum P' = P + c is exact iff
                    // (P' - P) - c == 0 and (P' - c) - P == 0 (Fast2Sum from the larger
                    // operand gives the non-zero rounding error otherwise)
                    uint32_t bad = 0;
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        const int b0 = 2 * q * BITS, b1 = (2 * q + 1) * BITS;
                        const uint32_t v0 = (b0 & 31) <= POS ? (wx.w[b0 >> 5] << (POS - (b0 & 31))) : (wx.w[b0 >> 5] >> ((b0 & 31) - POS));
                        const uint32_t v1 = (b1 & 31) <= POS ? (wx.w[b1 >> 5] << (POS - (b1 & 31))) : (wx.w[b1 >> 5] >> ((b1 & 31) - POS));
                        float2 P = __ffma2_rn(make_float2(__uint_as_float(lop3_and_or(v0, mhi, one)),
                                                          __uint_as_float(lop3_and_or(v1, mhi, one))), s_hi, s_off);
                        bool e0 = false, e1 = false;
#pragma unroll
                        for (int t = S - 1; t >= 1; t--) {
                            const float2 cc = *reinterpret_cast<const float2 *>(
                                tab + uint32_t(t * int(g.K) + ai[u][t]) * g.pitch + coff + 2 * q);
                            const float2 P2 = __fadd2_rn(P, cc);
                            const float2 d1 = __fadd2_rn(__fadd2_rn(P2, make_float2(-P.x, -P.y)), make_float2(-cc.x, -cc.y));
                            const float2 d2 = __fadd2_rn(__fadd2_rn(P2, make_float2(-cc.x, -cc.y)), make_float2(-P.x, -P.y));
                            e0 |= d1.x != 0.f || d2.x != 0.f;
                            e1 |= d1.y != 0.f || d2.y != 0.f;
                            P = P2;
                        }
                        bad |= (e0 ? 1u << (2 * q) : 0u) | (e1 ? 2u << (2 * q) : 0u);
                    }
#pragma unroll
                    for (int kk = 0; kk < 16; kk++) {   // rare: the element in the reference's float64 chain
                        if (!((bad >> kk) & 1u)) continue;
                        const int b = kk * BITS, wi = b >> 5, o = b & 31;
                        const uint32_t v = o <= POS ? (wx.w[wi] << (POS - o)) : (wx.w[wi] >> (o - POS));
                        const float qs = __fmaf_rn(__uint_as_float(lop3_and_or(v, mhi, one)), s_hi.x, s_off.x);
                        const float rr = exact_addback<S>(qs, tab, g.pitch, coff + kk, int(g.K), ai[u][0],
                                                          ai[u][SS > 1 ? 1 : 0], ai[u][SS > 2 ? 2 : 0],
                                                          ai[u][SS > 3 ? 3 : 0]);
                        if (kk & 1) y[kk >> 1].y = rr; else y[kk >> 1].x = rr;
                    }
                }
            }
            if (!valid) continue;
            const uint64_t o = obase + uint64_t(lr[u] * d);
            if constexpr (OBF16) {
                uint32_t v[8];
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    __nv_bfloat162 h = __floats2bfloat162_rn(y[q].x, y[q].y);
                    v[q] = *reinterpret_cast<uint32_t *>(&h);
                }
                uint4 *op = reinterpret_cast<uint4 *>(static_cast<uint16_t *>(a.out) + o);
                op[0] = make_uint4(v[0], v[1], v[2], v[3]);
                op[1] = make_uint4(v[4], v[5], v[6], v[7]);
            } else {
                float4 *op = reinterpret_cast<float4 *>(static_cast<float *>(a.out) + o);
#pragma unroll
                for (int q = 0; q < 4; q++) op[q] = make_float4(y[2 * q].x, y[2 * q].y, y[2 * q + 1].x, y[2 * q + 1].y);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.empty[k]);
    }
    const uint32_t stat = (bad_scale ? QVG_STATUS_NAN_SCALE : 0u) | (bad_asg ? QVG_STATUS_BAD_ASSIGN : 0u);
    const uint32_t all = __reduce_or_sync(0xffffffffu, stat);
    if (all && lane == 0) atomicOr(a.status, int(all));
}

// ============================================================================
// host: geometry and dispatch
// ============================================================================
static int ilog2i(int v) { int l = 0; while ((1 << l) < v) l++; return l; }

// smem: [bf16 staging][f32 padded tables][metadata][ring]; false when the
// configuration does not fit this kernel (callers fall back to v4/v5/v6)
static bool plan(bool quant, int64_t P, int64_t N, int d, int S, int K, int bits, int B, int xbytes,
                 uintptr_t align_probe, Geo &g, size_t &smem, int &grid, int cw = kCW, int ru = kU,
                 bool c32 = false) {
    if (S < 1 || S > 4 || d % 16 != 0 || d > 512 || N < 4 || N % 4 != 0) return false;
    const int n = d / 16;
    if (n & (n - 1)) return false;
    if ((align_probe & 3u) != 0) return false;
    if (P * N >= (int64_t(1) << 31) || N * d >= (int64_t(1) << 31)) return false;
    if (c32 && (d != 128 && d != 256)) return false;
    // c32: 32-channel slices of 36 floats (the 4-float pad holds the slice's
    // {unit, max |c|}), rows padded to a multiple of 32 floats (see k_quantize_ring32)
    const uint32_t R = uint32_t(cw * 32 / (c32 ? d / 32 : n) * ru);
    const uint32_t pitch = c32 ? uint32_t((36 * (d / 32) + 31) / 32 * 32) : uint32_t(16 * n + 4 * ((n + 1) / 2));
    const size_t tbytes = size_t(S) * K * d * 2;
    const size_t tabb = size_t(S) * K * pitch * 4;
    const size_t nchunk = c32 ? 0 : size_t(S) * K * n;
    size_t off_tab = (tbytes + 127) & ~size_t(127);
    size_t off_meta = off_tab + ((tabb + 127) & ~size_t(127));
    size_t off_ring = off_meta + ((nchunk * 8 + 1023) & ~size_t(1023));
    uint32_t stg_global = 0;
    uint32_t big_row, small_row;
    if (quant) {
        big_row = uint32_t(d * xbytes);
        small_row = 0;
    } else {
        if ((size_t(d) * bits) % 128 != 0) return false;       // 16-byte code rows
        big_row = uint32_t(d * bits / 8);
        small_row = uint32_t(d / B);
        if ((N * small_row) % 4 != 0) return false;
    }
    const size_t big = size_t(R) * big_row;
    const size_t small = size_t(R) * small_row + size_t(S) * R;
    const size_t stage = (big + ((small + 15) & ~size_t(15)) + 127) & ~size_t(127);
    const size_t budget = 227 * 1024 - 4096;      // dynamic smem; static arrays (barriers, sinks, tables) need the rest
    // c32 widens straight from global memory (L2-resident tables): the staging
    // copy's 32 KB buys one more ring stage (4 vs 3: 4.47 vs 4.58 ms)
    if (off_ring + 2 * stage > budget || (quant && c32)) {
        // no room for the bf16 staging copy: widen straight from global memory
        stg_global = 1;
        off_tab = 0;
        off_meta = (tabb + 127) & ~size_t(127);
        off_ring = off_meta + ((nchunk * 8 + 1023) & ~size_t(1023));
        if (off_ring + 2 * stage > budget) return false;
    }
    uint32_t nst = uint32_t((budget - off_ring) / stage);
    if (nst > 8) nst = 8;
    // work items: planes split into row ranges (multiples of R) until every
    // CTA has several
    const int64_t ctas = 148;
    int64_t ipp = 1;
    while (P * ipp < 6 * ctas && (N + ipp * 2 - 1) / (ipp * 2) >= int64_t(4 * R)) ipp *= 2;
    int64_t rpi = (N + ipp - 1) / ipp;
    rpi = (rpi + R - 1) / R * R;
    ipp = (N + rpi - 1) / rpi;
    g = Geo{uint32_t(P), uint32_t(N), uint32_t(d), uint32_t(K), R, nst, pitch, uint32_t(tbytes),
            uint32_t(nchunk), uint32_t(ilog2i(c32 ? d / 32 : n)), uint32_t(ipp), uint32_t(rpi), uint32_t(P * ipp),
            uint32_t(off_tab), uint32_t(off_meta), uint32_t(off_ring), uint32_t(stage), big_row, small_row,
            uint32_t(big), 0u, stg_global};
    if (const char *e = getenv("QVG_STREAM_DBG")) g.dbg = uint32_t(atoi(e));
    if (const char *e = getenv("QVG_STREAM_NST")) { const uint32_t v = uint32_t(atoi(e)); if (v >= 2 && v < nst) nst = v; g.nst = nst; }
    smem = off_ring + nst * stage;
    grid = int(P * ipp < ctas ? P * ipp : ctas);
    return true;
}

template <int BITS, int S, bool XB, int CW, int QU>
static int launch_q1(const QuantArgs &a, const Geo &g, size_t smem, int grid, cudaStream_t st) {
    cudaFuncSetAttribute(k_quantize_stream<BITS, S, XB, CW, QU>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k_quantize_stream<BITS, S, XB, CW, QU><<<grid, 32 * (CW + 1), smem, st>>>(a, g);
    return 1;
}

// 15 consumer warps x 2 rows per thread per stage: measured best on the bench
// cache (4.68 ms; 23 warps x 1 row at <= 80 registers spills: 5.7 ms, 20 x 1:
// 6.3 ms, 15 x 1: 4.9 ms)
template <int BITS, int S>
static int launch_q(const QuantArgs &a, bool xbf16, const Geo &g, size_t smem, int grid, cudaStream_t st) {
    return xbf16 ? launch_q1<BITS, S, true, kCW, kU>(a, g, smem, grid, st)
                 : launch_q1<BITS, S, false, kCW, kU>(a, g, smem, grid, st);
}

template <int BITS, int S>
static int launch_q32(const QuantArgs &a, bool xbf16, const Geo &g, size_t smem, int grid, cudaStream_t st) {
    if (xbf16) {
        cudaFuncSetAttribute(k_quantize_ring32<BITS, S, true, kCW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k_quantize_ring32<BITS, S, true, kCW><<<grid, 32 * (kCW + 1), smem, st>>>(a, g);
    } else {
        cudaFuncSetAttribute(k_quantize_ring32<BITS, S, false, kCW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k_quantize_ring32<BITS, S, false, kCW><<<grid, 32 * (kCW + 1), smem, st>>>(a, g);
    }
    return 1;
}

template <int BITS, int S>
static int launch_d(const DequantArgs &a, bool obf16, const Geo &g, size_t smem, int grid, cudaStream_t st) {
    if (obf16) {
        cudaFuncSetAttribute(k_dequant_stream<BITS, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k_dequant_stream<BITS, S, true><<<grid, kThreads, smem, st>>>(a, g);
    } else {
        cudaFuncSetAttribute(k_dequant_stream<BITS, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k_dequant_stream<BITS, S, false><<<grid, kThreads, smem, st>>>(a, g);
    }
    return 1;
}

}  // namespace stream

// returns 1 when the streaming kernel was launched, 0 when the caller must
// use another kernel for this configuration
int launch_quantize_stream(const QuantArgs &a, int64_t P, int bits, int S, bool xbf16, cudaStream_t st) {
    using namespace stream;
    Geo g;
    size_t smem;
    int grid;
    const uintptr_t probe = reinterpret_cast<uintptr_t>(a.asg) | reinterpret_cast<uintptr_t>(a.x);
    // 32 channels per thread for 2-bit, two-stage caches with 128 / 256-channel
    // rows and groups >= 32 (Self-Forcing: 4.54 vs 4.68 ms).  Everywhere else
    // the 16-channel kernel measured faster: its per-lane certificates cover
    // 16 channels (fewer lanes need the window test), and its f32 tables are
    // smaller per stage (the 32-channel tables of S = 4, K = 64 leave 2 ring
    // stages).  microbench N 4K/64K, K 64: S = 1 2-bit +15..70%, S = 2 4-bit
    // +9%, S = 3 +7% / +24%, S = 4 +32% / x2 (2-bit / 4-bit)
    static const bool no32 = [] { const char *e = getenv("QVG_QUANT_C16"); return e && atoi(e) == 1; }();
    if (!no32 && S == 2 && bits == 2 && a.B % 32 == 0 &&
        plan(true, P, a.N, a.d, S, a.K, bits, a.B, xbf16 ? 2 : 4, probe, g, smem, grid, kCW, 1, true)) {
#define QV_Q32(BB)                                                          \
        switch (S) {                                                        \
            case 1: return launch_q32<BB, 1>(a, xbf16, g, smem, grid, st); \
            case 2: return launch_q32<BB, 2>(a, xbf16, g, smem, grid, st); \
            case 3: return launch_q32<BB, 3>(a, xbf16, g, smem, grid, st); \
            default: return launch_q32<BB, 4>(a, xbf16, g, smem, grid, st); \
        }
        if (bits == 2) { QV_Q32(2) }
        if (bits == 4) { QV_Q32(4) }
        QV_Q32(8)
#undef QV_Q32
    }
    if (!plan(true, P, a.N, a.d, S, a.K, bits, a.B, xbf16 ? 2 : 4, probe, g, smem, grid)) return 0;
    if ((reinterpret_cast<uintptr_t>(a.x) & 15u) != 0) return 0;
#define QV_Q(BB)                                                      \
    switch (S) {                                                      \
        case 1: return launch_q<BB, 1>(a, xbf16, g, smem, grid, st); \
        case 2: return launch_q<BB, 2>(a, xbf16, g, smem, grid, st); \
        case 3: return launch_q<BB, 3>(a, xbf16, g, smem, grid, st); \
        default: return launch_q<BB, 4>(a, xbf16, g, smem, grid, st); \
    }
    if (bits == 2) { QV_Q(2) }
    if (bits == 4) { QV_Q(4) }
    QV_Q(8)
#undef QV_Q
}

int launch_dequantize_stream(const DequantArgs &a, int64_t P, int bits, int S, bool obf16, cudaStream_t st) {
    using namespace stream;
    Geo g;
    size_t smem;
    int grid;
    const uintptr_t probe = reinterpret_cast<uintptr_t>(a.asg) | reinterpret_cast<uintptr_t>(a.scales);
    if (!plan(false, P, a.N, a.d, S, a.K, bits, a.B, 0, probe, g, smem, grid)) return 0;
    if ((reinterpret_cast<uintptr_t>(a.payload) & 15u) != 0 || (a.pb % 16) != 0) return 0;
#define QV_D(BB)                                                      \
    switch (S) {                                                      \
        case 1: return launch_d<BB, 1>(a, obf16, g, smem, grid, st); \
        case 2: return launch_d<BB, 2>(a, obf16, g, smem, grid, st); \
        case 3: return launch_d<BB, 3>(a, obf16, g, smem, grid, st); \
        default: return launch_d<BB, 4>(a, obf16, g, smem, grid, st); \
    }
    if (bits == 2) { QV_D(2) }
    if (bits == 4) { QV_D(4) }
    QV_D(8)
#undef QV_D
}

}  // namespace qvg
