// qvg_dring.cu — K6 dequantize, 32 channels per thread (the default K6 for
// d = 128 / 256 and groups of >= 32 channels).
//
// The codec kernels are issue-bound (~13 instructions per element per thread
// is the budget at the HBM roofline), so the per-row work (codes, scale,
// assignments, certificate, addresses, loop control) is amortised over 32
// channels instead of 16: one persistent CTA per SM = 15 consumer warps + a
// producer warp streaming the packed code rows and the scale / assignment
// bytes through an mbarrier ring (as k_dequant_stream); the consumers widen
// each plane's bf16 centroid tables once into the padded f32 layout of
// each plane's bf16 centroid tables are re-laid once into a padded bf16 layout
// (32-channel slices at word 16c + 4(c/2), rows padded to a multiple of 128
// bytes, the slices' certificate metadata {unit, max |c|} per 16-channel half
// after the last slice) and added with FHADD.BF16 (`add.rn.f32.bf16`, f32 =
// bf16 + f32, one rounding): half the shared-memory wavefronts of f32 tables,
// which is what bounds this kernel (l1tex data pipe at ~90% with f32 tables).
// Bank conflicts: chunk k of slice c sits on bank quad 4c + c/2 + k (mod 8);
// the second row of a quarter-warp (d = 128) reads its upper half first, so
// the 8 threads of every LDS.128 hit 8 distinct quads.  Its code words are
// swapped to match and each 16-channel half is written back with one 256-bit
// store (STG.E.ENL2.256) to its own sector.
//
// Numerics are those of k_dequant_stream (Q/prq.py:113-132, Q/quant.py:151):
// q*s exact by one FFMA, the reference's float64 add-back order reproduced in
// f32 under a per-half exactness certificate (every non-final partial sum
// exact), the S = 2 swapped-order certificate, Fast2Sum-checked elements and
// the float64 chain otherwise; bf16 output = RNE(the f32 value).
#include "qvg_stream_dev.cuh"

namespace qvg {
namespace dring {

constexpr int kCW = 15;                    // consumer warps
constexpr int kThreads = 32 * (kCW + 1);   // + producer warp

struct DGeo {
    uint32_t P, N, d, K;
    uint32_t R;            // rows per stage = kCW * 32 / (d / 32)
    uint32_t nst;          // ring stages
    uint32_t pitch;        // padded bf16 table row pitch (32-bit words)
    uint32_t nslice;       // 32-channel table slices per plane (S*K*d/32)
    uint32_t lslc;         // log2(d / 32)
    uint32_t ipp, rpi, n_items;
    uint32_t off_stg, off_ring, stage_bytes, big_row, small_row, off_small;
    uint32_t tbytes;       // bf16 table bytes per plane (S*K*d*2)
    uint32_t stg_global;   // 1: no room for the staging copy, widen from global memory (L2)
};

struct DSched {
    uint32_t it, it1, p, r1, i0;
    __device__ __forceinline__ void init(const DGeo &g) {
        it = uint32_t((uint64_t(blockIdx.x) * g.n_items) / gridDim.x);
        it1 = uint32_t((uint64_t(blockIdx.x + 1) * g.n_items) / gridDim.x);
        start(g);
    }
    __device__ __forceinline__ void start(const DGeo &g) {
        if (it >= it1) return;
        p = it / g.ipp;
        i0 = (it - p * g.ipp) * g.rpi;
        r1 = min(g.N, i0 + g.rpi);
    }
    __device__ __forceinline__ bool valid() const { return it < it1; }
    __device__ __forceinline__ void next(const DGeo &g) {
        i0 += g.R;
        if (i0 >= r1) { it++; start(g); }
    }
};

// {ulp of the smallest non-zero |c| (+inf when all zero, 0 when that is not a
// normal bf16), max |c| (NaN-propagating)} of 16 values
__device__ __forceinline__ float2 meta16(const float *c) {
    float mx = 0.f, mn = __int_as_float(0x7F800000);
#pragma unroll
    for (int k = 0; k < 16; k++) {
        const float a = fabsf(c[k]);
        mx = stream::max_nan(mx, a);
        mn = a > 0.f ? fminf(mn, a) : mn;
    }
    float unit;
    if (mn == __int_as_float(0x7F800000)) unit = mn;
    else {
        const uint32_t eb = __float_as_uint(mn) & 0x7F800000u;
        unit = eb > (7u << 23) ? __uint_as_float(eb - (7u << 23)) : 0.f;
    }
    return make_float2(unit, mx);
}

// word offset of 32-channel slice c in a padded table row: 16 c + 4 (c / 2)
__host__ __device__ __forceinline__ uint32_t slice_w(uint32_t c) { return 16u * c + 4u * (c >> 1); }

// re-lay one plane's bf16 tables [S*K][d] (the staged copy, or global memory)
// into the padded layout: row pitch g.pitch words, slice c at slice_w(c), the
// slices' metadata {unit, max |c|} x 2 halves (float4) after the last slice
__device__ __forceinline__ void widen_h(const uint16_t *src, uint32_t *tab, const DGeo &g) {
    const uint32_t ns = g.d / 32, mo = slice_w(ns - 1) + 16u;
    for (uint32_t q = threadIdx.x; q < g.nslice; q += kCW * 32) {
        const uint4 *sp = reinterpret_cast<const uint4 *>(src + size_t(q) * 32);
        const uint4 v0 = sp[0], v1 = sp[1], v2 = sp[2], v3 = sp[3];
        float c[32];
        cvt16(v0, v1, c);
        cvt16(v2, v3, c + 16);
        const uint32_t cs = q % ns;
        uint32_t *row = tab + size_t(q / ns) * g.pitch;
        uint4 *dst = reinterpret_cast<uint4 *>(row + slice_w(cs));
        dst[0] = v0; dst[1] = v1; dst[2] = v2; dst[3] = v3;
        const float2 m0 = meta16(c), m1 = meta16(c + 16);
        *reinterpret_cast<float4 *>(row + mo + 4u * cs) = make_float4(m0.x, m0.y, m1.x, m1.y);
    }
}

// f32 = bf16 (low / high half of w) + y, one rounding (FHADD.BF16)
__device__ __forceinline__ float2 fhadd2(uint32_t w, float2 y) {
    float r0, r1;
    asm("{.reg .b16 l, h;\nmov.b32 {l, h}, %2;\nadd.rn.f32.bf16 %0, l, %3;\nadd.rn.f32.bf16 %1, h, %4;\n}"
        : "=f"(r0), "=f"(r1)
        : "r"(w), "f"(y.x), "f"(y.y));
    return make_float2(r0, r1);
}

// the reference's float64 add-back of one element (Q/prq.py:113-132), padded bf16 tables
template <int S>
__device__ __noinline__ float exact_addback_p(float qs, const uint32_t *tab, uint32_t pitch, uint32_t wo, uint32_t hsel,
                                              int K, int a0, int a1, int a2, int a3) {
    const int ai[4] = {a0, a1, a2, a3};
    double acc = double(qs);
#pragma unroll
    for (int t = S - 1; t >= 0; t--) {
        const uint32_t w = tab[uint32_t(t * K + ai[t]) * pitch + wo];
        acc = __dadd_rn(acc, double(__uint_as_float(hsel ? (w & 0xFFFF0000u) : (w << 16))));
    }
    return __double2float_rn(acc);
}

// one 256-bit global store (STG.E.ENL2.256) of 8 words to a 32-byte aligned address
__device__ __forceinline__ void st_global_v8(void *p, const uint32_t *v) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

__device__ __forceinline__ uint32_t lop3_and_xor(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0x6A;" : "=r"(d) : "r"(a), "r"(b), "r"(c));   // (a & b) ^ c
    return d;
}

// ============================================================================
// K6 dequantize
// ============================================================================
template <int BITS, int S, bool OBF16>
__global__ void __launch_bounds__(kThreads, 1) k_dequant_ring32(DequantArgs a, DGeo g) {
    constexpr int SS = S > 0 ? S : 1;
    constexpr uint32_t SIGNS = BITS == 2 ? 0xAAAAAAAAu : (BITS == 4 ? 0x88888888u : 0x80808080u);
    constexpr int POS = 23 - BITS;
    constexpr int HW = BITS / 2;                 // code words per 16-field half
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ stream::Bars bars;
    __shared__ uint32_t sink[kCW * 32];          // release-ordering stores, one word per thread
    uint32_t *const tab = reinterpret_cast<uint32_t *>(smem);           // padded bf16 tables (word view)
    uint16_t *const stg = reinterpret_cast<uint16_t *>(smem + g.off_stg);   // next plane's bf16 tables (TMA)
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
    DSched sc;
    sc.init(g);

    if (warp == kCW) {
        // ---------------- producer ----------------
        uint32_t s = 0, k = 0, ph = 0;
        for (; sc.valid(); sc.next(g), s++, k = k + 1 == g.nst ? (ph ^= 1u, 0u) : k + 1) {
            if (s >= g.nst) mbar_wait(&bars.empty[k], ph ^ 1u);
            const uint32_t nr = min(g.R, sc.r1 - sc.i0);
            uint8_t *st = ring + k * g.stage_bytes;
            if (lane == 0) {
                mbar_arrive_expect_tx(&bars.full[k], nr * g.big_row);
                stream::bulk_g2s_cta(st, a.payload + uint64_t(sc.p) * a.pb + uint64_t(sc.i0) * g.big_row,
                                     nr * g.big_row, &bars.full[k]);
            }
            const uint32_t nws = (nr * g.small_row) >> 2;
            for (uint32_t q = lane; q < nws; q += 32)
                stream::cp_async4(st + g.off_small + 4 * q, a.scales + (uint64_t(sc.p) * N + sc.i0) * g.small_row + 4 * q);
            const uint32_t nw = nr >> 2;
            uint8_t *sa = st + g.off_small + g.R * g.small_row;
#pragma unroll
            for (int t = 0; t < S; t++)
                for (uint32_t q = lane; q < nw; q += 32)
                    stream::cp_async4(sa + t * g.R + 4 * q, a.asg + (uint64_t(sc.p) * S + t) * N + sc.i0 + 4 * q);
            stream::cp_async_arrive_noinc(&bars.full[k]);
        }
        return;
    }

    // ---------------- consumers ----------------
    const uint32_t ls = g.lslc;
    const uint32_t c = threadIdx.x & ((1u << ls) - 1u);
    const uint32_t rslot = threadIdx.x >> ls;
    const uint32_t rho = d == 128 ? (uint32_t(lane) >> 2) & 1u : 0u;     // slot half 0 = channel half rho
    const uint32_t col = 32u * c, soff = slice_w(c), moff = slice_w((d >> 5) - 1) + 16u + 4u * c;
    const uint32_t mhi = ((1u << BITS) - 1u) << POS, one = 0x3F800000u;
    // field u at mantissa bits [POS, 23) of 1.0, its sign bit (bit 22) flipped
    // by the same LOP3: f = 1 + (u ^ 2^(b-1)) / 2^b
    const uint32_t kx = one | (1u << 22);
    const uint32_t KK = g.K, pitch = g.pitch;
    bool bad_scale = false, bad_asg = false;
    uint32_t cur = 0xFFFFFFFFu, k = 0, ph = 0, jp = 0;
    // the first plane's tables; each later plane's are staged by TMA while the
    // previous plane streams
    if (!g.stg_global && threadIdx.x == 0 && sc.valid()) stage_table(a.cent, sc.p, g.tbytes, stg, &bars.tab);
    for (; sc.valid(); sc.next(g), k = k + 1 == g.nst ? (ph ^= 1u, 0u) : k + 1) {
        if (sc.p != cur) {
            stream::named_sync_consumers<kCW>();
            if (!g.stg_global) mbar_wait(&bars.tab, jp & 1u);
            widen_h(g.stg_global ? a.cent + size_t(sc.p) * (g.tbytes / 2) : stg, tab, g);
            stream::named_sync_consumers<kCW>();
            if (!g.stg_global && threadIdx.x == 0 && (sc.p + 1) * g.ipp < sc.it1) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                stage_table(a.cent, sc.p + 1, g.tbytes, stg, &bars.tab);
            }
            jp++;
            cur = sc.p;
        }
        mbar_wait(&bars.full[k], ph);
        const uint8_t *st = ring + k * g.stage_bytes;
        const uint32_t nr = min(g.R, sc.r1 - sc.i0);
        const bool valid = rslot < nr;
        const uint32_t lr = valid ? rslot : nr - 1;
        uint32_t w[BITS];
        {
            const uint8_t *cp = st + lr * g.big_row + c * (4u * BITS);
            if constexpr (BITS == 2) {
                const uint2 v = *reinterpret_cast<const uint2 *>(cp);
                w[0] = v.x; w[1] = v.y;
            } else {
#pragma unroll
                for (int q = 0; q < BITS / 4; q++) {
                    const uint4 v = reinterpret_cast<const uint4 *>(cp)[q];
                    w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
                }
            }
        }
        const uint32_t scb = st[g.off_small + lr * g.small_row + (col >> a.lgB)];
        int ai[SS];
#pragma unroll
        for (int t = 0; t < S; t++) {
            const int at = st[g.off_small + g.R * g.small_row + t * g.R + lr];
            bad_asg |= at >= int(KK);
            ai[t] = at < int(KK) ? at : 0;
        }
        {   // every shared-memory read of the stage has landed before the release
            uint32_t dep = scb;
#pragma unroll
            for (int t = 0; t < S; t++) dep ^= uint32_t(ai[t]);
#pragma unroll
            for (int q = 0; q < BITS; q++) dep ^= w[q];
            reinterpret_cast<volatile uint32_t *>(sink)[threadIdx.x] = dep;
        }
        __syncwarp();
        if (lane == 0) stream::mbar_arrive(&bars.empty[k]);

        bad_scale |= (scb & 0x7Fu) == 0x7Fu;
        const float sv = e4m3_decode_fast(scb);
        // slot order: half 0 = channel half rho
        if (rho) {
#pragma unroll
            for (int q = 0; q < HW; q++) { const uint32_t t = w[q]; w[q] = w[q + HW]; w[q + HW] = t; }
        }
        const float2 s_hi = make_float2(sv * float(1 << BITS), sv * float(1 << BITS));
        const float2 s_off = make_float2(sv * (-1.5f * float(1 << BITS)), sv * (-1.5f * float(1 << BITS)));
        float2 y[16];
#pragma unroll
        for (int q = 0; q < 16; q++) {
            const int b0 = 2 * q * BITS, b1 = (2 * q + 1) * BITS;
            const uint32_t v0 = (b0 & 31) <= POS ? (w[b0 >> 5] << (POS - (b0 & 31))) : (w[b0 >> 5] >> ((b0 & 31) - POS));
            const uint32_t v1 = (b1 & 31) <= POS ? (w[b1 >> 5] << (POS - (b1 & 31))) : (w[b1 >> 5] >> ((b1 & 31) - POS));
            const float2 f = make_float2(__uint_as_float(lop3_and_xor(v0, mhi, kx)), __uint_as_float(lop3_and_xor(v1, mhi, kx)));
            y[q] = __ffma2_rn(f, s_hi, s_off);          // q*s, exact
        }
        const uint32_t *row[SS];
#pragma unroll
        for (int t = 0; t < S; t++) row[t] = tab + (uint32_t(t) * KK + uint32_t(ai[t])) * pitch;
        // per slot half: certificate (every non-final partial sum exact in f32,
        // see k_dequant_stream), S = 2 swapped order, add-back
        bool certh[2];
#pragma unroll
        for (int sh = 0; sh < 2; sh++) {
            const uint32_t chh = uint32_t(sh) ^ rho;                 // channel half
            bool cert = true, swap01 = false;
            if constexpr (S >= 2) {
                uint32_t anyq = 0;
#pragma unroll
                for (int q = 0; q < HW; q++) anyq |= w[sh * HW + q];
                const float unit_s = anyq ? fmaxf(__uint_as_float((__float_as_uint(sv) & 0x7F800000u) - (3u << 23)), 0.001953125f)
                                          : __int_as_float(0x7F800000);
                const float bound_s = anyq ? sv * float(1 << (BITS - 1)) : 0.f;
                float unit = unit_s, bound = bound_s;
#pragma unroll
                for (int t = 1; t < S; t++) {
                    const float4 m = *reinterpret_cast<const float4 *>(row[t] + moff);
                    unit = fminf(unit, chh ? m.z : m.x);
                    bound = __fadd_ru(bound, chh ? m.w : m.y);
                }
                cert = S == 2 && !anyq ? true : bound < unit * 16777216.f;
                if constexpr (S == 2) {
                    const float4 m = *reinterpret_cast<const float4 *>(row[0] + moff);
                    const float u0 = chh ? m.z : m.x, m0 = chh ? m.w : m.y;
                    swap01 = !cert && __fadd_ru(bound_s, m0) < fminf(unit_s, u0) * 16777216.f &&
                             __fadd_ru(bound, m0) < fminf(unit, u0) * 9007199254740992.f;
                    cert = cert || swap01;
                }
            }
            certh[sh] = cert;
            const uint32_t *r1 = row[SS > 1 ? 1 : 0], *r0 = row[0];
            if constexpr (S == 2) {
                if (swap01) { const uint32_t *tmp = r1; r1 = r0; r0 = tmp; }
            }
#pragma unroll
            for (int t = S - 1; t >= 0; t--) {
                const uint32_t *rr = (S == 2 ? (t == 1 ? r1 : r0) : row[t]) + soff + 8u * chh;
#pragma unroll
                for (int j = 0; j < 2; j++) {
                    const uint4 cv = *reinterpret_cast<const uint4 *>(rr + 4 * j);
                    y[8 * sh + 4 * j] = fhadd2(cv.x, y[8 * sh + 4 * j]);
                    y[8 * sh + 4 * j + 1] = fhadd2(cv.y, y[8 * sh + 4 * j + 1]);
                    y[8 * sh + 4 * j + 2] = fhadd2(cv.z, y[8 * sh + 4 * j + 2]);
                    y[8 * sh + 4 * j + 3] = fhadd2(cv.w, y[8 * sh + 4 * j + 3]);
                }
            }
        }
        if constexpr (S >= 2) {
            if (!certh[0] || !certh[1]) {
                // rare: per element of an uncertified half, every non-final partial
                // sum P' = P + c checked by Fast2Sum; inexact elements take the
                // reference's float64 chain
#pragma unroll
                for (int e = 0; e < 32; e++) {
                    if (certh[e >> 4]) continue;
                    const uint32_t cof = 16u * (uint32_t(e >> 4) ^ rho) + (uint32_t(e) & 15u);
                    const int bb = e * BITS;
                    const uint32_t u = ((w[bb >> 5] >> (bb & 31)) & ((1u << BITS) - 1u)) ^ (1u << (BITS - 1));
                    const float qs = float(int(u) - (1 << (BITS - 1))) * sv;
                    float P = qs;
                    bool bad = false;
#pragma unroll
                    for (int t = S - 1; t >= 1; t--) {
                        const uint32_t cw = row[t][soff + (cof >> 1)];
                        const float cc = __uint_as_float((cof & 1u) ? (cw & 0xFFFF0000u) : (cw << 16));
                        const float P2 = __fadd_rn(P, cc);
                        bad |= __fadd_rn(__fadd_rn(P2, -P), -cc) != 0.f || __fadd_rn(__fadd_rn(P2, -cc), -P) != 0.f;
                        P = P2;
                    }
                    if (bad) {
                        const float rr = exact_addback_p<S>(qs, tab, pitch, soff + (cof >> 1), cof & 1u, int(KK), ai[0],
                                                                  ai[SS > 1 ? 1 : 0], ai[SS > 2 ? 2 : 0], ai[SS > 3 ? 3 : 0]);
                        if (e & 1) y[e >> 1].y = rr; else y[e >> 1].x = rr;
                    }
                }
            }
        }
        if (!valid) continue;
        const uint64_t o = (uint64_t(cur) * N + sc.i0 + lr) * d + col;
#pragma unroll
        for (int sh = 0; sh < 2; sh++) {
            const uint32_t chh = uint32_t(sh) ^ rho;
            if constexpr (OBF16) {
                uint32_t v[8];
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    __nv_bfloat162 h = __floats2bfloat162_rn(y[8 * sh + q].x, y[8 * sh + q].y);
                    v[q] = *reinterpret_cast<uint32_t *>(&h);
                }
                st_global_v8(static_cast<uint16_t *>(a.out) + o + 16u * chh, v);
            } else {
#pragma unroll
                for (int hh = 0; hh < 2; hh++) {
                    uint32_t v[8];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        v[2 * q] = __float_as_uint(y[8 * sh + 4 * hh + q].x);
                        v[2 * q + 1] = __float_as_uint(y[8 * sh + 4 * hh + q].y);
                    }
                    st_global_v8(static_cast<float *>(a.out) + o + 16u * chh + 8u * hh, v);
                }
            }
        }
    }
    const uint32_t stat = (bad_scale ? QVG_STATUS_NAN_SCALE : 0u) | (bad_asg ? QVG_STATUS_BAD_ASSIGN : 0u);
    const uint32_t all = __reduce_or_sync(0xffffffffu, stat);
    if (all && lane == 0) atomicOr(a.status, int(all));
}

// ============================================================================
// host: geometry and dispatch
// ============================================================================
static int ilog2i(int v) { int l = 0; while ((1 << l) < v) l++; return l; }

// smem: [padded bf16 tables][bf16 staging copy of the next plane's tables][ring]; false when the configuration does not fit
// (callers fall back to the 16-channel ring kernel)
static bool plan(int64_t P, int64_t N, int d, int S, int K, int bits, int B, DGeo &g, size_t &smem, int &grid) {
    if (S < 1 || S > 4 || (d != 128 && d != 256) || B % 32 != 0 || N < 4 || N % 4 != 0) return false;
    if (P * N >= (int64_t(1) << 31) || N * d >= (int64_t(1) << 31)) return false;
    const int nslc = d / 32;
    const uint32_t R = uint32_t(kCW * 32 / nslc);
    const uint32_t pitch = (slice_w(uint32_t(nslc) - 1) + 16u + 4u * uint32_t(nslc) + 31u) / 32u * 32u;
    const size_t tabb = size_t(S) * K * pitch * 4;
    const size_t tbytes = size_t(S) * K * d * 2;
    const size_t off_stg = (tabb + 127) & ~size_t(127);
    size_t off_ring = (off_stg + tbytes + 1023) & ~size_t(1023);
    const uint32_t big_row = uint32_t(d * bits / 8), small_row = uint32_t(d / B);
    if ((N * small_row) % 4 != 0) return false;
    const size_t big = size_t(R) * big_row;
    const size_t small = size_t(R) * small_row + size_t(S) * R;
    const size_t stage = (big + ((small + 15) & ~size_t(15)) + 127) & ~size_t(127);
    const size_t budget = 227 * 1024 - 4096;      // dynamic smem; static arrays (barriers, sinks, tables) need the rest
    uint32_t stg_global = 0;
    if (off_ring + 2 * stage > budget) {       // no room for the staging copy
        stg_global = 1;
        off_ring = (tabb + 1023) & ~size_t(1023);
        if (off_ring + 2 * stage > budget) return false;
    }
    uint32_t nst = uint32_t((budget - off_ring) / stage);
    if (nst > 16) nst = 16;
    const int64_t ctas = 148;
    int64_t ipp = 1;
    while (P * ipp < 6 * ctas && (N + ipp * 2 - 1) / (ipp * 2) >= int64_t(4 * R)) ipp *= 2;
    int64_t rpi = (N + ipp - 1) / ipp;
    rpi = (rpi + R - 1) / R * R;
    ipp = (N + rpi - 1) / rpi;
    g = DGeo{uint32_t(P), uint32_t(N), uint32_t(d), uint32_t(K), R, nst, pitch, uint32_t(size_t(S) * K * nslc),
             uint32_t(ilog2i(nslc)), uint32_t(ipp), uint32_t(rpi), uint32_t(P * ipp), uint32_t(off_stg),
             uint32_t(off_ring), uint32_t(stage), big_row, small_row, uint32_t(big), uint32_t(tbytes), stg_global};
    smem = off_ring + g.nst * stage;
    grid = int(P * ipp < ctas ? P * ipp : ctas);
    return true;
}

template <int BITS, int S>
static int launch_d(const DequantArgs &a, bool obf16, const DGeo &g, size_t smem, int grid, cudaStream_t st) {
    if (obf16) {
        cudaFuncSetAttribute(k_dequant_ring32<BITS, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k_dequant_ring32<BITS, S, true><<<grid, kThreads, smem, st>>>(a, g);
    } else {
        cudaFuncSetAttribute(k_dequant_ring32<BITS, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k_dequant_ring32<BITS, S, false><<<grid, kThreads, smem, st>>>(a, g);
    }
    return 1;
}

}  // namespace dring

// returns 1 when the 32-channel kernel was launched, 0 when the caller must
// use another kernel for this configuration
int launch_dequantize_ring32(const DequantArgs &a, int64_t P, int bits, int S, bool obf16, cudaStream_t st) {
    using namespace dring;
    static const bool off = [] { const char *e = getenv("QVG_DEQ_C16"); return e && atoi(e) == 1; }();
    // S >= 3: the 16-channel kernel's finer certificates leave fewer rows to the
    // per-element Fast2Sum fallback (microbench N 64K, K 64, S = 3: 1.90 vs
    // 1.32 TB/s; S = 4 equal); S <= 2: this kernel (S = 2, K 256: 4.49 vs 2.84)
    if (off || S > 2) return 0;
    DGeo g;
    size_t smem;
    int grid;
    if ((reinterpret_cast<uintptr_t>(a.asg) | reinterpret_cast<uintptr_t>(a.scales)) & 3u) return 0;
    if ((reinterpret_cast<uintptr_t>(a.payload) & 15u) != 0 || (a.pb % 16) != 0) return 0;
    if ((reinterpret_cast<uintptr_t>(a.out) & 31u) != 0 || (reinterpret_cast<uintptr_t>(a.cent) & 15u) != 0) return 0;
    if (!plan(P, a.N, a.d, S, a.K, bits, a.B, g, smem, grid)) return 0;
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
