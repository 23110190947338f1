// qvg_wring.cu — K5 quantize with per-warp TMA rings (the fast path for
// bf16/f32 K/V planes, d = 128-class rows).
//
// The producer/consumer ring of qvg_stream.cu couples all warps of a CTA:
// a slot is refilled only after the slowest warp released it, so one warp in
// a rare exact fallback stalls the others.  Here every warp owns a private
// ring of D slots of 8 rows (one cp.async.bulk of the rows + 4-byte cp.async
// of the assignment bytes per slot, completing on the slot's mbarrier) and
// refills a slot itself right after consuming it: warps only meet at plane
// boundaries, where the f32 centroid tables are re-widened.
//
// Work: the CTA's contiguous items (plane, row range) are cut into tiles of
// 8 rows; tile g of the CTA goes to warp g % 16.  Element math and the
// certified exact fallbacks are those of k_quantize_stream (qvg_stream.cu).
#include "qvg_stream_dev.cuh"

namespace qvg {
namespace stream {

constexpr int kWW = 16;                  // warps per CTA (all compute)
constexpr int kWThreads = 32 * kWW;

struct WGeo {
    Geo g;                 // tables, items (rpi multiple of the tile), g.R = rows per tile
    uint32_t D;            // slots per warp ring
    uint32_t slot_bytes;   // x rows + S*8 assignment bytes, 128-aligned
    uint32_t tpi;          // tile slots per item (ceil(rpi / 8))
    uint32_t off_rings;    // smem offset of the rings
};

struct WTile {
    uint32_t p, r0, nr;    // plane, first row, rows (0: empty tile slot)
};

// walks this warp's tiles (every kWW-th tile slot of the CTA's items) with
// incremental counters: item it = p * ipp + q, tile t inside the item
struct TileIt {
    uint32_t it, p, q, t;
    __device__ __forceinline__ void init(const WGeo &w, uint32_t it0, uint32_t first) {
        it = it0 + first / w.tpi;      // once per kernel
        t = first % w.tpi;
        p = it / w.g.ipp;
        q = it - p * w.g.ipp;
    }
    __device__ __forceinline__ void advance(const WGeo &w) {
        t += kWW;
        while (t >= w.tpi) {
            t -= w.tpi;
            it++;
            if (++q == w.g.ipp) { q = 0; p++; }
        }
    }
    __device__ __forceinline__ WTile tile(const WGeo &w) const {
        const uint32_t rs = q * w.g.rpi;
        const uint32_t re = min(w.g.N, rs + w.g.rpi);
        const uint32_t r0 = rs + t * w.g.R;
        return WTile{p, r0, r0 < re ? min(w.g.R, re - r0) : 0u};
    }
};

// one bulk copy of the tile's rows into a ring slot (lane 0 of the warp)
__device__ __forceinline__ void issue_tile(const QuantArgs &a, const WGeo &w, const WTile &tl, uint8_t *slot,
                                           uint64_t *bar) {
    const uint32_t row_b = w.g.big_row;
    mbar_arrive_expect_tx(bar, tl.nr * row_b);
    if (tl.nr)
        bulk_g2s_cta(slot, static_cast<const uint8_t *>(a.x) + (uint64_t(tl.p) * w.g.N + tl.r0) * row_b,
                     tl.nr * row_b, bar);
}

template <int BITS, int S, bool XBF16, int kU>
__global__ void __launch_bounds__(kWThreads, 1) k_quantize_wring(QuantArgs a, WGeo w) {
    constexpr int QMAX = (1 << (BITS - 1)) - 1;
    constexpr int SS = S > 0 ? S : 1;
    constexpr int FPW = 32 / BITS;
    constexpr uint32_t SIGNS = BITS == 2 ? 0xAAAAAAAAu : (BITS == 4 ? 0x88888888u : 0x80808080u);
    constexpr float MAGIC = 12582912.f + float(1 << (BITS - 1));   // 1.5*2^23 + bias
    constexpr uint32_t XB = XBF16 ? 2 : 4;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t ring_bar[kWW][8];
    __shared__ uint64_t tab_bar;
    __shared__ float rcp_tab[128];
    const Geo &g = w.g;
    uint16_t *const stg = reinterpret_cast<uint16_t *>(smem);
    float *const tab = reinterpret_cast<float *>(smem + g.off_tab);
    float2 *const meta = reinterpret_cast<float2 *>(smem + g.off_meta);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t *const ring = smem + w.off_rings + size_t(warp) * w.D * w.slot_bytes;
    uint64_t *const bars = ring_bar[warp];
    const uint32_t d = g.d;

    if (threadIdx.x < 128) rcp_tab[threadIdx.x] = __frcp_rn(e4m3_decode_fast(threadIdx.x));
    if (lane == 0)
        for (uint32_t k = 0; k < w.D; k++) mbar_init(&bars[k], 1);
    if (threadIdx.x == 0) mbar_init(&tab_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    const uint32_t it0 = uint32_t((uint64_t(blockIdx.x) * g.n_items) / gridDim.x);
    const uint32_t it1 = uint32_t((uint64_t(blockIdx.x + 1) * g.n_items) / gridDim.x);
    const uint32_t ntile = (it1 - it0) * w.tpi;            // tile slots of this CTA
    // this warp's tiles: gt = warp, warp + 16, ...; prologue fills D-1 slots
    TileIt iss, con;                                       // issue / consume iterators
    iss.init(w, it0, warp);
    con = iss;
    uint32_t n_iss = 0, slot_i = 0;                        // tiles issued, next slot to fill
    const uint32_t my_tiles = warp < ntile ? (ntile - 1 - warp) / kWW + 1 : 0;
    for (; n_iss + 1 < w.D && n_iss < my_tiles; n_iss++) {
        if (lane == 0) issue_tile(a, w, iss.tile(w), ring + slot_i * w.slot_bytes, &bars[slot_i]);
        iss.advance(w);
        slot_i = slot_i + 1 == w.D ? 0 : slot_i + 1;
    }
    if (threadIdx.x == 0 && it0 < it1) stage_table(a.cent, it0 / g.ipp, g.tbytes, stg, &tab_bar);

    const uint32_t lvpr = g.lchunk;
    const uint32_t c = lane & ((1u << lvpr) - 1u);
    const uint32_t col = c << 4;
    const uint32_t coff = blk_off(c);
    const uint32_t rslot = uint32_t(lane) >> lvpr, rpp = 32u >> lvpr;   // rows per pass per warp
    const int glanes = 1 << a.gshift;
    bool nonfinite = false;
    uint32_t cur = 0xFFFFFFFFu, jp = 0;

    // assignment bytes of this thread's rows (byte u of word t = row u, stage t),
    // loaded one tile ahead
    uint32_t aw_nx[SS];
    auto load_ai = [&](const WTile &tl) {
#pragma unroll
        for (int t = 0; t < S; t++) aw_nx[t] = 0u;
#pragma unroll
        for (int u = 0; u < kU; u++) {
            const uint32_t l = u * rpp + rslot;
            const uint32_t lr = tl.nr ? (l < tl.nr ? l : tl.nr - 1) : 0u;
#pragma unroll
            for (int t = 0; t < S; t++)
                aw_nx[t] |= (tl.nr ? uint32_t(__ldg(a.asg + (uint64_t(tl.p) * S + t) * g.N + tl.r0 + lr)) : 0u)
                            << (8 * u);
        }
    };
    if (my_tiles) load_ai(con.tile(w));
    uint32_t n_con = 0, slot_c = 0, phase = 0;
    uint32_t pl = it0 / g.ipp, ql = it0 - pl * g.ipp;      // plane / part of item `it`
    for (uint32_t it = it0; it < it1; it++) {
        const uint32_t p = pl;
        if (++ql == g.ipp) { ql = 0; pl++; }
        if (p != cur) {                                    // new plane: re-widen the tables
            __syncthreads();
            mbar_wait(&tab_bar, jp & 1u);
            widen(stg, tab, meta, g, kWThreads);
            __syncthreads();
            if (threadIdx.x == 0 && int64_t(p + 1) * g.ipp < int64_t(it1)) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                stage_table(a.cent, p + 1, g.tbytes, stg, &tab_bar);
            }
            cur = p;
            jp++;
        }
        // this warp's tiles inside item `it`
        while (n_con < my_tiles && con.it == it) {
            // refill: the slot of the previous tile was released at the end of the
            // previous iteration (__syncwarp), so the next tile can stream into it
            if (n_iss < my_tiles) {
                if (lane == 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue_tile(a, w, iss.tile(w), ring + slot_i * w.slot_bytes, &bars[slot_i]);
                }
                iss.advance(w);
                slot_i = slot_i + 1 == w.D ? 0 : slot_i + 1;
                n_iss++;
            }
            const WTile tl = con.tile(w);
            con.advance(w);
            uint32_t aw[SS];
#pragma unroll
            for (int t = 0; t < S; t++) aw[t] = aw_nx[t];
            if (n_con + 1 < my_tiles) load_ai(con.tile(w));
            const uint32_t k = slot_c;
            mbar_wait(&bars[k], phase);
            n_con++;
            if (++slot_c == w.D) { slot_c = 0; phase ^= 1u; }
            if (tl.nr == 0) continue;
            const uint8_t *st = ring + k * w.slot_bytes;
            const uint32_t nr = tl.nr;
            // rows of this thread: rslot, rslot + 4, ... (one at a time: low register
            // pressure, per-row state reused across the loop)
            const uint8_t *xr = st + rslot * g.big_row + col * XB;
            uint8_t *pay = a.payload + uint64_t(p) * a.pb + (((tl.r0 + rslot) * d + col) * BITS >> 3);
            uint8_t *scp = a.scales + uint64_t(p) * a.ng + (((tl.r0 + rslot) * d + col) >> a.lgB);
            const bool swr = (lane & (glanes - 1)) == 0;
#pragma unroll 1
            for (int u = 0; u < kU; u++, xr += rpp * g.big_row, pay += rpp * (d * BITS / 8),
                     scp += rpp * (d >> a.lgB)) {
                const bool valid = u * rpp + rslot < nr;      // warp-divergent only in a tail tile
                float2 r[8];
                float xmin = 0.f;
                if constexpr (XBF16) {
                    const uint4 w0 = *reinterpret_cast<const uint4 *>(xr);
                    const uint4 w1 = *reinterpret_cast<const uint4 *>(xr + 16);
                    cvt16(w0, w1, reinterpret_cast<float *>(r));
                    float mv[8];
#pragma unroll
                    for (int q = 0; q < 8; q++) mv[q] = fminf(fabsf(r[q].x), fabsf(r[q].y));
#pragma unroll
                    for (int span = 1; span < 8; span *= 2)
#pragma unroll
                        for (int q = 0; q < 8; q += 2 * span) mv[q] = fminf(mv[q], mv[q + span]);
                    xmin = mv[0];
                } else {
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        const float4 v = *reinterpret_cast<const float4 *>(xr + 16 * j);
                        r[2 * j] = make_float2(v.x, v.y);
                        r[2 * j + 1] = make_float2(v.z, v.w);
                    }
                }
                int ar[SS];
#pragma unroll
                for (int t = 0; t < S; t++) ar[t] = int((aw[t] >> (8 * u)) & 0xFFu);
                // residual, error-bound inputs and the exactness certificate (see K5 in qvg_stream.cu)
                float cb = 0.f, csum = 0.f, cunit = __int_as_float(0x7F800000);
#pragma unroll
                for (int t = 0; t < S; t++) {
                    const float *row = tab + uint32_t(t * int(g.K) + ar[t]) * g.pitch + coff;
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        const float4 cv = *reinterpret_cast<const float4 *>(row + 4 * j);
                        r[2 * j] = __fadd2_rn(r[2 * j], make_float2(-cv.x, -cv.y));
                        r[2 * j + 1] = __fadd2_rn(r[2 * j + 1], make_float2(-cv.z, -cv.w));
                    }
                    const float2 m = meta[(uint32_t(t * int(g.K) + ar[t]) << lvpr) + c];
                    if (t > 0) cb = __fmaf_ru(float(t), m.y, cb);
                    csum = __fadd_ru(csum, m.y);
                    cunit = fminf(cunit, m.x);
                }
                float mv[8];
#pragma unroll
                for (int q = 0; q < 8; q++) mv[q] = max3_nan_abs(0.f, r[q].x, r[q].y);
#pragma unroll
                for (int span = 1; span < 8; span *= 2)
#pragma unroll
                    for (int q = 0; q < 8; q += 2 * span) mv[q] = max_nan(mv[q], mv[q + span]);
                float am = mv[0];
                nonfinite |= valid && (!(am <= 3.402823466e38f) || !(cb <= 3.402823466e38f));
                bool cert = false;
                if constexpr (XBF16) {
                    const uint32_t eb8 = __float_as_uint(xmin) & 0x7F800000u;
                    const float xunit = eb8 > (7u << 23) ? __uint_as_float(eb8 - (7u << 23)) : 0.f;
                    cert = __fmaf_ru(2.f, csum, am) < fminf(xunit, cunit) * 16777216.f;
                }
                float eb = (S > 0 && !cert) ? __fmaf_ru(float(S), am, cb) : 0.f;
                for (int m = 1; m < glanes; m <<= 1) {
                    am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, m));
                    eb = fmaxf(eb, __shfl_xor_sync(0xffffffffu, eb, m));
                }
                const float E = __fmul_ru(eb, 2.38418579e-7f);      // 2^-22
                const float lo = __fsub_rd(am, E), hi = __fadd_ru(am, E);
                bool cbm = false;
                uint32_t code = scale_code<QMAX>(lo > 0.f ? lo : hi, hi, cbm);
                const bool zero = am == 0.f && E == 0.f;
                code = zero || !(lo > 0.f) ? 0x38u : code;
                const bool camb = valid && !zero && (cbm || !(lo > 0.f));
                if (__any_sync(0xffffffffu, camb))          // exact scale (rare, out of line)
                    code = fix_scale<QMAX, S, XBF16>(xr, tab, g.pitch, coff, int(g.K), ar[0], ar[SS > 1 ? 1 : 0],
                                                     ar[SS > 2 ? 2 : 0], ar[SS > 3 ? 3 : 0], am, E, camb, glanes,
                                                     code);
                const float sv = e4m3_decode_fast(code);
                const float inv = rcp_tab[code & 0x7Fu];
                const float2 inv2 = make_float2(inv, inv);
                uint32_t f[16];
                float2 yv[8];
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    yv[q] = __ffma2_rn(r[q], inv2, make_float2(MAGIC, MAGIC));
                    f[2 * q] = __float_as_uint(yv[q].x);
                    f[2 * q + 1] = __float_as_uint(yv[q].y);
                }
                Words4 b32;
#pragma unroll
                for (int wd = 0; wd < BITS / 2; wd++) {
                    uint32_t v[FPW];
#pragma unroll
                    for (int k2 = 0; k2 < FPW; k2++) v[k2] = f[wd * FPW + k2];
#pragma unroll
                    for (int span = 1; span < FPW; span *= 2)
#pragma unroll
                        for (int k2 = 0; k2 < FPW; k2 += 2 * span) v[k2] += v[k2 + span] << (BITS * span);
                    b32.w[wd] = (v[0] - magic_sum<BITS>()) ^ SIGNS;
                }
                const bool allv = !(E < 0.125f * sv) || code == 0x7Eu;
                const float thr = window_thr<QMAX>(sv, inv, E);
                float wv[8];
                bool amb;
                if constexpr (QMAX == 1) {
                    const float h = 0.5f * sv;
                    const float2 pa = make_float2(-h * h, -h * h);
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        const float2 gg = __ffma2_rn(r[q], r[q], pa);
                        wv[q] = fminf(fabsf(gg.x), fabsf(gg.y));
                    }
#pragma unroll
                    for (int span = 1; span < 8; span *= 2)
#pragma unroll
                        for (int q = 0; q < 8; q += 2 * span) wv[q] = fminf(wv[q], wv[q + span]);
                    amb = allv || wv[0] <= thr;
                } else {
                    const float2 pa = make_float2(-MAGIC, -MAGIC);
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        const float2 qf = __fadd2_rn(yv[q], pa);
                        const float2 dist = __ffma2_rn(r[q], inv2, make_float2(-qf.x, -qf.y));
                        wv[q] = fmaxf(fabsf(dist.x), fabsf(dist.y));
                    }
#pragma unroll
                    for (int span = 1; span < 8; span *= 2)
#pragma unroll
                        for (int q = 0; q < 8; q += 2 * span) wv[q] = fmaxf(wv[q], wv[q + span]);
                    amb = allv || wv[0] >= thr;
                }
                if (amb && valid)      // exact codes (rare, out of line)
                    b32 = fix_codes<BITS, S, XBF16>(xr, tab, g.pitch, coff, int(g.K), ar[0], ar[SS > 1 ? 1 : 0],
                                                    ar[SS > 2 ? 2 : 0], ar[SS > 3 ? 3 : 0], sv, inv, E, thr, allv,
                                                    b32);
                if (valid) {
                    if constexpr (BITS == 2) *reinterpret_cast<uint32_t *>(pay) = b32.w[0];
                    else if constexpr (BITS == 4) *reinterpret_cast<uint2 *>(pay) = make_uint2(b32.w[0], b32.w[1]);
                    else *reinterpret_cast<uint4 *>(pay) = make_uint4(b32.w[0], b32.w[1], b32.w[2], b32.w[3]);
                    if (swr) *scp = uint8_t(code);
                }
            }
            __syncwarp();          // slot k fully read: it may be refilled next iteration
        }
    }
    const uint32_t all = __reduce_or_sync(0xffffffffu, nonfinite ? uint32_t(QVG_STATUS_NONFINITE) : 0u);
    if (all && lane == 0) atomicOr(a.status, int(all));
}

// geometry: tables as in the shared-ring kernel; rings of D slots per warp
static bool wplan(int64_t P, int64_t N, int d, int S, int K, int xbytes, int TR, WGeo &w, size_t &smem, int &grid) {
    if (S < 1 || S > 4 || d != 128 || N < 4 || N % 4 != 0) return false;
    if (P * N >= (int64_t(1) << 31)) return false;
    const int n = d / 16;
    const uint32_t pitch = uint32_t(16 * n + 4 * ((n + 1) / 2));
    const size_t tbytes = size_t(S) * K * d * 2;
    const size_t tabb = size_t(S) * K * pitch * 4;
    const size_t nchunk = size_t(S) * K * n;
    const size_t off_tab = (tbytes + 127) & ~size_t(127);
    const size_t off_meta = off_tab + ((tabb + 127) & ~size_t(127));
    const size_t off_rings = off_meta + ((nchunk * 8 + 127) & ~size_t(127));
    const size_t big_row = size_t(d) * xbytes;
    const size_t slot = (size_t(TR) * big_row + 127) & ~size_t(127);
    const size_t budget = 227 * 1024 - 4096;
    if (off_rings + size_t(kWW) * 2 * slot > budget) return false;
    uint32_t D = uint32_t((budget - off_rings) / (size_t(kWW) * slot));
    if (D > 8) D = 8;
    if (D < 2) return false;
    if (const char *e = getenv("QVG_WRING_D")) { const uint32_t v = uint32_t(atoi(e)); if (v >= 2 && v < D) D = v; }
    // items: planes split into row ranges (multiples of the tile) until every
    // CTA has several; then tile slots per item
    const int64_t ctas = 148;
    int64_t ipp = 1;
    while (P * ipp < 4 * ctas && (N + ipp * 2 - 1) / (ipp * 2) >= 1024) ipp *= 2;
    int64_t rpi = (N + ipp - 1) / ipp;
    rpi = (rpi + TR - 1) / TR * TR;
    ipp = (N + rpi - 1) / rpi;
    Geo g{uint32_t(P), uint32_t(N), uint32_t(d), uint32_t(K), uint32_t(TR), 0u, pitch, uint32_t(tbytes),
          uint32_t(nchunk), uint32_t(n == 8 ? 3 : 0), uint32_t(ipp), uint32_t(rpi), uint32_t(P * ipp),
          uint32_t(off_tab), uint32_t(off_meta), 0u, 0u, uint32_t(big_row), 0u, 0u, 0u};
    w = WGeo{g, D, uint32_t(slot), uint32_t(rpi / TR), uint32_t(off_rings)};
    smem = off_rings + size_t(kWW) * D * slot;
    grid = int(P * ipp < ctas ? P * ipp : ctas);
    return true;
}

constexpr int kWU = 4;     // rows per thread per tile (tile = 4 * kWU rows)

template <int BITS, int S>
static int launch_wq(const QuantArgs &a, bool xbf16, const WGeo &w, size_t smem, int grid, cudaStream_t st) {
    if (xbf16) {
        cudaFuncSetAttribute(k_quantize_wring<BITS, S, true, kWU>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k_quantize_wring<BITS, S, true, kWU><<<grid, kWThreads, smem, st>>>(a, w);
    } else {
        cudaFuncSetAttribute(k_quantize_wring<BITS, S, false, kWU>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k_quantize_wring<BITS, S, false, kWU><<<grid, kWThreads, smem, st>>>(a, w);
    }
    return 1;
}

}  // namespace stream

int launch_quantize_wring(const QuantArgs &a, int64_t P, int bits, int S, bool xbf16, cudaStream_t st) {
    using namespace stream;
    WGeo w;
    size_t smem;
    int grid;
    if ((reinterpret_cast<uintptr_t>(a.x) & 15u) != 0 || (reinterpret_cast<uintptr_t>(a.asg) & 3u) != 0) return 0;
    if (!wplan(P, a.N, a.d, S, a.K, xbf16 ? 2 : 4, 4 * kWU, w, smem, grid)) return 0;
#define QV_W(BB)                                                       \
    switch (S) {                                                       \
        case 1: return launch_wq<BB, 1>(a, xbf16, w, smem, grid, st); \
        case 2: return launch_wq<BB, 2>(a, xbf16, w, smem, grid, st); \
        case 3: return launch_wq<BB, 3>(a, xbf16, w, smem, grid, st); \
        default: return launch_wq<BB, 4>(a, xbf16, w, smem, grid, st); \
    }
    if (bits == 2) { QV_W(2) }
    if (bits == 4) { QV_W(4) }
    QV_W(8)
#undef QV_W
}

}  // namespace qvg
