// qvg_assign_tc.cu — K2 k-means assignment (Q/clustering.py:66-71) as a
// tcgen05 distance GEMM with a fused, certified argmin.
//
//   D[i, j] = c2[j] - 2 * (x_i . c_j),   pi_i = first argmin_j D[i, j]
//
// The reference computes x_i . c_j as ONE sequential float64 FMA chain over
// the 128 channels (OpenBLAS dgemm).  Here:
//  1. k_split_rows (once per SAS stage: the rows do not change across the
//     Lloyd iterations) writes every 128-row tile of the float64 rows as three
//     bf16 tiles hi + mid + lo (|x - hi - mid - lo| <= 2^-24 |x|), already in
//     the UMMA canonical K-major layout, so a tile is ONE contiguous bulk copy;
//  2. k_assign_tc (persistent, one CTA per SM) widens the plane's centroids to
//     the same three-way split in shared memory, streams row tiles in with
//     cp.async.bulk, and issues tcgen05.mma (kind::f16, M = 128 rows,
//     N = centroid block, K = 16) for the six significant split products
//     hi.hi + hi.mid + mid.hi + hi.lo + lo.hi + mid.mid into four TMEM
//     accumulators (one per 32-channel slice, which bounds the fp32
//     accumulation error);
//  3. the epilogue (thread = row = TMEM lane) forms D'[j] = c2[j] - 2 cross'[j]
//     with the exact float64 c2 and keeps, online, the first argmin j* and
//     min_{j != j*} (D'[j] - E[j]) with the rigorous error bound
//     E[j] = 2^-15 ||x_i|| ||c_j|| + 2^-100 (Cauchy-Schwarz on sum |x_k c_jk|, an
//     absolute floor for underflow of tiny data; covers the
//     split, the fp32 accumulation and summation, and the reference's own
//     float64 rounding).  The row is certified when that minimum exceeds
//     D'[j*] + E[j*]: then the reference's argmin is j* (exact ties are never
//     certified, so the first-min rule cannot be violated);
//  4. uncertified rows are appended to a list and recomputed by
//     k_assign_recheck with the reference's exact float64 FMA chain.
#include <cstdio>
#include <cstdlib>

#include "qvg_common.cuh"
#include "qvg_internal.h"

namespace qvg {
namespace atc {

constexpr int kM = 128;                // rows per tile (UMMA M)
constexpr int kD = 128;                // channels (UMMA K total)
constexpr int kNB = 128;               // centroids per block (UMMA N <= 128)
constexpr int kTileB = kM * kD * 2;    // one bf16 split tile (32 KB)
constexpr int kSplit = 3;
constexpr int kAcc = 4;                // TMEM accumulators = 32-channel slices
constexpr uint32_t kSbo = 2048, kLbo = 128;

__device__ __forceinline__ uint32_t su32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }

// UMMA canonical K-major, no swizzle: (r, k) of a [rows][128] bf16 tile
__host__ __device__ __forceinline__ uint32_t kmaj_off(uint32_t r, uint32_t k) {
    return (r >> 3) * kSbo + (k >> 3) * kLbo + (r & 7u) * 16u + (k & 7u) * 2u;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFFu);
    d |= uint64_t((kLbo >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((kSbo >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;
    return d;
}

// kind::f16, A = B = bf16, D = f32, both K-major, M = 128, N = n
__device__ __forceinline__ uint32_t idesc(uint32_t n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((uint32_t(kM) >> 4) << 24);
}

__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void bar_init(uint64_t *bar, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(n));
}
__device__ __forceinline__ void bar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n}" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float v[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}

// the kAcc accumulator chunks of 32 columns with one wait (the loads overlap)
__device__ __forceinline__ void tmem_ld32x4(uint32_t taddr, uint32_t stride, float v[4][32]) {
#pragma unroll
    for (int c = 0; c < 4; c++) {
        uint32_t *r = reinterpret_cast<uint32_t *>(v[c]);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
              "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
              "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
              "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr + c * stride));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// x = hi + mid + lo (+ <= 2^-24 |x|), each RN to bf16 (bits)
__device__ __forceinline__ void split3(double x, uint16_t &hi, uint16_t &mid, uint16_t &lo) {
    const __nv_bfloat16 h = __double2bfloat16(x);
    const double r1 = x - double(__bfloat162float(h));
    const __nv_bfloat16 m = __double2bfloat16(r1);
    const double r2 = r1 - double(__bfloat162float(m));
    const __nv_bfloat16 l = __double2bfloat16(r2);
    hi = __bfloat16_as_ushort(h);
    mid = __bfloat16_as_ushort(m);
    lo = __bfloat16_as_ushort(l);
}

// ---------------------------------------------------------------------------
// rows [P][N][128] f64 -> [P][T][3][128x128 UMMA tile] bf16 + row norms
// ---------------------------------------------------------------------------
// x16 (optional): the bf16 input when the rows are exactly it (stage 1 of a bf16
// chunk) -- read instead of the float64 rows (a quarter of the bytes); the mid /
// lo splits are then zero and are written only when write_lo (the assignment
// kernel reads them unless it runs in its hi-split-only mode)
__global__ void k_split_rows(const double *rows, const uint16_t *x16, int write_lo, uint16_t *split, float *xnorm,
                             float *rows32, int32_t *rows32_ok, int64_t P, int64_t N, int T) {
    // one thread = 8 channels (one 16-byte chunk of the tile) of one row
    const int64_t total = P * int64_t(T) * kM * (kD / 8);
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int ch = int(e % (kD / 8));
        const int64_t rt = e / (kD / 8);               // global (plane, tile, row)
        const int r = int(rt % kM);
        const int64_t pt = rt / kM;
        const int t = int(pt % T);
        const int64_t p = pt / T;
        const int64_t row = int64_t(t) * kM + r;
        uint16_t v[kSplit][8];
        double ss = 0.0;
        if (row < N && x16) {
            const uint4 w = *reinterpret_cast<const uint4 *>(x16 + (p * N + row) * kD + ch * 8);
            const uint32_t u[4] = {w.x, w.y, w.z, w.w};
            float f[8];
#pragma unroll
            for (int h = 0; h < 4; h++) {
                v[0][2 * h] = uint16_t(u[h] & 0xFFFFu);
                v[0][2 * h + 1] = uint16_t(u[h] >> 16);
                f[2 * h] = __uint_as_float(u[h] << 16);
                f[2 * h + 1] = __uint_as_float(u[h] & 0xFFFF0000u);
            }
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const double x = double(f[k]);
                ss = fma(x, x, ss);
                v[1][k] = v[2][k] = 0;
            }
            float4 *dst32 = reinterpret_cast<float4 *>(rows32 + (p * N + row) * kD + ch * 8);
            dst32[0] = make_float4(f[0], f[1], f[2], f[3]);
            dst32[1] = make_float4(f[4], f[5], f[6], f[7]);
        } else if (row < N) {
            const double *src = rows + (p * N + row) * kD + ch * 8;
            float f[8];
            bool exact = true;
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const double x = src[k];
                ss = fma(x, x, ss);
                split3(x, v[0][k], v[1][k], v[2][k]);
                f[k] = float(x);
                exact &= double(f[k]) == x;
            }
            float4 *dst32 = reinterpret_cast<float4 *>(rows32 + (p * N + row) * kD + ch * 8);
            dst32[0] = make_float4(f[0], f[1], f[2], f[3]);
            dst32[1] = make_float4(f[4], f[5], f[6], f[7]);
            if (!exact) rows32_ok[p] = 0;
        } else {
#pragma unroll
            for (int k = 0; k < 8; k++) v[0][k] = v[1][k] = v[2][k] = 0;
        }
        uint8_t *tile = reinterpret_cast<uint8_t *>(split) + pt * (kSplit * size_t(kTileB));
        const int ns = (x16 && !write_lo) ? 1 : kSplit;
#pragma unroll
        for (int s = 0; s < kSplit; s++) {
            if (s >= ns) break;
            uint4 w;
            w.x = uint32_t(v[s][0]) | (uint32_t(v[s][1]) << 16);
            w.y = uint32_t(v[s][2]) | (uint32_t(v[s][3]) << 16);
            w.z = uint32_t(v[s][4]) | (uint32_t(v[s][5]) << 16);
            w.w = uint32_t(v[s][6]) | (uint32_t(v[s][7]) << 16);
            *reinterpret_cast<uint4 *>(tile + s * kTileB + kmaj_off(r, ch * 8)) = w;
        }
        // ||x||^2 over the 16 chunks of the row (consecutive threads)
#pragma unroll
        for (int m = 1; m < 16; m <<= 1) ss += __shfl_xor_sync(0xffffffffu, ss, m);
        if (ch == 0 && row < N) xnorm[p * N + row] = float(sqrt(ss) * (1.0 + 1e-6));   // rounded up
    }
}

struct TcArgs {
    const uint16_t *split;     // [P][T][3][tile]
    const float *xnorm;        // [P][N]
    const double *cent;        // [P][K][128]
    const double *c2;          // [P][K] exact (reference pairwise)
    int32_t *assign;           // [P][N]
    int32_t *recheck;          // [P*N] list of p*N + row
    int32_t *n_recheck;
    const PlaneState *st;      // skip converged planes (nullable)
    int64_t P, N;
    int K, T, skip_done;
    int a_one;                 // rows exactly bf16 (stage 1 of a bf16 chunk): splits 1, 2 are zero
};

// smem: A tiles (3 x 32 KB) | B tiles (3 x kNB x 128 bf16 = 96 KB) | c2, cnorm
constexpr size_t kSmemA = size_t(kSplit) * kTileB;
constexpr size_t kSmemB = size_t(kSplit) * kNB * kD * 2;
constexpr size_t kSmem = kSmemA + kSmemB + 2 * kNB * sizeof(float) + kNB * sizeof(double) + 1024;

// 8 warps: warp w reads TMEM lanes 32 (w & 3) (its rows) and takes the 32-centroid
// chunks c with c % 2 == w >> 2; the two halves' certified states merge in smem
constexpr int kTcThreads = 256;
__global__ void __launch_bounds__(kTcThreads, 1) k_assign_tc(TcArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem, *sB = smem + kSmemA;
    // per centroid of the block: c2 rounded to f32, and the two bound coefficients
    // t1 = 2^-15 |c| and t2 = 2^-22 |c2f| (both rounded up)
    float *c2f = reinterpret_cast<float *>(sB + kSmemB);
    float *t2s = c2f + kNB;
    float *t1s = t2s + kNB;
    __shared__ uint64_t bar_a, bar_mma;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int K = a.K;
    const int64_t n_items = a.P * a.T;

    if (tid == 0) {
        bar_init(&bar_a, 1);
        bar_init(&bar_mma, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t t_lane = uint32_t((warp & 3) * 32) << 16;
    const int hh = warp >> 2, rl = tid & 127;         // centroid-chunk half, row in the tile
    __shared__ float mD[kM], mE[kM], mO[kM];
    __shared__ int mJ[kM];

    // this CTA's contiguous items (plane, tile)
    const int64_t it0 = (int64_t(blockIdx.x) * n_items) / gridDim.x;
    const int64_t it1 = (int64_t(blockIdx.x + 1) * n_items) / gridDim.x;
    int64_t cur_p = -1;
    uint32_t pa = 0, pm = 0;          // barrier phases
    // the next item this CTA processes (planes already converged are skipped)
    auto next_item = [&](int64_t from) {
        while (from < it1 && a.skip_done && a.st[from / a.T].done) from++;
        return from;
    };
    // stream a row tile (3 splits, one contiguous bulk copy); the next item's tile
    // is requested as soon as the current item's last MMAs are done, so its
    // transfer overlaps the epilogue
    auto load_tile = [&](int64_t item) {
        if (tid == 0 && item < it1) {
            // bf16-exact rows: only the hi split is nonzero (a third of the bytes)
            const uint32_t nbytes = a.a_one ? uint32_t(kTileB) : uint32_t(kSmemA);
            expect_tx(&bar_a, nbytes);
            bulk_g2s(sA, reinterpret_cast<const uint8_t *>(a.split) + size_t(item) * kSmemA, nbytes, &bar_a);
        }
    };
    int64_t it = next_item(it0);
    load_tile(it);
    for (; it < it1;) {
        const int64_t p = it / a.T;
        const int t = int(it - p * a.T);
        const int64_t it_next = next_item(it + 1);
        const int nblk = (K + kNB - 1) / kNB;
        const int64_t row = int64_t(t) * kM + rl;
        const float xn = row < a.N ? a.xnorm[p * a.N + row] : 0.f;
        // online certified argmin state (thread = row)
        float bestD = 0.f, bestE = 0.f, others = INFINITY;
        int bestj = -1;
        for (int blk = 0; blk < nblk; blk++) {
            const int j0 = blk * kNB, nb = min(kNB, K - j0);
            const int nbp = (nb + 15) & ~15;            // UMMA N multiple of 16
            if (p != cur_p || nblk > 1) {
                // centroid block -> 3 bf16 splits (UMMA K-major) + c2 + norms
                __syncthreads();                        // previous users of sB / c2s done
                for (int e = tid; e < nbp * (kD / 8); e += blockDim.x) {
                    const int j = e / (kD / 8), ch = e % (kD / 8);
                    uint16_t v[kSplit][8];
#pragma unroll
                    for (int k = 0; k < 8; k++) {
                        const double x = j < nb ? a.cent[(p * K + j0 + j) * kD + ch * 8 + k] : 0.0;
                        split3(x, v[0][k], v[1][k], v[2][k]);
                    }
#pragma unroll
                    for (int s = 0; s < kSplit; s++) {
                        uint4 w;
                        w.x = uint32_t(v[s][0]) | (uint32_t(v[s][1]) << 16);
                        w.y = uint32_t(v[s][2]) | (uint32_t(v[s][3]) << 16);
                        w.z = uint32_t(v[s][4]) | (uint32_t(v[s][5]) << 16);
                        w.w = uint32_t(v[s][6]) | (uint32_t(v[s][7]) << 16);
                        *reinterpret_cast<uint4 *>(sB + s * (kNB * kD * 2) + kmaj_off(j, ch * 8)) = w;
                    }
                }
                for (int j = tid; j < nbp; j += blockDim.x) {
                    double ss = 0.0;
                    if (j < nb)
                        for (int k = 0; k < kD; k++) {
                            const double c = a.cent[(p * K + j0 + j) * kD + k];
                            ss = fma(c, c, ss);
                        }
                    const float cf = j < nb ? __double2float_rn(a.c2[p * K + j0 + j]) : 0.f;
                    c2f[j] = cf;
                    // 2^-22 |c2f| plus an absolute floor of 2^-100: bf16 splits, f32 products
                    // and c2 -> f32 lose at most ~2^-130 absolutely to underflow, so rows of
                    // tiny data are never certified and take the exact float64 recheck
                    t2s[j] = __fadd_ru(__fmul_ru(fabsf(cf), 2.384185791015625e-07f), 7.888609052210118e-31f);
                    t1s[j] = __fmul_ru(float(sqrt(ss) * (1.0 + 1e-6)), 3.0517578125e-05f);   // 2^-15
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> tensor core
                __syncthreads();
                cur_p = p;
            }
            if (blk == 0) { bar_wait(&bar_a, pa); pa ^= 1u; }
            // ---- MMAs: acc[q] = sum over slice q (32 channels = 2 K-steps) of the 6 products
            if (tid == 0) {
                fence_after();
                const uint32_t id = idesc(uint32_t(nbp));
                // bf16-exact rows (a_one): the products of the zero A splits (1, 0),
                // (2, 0), (1, 1) vanish exactly and are skipped; order kept otherwise
                const int prod6[6][2] = {{0, 0}, {0, 1}, {1, 0}, {0, 2}, {2, 0}, {1, 1}};
                const int prod3[6][2] = {{0, 0}, {0, 1}, {0, 2}, {0, 0}, {0, 0}, {0, 0}};
                const int (*prod)[2] = a.a_one ? prod3 : prod6;
                const int npr = a.a_one ? 3 : 6;
#pragma unroll
                for (int q = 0; q < kAcc; q++) {
                    int first = 1;
#pragma unroll
                    for (int ks = 0; ks < 2; ks++) {
                        const int k = (q * 2 + ks) * 16;
#pragma unroll
                        for (int pr = 0; pr < 6; pr++) {
                            if (pr >= npr) break;
                            const uint64_t ad = sdesc(su32(sA + prod[pr][0] * kTileB + kmaj_off(0, k)));
                            const uint64_t bd = sdesc(su32(sB + prod[pr][1] * (kNB * kD * 2) + kmaj_off(0, k)));
                            mma(tmem + q * kNB, ad, bd, id, first ? 0u : 1u);
                            first = 0;
                        }
                    }
                }
                commit(&bar_mma);
            }
            bar_wait(&bar_mma, pm);
            pm ^= 1u;
            fence_after();
            if (blk == nblk - 1) load_tile(it_next);     // sA no longer read by this item's MMAs
            // ---- epilogue: 32 centroids at a time
            for (int c0 = 32 * hh; c0 < nb; c0 += 64) {
                static_assert(kAcc == 4, "tmem_ld32x4 loads four accumulators");
                float acc[4][32];
                tmem_ld32x4(tmem + t_lane + c0, kNB, acc);
                float cr[32];
#pragma unroll
                for (int i = 0; i < 32; i++) cr[i] = ((acc[0][i] + acc[1][i]) + acc[2][i]) + acc[3][i];
                const int nn = min(32, nb - c0);
                // certified argmin in f32 with directed rounding: D = c2f - 2 cross (one
                // rounding), E = 2^-15 |x||c| + 2^-22 (|c2f| + 2 |cross|) covers the split /
                // accumulation error of the cross term, c2 -> f32 and the rounding of D;
                // two independent chains (even / odd centroids), merged below
                float bD[2], bE[2], oth[2] = {INFINITY, INFINITY};
                int bj[2] = {-1, -1};
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    if (i >= nn) break;
                    const int j = c0 + i, ch = i & 1;
                    const float D = __fmaf_rn(-2.f, cr[i], c2f[j]);
                    const float E = __fmaf_ru(xn, t1s[j], __fmaf_ru(fabsf(cr[i]), 4.76837158203125e-07f, t2s[j]));
                    if (bj[ch] < 0) { bD[ch] = D; bE[ch] = E; bj[ch] = j0 + j; }
                    else if (D < bD[ch]) {
                        oth[ch] = fminf(oth[ch], __fsub_rd(bD[ch], bE[ch]));
                        bD[ch] = D; bE[ch] = E; bj[ch] = j0 + j;
                    } else {
                        oth[ch] = fminf(oth[ch], __fsub_rd(D, E));
                    }
                }
                // merge the chains and the running state (ties are never certified:
                // the loser's D - E <= the winner's D keeps `others` below bestD + bestE)
#pragma unroll
                for (int ch = 0; ch < 2; ch++) {
                    if (bj[ch] < 0) continue;
                    others = fminf(others, oth[ch]);
                    if (bestj < 0) { bestD = bD[ch]; bestE = bE[ch]; bestj = bj[ch]; }
                    else if (bD[ch] < bestD || (bD[ch] == bestD && bj[ch] < bestj)) {
                        others = fminf(others, __fsub_rd(bestD, bestE));
                        bestD = bD[ch]; bestE = bE[ch]; bestj = bj[ch];
                    } else {
                        others = fminf(others, __fsub_rd(bD[ch], bE[ch]));
                    }
                }
            }
            fence_before();
            __syncthreads();                 // TMEM / sB reads done before the next MMAs
        }
        // merge the two chunk halves of each row (half 1 hands its state to half 0)
        if (hh == 1) { mD[rl] = bestD; mE[rl] = bestE; mO[rl] = others; mJ[rl] = bestj; }
        __syncthreads();
        if (hh == 0) {
            others = fminf(others, mO[rl]);
            const int oj = mJ[rl];
            if (oj >= 0) {
                const float oD = mD[rl], oE = mE[rl];
                if (bestj < 0) { bestD = oD; bestE = oE; bestj = oj; }
                else if (oD < bestD || (oD == bestD && oj < bestj)) {
                    others = fminf(others, __fsub_rd(bestD, bestE));
                    bestD = oD; bestE = oE; bestj = oj;
                } else {
                    others = fminf(others, __fsub_rd(oD, oE));
                }
            }
        }
        if (hh == 0 && row < a.N) {
            const bool ok = others > __fadd_ru(bestD, bestE);
            a.assign[p * a.N + row] = ok ? bestj : -1;
            if (!ok) a.recheck[atomicAdd(a.n_recheck, 1)] = int32_t(p * a.N + row);
        }
        it = it_next;
    }
    fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// exact float64 argmin of the listed rows (warp per row): the reference's
// sequential FMA chain per centroid, D = c2 - 2 cross, first minimum
__global__ void k_assign_recheck(const double *rows, const double *cent, const double *c2, int32_t *assign,
                                 const int32_t *list, const int32_t *n_list, int64_t N, int K) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const int n = *n_list;
    for (int64_t w = wid; w < n; w += nw) {
        const int64_t pr = list[w];
        const int64_t p = pr / N;
        const double *x = rows + pr * kD;
        double bv = 0.0;
        int bj = -1;
        for (int j = lane; j < K; j += 32) {
            const double *c = cent + (p * K + j) * kD;
            double acc = 0.0;
#pragma unroll 8
            for (int k = 0; k < kD; k++) acc = __fma_rn(x[k], c[k], acc);
            const double D = __dsub_rn(c2[p * K + j], __dmul_rn(2.0, acc));
            if (bj < 0 || D < bv) { bv = D; bj = j; }
        }
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, m);
            const int oj = __shfl_xor_sync(0xffffffffu, bj, m);
            const bool take = oj >= 0 && (bj < 0 || ov < bv || (ov == bv && oj < bj));
            if (take) { bv = ov; bj = oj; }
        }
        if (lane == 0) assign[pr] = bj;
    }
}

}  // namespace atc

size_t assign_tc_split_elems(int64_t P, int64_t N) {
    const int64_t T = (N + atc::kM - 1) / atc::kM;
    return size_t(P) * T * atc::kSplit * atc::kM * atc::kD;
}

bool assign_tc_ok(int d, int K) { return d == atc::kD && K >= 1 && K <= 256; }

static bool assign_one_enabled() {
    static const bool v = [] { const char *e = getenv("QVG_ASSIGN_ONE"); return !e || atoi(e) != 0; }();
    return v;
}

int launch_split_rows(const double *rows, const uint16_t *x16, uint16_t *split, float *xnorm, float *rows32,
                      int32_t *rows32_ok, int64_t P, int64_t N, cudaStream_t st) {
    const int T = int((N + atc::kM - 1) / atc::kM);
    cudaMemsetAsync(rows32_ok, 1, size_t(P) * sizeof(int32_t), st);      // nonzero = exact until shown otherwise
    const int64_t total = P * T * atc::kM * (atc::kD / 8);
    int64_t g = (total + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    const bool xs = x16 && (reinterpret_cast<uintptr_t>(x16) & 15) == 0;
    atc::k_split_rows<<<unsigned(g), 256, 0, st>>>(rows, xs ? x16 : nullptr, assign_one_enabled() ? 0 : 1, split, xnorm,
                                                  rows32, rows32_ok, P, N, T);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

int launch_assign_tc(const uint16_t *split, const float *xnorm, const double *rows, const double *cent,
                     const double *c2, int32_t *assign, int32_t *recheck, int32_t *n_recheck,
                     const PlaneState *st_planes, int skip_done, int64_t P, int64_t N, int K, int a_one,
                     cudaStream_t st) {
    using namespace atc;
    const int T = int((N + kM - 1) / kM);
    cudaMemsetAsync(n_recheck, 0, sizeof(int32_t), st);
    TcArgs ta{split, xnorm, cent, c2, assign, recheck, n_recheck, st_planes, P, N, K, T, skip_done,
              (a_one && assign_one_enabled()) ? 1 : 0};
    cudaFuncSetAttribute(k_assign_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmem));
    const int64_t items = P * T;
    const int grid = int(items < 148 ? items : 148);
    k_assign_tc<<<grid, kTcThreads, kSmem, st>>>(ta);
    k_assign_recheck<<<148 * 4, 256, 0, st>>>(rows, cent, c2, assign, recheck, n_recheck, N, K);
    static const bool stats = getenv("QVG_ASSIGN_STATS") != nullptr;
    if (stats) {   // measurement aid: fraction of rows the filter could not certify
        int32_t n = 0;
        cudaMemcpyAsync(&n, n_recheck, sizeof(n), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        fprintf(stderr, "qvg assign_tc: %d of %lld rows rechecked (%.4f%%)\n", n, (long long)(P * N),
                100.0 * n / double(P * N));
    }
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

}  // namespace qvg
