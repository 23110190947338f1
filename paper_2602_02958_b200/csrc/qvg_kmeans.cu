// qvg_kmeans.cu — Semantic-Aware Smoothing on sm_100a: deterministic Lloyd
// k-means (Q/clustering.py) reproduced bit for bit on the GPU.
//
//  K1 k_kmeanspp        k-means++ seeding, one CTA per plane (Q/clustering.py:47-63);
//                       the sequential-cumsum inverse-CDF pick is decided from a
//                       parallel prefix with a rigorous error certificate, with an
//                       exact sequential fallback when the certificate fails.
//  K2 k_assign          distance GEMM (fp64 FMA chain in k order, as OpenBLAS
//                       dgemm) fused with c2 = pairwise(C^2) and first-min argmin
//                       (Q/clustering.py:66-71).
//  K3 k_members/k_sums  stable counting sort of rows by cluster, then one ordered
//                       fp64 chain per (cluster, channel) = np.add.at, divide,
//                       keep-old for empties (Q/clustering.py:89-95);
//     k_repair          farthest-row empty-cluster repair (Q/clustering.py:97-104).
//  K4 k_obj_leaves /    numpy pairwise flat sum of the SSE (Q/clustering.py:106,
//     k_obj_combine     143) over a host-built copy of numpy's recursion tree, and
//                       the tol test (Q/clustering.py:148-151) on device.
// Every kernel reads a per-plane `done` flag, so one launch sequence of
// max_iters Lloyd steps serves planes that converge at different iterations.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "qvg_common.cuh"
#include "qvg_internal.h"

namespace qvg {

// ---- pairwise over one row of d <= 128 values, 8 lanes per row ----------
// v(k) supplies element k.  Result valid in every lane of the 8-lane group.
template <typename F>
__device__ __forceinline__ double row_pairwise8(int d, int j, F v) {
    if (d < 8) {
        double s = 0.0;
        for (int k = 0; k < d; k++) s = __dadd_rn(s, v(k));
        return __shfl_sync(0xffffffffu, s, (threadIdx.x & 31) & ~7);
    }
    const int m = d >> 3;
    double acc = v(j);
    for (int i = 1; i < m; i++) acc = __dadd_rn(acc, v(i * 8 + j));
    acc = pairwise8_tree(acc);
    for (int k = m * 8; k < d; k++) acc = __dadd_rn(acc, v(k));   // tail, all lanes equal
    return acc;
}

// leaf sum of v over [off, off+len), 8 lanes (len <= 128); numpy leaf rule.
template <typename F>
__device__ __forceinline__ double leaf_sum8(int64_t off, int len, int j, F v) {
    if (len < 8) {
        double s = 0.0;
        for (int k = 0; k < len; k++) s = __dadd_rn(s, v(off + k));
        return s;
    }
    const int m = len >> 3;
    double acc = v(off + j);
#pragma unroll 4
    for (int i = 1; i < m; i++) acc = __dadd_rn(acc, v(off + i * 8 + j));   // loads of 4 terms in flight
    acc = pairwise8_tree(acc);
    for (int k = m * 8; k < len; k++) acc = __dadd_rn(acc, v(off + k));
    return acc;
}

template <int U, typename F>
__device__ __forceinline__ double leaf_sum8u(int64_t off, int len, int j, F v) {
    if (len < 8) {
        double s = 0.0;
        for (int k = 0; k < len; k++) s = __dadd_rn(s, v(off + k));
        return s;
    }
    const int m = len >> 3;
    double acc = v(off + j);
#pragma unroll U
    for (int i = 1; i < m; i++) acc = __dadd_rn(acc, v(off + i * 8 + j));
    acc = pairwise8_tree(acc);
    for (int k = m * 8; k < len; k++) acc = __dadd_rn(acc, v(off + k));
    return acc;
}

// ------------------------------------------------------------------------
// widen input to the f64 stage-1 rows (plane.data.astype(np.float64)) + NaN scan
// ------------------------------------------------------------------------
__global__ void k_widen(const void *x, int xbf16, double *rows, int64_t n, int32_t *status) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        float f = xbf16 ? bf16_to_f32(static_cast<const uint16_t *>(x)[i]) : static_cast<const float *>(x)[i];
        if (!isfinite(f)) atomicOr(status, QVG_STATUS_NONFINITE);
        rows[i] = double(f);
    }
}

// ------------------------------------------------------------------------
// K1: k-means++ (one CTA of 1024 threads per plane)
// ------------------------------------------------------------------------
struct PPArgs {
    const double *rows;      // [P][N][d]
    const float *rows32;     // [P][N][d] float32 copy (nullable)
    const uint16_t *rows16;  // [P][N][d] the bf16 input when the rows are exactly it (nullable)
    const int32_t *rows32_ok;   // [P] 1: the copy is exact
    const double *draws;     // this stage's draws of plane 0; plane p at + p*draws_stride
    int64_t draws_stride;
    double *cent;            // [P][K][d]
    double *d2;              // [P][N]
    const int64_t *lf_off;   // pick-tree leaves over N
    const int32_t *lf_len;
    int n_leaves;
    int64_t N;
    int d, K;
    const int32_t *nd_l, *nd_r, *h_start;   // internal nodes of the pick tree, by height
    int n_heights;
    int d2_smem;             // 1: the N pick weights live in shared memory (after the draws)
    // stage 2 of a bf16 chunk: rows rebuilt from the input and the stage-1 table
    const uint16_t *x16;     // [P][N][d] bf16 input (nullable)
    const uint16_t *c1;      // stage-1 bf16 centroids of plane 0; plane p at + p*c1_stride
    int64_t c1_stride;
    const uint8_t *a1;       // stage-1 assignments of plane 0; plane p at + p*a1_stride
    int64_t a1_stride;
    int64_t c1_off;          // shared-memory offset (in doubles) of the padded table copy
};

// rows read as T (double, or float when the plane's float64 rows are all exactly
// representable in float32, see k_split_rows): identical values, half the bytes
// a bf16 element read as its exact double value
struct Bf16 {
    uint16_t v;
    __device__ __forceinline__ operator double() const { return double(__uint_as_float(uint32_t(v) << 16)); }
};

__device__ __forceinline__ void bf16x8_to_f64(uint4 w, double v[8]) {
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int h = 0; h < 4; h++) {
        v[2 * h] = double(__uint_as_float(u[h] << 16));
        v[2 * h + 1] = double(__uint_as_float(u[h] & 0xFFFF0000u));
    }
}

// Row sources: row(i)[k] is the exact double value of element (i, k);
// load8(i, k0, v) fetches elements k0..k0+7 (k0 % 8 == 0) with vector loads.
template <typename T>
struct SrcPlain {                       // rows stored as T (double / float / bf16)
    static constexpr int kBytes = sizeof(T);
    static constexpr bool kResid = false;
    const T *rows;
    int d;
    struct Row {
        const T *r;
        __device__ __forceinline__ double operator[](int k) const { return double(r[k]); }
        __device__ __forceinline__ void load8(int k0, double v[8]) const {   // 2-byte T
            bf16x8_to_f64(*reinterpret_cast<const uint4 *>(r + k0), v);
        }
    };
    __device__ __forceinline__ Row row(int64_t i) const { return Row{rows + i * d}; }
    __device__ __forceinline__ void load8(int64_t i, int k0, double v[8]) const {
        const T *r = rows + i * d + k0;
        if constexpr (sizeof(T) == 2) {
            bf16x8_to_f64(*reinterpret_cast<const uint4 *>(r), v);
        } else if constexpr (sizeof(T) == 4) {
            const float4 a = reinterpret_cast<const float4 *>(r)[0], b = reinterpret_cast<const float4 *>(r)[1];
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
#pragma unroll
            for (int h = 0; h < 4; h++) {
                const double2 t = reinterpret_cast<const double2 *>(r)[h];
                v[2 * h] = t.x;
                v[2 * h + 1] = t.y;
            }
        }
    }
};
struct SrcResid {                       // stage-2 rows x - C1_bf16[pi1] rebuilt from the bf16 input
    static constexpr int kBytes = 2;    // (the f64 difference of two bf16 values is exact)
    static constexpr bool kResid = true;
    const uint16_t *x;
    const uint16_t *c1;                 // shared copy of this plane's stage-1 table, row pitch `cp`
    const uint8_t *a1;
    int d, cp;
    struct Row {
        const uint16_t *xr, *cr;
        __device__ __forceinline__ double operator[](int k) const {
            return __dsub_rn(double(__uint_as_float(uint32_t(xr[k]) << 16)), double(__uint_as_float(uint32_t(cr[k]) << 16)));
        }
        __device__ __forceinline__ void load8(int k0, double v[8]) const {
            const uint4 xw = *reinterpret_cast<const uint4 *>(xr + k0);
            const uint4 cw = *reinterpret_cast<const uint4 *>(cr + k0);
            const uint32_t xu[4] = {xw.x, xw.y, xw.z, xw.w}, cu[4] = {cw.x, cw.y, cw.z, cw.w};
#pragma unroll
            for (int h = 0; h < 4; h++) {
                v[2 * h] = __dsub_rn(double(__uint_as_float(xu[h] << 16)), double(__uint_as_float(cu[h] << 16)));
                v[2 * h + 1] = __dsub_rn(double(__uint_as_float(xu[h] & 0xFFFF0000u)),
                                         double(__uint_as_float(cu[h] & 0xFFFF0000u)));
            }
        }
    };
    __device__ __forceinline__ Row row(int64_t i) const { return Row{x + i * d, c1 + int(a1[i]) * cp}; }
    __device__ __forceinline__ void load8(int64_t i, int k0, double v[8]) const {
        const uint4 xw = *reinterpret_cast<const uint4 *>(x + i * d + k0);
        const uint4 cw = *reinterpret_cast<const uint4 *>(c1 + int(a1[i]) * cp + k0);
        const uint32_t xu[4] = {xw.x, xw.y, xw.z, xw.w}, cu[4] = {cw.x, cw.y, cw.z, cw.w};
#pragma unroll
        for (int h = 0; h < 4; h++) {
            v[2 * h] = __dsub_rn(double(__uint_as_float(xu[h] << 16)), double(__uint_as_float(cu[h] << 16)));
            v[2 * h + 1] = __dsub_rn(double(__uint_as_float(xu[h] & 0xFFFF0000u)),
                                     double(__uint_as_float(cu[h] & 0xFFFF0000u)));
        }
    }
};

template <typename Src>
__device__ __forceinline__ void kmeanspp_body(const PPArgs &a, const Src src, double *sm) {
    double *xc = sm;                       // [d]
    double *leaf = sm + 128;               // [n_leaves] leaves, then the internal nodes
    double *dr = leaf + 2 * a.n_leaves - 1;   // [K] this plane's draws
    __shared__ int64_t s_pick;
    const int64_t p = blockIdx.x;
    const int64_t N = a.N;
    const int d = a.d, K = a.K;
    double *d2 = a.d2_smem ? sm + 128 + 2 * a.n_leaves - 1 + K : a.d2 + p * N;
    double *cent = a.cent + p * int64_t(K) * d;
    const double *draws = a.draws + p * a.draws_stride;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int j8 = lane & 7;

    for (int k = tid; k < K; k += blockDim.x) dr[k] = draws[k];
    if (tid == 0) {
        int64_t c = int64_t(draws[0] * double(N));
        s_pick = c < N - 1 ? c : N - 1;
    }
    __syncthreads();
    for (int pk = 0; pk < K; pk++) {
        const int64_t c = s_pick;
        const auto rc = src.row(c);
        for (int k = tid; k < d; k += blockDim.x) {
            double v = rc[k];
            xc[k] = v;
            cent[int64_t(pk) * d + k] = v;
        }
        __syncthreads();
        if (pk == K - 1) break;
        // d2 = min(d2, ((rows - rows[c])**2).sum(axis=1))
        auto generic_rows = [&]() {
            for (int64_t i0 = int64_t(warp) * 4; i0 < N; i0 += blockDim.x >> 3) {  // warp-uniform
                const int64_t i = i0 + (lane >> 3);
                const int64_t ii = i < N ? i : N - 1;
                const auto ri = src.row(ii);
                double dist = row_pairwise8(d, j8, [&](int k) {
                    double t = __dsub_rn(ri[k], xc[k]);
                    return __dmul_rn(t, t);
                });
                dist = __dadd_rn(0.0, dist);
                if (j8 == 0 && i < N) d2[i] = (pk == 0 || dist < d2[i]) ? dist : d2[i];
            }
        };
        if constexpr (Src::kBytes == 2) {
            if (d == 128) {
            // head_dim 128, bf16 rows: one row per thread, the eight numpy pairwise-8
            // accumulators in registers (r_j = sum over i of t(8i + j), i = 0..15, in
            // order, then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))); 16-byte loads
            for (int64_t i = tid; i < N; i += blockDim.x) {
                double r[8];
                const auto rw = src.row(i);                  // row pointers (and pi1) once
#pragma unroll
                for (int q = 0; q < 16; q++) {
                    double v[8];
                    rw.load8(q * 8, v);
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        const double t = __dsub_rn(v[j], xc[q * 8 + j]);
                        r[j] = q == 0 ? __dmul_rn(t, t) : __dadd_rn(r[j], __dmul_rn(t, t));
                    }
                }
                const double sum = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                                             __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
                const double dist = __dadd_rn(0.0, sum);
                d2[i] = (pk == 0 || dist < d2[i]) ? dist : d2[i];
            }
            } else {
                generic_rows();
            }
        } else if (d == 128) {
            // head_dim 128, float / double rows: 8 lanes per row, all 16 loads of a lane
            // issued before the (ordered) sums, two rows per 8-lane group in flight
            double xcl[16];
#pragma unroll
            for (int q = 0; q < 16; q++) xcl[q] = xc[q * 8 + j8];
            const int64_t step = blockDim.x >> 3;                      // rows per CTA pass
            for (int64_t i0 = int64_t(warp) * 4; i0 < N; i0 += 2 * step) {   // warp-uniform
                const int64_t ia = i0 + (lane >> 3), ib = ia + step;
                const auto ra = src.row(ia < N ? ia : N - 1), rb = src.row(ib < N ? ib : N - 1);
                double va[16], vb[16];
#pragma unroll
                for (int q = 0; q < 16; q++) { va[q] = ra[q * 8 + j8]; vb[q] = rb[q * 8 + j8]; }
                double sa, sb;
                {
                    double t = __dsub_rn(va[0], xcl[0]);
                    sa = __dmul_rn(t, t);
                    t = __dsub_rn(vb[0], xcl[0]);
                    sb = __dmul_rn(t, t);
                }
#pragma unroll
                for (int q = 1; q < 16; q++) {
                    double t = __dsub_rn(va[q], xcl[q]);
                    sa = __dadd_rn(sa, __dmul_rn(t, t));
                    t = __dsub_rn(vb[q], xcl[q]);
                    sb = __dadd_rn(sb, __dmul_rn(t, t));
                }
                sa = __dadd_rn(0.0, pairwise8_tree(sa));
                sb = __dadd_rn(0.0, pairwise8_tree(sb));
                if (j8 == 0 && ia < N) d2[ia] = (pk == 0 || sa < d2[ia]) ? sa : d2[ia];
                if (j8 == 0 && ib < N) d2[ib] = (pk == 0 || sb < d2[ib]) ? sb : d2[ib];
            }
        } else {
            generic_rows();
        }
        __syncthreads();
        // total = weights.sum() : leaves then numpy recursion
        for (int L0 = warp * 4; L0 < a.n_leaves; L0 += blockDim.x >> 3) {     // warp-uniform
            const int L = L0 + (lane >> 3);
            const int LL = L < a.n_leaves ? L : a.n_leaves - 1;
            double s = leaf_sum8(a.lf_off[LL], a.lf_len[LL], j8, [&](int64_t e) { return d2[e]; });
            if (j8 == 0 && L < a.n_leaves) leaf[L] = s;
        }
        __syncthreads();
        if (warp == 0) {
            // (1) total = the numpy recursion over the leaves, level by level (host-built tree)
            const int nl = a.n_leaves;
            for (int hh = 0; hh < a.n_heights; hh++) {
                for (int i = a.h_start[hh] + lane; i < a.h_start[hh + 1]; i += 32)
                    leaf[nl + i] = __dadd_rn(leaf[a.nd_l[i]], leaf[a.nd_r[i]]);
                __syncwarp();
            }
            const double total = __dadd_rn(0.0, leaf[nl > 1 ? 2 * nl - 2 : 0]);
            const double r = dr[pk + 1];
            int64_t pick;
            if (!(total > 0.0)) {                         // uniform fallback (Q/clustering.py:41-42)
                pick = int64_t(r * double(N));
            } else {
                // (2) searchsorted(cumsum(d2), target, 'right') = #{j : cum_seq[j] <= target}.
                // cum_seq (sequential f64) and every prefix computed here (sums of
                // non-negative terms in another order) lie within gamma_N * S_j of the
                // exact prefix S_j, so a prefix farther than 2 gamma_N from target decides
                // its element exactly; undecided elements replay the sequential cumsum.
                // Leaf level first (whole leaves certainly below target), then the
                // elements from the first undecided leaf on, 32 at a time.
                const double target = __dmul_rn(r, total);
                const double eps = double(2 * N + 64) * 2.220446049250313e-16;
                double base = 0.0;
                int lo = nl;
                for (int L0 = 0; L0 < nl; L0 += 32) {
                    const int L = L0 + lane;
                    double incl = L < nl ? leaf[L] : 0.0;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const double t = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += t;
                    }
                    const double q = base + incl;
                    const unsigned und = __ballot_sync(0xffffffffu, L < nl && !(q + q * eps < target));
                    if (und) {
                        const int f = __ffs(und) - 1;
                        lo = L0 + f;
                        const double before = __shfl_sync(0xffffffffu, incl, f > 0 ? f - 1 : 0);
                        base = f > 0 ? base + before : base;
                        break;
                    }
                    base += __shfl_sync(0xffffffffu, incl, 31);
                }
                int64_t cnt = lo < nl ? a.lf_off[lo] : N;
                bool amb = false;
                if (lo < nl) {
                    for (int64_t e0 = cnt; e0 < N; e0 += 32) {
                        const int64_t i = e0 + lane;
                        double incl = i < N ? d2[i] : 0.0;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const double t = __shfl_up_sync(0xffffffffu, incl, o);
                            if (lane >= o) incl += t;
                        }
                        const double pre = base + incl, m = pre * eps;
                        const bool le = i < N && pre + m < target;
                        const bool gt = i >= N || pre - m > target;
                        cnt += __popc(__ballot_sync(0xffffffffu, le));
                        amb |= __any_sync(0xffffffffu, !le && !gt);
                        if (__any_sync(0xffffffffu, gt)) break;      // monotone: the rest is above
                        base += __shfl_sync(0xffffffffu, incl, 31);
                    }
                }
                pick = cnt;
                if (amb && lane == 0) {                  // exact sequential cumsum (rare)
                    double cs = 0.0;
                    int64_t i = 0;
                    for (; i < N; i++) {
                        cs = __dadd_rn(cs, d2[i]);
                        if (cs > target) break;
                    }
                    pick = i;
                }
            }
            if (lane == 0) s_pick = pick < N - 1 ? pick : N - 1;
        }
        __syncthreads();
    }
}


template <int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) k_kmeanspp(PPArgs a) {
    extern __shared__ double sm[];
    const int64_t p = blockIdx.x, nd = a.N * a.d;
    if (a.rows16) {
        kmeanspp_body(a, SrcPlain<Bf16>{reinterpret_cast<const Bf16 *>(a.rows16) + p * nd, a.d}, sm);
    } else if (a.x16) {
        // padded pitch (d + 8): the lanes' 16-byte reads of random table rows spread
        // over the banks instead of all hitting the same ones
        const int cp = a.d + 8;
        uint16_t *c1s = reinterpret_cast<uint16_t *>(sm + a.c1_off);
        const uint16_t *c1g = a.c1 + p * a.c1_stride;
        for (int e = threadIdx.x; e < a.K * a.d; e += blockDim.x) c1s[(e / a.d) * cp + e % a.d] = c1g[e];
        __syncthreads();
        kmeanspp_body(a, SrcResid{a.x16 + p * nd, c1s, a.a1 + p * a.a1_stride, a.d, cp}, sm);
    } else if (a.rows32 && a.rows32_ok[p]) {
        kmeanspp_body(a, SrcPlain<float>{a.rows32 + p * nd, a.d}, sm);
    } else {
        kmeanspp_body(a, SrcPlain<double>{a.rows + p * nd, a.d}, sm);
    }
}

// ------------------------------------------------------------------------
// K2: assignment — fp64 FMA-chain distance GEMM fused with argmin
// ------------------------------------------------------------------------
constexpr int AR = 64, AC = 64, AK = 32;

struct AssignArgs {
    const double *rows;
    const double *cent;
    int32_t *assign;       // [P][N]
    const PlaneState *st;
    int64_t N;
    int d, K;
    int skip_done;
};

__global__ void __launch_bounds__(256) k_assign(AssignArgs a) {
    const int64_t p = blockIdx.y;
    if (a.skip_done && a.st[p].done) return;
    __shared__ double Xs[AR][AK + 1];
    __shared__ double Cs[AC][AK + 1];
    __shared__ double c2s[kMaxK];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int d = a.d, K = a.K;
    const int64_t N = a.N;
    const double *rows = a.rows + p * N * d;
    const double *cent = a.cent + p * int64_t(K) * d;
    const int64_t r0 = int64_t(blockIdx.x) * AR;

    // c2 = (centroids ** 2).sum(axis=1), numpy pairwise per centroid
    for (int c0 = (tid >> 5) * 4; c0 < K; c0 += 32) {          // warp-uniform trip count
        const int c = c0 + ((tid & 31) >> 3);
        const double *cc = cent + int64_t(c < K ? c : K - 1) * d;
        double s = row_pairwise8(d, tid & 7, [&](int k) { return __dmul_rn(cc[k], cc[k]); });
        if ((tid & 7) == 0 && c < K) c2s[c] = __dadd_rn(0.0, s);
    }
    double bv[4];
    int bj[4];
#pragma unroll
    for (int i = 0; i < 4; i++) { bv[i] = 0.0; bj[i] = -1; }

    for (int c0 = 0; c0 < K; c0 += AC) {
        double acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int j = 0; j < 4; j++) acc[i][j] = 0.0;
        for (int k0 = 0; k0 < d; k0 += AK) {
            __syncthreads();
            for (int e = tid; e < AR * AK; e += 256) {
                int rr = e / AK, kk = e % AK;
                int64_t row = r0 + rr;
                Xs[rr][kk] = (row < N && k0 + kk < d) ? rows[row * d + k0 + kk] : 0.0;
                int cc = c0 + rr;
                Cs[rr][kk] = (cc < K && k0 + kk < d) ? cent[int64_t(cc) * d + k0 + kk] : 0.0;
            }
            __syncthreads();
            const int kmax = min(AK, d - k0);
            for (int kk = 0; kk < kmax; kk++) {
                double xv[4], cv[4];
#pragma unroll
                for (int i = 0; i < 4; i++) xv[i] = Xs[ty + 16 * i][kk];
#pragma unroll
                for (int j = 0; j < 4; j++) cv[j] = Cs[tx + 16 * j][kk];
#pragma unroll
                for (int i = 0; i < 4; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) acc[i][j] = __fma_rn(xv[i], cv[j], acc[i][j]);
            }
        }
        // D = c2 - 2*cross; first minimum (np.argmin)
#pragma unroll
        for (int j = 0; j < 4; j++) {
            int cj = c0 + tx + 16 * j;
            if (cj >= K) continue;
            double c2 = c2s[cj];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                double D = __dsub_rn(c2, __dmul_rn(2.0, acc[i][j]));
                if (bj[i] < 0 || D < bv[i]) { bv[i] = D; bj[i] = cj; }
            }
        }
    }
    // reduce over the 16 tx lanes: lexicographic (value, index)
#pragma unroll
    for (int i = 0; i < 4; i++) {
        double v = bv[i];
        int j = bj[i];
#pragma unroll
        for (int m = 1; m < 16; m <<= 1) {
            double ov = __shfl_xor_sync(0xffffffffu, v, m);
            int oj = __shfl_xor_sync(0xffffffffu, j, m);
            bool take = oj >= 0 && (j < 0 || ov < v || (ov == v && oj < j));
            if (take) { v = ov; j = oj; }
        }
        int64_t row = r0 + ty + 16 * i;
        if (tx == 0 && row < N) a.assign[p * N + row] = j;
    }
}

// exact c2 = (centroids ** 2).sum(axis=1) (numpy pairwise, as k_assign) for the
// tensor-core assignment path; 8 lanes per centroid
__global__ void k_c2(const double *cent, double *c2, const PlaneState *st, int skip_done, int64_t P, int d, int K) {
    const int64_t g = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 3;   // (plane, centroid)
    const int64_t gc = g < P * K ? g : P * K - 1;
    const int64_t p = gc / K;
    const double *cc = cent + gc * d;
    double s = row_pairwise8(d, threadIdx.x & 7, [&](int k) { return __dmul_rn(cc[k], cc[k]); });
    if ((threadIdx.x & 7) == 0 && g < P * K && !(skip_done && st[p].done)) c2[g] = __dadd_rn(0.0, s);
}

// ------------------------------------------------------------------------
// K3a: stable counting sort of rows by cluster (one CTA of 1024 per plane)
// ------------------------------------------------------------------------
struct MemberArgs {
    const int32_t *assign;
    int32_t *counts;       // [P][K]
    int32_t *offsets;      // [P][K+1]
    int32_t *members;      // [P][N]
    const PlaneState *st;
    int64_t N;
    int K;
};

__global__ void __launch_bounds__(1024) k_members(MemberArgs a) {
    const int64_t p = blockIdx.x;
    if (a.st[p].done) return;
    extern __shared__ int32_t smi[];
    const int K = a.K;
    int32_t *cnt = smi;                 // [K]
    int32_t *base = smi + K;            // [K]
    int32_t *wcnt = smi + 2 * K;        // [32][K]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t N = a.N;
    const int32_t *asg = a.assign + p * N;
    int32_t *mem = a.members + p * N;
    for (int j = tid; j < K; j += blockDim.x) cnt[j] = 0;
    for (int j = tid; j < 32 * K; j += blockDim.x) wcnt[j] = 0;
    __syncthreads();
    for (int64_t i = tid; i < N; i += blockDim.x) atomicAdd(&cnt[asg[i]], 1);
    __syncthreads();
    if (tid == 0) {
        int run = 0;
        for (int j = 0; j < K; j++) {
            a.counts[p * K + j] = cnt[j];
            a.offsets[p * (K + 1) + j] = run;
            base[j] = run;
            run += cnt[j];
        }
        a.offsets[p * (K + 1) + K] = run;
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t b0 = 0; b0 < N; b0 += blockDim.x) {
        const int64_t i = b0 + tid;
        const int c = i < N ? asg[i] : -1;
        const unsigned same = __match_any_sync(0xffffffffu, c);
        const int rank = __popc(same & lt);
        if (c >= 0 && rank == 0) wcnt[warp * K + c] = __popc(same);
        __syncthreads();
        for (int j = tid; j < K; j += blockDim.x) {     // per-cluster prefix over warps
            int run = base[j];
            for (int w = 0; w < 32; w++) {
                int t = wcnt[w * K + j];
                wcnt[w * K + j] = run;
                run += t;
            }
            base[j] = run;
        }
        __syncthreads();
        if (c >= 0) mem[wcnt[warp * K + c] + rank] = int32_t(i);
        __syncthreads();
        for (int j = tid; j < 32 * K; j += blockDim.x) wcnt[j] = 0;
        __syncthreads();
    }
}

// K3b: per (cluster, channel) ordered sums = np.add.at, then / count.
// The stage rows of a bf16 chunk rebuilt from the input (exact in f64): stage 1
// = x, stage 2 = x - C1_bf16[pi1] (c1 != nullptr).  2 bytes per element read
// instead of the 4/8-byte stage rows.
struct BfSrc {
    const uint16_t *x16;       // [P][N][d] (nullptr: not available)
    const uint16_t *c1;        // stage-1 bf16 table of plane 0, plane p at + p * c1_stride
    int64_t c1_stride;
    const uint8_t *a1;         // stage-1 assignments of plane 0, plane p at + p * a1_stride
    int64_t a1_stride;
    __device__ __forceinline__ double at(int64_t p, int64_t N, int d, int64_t row, int col) const {
        double v = double(__uint_as_float(uint32_t(x16[(p * N + row) * d + col]) << 16));
        if (c1) {
            const int c = a1[p * a1_stride + row];
            v = __dsub_rn(v, double(__uint_as_float(uint32_t(c1[p * c1_stride + int64_t(c) * d + col]) << 16)));
        }
        return v;
    }
};

struct SumArgs {
    const double *rows;
    const float *rows32;        // exact float32 copy when rows32_ok[p] (half the bytes)
    const int32_t *rows32_ok;
    double *cent;
    const int32_t *counts, *offsets, *members;
    const PlaneState *st;
    int64_t N;
    int d, K;
};

__global__ void __launch_bounds__(128) k_sums(SumArgs a) {
    const int64_t p = blockIdx.y;
    const int j = blockIdx.x;
    if (a.st[p].done) return;
    const int K = a.K, d = a.d;
    const int cnt = a.counts[p * K + j];
    if (cnt == 0) return;                         // keep the old centroid
    const int32_t *mem = a.members + p * a.N + a.offsets[p * (K + 1) + j];
    auto body = [&](auto val) {
        for (int k = threadIdx.x; k < d; k += blockDim.x) {
            double acc = 0.0;
            int t = 0;
            for (; t + 8 <= cnt; t += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; u++) v[u] = val(mem[t + u], k);
#pragma unroll
                for (int u = 0; u < 8; u++) acc = __dadd_rn(acc, v[u]);
            }
            for (; t < cnt; t++) acc = __dadd_rn(acc, val(mem[t], k));
            a.cent[(p * K + j) * int64_t(d) + k] = __ddiv_rn(acc, double(cnt));
        }
    };
    // (the bf16 source measured slower here: 2-byte member gathers)
    if (a.rows32 && a.rows32_ok[p]) {
        const float *rw = a.rows32 + p * a.N * d;
        body([&](int64_t r, int k) { return double(rw[r * d + k]); });
    } else {
        const double *rw = a.rows + p * a.N * d;
        body([&](int64_t r, int k) { return rw[r * d + k]; });
    }
}

// K3c: empty-cluster repair (one CTA of 1024 per plane; returns at once when
// no cluster is empty, the common case).
struct RepairArgs {
    const double *rows;
    double *cent;
    const float *rows32;        // exact float32 copy when rows32_ok[p] (half the bytes; nullable)
    const int32_t *rows32_ok;
    int32_t *assign;
    const int32_t *counts;
    double *dist;          // [P][N] scratch
    const PlaneState *st;
    int64_t N;
    int d, K;
};

__global__ void __launch_bounds__(1024) k_repair(RepairArgs a) {
    const int64_t p = blockIdx.x;
    if (a.st[p].done) return;
    const int K = a.K, d = a.d;
    const int64_t N = a.N;
    const int32_t *cnt = a.counts + p * K;
    int any = 0;
    for (int j = threadIdx.x; j < K; j += blockDim.x) any |= cnt[j] == 0;
    if (!__syncthreads_or(any)) return;
    double *cent = a.cent + p * int64_t(K) * d;
    int32_t *asg = a.assign + p * N;
    double *dist = a.dist + p * N;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, j8 = lane & 7;
    // a CTA streams its whole plane here (one SM's share of HBM), so the exact
    // float32 copy of the rows is read when there is one: identical values
    const bool r32 = a.rows32 && a.rows32_ok[p];
    auto pass = [&](auto rowp) {
        for (int64_t i0 = int64_t(warp) * 4; i0 < N; i0 += blockDim.x >> 3) {    // warp-uniform
            const int64_t i = i0 + (lane >> 3);
            const int64_t ii = i < N ? i : N - 1;
            const auto ri = rowp + ii * d;
            const double *ci = cent + int64_t(asg[ii]) * d;
            double s = row_pairwise8(d, j8, [&](int k) {
                double t = __dsub_rn(double(ri[k]), ci[k]);
                return __dmul_rn(t, t);
            });
            if (j8 == 0 && i < N) dist[i] = __dadd_rn(0.0, s);
        }
    };
    if (r32) pass(a.rows32 + p * N * d);
    else pass(a.rows + p * N * d);
    __syncthreads();
    __shared__ double wv[32];
    __shared__ int64_t wi[32];
    __shared__ int64_t s_r;
    for (int j = 0; j < K; j++) {
        if (cnt[j] != 0) continue;
        double bv = -1.0 / 0.0;
        int64_t bi = -1;
        for (int64_t i = tid; i < N; i += blockDim.x) {
            double v = dist[i];
            if (bi < 0 || v > bv) { bv = v; bi = i; }
        }
        for (int m = 1; m < 32; m <<= 1) {
            double ov = __shfl_xor_sync(0xffffffffu, bv, m);
            int64_t oi = __shfl_xor_sync(0xffffffffu, bi, m);
            if (oi >= 0 && (bi < 0 || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
        }
        if (lane == 0) { wv[warp] = bv; wi[warp] = bi; }
        __syncthreads();
        if (tid == 0) {
            double v = wv[0];
            int64_t r = wi[0];
            for (int w = 1; w < (int)(blockDim.x >> 5); w++)
                if (wi[w] >= 0 && (r < 0 || wv[w] > v || (wv[w] == v && wi[w] < r))) { v = wv[w]; r = wi[w]; }
            s_r = r;
            asg[r] = j;
            dist[r] = -1.0;
        }
        __syncthreads();
        const int64_t r = s_r;
        for (int k = tid; k < d; k += blockDim.x)
            cent[int64_t(j) * d + k] = r32 ? double(a.rows32[(p * N + r) * d + k]) : a.rows[(p * N + r) * d + k];
        __syncthreads();
    }
}

// ------------------------------------------------------------------------
// K4: objective = ((rows - cent[assign])**2).sum() (flat numpy pairwise)
// ------------------------------------------------------------------------
struct ObjArgs {
    BfSrc bf;
    const double *rows;
    const float *rows32;        // exact float32 copy when rows32_ok[p]
    const int32_t *rows32_ok;
    const double *cent;
    const int32_t *assign;
    double *nodes;            // [P][n_nodes]
    PlaneState *st;
    const int64_t *lf_off;
    const int32_t *lf_len;
    const int32_t *nd_l, *nd_r, *h_start;
    int n_leaves, n_heights;
    int64_t N;
    int d, K;
    int mode;                 // 0: initial objective -> prev; 1: Lloyd step + tol test; 2: objective only
    double tol;
    int lgd;                  // log2(d) when d is a power of two, else -1
};

__global__ void __launch_bounds__(256) k_obj_leaves(ObjArgs a) {
    const int64_t p = blockIdx.y;
    if (a.mode == 1 && a.st[p].done) return;
    const int d = a.d;
    const double *rows = a.rows + p * a.N * d;
    const double *cent = a.cent + p * int64_t(a.K) * d;
    const int32_t *asg = a.assign + p * a.N;
    const int n_nodes = 2 * a.n_leaves - 1;
    const int j8 = threadIdx.x & 7;
    const int64_t wg = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;   // global warp
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    auto run = [&](auto rw, auto pow2) {
        constexpr bool P2 = decltype(pow2)::value;
        for (int64_t L0 = wg * 4; L0 < a.n_leaves; L0 += nw * 4) {            // warp-uniform
            const int64_t L = L0 + ((threadIdx.x & 31) >> 3);
            const int64_t LL = L < a.n_leaves ? L : a.n_leaves - 1;
            double s = leaf_sum8(a.lf_off[LL], a.lf_len[LL], j8, [&](int64_t e) {
                const int64_t row = P2 ? e >> a.lgd : e / d;
                const int col = P2 ? int(e & (d - 1)) : int(e - row * d);
                double t = __dsub_rn(double(rw[e]), cent[int64_t(asg[row]) * d + col]);
                return __dmul_rn(t, t);
            });
            if (j8 == 0 && L < a.n_leaves) a.nodes[p * n_nodes + L] = s;
        }
    };
    if (a.bf.x16 && a.lgd >= 7) {                    // rows rebuilt from the bf16 input
        // d >= 128: a leaf (<= 128 elements) spans at most two rows, whose
        // assignments (and stage-1 table rows) are looked up once per leaf
        const uint16_t *xp = a.bf.x16 + p * a.N * d;
        const uint16_t *c1p = a.bf.c1 ? a.bf.c1 + p * a.bf.c1_stride : nullptr;
        const uint8_t *a1p = a.bf.c1 ? a.bf.a1 + p * a.bf.a1_stride : nullptr;
        for (int64_t L0 = wg * 4; L0 < a.n_leaves; L0 += nw * 4) {            // warp-uniform
            const int64_t L = L0 + ((threadIdx.x & 31) >> 3);
            const int64_t LL = L < a.n_leaves ? L : a.n_leaves - 1;
            const int64_t off = a.lf_off[LL];
            const int64_t r0 = off >> a.lgd, r1 = r0 + 1 < a.N ? r0 + 1 : r0;
            const double *ce0 = cent + int64_t(asg[r0]) * d, *ce1 = cent + int64_t(asg[r1]) * d;
            const uint16_t *cb0 = c1p ? c1p + int64_t(a1p[r0]) * d : nullptr;
            const uint16_t *cb1 = c1p ? c1p + int64_t(a1p[r1]) * d : nullptr;
            double s = leaf_sum8u<8>(off, a.lf_len[LL], j8, [&](int64_t e) {
                const bool first = (e >> a.lgd) == r0;
                const int col = int(e & (d - 1));
                double v = double(__uint_as_float(uint32_t(xp[e]) << 16));
                if (c1p) v = __dsub_rn(v, double(__uint_as_float(uint32_t((first ? cb0 : cb1)[col]) << 16)));
                double t = __dsub_rn(v, (first ? ce0 : ce1)[col]);
                return __dmul_rn(t, t);
            });
            if (j8 == 0 && L < a.n_leaves) a.nodes[p * n_nodes + L] = s;
        }
        return;
    }
    const bool r32 = a.rows32 && a.rows32_ok[p];
    if (a.lgd >= 0) {
        if (r32) run(a.rows32 + p * a.N * d, std::true_type{});
        else run(rows, std::true_type{});
    } else {
        if (r32) run(a.rows32 + p * a.N * d, std::false_type{});
        else run(rows, std::false_type{});
    }
}

// K4 leaves over bf16 planes (d >= 128, a power of two), one CTA per plane,
// one thread per leaf: the plane's float64 centroid table and bf16 stage-1
// table are staged in shared memory (rows padded by 16 bytes, so the lanes'
// 16-byte reads of unrelated rows spread over the banks), numpy's eight
// accumulators r[0..7] live in registers, and each step of 8 consecutive
// elements (leaf offsets are multiples of 8, so a step never crosses a row)
// is one 16-byte load of x plus shared-memory reads -- the same float64
// operations in the same order as k_obj_leaves' 8-lane groups (r[j]
// sequential over the steps, then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then
// the tail).  k_obj_leaves' global-memory version was bound by L1 wavefronts
// of the per-lane centroid-row reads.
constexpr int kObjThreads = 512;

__device__ __forceinline__ void bf16x8(uint4 w, float f[8]) {
    const uint32_t v[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < 4; i++) {
        f[2 * i] = __uint_as_float(v[i] << 16);
        f[2 * i + 1] = __uint_as_float(v[i] & 0xFFFF0000u);
    }
}

static size_t obj_plane_smem(int K, int d, bool c1) {
    return size_t(K) * (size_t(d) * 8 + 16) + (c1 ? size_t(K) * (size_t(d) * 2 + 16) : 0);
}

__global__ void __launch_bounds__(kObjThreads, 2) k_obj_plane(ObjArgs a) {
    extern __shared__ __align__(16) uint8_t osm[];
    const int64_t p = blockIdx.x;
    if (a.mode == 1 && a.st[p].done) return;
    const int d = a.d, K = a.K;
    const int cp = d * 8 + 16, bp = d * 2 + 16;       // padded row pitches (bytes)
    uint8_t *sc = osm, *sb = osm + size_t(K) * cp;
    const uint16_t *c1p = a.bf.c1 ? a.bf.c1 + p * a.bf.c1_stride : nullptr;
    const uint8_t *a1p = a.bf.c1 ? a.bf.a1 + p * a.bf.a1_stride : nullptr;
    {
        const uint4 *cg = reinterpret_cast<const uint4 *>(a.cent + p * int64_t(K) * d);
        const int per = d / 2;                        // 16-byte words per f64 row
        for (int i = threadIdx.x; i < K * per; i += blockDim.x)
            *reinterpret_cast<uint4 *>(sc + (i / per) * cp + (i % per) * 16) = cg[i];
        if (c1p) {
            const uint4 *bg = reinterpret_cast<const uint4 *>(c1p);
            const int pb = d / 8;
            for (int i = threadIdx.x; i < K * pb; i += blockDim.x)
                *reinterpret_cast<uint4 *>(sb + (i / pb) * bp + (i % pb) * 16) = bg[i];
        }
    }
    __syncthreads();
    const int32_t *asg = a.assign + p * a.N;
    const uint16_t *xp = a.bf.x16 + p * a.N * d;
    const int n_nodes = 2 * a.n_leaves - 1;
    auto elem1 = [&](int64_t e) {
        const int64_t row = e >> a.lgd;
        const int col = int(e & (d - 1));
        double v = double(__uint_as_float(uint32_t(xp[e]) << 16));
        if (c1p) v = __dsub_rn(v, double(__uint_as_float(uint32_t(
                                    *reinterpret_cast<const uint16_t *>(sb + a1p[row] * bp + col * 2)) << 16)));
        const double t = __dsub_rn(v, *reinterpret_cast<const double *>(sc + asg[row] * cp + col * 8));
        return __dmul_rn(t, t);
    };
    for (int L = threadIdx.x; L < a.n_leaves; L += blockDim.x) {
        const int64_t off = a.lf_off[L];
        const int len = a.lf_len[L];
        double s;
        if (len < 8 || (off & 7) != 0) {
            s = 0.0;
            if (len < 8) {
                for (int k = 0; k < len; k++) s = __dadd_rn(s, elem1(off + k));
            } else {
                const int m = len >> 3;
                double r[8];
                for (int k = 0; k < 8; k++) r[k] = elem1(off + k);
                for (int i = 1; i < m; i++)
                    for (int k = 0; k < 8; k++) r[k] = __dadd_rn(r[k], elem1(off + 8 * i + k));
                s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                              __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
                for (int k = m * 8; k < len; k++) s = __dadd_rn(s, elem1(off + k));
            }
        } else {
            const int64_t r0 = off >> a.lgd, r1 = (off + len - 1) >> a.lgd;   // a leaf spans <= 2 rows
            const uint8_t *ce0 = sc + asg[r0] * cp, *ce1 = sc + asg[r1] * cp;
            const uint8_t *cb0 = c1p ? sb + a1p[r0] * bp : nullptr, *cb1 = c1p ? sb + a1p[r1] * bp : nullptr;
            auto elem8 = [&](int64_t e, double v[8]) {
                const bool first = (e >> a.lgd) == r0;
                const int col = int(e & (d - 1));
                float xf[8];
                bf16x8(*reinterpret_cast<const uint4 *>(xp + e), xf);
                double xv[8];
#pragma unroll
                for (int k = 0; k < 8; k++) xv[k] = double(xf[k]);
                if (c1p) {
                    float cf[8];
                    bf16x8(*reinterpret_cast<const uint4 *>((first ? cb0 : cb1) + col * 2), cf);
#pragma unroll
                    for (int k = 0; k < 8; k++) xv[k] = __dsub_rn(xv[k], double(cf[k]));
                }
                const double2 *ce = reinterpret_cast<const double2 *>((first ? ce0 : ce1) + col * 8);
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const double2 c = ce[k];
                    const double t0 = __dsub_rn(xv[2 * k], c.x), t1 = __dsub_rn(xv[2 * k + 1], c.y);
                    v[2 * k] = __dmul_rn(t0, t0);
                    v[2 * k + 1] = __dmul_rn(t1, t1);
                }
            };
            const int m = len >> 3;
            double r[8];
            elem8(off, r);
#pragma unroll 2
            for (int i = 1; i < m; i++) {
                double v[8];
                elem8(off + 8 * i, v);
#pragma unroll
                for (int k = 0; k < 8; k++) r[k] = __dadd_rn(r[k], v[k]);
            }
            s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                          __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
            for (int k = m * 8; k < len; k++) s = __dadd_rn(s, elem1(off + k));
        }
        a.nodes[p * n_nodes + L] = s;
    }
}

__global__ void __launch_bounds__(1024) k_obj_combine(ObjArgs a) {
    const int64_t p = blockIdx.x;
    if (a.mode == 1 && a.st[p].done) return;
    const int nl = a.n_leaves;
    double *nodes = a.nodes + p * (2 * nl - 1);
    for (int h = 0; h < a.n_heights; h++) {
        for (int i = a.h_start[h] + threadIdx.x; i < a.h_start[h + 1]; i += blockDim.x)
            nodes[nl + i] = __dadd_rn(nodes[a.nd_l[i]], nodes[a.nd_r[i]]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double obj = __dadd_rn(0.0, nodes[nl > 1 ? 2 * nl - 2 : 0]);
        PlaneState &s = a.st[p];
        s.obj = obj;
        if (a.mode == 0) {
            s.prev = obj;
        } else if (a.mode == 2) {
            // objective only (kmeans result / lloyd_step return value)
        } else {
            s.iters += 1;
            const double tiny = 2.2250738585072014e-308;
            double den = s.prev > tiny ? s.prev : tiny;
            if (__ddiv_rn(__dsub_rn(s.prev, obj), den) < a.tol) s.done = 1;
            else s.prev = obj;
        }
    }
}

// ------------------------------------------------------------------------
// stage finalisation: bf16 centroids, u8 assignments, residual update
// ------------------------------------------------------------------------
__global__ void k_finalize_cent(const double *cent, uint16_t *cent_out, double *cent64_out,
                                int64_t P, int S, int t, int K, int d) {
    const int64_t n = P * K * d;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        int64_t p = i / (int64_t(K) * d), r = i - p * K * d;
        int64_t o = (p * S + t) * int64_t(K) * d + r;
        double c = cent[i];
        cent_out[o] = f32_to_bf16_bits_rne(__double2float_rn(c));
        if (cent64_out) cent64_out[o] = c;
    }
}

// update_rows = 0: only the u8 assignments / iteration counts (the last stage of
// prq_compress: its residual is never read -- the quantizer works from x and the
// tables)
__global__ void k_residual(double *rows, const double *cent, const int32_t *assign,
                           uint8_t *assign_out, int32_t *iters_out, const PlaneState *st,
                           int64_t P, int64_t N, int S, int t, int K, int d, int update_rows) {
    // grid.y = plane, one row per 32-thread group (no 64-bit divisions per element)
    const int64_t p = blockIdx.y;
    double *pr = rows + p * N * d;
    const double *pc = cent + p * int64_t(K) * d;
    const int32_t *pa = assign + p * N;
    const int lane = threadIdx.x & 31;
    for (int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < N;
         row += (int64_t(gridDim.x) * blockDim.x) >> 5) {
        const int c = pa[row];
        const double *cr = pc + int64_t(c) * d;
        double *rr = pr + row * d;
        for (int col = lane; update_rows && col < d; col += 32) {
            const float cb = bf16_to_f32(f32_to_bf16_bits_rne(__double2float_rn(cr[col])));
            rr[col] = __dsub_rn(rr[col], double(cb));
        }
        if (lane == 0) assign_out[(p * S + t) * N + row] = uint8_t(c);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && iters_out) iters_out[p * S + t] = st[p].iters;
}

__global__ void k_stage_reset(PlaneState *st, int64_t P) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P; i += int64_t(gridDim.x) * blockDim.x)
        st[i] = PlaneState{0.0, 0.0, 0, 0};
}

// ------------------------------------------------------------------------
// host-side orchestration (called from qvg_capi.cu)
// ------------------------------------------------------------------------

static int g1d(int64_t n, int b) {
    int64_t g = (n + b - 1) / b;
    return int(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

int launch_widen(const void *x, int xbf16, double *rows, int64_t n, int32_t *status, cudaStream_t st) {
    k_widen<<<g1d(n, 256), 256, 0, st>>>(x, xbf16, rows, n, status);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

static BfSrc bf_src(const KMeansBuffers &b) {
    if (b.src16) return BfSrc{b.src16, nullptr, 0, nullptr, 0};
    if (b.res_x16) return BfSrc{b.res_x16, b.res_c1, b.res_c1_stride, b.res_a1, b.res_a1_stride};
    return BfSrc{nullptr, nullptr, 0, nullptr, 0};
}

static void objective(const KMeansBuffers &b, int64_t P, int64_t N, int d, int K, int mode,
                      double tol, cudaStream_t st) {
    const int lgd = (d & (d - 1)) == 0 ? __builtin_ctz(unsigned(d)) : -1;
    ObjArgs o{bf_src(b), b.rows, b.rows32_valid ? b.rows32 : nullptr, b.rows32_ok, b.cent, b.assign, b.nodes, b.st,
              b.ob_off, b.ob_len, b.nd_l, b.nd_r, b.h_start, b.ob_leaves, b.ob_heights, N, d, K, mode, tol,
              lgd};
    static const bool staged = [] { const char *e = getenv("QVG_OBJ_THREAD"); return !e || atoi(e) != 0; }();
    const size_t osm = obj_plane_smem(K, d, o.bf.c1 != nullptr);
    if (staged && o.bf.x16 && lgd >= 7 && osm <= 110 * 1024 && (!o.bf.c1 || o.bf.c1_stride % 8 == 0) &&
        (reinterpret_cast<uintptr_t>(o.bf.x16) & 15) == 0 && (reinterpret_cast<uintptr_t>(o.bf.c1) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(o.cent) & 15) == 0) {
        cudaFuncSetAttribute(k_obj_plane, cudaFuncAttributeMaxDynamicSharedMemorySize, int(osm));
        k_obj_plane<<<(unsigned)P, kObjThreads, osm, st>>>(o);
    } else {
        dim3 g((unsigned)((int64_t(b.ob_leaves) * 8 + 255) / 256 < 4096 ? (int64_t(b.ob_leaves) * 8 + 255) / 256 : 4096),
               (unsigned)P);
        k_obj_leaves<<<g, 256, 0, st>>>(o);
    }
    k_obj_combine<<<(unsigned)P, 1024, 0, st>>>(o);
}

// QVG_ASSIGN=exact forces the float64 kernel (A/B measurements)
static bool assign_tc_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("QVG_ASSIGN");
        v = (e && !strcmp(e, "exact")) ? 0 : 1;
    }
    return v == 1;
}

static void assign_step(const KMeansBuffers &b, int64_t P, int64_t N, int d, int K, int skip,
                        cudaStream_t st) {
    if (b.rsplit && assign_tc_enabled()) {
        // tensor-core filter with certified argmin + exact recheck (qvg_assign_tc.cu)
        const int64_t n8 = P * K * 8;
        k_c2<<<unsigned((n8 + 255) / 256), 256, 0, st>>>(b.cent, b.c2, b.st, skip, P, d, K);
        launch_assign_tc(b.rsplit, b.xnorm, b.rows, b.cent, b.c2, b.assign, b.recheck, b.n_recheck, b.st, skip,
                         P, N, K, b.src16 != nullptr, st);
        return;
    }
    AssignArgs aa{b.rows, b.cent, b.assign, b.st, N, d, K, skip};
    k_assign<<<dim3((unsigned)((N + AR - 1) / AR), (unsigned)P), 256, 0, st>>>(aa);
}

int run_kmeanspp(const KMeansBuffers &b, int64_t P, int64_t N, int d, int K, const double *draws,
                 int64_t draws_stride, cudaStream_t st) {
    PPArgs pa{b.rows, b.rows32_valid ? b.rows32 : nullptr, b.src16, b.rows32_ok, draws, draws_stride, b.cent, b.d2, b.pk_off, b.pk_len, b.pk_leaves, N, d, K,
              b.pk_l, b.pk_r, b.pk_hstart, b.pk_heights, 0, nullptr, nullptr, 0, nullptr, 0, 0};
    size_t smem = sizeof(double) * (128 + 2 * b.pk_leaves - 1 + K);
    // the pick weights in shared memory while two 1024-thread CTAs still fit per SM
    if (smem + sizeof(double) * N <= 100 * 1024) {
        smem += sizeof(double) * N;
        pa.d2_smem = 1;
    }
    // stage 2 of a bf16 chunk (d = 128): rebuild the rows x - C1_bf16[pi1] exactly in
    // f64 from the bf16 input and a shared copy of the stage-1 table (2 bytes per
    // element instead of the 4- or 8-byte stage rows)
    const size_t tab = (size_t(K) * (d + 8) * 2 + 15) & ~size_t(15);
    if (b.res_x16 && d == 128 && ((smem + 15) & ~size_t(15)) + tab <= 100 * 1024) {
        smem = (smem + 15) & ~size_t(15);
        pa.x16 = b.res_x16;
        pa.c1 = b.res_c1;
        pa.c1_stride = b.res_c1_stride;
        pa.a1 = b.res_a1;
        pa.a1_stride = b.res_a1_stride;
        pa.c1_off = int64_t(smem / sizeof(double));
        smem += tab;
    }
    // 512-thread CTAs, two planes per SM (64 registers): 85.7 ms per cold chunk
    // vs 87.9 with one 1024-thread CTA per SM and 88.8 with 512 threads at 128
    // registers (one plane per SM); 256 threads: 85.9
    static const int nt = [] { const char *e = getenv("QVG_KPP_THREADS"); return e ? atoi(e) : 512; }();
    if (nt == 512) {
        cudaFuncSetAttribute(k_kmeanspp<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_kmeanspp<512><<<(unsigned)P, 512, smem, st>>>(pa);
    } else if (nt == 256) {
        cudaFuncSetAttribute(k_kmeanspp<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_kmeanspp<256><<<(unsigned)P, 256, smem, st>>>(pa);
    } else {
        cudaFuncSetAttribute(k_kmeanspp<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_kmeanspp<1024><<<(unsigned)P, 1024, smem, st>>>(pa);
    }
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

static void lloyd_body(const KMeansBuffers &b, int64_t P, int64_t N, int d, int K, int mode,
                       double tol, cudaStream_t st) {
    size_t msmem = sizeof(int32_t) * (34 * K);
    if (msmem > 48 * 1024)
        cudaFuncSetAttribute(k_members, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msmem);
    assign_step(b, P, N, d, K, 1, st);
    MemberArgs ma{b.assign, b.counts, b.offsets, b.members, b.st, N, K};
    k_members<<<(unsigned)P, 1024, msmem, st>>>(ma);
    SumArgs sa{b.rows, b.rows32_valid ? b.rows32 : nullptr, b.rows32_ok, b.cent, b.counts, b.offsets, b.members, b.st, N, d, K};
    k_sums<<<dim3((unsigned)K, (unsigned)P), 128, 0, st>>>(sa);
    RepairArgs ra{b.rows, b.cent, b.rows32_valid ? b.rows32 : nullptr, b.rows32_ok, b.assign, b.counts, b.d2, b.st, N, d, K};
    k_repair<<<(unsigned)P, 1024, 0, st>>>(ra);
    objective(b, P, N, d, K, mode, tol, st);
}

// The rows are fixed for a whole stage (or Lloyd step): split them once into the
// bf16 hi/mid/lo tiles of the tensor-core assignment (every assign_step reads them).
static int split_rows(KMeansBuffers &b, int64_t P, int64_t N, cudaStream_t st) {
    b.rows32_valid = 0;
    if (b.rsplit && assign_tc_enabled()) {
        if (launch_split_rows(b.rows, b.src16, b.rsplit, b.xnorm, b.rows32, b.rows32_ok, P, N, st)) return QVG_ERR_CUDA;
        b.rows32_valid = 1;
    }
    return QVG_OK;
}

// One SAS stage's k-means for all planes (Q/clustering.py:110-160); leaves
// the final assignment in b.assign and the iteration count in b.st.
int run_kmeans_stage(KMeansBuffers &b, int64_t P, int64_t N, int d, int K, int max_iters,
                     double tol, const double *draws_stage, int64_t draws_stride, bool warm,
                     cudaStream_t st) {
    k_stage_reset<<<g1d(P, 256), 256, 0, st>>>(b.st, P);
    if (split_rows(b, P, N, st)) return QVG_ERR_CUDA;
    if (!warm && run_kmeanspp(b, P, N, d, K, draws_stage, draws_stride, st)) return QVG_ERR_CUDA;
    // objective of the starting centroids (Q/clustering.py:142-143)
    assign_step(b, P, N, d, K, 0, st);
    objective(b, P, N, d, K, 0, tol, st);
    for (int it = 0; it < max_iters; it++) lloyd_body(b, P, N, d, K, 1, tol, st);
    // final assignment (Q/clustering.py:153)
    assign_step(b, P, N, d, K, 0, st);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

__global__ void k_km_outputs(const int32_t *assign, uint8_t *assign_out, const PlaneState *st,
                             double *obj_out, int32_t *iters_out, int64_t P, int64_t N) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P * N; i += int64_t(gridDim.x) * blockDim.x) {
        if (assign_out) assign_out[i] = uint8_t(assign[i]);
        if (i % N == 0) {
            int64_t p = i / N;
            if (obj_out) obj_out[p] = st[p].obj;
            if (iters_out) iters_out[p] = st[p].iters;
        }
    }
}

int kmeans_outputs(const KMeansBuffers &b, int64_t P, int64_t N, int d, int K, uint8_t *assign,
                   double *objective_out, int32_t *iters, cudaStream_t st) {
    objective(b, P, N, d, K, 2, 0.0, st);   // Q/clustering.py:154
    k_km_outputs<<<g1d(P * N, 256), 256, 0, st>>>(b.assign, assign, b.st, objective_out, iters, P, N);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

int lloyd_once(KMeansBuffers &b, int64_t P, int64_t N, int d, int K, uint8_t *assign,
               double *objective_out, cudaStream_t st) {
    k_stage_reset<<<g1d(P, 256), 256, 0, st>>>(b.st, P);
    if (split_rows(b, P, N, st)) return QVG_ERR_CUDA;
    lloyd_body(b, P, N, d, K, 2, 0.0, st);
    k_km_outputs<<<g1d(P * N, 256), 256, 0, st>>>(b.assign, assign, b.st, objective_out, nullptr, P, N);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

int run_assign(const double *rows, const double *cent, int32_t *assign, int64_t P, int64_t N, int d,
               int K, cudaStream_t st) {
    AssignArgs aa{rows, cent, assign, nullptr, N, d, K, 0};
    k_assign<<<dim3((unsigned)((N + AR - 1) / AR), (unsigned)P), 256, 0, st>>>(aa);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

// add_back (Q/smoothing.py:44-54): residual + f64(C_bf16[pi])
__global__ void k_add_back(const double *res, const uint16_t *cent, const uint8_t *asg, int64_t P,
                           int64_t N, int d, int K, double *out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P * N * d; i += int64_t(gridDim.x) * blockDim.x) {
        int64_t p = i / (N * d), e = i - p * N * d, row = e / d;
        int col = int(e - row * d);
        int c = asg[p * N + row];
        out[i] = __dadd_rn(res[i], double(bf16_to_f32(cent[(p * K + c) * int64_t(d) + col])));
    }
}

int run_add_back(const double *residual, const uint16_t *cent, const uint8_t *assign, int64_t P,
                 int64_t N, int d, int K, double *out, cudaStream_t st) {
    k_add_back<<<g1d(P * N * d, 256), 256, 0, st>>>(residual, cent, assign, P, N, d, K, out);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

int finalize_stage(const KMeansBuffers &b, int64_t P, int64_t N, int d, int K, int S, int t,
                   uint16_t *cent_out, double *cent64_out, uint8_t *assign_out, int32_t *iters_out,
                   cudaStream_t st, bool update_rows) {
    k_finalize_cent<<<g1d(P * K * d, 256), 256, 0, st>>>(b.cent, cent_out, cent64_out, P, S, t, K, d);
    const int64_t rb = (N + 7) / 8;                       // 8 rows per 256-thread CTA
    k_residual<<<dim3(unsigned(rb < 4096 ? rb : 4096), unsigned(P)), 256, 0, st>>>(
        b.rows, b.cent, b.assign, assign_out, iters_out, b.st, P, N, S, t, K, d, update_rows ? 1 : 0);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

}  // namespace qvg
