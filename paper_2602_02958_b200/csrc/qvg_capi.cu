// qvg_capi.cu — the extern "C" boundary declared in include/qvg.h.
//
// Validation mirrors the reference's raises (Q/types.py:88-102,202-214,
// Q/quant.py:139-145, Q/clustering.py:126-129) as integer codes; the work is
// stream-ordered and asynchronous; the caller owns every buffer.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "qvg_common.cuh"
#include "qvg_internal.h"

namespace qvg {

static thread_local char g_err[512] = "";

int set_err(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

static int cuda_check(const char *where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(QVG_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
    return QVG_OK;
}

// ---- numpy pairwise-recursion plans ---------------------------------------
struct Plan {
    std::vector<int64_t> off;
    std::vector<int32_t> len;
    std::vector<int32_t> l, r, hstart;
    int heights = 0;
};

namespace {
struct Node { int32_t a, b, h; };
// returns encoded id: >= 0 leaf index, < 0 -(internal index + 1); height via *h
int32_t plan_rec(int64_t off, int64_t n, Plan &pl, std::vector<Node> &in, int *h) {
    if (n <= 128) {
        pl.off.push_back(off);
        pl.len.push_back(int32_t(n));
        *h = 0;
        return int32_t(pl.off.size() - 1);
    }
    int64_t hh = n / 2;
    hh -= hh % 8;
    int ha, hb;
    int32_t a = plan_rec(off, hh, pl, in, &ha);
    int32_t b = plan_rec(off + hh, n - hh, pl, in, &hb);
    in.push_back(Node{a, b, 1 + std::max(ha, hb)});
    *h = in.back().h;
    return -int32_t(in.size());
}
}  // namespace

static void build_plan(int64_t n, Plan &pl) {
    std::vector<Node> in;
    int h;
    plan_rec(0, n, pl, in, &h);
    const int32_t L = int32_t(pl.off.size());
    std::vector<int32_t> order(in.size());
    for (size_t i = 0; i < in.size(); i++) order[i] = int32_t(i);
    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return in[x].h < in[y].h; });
    std::vector<int32_t> rank(in.size());
    for (size_t i = 0; i < order.size(); i++) rank[order[i]] = int32_t(i);
    auto remap = [&](int32_t id) { return id >= 0 ? id : L + rank[-id - 1]; };
    pl.heights = in.empty() ? 0 : in[order.back()].h;
    pl.hstart.assign(pl.heights + 1, 0);
    for (size_t i = 0; i < order.size(); i++) {
        const Node &nd = in[order[i]];
        pl.l.push_back(remap(nd.a));
        pl.r.push_back(remap(nd.b));
    }
    // hstart[h-1] = first internal (sorted) index of height h; hstart[H] = count
    int cur = 0;
    for (int hgt = 1; hgt <= pl.heights; hgt++) {
        pl.hstart[hgt - 1] = cur;
        while (cur < int(order.size()) && in[order[cur]].h == hgt) cur++;
    }
    pl.hstart[pl.heights] = cur;
}

static int64_t n_leaves(int64_t n) {
    if (n <= 128) return 1;
    int64_t h = n / 2;
    h -= h % 8;
    return n_leaves(h) + n_leaves(n - h);
}

// ---- workspace carving ------------------------------------------------------
struct Carver {
    char *base;
    size_t off = 0;
    template <typename T>
    T *take(int64_t count) {
        off = (off + 255) & ~size_t(255);
        T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += size_t(count) * sizeof(T);
        return p;
    }
};

// kmeans scratch (+ rows/cent when own_rows)
static void carve_kmeans(Carver &c, int64_t P, int64_t N, int d, int K, bool own_rows,
                         bool own_cent, KMeansBuffers &b) {
    const int64_t Lo = n_leaves(N * d), Lp = n_leaves(N);
    if (own_rows) b.rows = c.take<double>(P * N * d);
    if (own_cent) b.cent = c.take<double>(P * K * d);
    b.d2 = c.take<double>(P * N);
    b.nodes = c.take<double>(P * (2 * Lo - 1));
    b.assign = c.take<int32_t>(P * N);
    b.counts = c.take<int32_t>(P * K);
    b.offsets = c.take<int32_t>(P * (K + 1));
    b.members = c.take<int32_t>(P * N);
    b.st = c.take<PlaneState>(P);
    b.pk_off = c.take<int64_t>(Lp);
    b.pk_len = c.take<int32_t>(Lp);
    b.pk_leaves = int(Lp);
    b.pk_l = c.take<int32_t>(Lp);
    b.pk_r = c.take<int32_t>(Lp);
    b.pk_hstart = c.take<int32_t>(80);
    b.ob_off = c.take<int64_t>(Lo);
    b.ob_len = c.take<int32_t>(Lo);
    b.nd_l = c.take<int32_t>(Lo);
    b.nd_r = c.take<int32_t>(Lo);
    b.h_start = c.take<int32_t>(80);
    b.ob_leaves = int(Lo);
    if (assign_tc_ok(d, K)) {
        b.rsplit = c.take<uint16_t>(int64_t(assign_tc_split_elems(P, N)));
        b.xnorm = c.take<float>(P * N);
        b.c2 = c.take<double>(P * K);
        b.recheck = c.take<int32_t>(P * N);
        b.n_recheck = c.take<int32_t>(8);
        b.rows32 = c.take<float>(P * N * d);
        b.rows32_ok = c.take<int32_t>(P);
    }
}

static int upload_plans(KMeansBuffers &b, int64_t N, int d, cudaStream_t st) {
    Plan po, pp;
    build_plan(N * d, po);
    build_plan(N, pp);
    if (po.heights > 78) return set_err(QVG_ERR_UNSUPPORTED, "pairwise tree too deep");
    b.ob_heights = po.heights;
    if (pp.heights > 78) return set_err(QVG_ERR_UNSUPPORTED, "pairwise tree too deep");
    b.pk_heights = pp.heights;
    if (!pp.l.empty()) {
        cudaMemcpyAsync(b.pk_l, pp.l.data(), pp.l.size() * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(b.pk_r, pp.r.data(), pp.r.size() * 4, cudaMemcpyHostToDevice, st);
    }
    cudaMemcpyAsync(b.pk_hstart, pp.hstart.data(), pp.hstart.size() * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(b.pk_off, pp.off.data(), pp.off.size() * 8, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(b.pk_len, pp.len.data(), pp.len.size() * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(b.ob_off, po.off.data(), po.off.size() * 8, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(b.ob_len, po.len.data(), po.len.size() * 4, cudaMemcpyHostToDevice, st);
    if (!po.l.empty()) {
        cudaMemcpyAsync(b.nd_l, po.l.data(), po.l.size() * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(b.nd_r, po.r.data(), po.r.size() * 4, cudaMemcpyHostToDevice, st);
    }
    cudaMemcpyAsync(b.h_start, po.hstart.data(), po.hstart.size() * 4, cudaMemcpyHostToDevice, st);
    return cuda_check("plan upload");
}

// ---- validation -------------------------------------------------------------
static int check_config(const qvg_config *cfg, bool need_kmeans) {
    if (!cfg) return set_err(QVG_ERR_BAD_CONFIG, "config is NULL");
    if (cfg->bits != 2 && cfg->bits != 4 && cfg->bits != 8)
        return set_err(QVG_ERR_BAD_CONFIG, "bits must be one of (2, 4, 8), got %d", cfg->bits);
    if (cfg->group_size < 1) return set_err(QVG_ERR_BAD_CONFIG, "group_size must be >= 1");
    if (cfg->stages < 0) return set_err(QVG_ERR_BAD_CONFIG, "stages must be >= 0");
    if (cfg->centroids < 1 || cfg->centroids > kMaxK)
        return set_err(QVG_ERR_BAD_CONFIG, "centroids must be in [1, 256]");
    if (need_kmeans && cfg->kmeans_max_iters < 1)
        return set_err(QVG_ERR_BAD_CONFIG, "kmeans_max_iters must be >= 1");
    if (need_kmeans && !(cfg->kmeans_tol >= 0)) return set_err(QVG_ERR_BAD_CONFIG, "kmeans_tol must be >= 0");
    return QVG_OK;
}

static int check_plane(int64_t P, int64_t N, int d, const qvg_config *cfg) {
    if (P < 0) return set_err(QVG_ERR_BAD_CONFIG, "n_planes must be >= 0");
    if (N < 1 || d < 1) return set_err(QVG_ERR_EMPTY_PLANE, "plane has no data (%lld x %d)", (long long)N, d);
    if (d % cfg->group_size != 0)
        return set_err(QVG_ERR_DIMENSION_MISMATCH, "group_size %d does not divide head_dim %d", cfg->group_size, d);
    return QVG_OK;
}

}  // namespace qvg

using namespace qvg;

extern "C" {

int qvg_abi_version(void) { return QVG_ABI_VERSION; }
const char *qvg_last_error(void) { return g_err; }

size_t qvg_compress_workspace_size(int64_t P, int64_t N, int32_t d, const qvg_config *cfg) {
    if (!cfg || P < 1 || N < 1 || d < 1) return 0;
    Carver c{nullptr};
    KMeansBuffers b{};
    carve_kmeans(c, P, N, d, cfg->centroids, true, true, b);
    return c.off + 256;
}

int qvg_compress(const void *x, int32_t x_dtype, int64_t P, int64_t N, int32_t d,
                 const qvg_config *cfg, const double *pp_draws, const double *warm_init,
                 uint8_t *payload, uint8_t *scales, uint16_t *centroids, uint8_t *assign,
                 double *centroids_f64, int32_t *iters, int32_t *status, void *workspace,
                 size_t workspace_bytes, void *stream) {
    int rc;
    if ((rc = check_config(cfg, true)) || (rc = check_plane(P, N, d, cfg))) return rc;
    if (x_dtype != QVG_DTYPE_F32 && x_dtype != QVG_DTYPE_BF16)
        return set_err(QVG_ERR_BAD_CONFIG, "x_dtype must be f32 or bf16");
    if (P == 0) return QVG_OK;
    const int S = cfg->stages, K = cfg->centroids;
    if (S > 0 && d > 128) return set_err(QVG_ERR_UNSUPPORTED, "k-means kernels support head_dim <= 128");
    if (S > 0 && !pp_draws && !warm_init) return set_err(QVG_ERR_BAD_CONFIG, "need pp_draws or warm_init");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (S > 0) {
        size_t need = qvg_compress_workspace_size(P, N, d, cfg);
        if (!workspace || workspace_bytes < need)
            return set_err(QVG_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", need, workspace_bytes);
        char *base = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
        Carver c{base};
        KMeansBuffers b{};
        carve_kmeans(c, P, N, d, K, true, true, b);
        if ((rc = upload_plans(b, N, d, st))) return rc;
        if ((rc = launch_widen(x, x_dtype == QVG_DTYPE_BF16, b.rows, P * N * d, status, st)))
            return set_err(rc, "widen launch failed");
        for (int t = 0; t < S; t++) {
            bool warm = warm_init != nullptr;
            if (warm)
                cudaMemcpy2DAsync(b.cent, size_t(K) * d * 8, warm_init + int64_t(t) * K * d,
                                  size_t(S) * K * d * 8, size_t(K) * d * 8, size_t(P),
                                  cudaMemcpyDeviceToDevice, st);
            b.src16 = (t == 0 && x_dtype == QVG_DTYPE_BF16) ? static_cast<const uint16_t *>(x) : nullptr;
            const bool r2 = t == 1 && x_dtype == QVG_DTYPE_BF16;
            b.res_x16 = r2 ? static_cast<const uint16_t *>(x) : nullptr;
            b.res_c1 = r2 ? centroids : nullptr;
            b.res_a1 = r2 ? assign : nullptr;
            b.res_c1_stride = int64_t(S) * K * d;
            b.res_a1_stride = int64_t(S) * N;
            rc = run_kmeans_stage(b, P, N, d, K, cfg->kmeans_max_iters, cfg->kmeans_tol,
                                  warm ? nullptr : pp_draws + int64_t(t) * K, int64_t(S) * K, warm, st);
            if (rc) return set_err(rc, "k-means stage %d: %s", t, cudaGetErrorString(cudaGetLastError()));
            rc = finalize_stage(b, P, N, d, K, S, t, centroids, centroids_f64, assign, iters, st, t + 1 < S);
            if (rc) return set_err(rc, "stage finalize failed");
        }
    }
    rc = launch_quantize(x, x_dtype, P, N, d, cfg->bits, cfg->group_size, S, K, centroids, assign,
                         payload, scales, status, st);
    if (rc) return set_err(rc, "quantize launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return QVG_OK;
}

int qvg_quantize(const void *x, int32_t x_dtype, int64_t P, int64_t N, int32_t d,
                 const qvg_config *cfg, const uint16_t *centroids, const uint8_t *assign,
                 uint8_t *payload, uint8_t *scales, int32_t *status, void *stream) {
    int rc;
    if ((rc = check_config(cfg, false)) || (rc = check_plane(P, N, d, cfg))) return rc;
    if (x_dtype != QVG_DTYPE_F32 && x_dtype != QVG_DTYPE_BF16 && x_dtype != QVG_DTYPE_F64)
        return set_err(QVG_ERR_BAD_CONFIG, "x_dtype must be f32, bf16 or f64");
    if (P == 0) return QVG_OK;
    if (cfg->stages > 0 && (!centroids || !assign)) return set_err(QVG_ERR_BAD_CONFIG, "stage metadata is NULL");
    rc = launch_quantize(x, x_dtype, P, N, d, cfg->bits, cfg->group_size, cfg->stages, cfg->centroids,
                         centroids, assign, payload, scales, status, static_cast<cudaStream_t>(stream));
    return rc ? set_err(rc, "quantize launch failed: %s", cudaGetErrorString(cudaGetLastError())) : QVG_OK;
}

int qvg_dequantize(const uint8_t *payload, const uint8_t *scales, const uint16_t *centroids,
                   const uint8_t *assign, int64_t P, int64_t N, int32_t d, const qvg_config *cfg,
                   void *out, int32_t out_dtype, int32_t *status, void *stream) {
    int rc;
    if ((rc = check_config(cfg, false)) || (rc = check_plane(P, N, d, cfg))) return rc;
    if (out_dtype != QVG_DTYPE_F32 && out_dtype != QVG_DTYPE_BF16)
        return set_err(QVG_ERR_BAD_CONFIG, "out_dtype must be f32 or bf16");
    if (P == 0) return QVG_OK;
    if (cfg->stages > 0 && (!centroids || !assign)) return set_err(QVG_ERR_BAD_CONFIG, "stage metadata is NULL");
    rc = launch_dequantize(payload, scales, centroids, assign, P, N, d, cfg->bits, cfg->group_size,
                           cfg->stages, cfg->centroids, out, out_dtype, status,
                           static_cast<cudaStream_t>(stream));
    return rc ? set_err(rc, "dequantize launch failed: %s", cudaGetErrorString(cudaGetLastError())) : QVG_OK;
}

int qvg_pack_codes(const int8_t *q, int64_t n, int32_t bits, uint8_t *out, int32_t *status, void *stream) {
    if (bits != 2 && bits != 4 && bits != 8) return set_err(QVG_ERR_BAD_CONFIG, "bits must be 2, 4 or 8");
    if (n < 0) return set_err(QVG_ERR_BAD_CONFIG, "n must be >= 0");
    int rc = launch_pack(q, n, bits, out, status, static_cast<cudaStream_t>(stream));
    return rc ? set_err(rc, "pack launch failed") : QVG_OK;
}

int qvg_unpack_codes(const uint8_t *in, int64_t n, int32_t bits, int8_t *out, void *stream) {
    if (bits != 2 && bits != 4 && bits != 8) return set_err(QVG_ERR_BAD_CONFIG, "bits must be 2, 4 or 8");
    if (n < 0) return set_err(QVG_ERR_BAD_CONFIG, "n must be >= 0");
    int rc = launch_unpack(in, n, bits, out, static_cast<cudaStream_t>(stream));
    return rc ? set_err(rc, "unpack launch failed") : QVG_OK;
}

// ---- clustering / smoothing entry points ------------------------------------
size_t qvg_kmeans_workspace_size(int64_t P, int64_t N, int32_t d, int32_t K) {
    if (P < 1 || N < 1 || d < 1 || K < 1) return 0;
    Carver c{nullptr};
    KMeansBuffers b{};
    carve_kmeans(c, P, N, d, K, false, false, b);
    return c.off + 256;
}

static int kmeans_setup(const double *rows, int64_t P, int64_t N, int32_t d, int32_t K,
                        const double *init, double *cent, void *workspace, size_t wbytes,
                        cudaStream_t st, KMeansBuffers &b) {
    if (N < 1) return set_err(QVG_ERR_EMPTY_INPUT, "need at least one row");
    if (K < 1 || K > kMaxK) return set_err(QVG_ERR_BAD_CONFIG, "k must be in [1, 256] (one-byte assignments)");
    if (d < 1 || d > 128) return set_err(QVG_ERR_UNSUPPORTED, "k-means kernels support 1 <= d <= 128");
    size_t need = qvg_kmeans_workspace_size(P, N, d, K);
    if (!workspace || wbytes < need) return set_err(QVG_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", need, wbytes);
    char *base = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    Carver c{base};
    carve_kmeans(c, P, N, d, K, false, false, b);
    b.rows = const_cast<double *>(rows);
    b.cent = cent;
    int rc;
    if ((rc = upload_plans(b, N, d, st))) return rc;
    if (init && init != cent) cudaMemcpyAsync(cent, init, size_t(P * K * d) * 8, cudaMemcpyDeviceToDevice, st);
    return cuda_check("k-means setup");
}

int qvg_kmeans(const double *rows, int64_t P, int64_t N, int32_t d, int32_t K, int32_t max_iters,
               double tol, const double *draws, const double *init, double *centroids,
               uint8_t *assign, double *objective, int32_t *iters, void *workspace,
               size_t workspace_bytes, void *stream) {
    if (P == 0) return QVG_OK;
    if (max_iters < 1) return set_err(QVG_ERR_BAD_CONFIG, "max_iters must be >= 1");
    if (!(tol >= 0)) return set_err(QVG_ERR_BAD_CONFIG, "tol must be >= 0");
    if (!draws && !init) return set_err(QVG_ERR_BAD_CONFIG, "need draws or init");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    KMeansBuffers b{};
    int rc = kmeans_setup(rows, P, N, d, K, init, centroids, workspace, workspace_bytes, st, b);
    if (rc) return rc;
    if (run_kmeans_stage(b, P, N, d, K, max_iters, tol, draws, K, init != nullptr, st) ||
        kmeans_outputs(b, P, N, d, K, assign, objective, iters, st))
        return set_err(QVG_ERR_CUDA, "k-means launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return QVG_OK;
}

int qvg_kmeanspp(const double *rows, int64_t P, int64_t N, int32_t d, int32_t K,
                 const double *draws, double *centroids, void *workspace, size_t workspace_bytes,
                 void *stream) {
    if (P == 0) return QVG_OK;
    if (N < 1) return set_err(QVG_ERR_EMPTY_INPUT, "need at least one row");
    if (K < 1 || K > kMaxK) return set_err(QVG_ERR_BAD_CONFIG, "k must be >= 1");
    if (d < 1 || d > 128) return set_err(QVG_ERR_UNSUPPORTED, "k-means kernels support 1 <= d <= 128");
    size_t need = qvg_kmeans_workspace_size(P, N, d, K);
    if (!workspace || workspace_bytes < need) return set_err(QVG_ERR_WORKSPACE, "workspace needs %zu bytes", need);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    char *base = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    Carver c{base};
    KMeansBuffers b{};
    carve_kmeans(c, P, N, d, K, false, false, b);
    b.rows = const_cast<double *>(rows);
    b.cent = centroids;
    int rc;
    if ((rc = upload_plans(b, N, d, st))) return rc;
    rc = run_kmeanspp(b, P, N, d, K, draws, K, st);
    return rc ? set_err(rc, "k-means++ launch failed") : QVG_OK;
}

int qvg_assign(const double *rows, const double *centroids, int64_t P, int64_t N, int32_t d,
               int32_t K, int32_t *assign, void *stream) {
    if (P == 0) return QVG_OK;
    if (N < 1) return set_err(QVG_ERR_EMPTY_INPUT, "need at least one row");
    if (d < 1 || d > 128) return set_err(QVG_ERR_UNSUPPORTED, "k-means kernels support 1 <= d <= 128");
    if (K < 1 || K > kMaxK) return set_err(QVG_ERR_BAD_CONFIG, "k must be in [1, 256]");
    int rc = run_assign(rows, centroids, assign, P, N, d, K, static_cast<cudaStream_t>(stream));
    return rc ? set_err(rc, "assign launch failed") : QVG_OK;
}

int qvg_lloyd_step(const double *rows, double *centroids, int64_t P, int64_t N, int32_t d,
                   int32_t K, uint8_t *assign, double *objective, void *workspace,
                   size_t workspace_bytes, void *stream) {
    if (P == 0) return QVG_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    KMeansBuffers b{};
    int rc = kmeans_setup(rows, P, N, d, K, nullptr, centroids, workspace, workspace_bytes, st, b);
    if (rc) return rc;
    rc = lloyd_once(b, P, N, d, K, assign, objective, st);
    return rc ? set_err(rc, "lloyd step failed: %s", cudaGetErrorString(cudaGetLastError())) : QVG_OK;
}

size_t qvg_sa_smoothing_workspace_size(int64_t P, int64_t N, int32_t d, int32_t K) {
    size_t w = qvg_kmeans_workspace_size(P, N, d, K);
    return w ? w + size_t(P) * K * d * 8 + 512 : 0;
}

int qvg_sa_smoothing(const double *x, int64_t P, int64_t N, int32_t d, int32_t K,
                     int32_t max_iters, double tol, const double *draws, const double *warm_init,
                     double *residual, uint16_t *centroids, uint8_t *assign, double *centroids_f64,
                     int32_t *iters, void *workspace, size_t workspace_bytes, void *stream) {
    if (P == 0) return QVG_OK;
    if (max_iters < 1) return set_err(QVG_ERR_BAD_CONFIG, "max_iters must be >= 1");
    if (!(tol >= 0)) return set_err(QVG_ERR_BAD_CONFIG, "tol must be >= 0");
    if (!draws && !warm_init) return set_err(QVG_ERR_BAD_CONFIG, "need draws or warm_init");
    if (N < 1) return set_err(QVG_ERR_EMPTY_INPUT, "need at least one row");
    if (K < 1 || K > kMaxK) return set_err(QVG_ERR_BAD_CONFIG, "k must be in [1, 256] (one-byte assignments)");
    if (d < 1 || d > 128) return set_err(QVG_ERR_UNSUPPORTED, "k-means kernels support 1 <= d <= 128");
    size_t need = qvg_sa_smoothing_workspace_size(P, N, d, K);
    if (!workspace || workspace_bytes < need) return set_err(QVG_ERR_WORKSPACE, "workspace needs %zu bytes", need);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double *cent = reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    char *rest = reinterpret_cast<char *>(cent + P * K * d);
    size_t rest_bytes = workspace_bytes - size_t(rest - static_cast<char *>(workspace));
    cudaMemcpyAsync(residual, x, size_t(P * N * d) * 8, cudaMemcpyDeviceToDevice, st);
    KMeansBuffers b{};
    int rc = kmeans_setup(residual, P, N, d, K, warm_init, cent, rest, rest_bytes, st, b);
    if (rc) return rc;
    if (run_kmeans_stage(b, P, N, d, K, max_iters, tol, draws, K, warm_init != nullptr, st) ||
        finalize_stage(b, P, N, d, K, 1, 0, centroids, centroids_f64, assign, iters, st))
        return set_err(QVG_ERR_CUDA, "smoothing launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return QVG_OK;
}

int qvg_add_back(const double *residual, const uint16_t *centroids, const uint8_t *assign,
                 int64_t P, int64_t N, int32_t d, int32_t K, double *out, void *stream) {
    if (P == 0) return QVG_OK;
    int rc = run_add_back(residual, centroids, assign, P, N, d, K, out, static_cast<cudaStream_t>(stream));
    return rc ? set_err(rc, "add_back launch failed") : QVG_OK;
}

size_t qvg_attention_workspace_size(int64_t nq, int64_t n_cache, int64_t n_cur, int32_t H,
                                    int32_t d, const qvg_config *cfg) {
    return attention_workspace_size(nq, n_cache, n_cur, H, d, cfg);
}

int qvg_attention(const uint16_t *q, const uint8_t *payload, const uint8_t *scales,
                  const uint16_t *centroids, const uint8_t *assign, const uint16_t *kv_bf16,
                  const uint16_t *k_cur, const uint16_t *v_cur, int64_t nq, int64_t n_cache,
                  int64_t n_cur, int32_t H, int32_t d, const qvg_config *cfg, float softmax_scale,
                  uint16_t *out, void *workspace, size_t workspace_bytes, int32_t *status, void *stream) {
    int rc;
    if ((rc = check_config(cfg, false))) return rc;
    if (nq < 0 || n_cache < 0 || n_cur < 0 || H < 1) return set_err(QVG_ERR_BAD_CONFIG, "bad attention sizes");
    if (n_cache + n_cur < 1) return set_err(QVG_ERR_EMPTY_INPUT, "no keys");
    if (nq == 0) return QVG_OK;
    if (n_cache > 0 && d % cfg->group_size != 0)
        return set_err(QVG_ERR_DIMENSION_MISMATCH, "group_size %d does not divide head_dim %d", cfg->group_size, d);
    return run_attention(q, payload, scales, centroids, assign, kv_bf16, k_cur, v_cur, nq, n_cache,
                         n_cur, H, d, cfg, softmax_scale, out, workspace, workspace_bytes, status,
                         static_cast<cudaStream_t>(stream));
}

int qvg_attention_rope(const uint16_t *q, const uint8_t *payload, const uint8_t *scales,
                       const uint16_t *centroids, const uint8_t *assign, const uint16_t *kv_bf16,
                       const uint16_t *k_cur, const uint16_t *v_cur, int64_t nq, int64_t n_cache,
                       int64_t n_cur, int32_t H, int32_t d, const qvg_config *cfg, float softmax_scale,
                       const float *rope_cos, const float *rope_sin, int32_t rope_mode, uint16_t *out,
                       void *workspace, size_t workspace_bytes, int32_t *status, void *stream) {
    int rc;
    if ((rc = check_config(cfg, false))) return rc;
    if (nq < 0 || n_cache < 0 || n_cur < 0 || H < 1) return set_err(QVG_ERR_BAD_CONFIG, "bad attention sizes");
    if (n_cache + n_cur < 1) return set_err(QVG_ERR_EMPTY_INPUT, "no keys");
    if (nq == 0) return QVG_OK;
    if (n_cache > 0 && payload && d % cfg->group_size != 0)
        return set_err(QVG_ERR_DIMENSION_MISMATCH, "group_size %d does not divide head_dim %d", cfg->group_size, d);
    return run_attention(q, payload, scales, centroids, assign, kv_bf16, k_cur, v_cur, nq, n_cache,
                         n_cur, H, d, cfg, softmax_scale, out, workspace, workspace_bytes, status,
                         static_cast<cudaStream_t>(stream), rope_cos, rope_sin, rope_mode);
}

}  // extern "C"
