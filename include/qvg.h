/*
 * qvg.h — C ABI of libqvg_b200.so, the sm_100a implementation of the QVG
 * KV-cache hot path (arXiv 2602.02958; reference package `qvgcodec`).
 *
 * The reference has no native boundary of its own: its hot path is the
 * Python API in /root/reference/pkg/src/qvgcodec, and its SPEC describes
 * (but never ships) a "flat procedural ABI … all errors as integer codes
 * with a last-error message accessor", reentrant, buffers + plain-scalar
 * config.  This header is that ABI, generalised from one
 * host plane to P device-resident planes.  Each entry point names the
 * reference function it replaces.
 *
 * Conventions
 *  - Every pointer argument is a DEVICE pointer unless marked (host).
 *    The library never allocates: the caller owns every buffer, sized by
 *    the layouts below and by qvg_*_workspace_size().
 *  - `stream` is a cudaStream_t (void* here to keep CUDA types out of the
 *    ABI).  Calls are stream-ordered and asynchronous; argument errors are
 *    returned immediately, data-dependent errors (NaN/Inf input) are
 *    OR-ed into the device word `*status` (QVG_STATUS_* bits).
 *  - Return value: QVG_OK or one QVG_ERR_* code; qvg_last_error() gives a
 *    thread-local message.  No global mutable state: calls are reentrant.
 *
 * Plane layouts (plane = one (layer, head, K|V) matrix of N tokens x d;
 * P planes are stored back to back, plane-major):
 *   x            [P][N][d]       f32 or bf16 (QVG_DTYPE_*)
 *   payload      [P][PB]         u8, PB = ceil(N*d*bits/8); element i of a
 *                                plane -> byte i*bits/8, bit (i*bits)%8,
 *                                two's complement (Q/quant.py:78-100)
 *   scales       [P][N*d/B]      u8 E4M3 codes, row-major group order
 *   centroids    [P][S][K][d]    u16 = bf16 bit patterns (StageMeta.centroids)
 *   assign       [P][S][N]       u8 (StageMeta.assignments)
 *   pp_draws     [P][S][K]       f64, Generator(Philox(stage_seed)).random(K)
 *                                for each plane's chunk (Q/clustering.py:32-63)
 */
#ifndef QVG_B200_H
#define QVG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QVG_ABI_VERSION 2

#if defined(__GNUC__)
#define QVG_API __attribute__((visibility("default")))
#else
#define QVG_API
#endif

/* Error codes; the Python layer maps each to the reference exception class
 * (Q/errors.py:8-73). */
enum {
    QVG_OK = 0,
    QVG_ERR_DIMENSION_MISMATCH = 1, /* DimensionMismatch  (Q/errors.py:12)  */
    QVG_ERR_NONFINITE_INPUT = 2,    /* NonFiniteInput     (Q/errors.py:16)  */
    QVG_ERR_EMPTY_PLANE = 3,        /* EmptyPlane         (Q/errors.py:20)  */
    QVG_ERR_EMPTY_INPUT = 4,        /* EmptyInput         (Q/errors.py:24)  */
    QVG_ERR_BAD_CONFIG = 5,         /* ValueError         (Q/types.py:88-102) */
    QVG_ERR_RANGE_OVERFLOW = 6,     /* RangeOverflow      (Q/errors.py:36)  */
    QVG_ERR_TRUNCATED = 7,          /* Truncated          (Q/errors.py:40)  */
    QVG_ERR_NAN_PATTERN = 8,        /* NaNPattern         (Q/errors.py:32)  */
    QVG_ERR_CUDA = 9,               /* CUDA runtime failure                  */
    QVG_ERR_WORKSPACE = 10,         /* workspace too small / misaligned      */
    QVG_ERR_UNSUPPORTED = 11        /* shape outside the compiled kernels    */
};

/* Bits OR-ed into *status by the kernels. */
enum {
    QVG_STATUS_NONFINITE = 1,   /* NaN/Inf seen in x                         */
    QVG_STATUS_NAN_SCALE = 2,   /* an E4M3 NaN pattern (0x7F/0xFF) in scales */
    QVG_STATUS_BAD_ASSIGN = 4,  /* assignment >= K in a decode input          */
    QVG_STATUS_RANGE = 8        /* code outside the symmetric b-bit range     */
};

enum { QVG_DTYPE_F32 = 0, QVG_DTYPE_BF16 = 1, QVG_DTYPE_F64 = 2 /* qvg_quantize only */ };

/* QuantConfig (Q/types.py:76-107), POD form. */
typedef struct {
    int32_t bits;             /* 2, 4 or 8                                 */
    int32_t group_size;       /* B, divides d                              */
    int32_t stages;           /* S >= 0                                    */
    int32_t centroids;        /* K in [1, 256]                             */
    int32_t kmeans_max_iters; /* >= 1                                      */
    int32_t reserved;
    double kmeans_tol;        /* >= 0                                      */
    uint64_t seed;            /* stage seeds are derived on the host       */
} qvg_config;

QVG_API int qvg_abi_version(void);
QVG_API const char *qvg_last_error(void);

/* Replaces prq_compress(plane, config, warm_init) (Q/prq.py:58-80) for P
 * planes: validate (Q/types.py:202-214), S stages of Semantic-Aware
 * Smoothing (k-means++ / warm start, Lloyd iterations, bf16 centroid
 * subtraction; Q/smoothing.py:23-41, Q/clustering.py:47-160), then the
 * per-group quantizer (Q/quant.py:134-148).
 *   pp_draws       [P][S][K] f64 (ignored where warm_init is given)
 *   warm_init      [P][S][K][d] f64 or NULL (Q/prq.py:61-71)
 *   centroids_f64  [P][S][K][d] f64 or NULL: the unrounded k-means result,
 *                  the warm start for the next chunk (Q/clustering.py:163)
 *   iters          [P][S] i32 or NULL: Lloyd iterations used per stage
 * Bit-exact with the reference (assignments, centroids, payload, scales). */
QVG_API size_t qvg_compress_workspace_size(int64_t n_planes, int64_t n_tokens, int32_t head_dim,
                                   const qvg_config *cfg /* host */);
QVG_API int qvg_compress(const void *x, int32_t x_dtype, int64_t n_planes, int64_t n_tokens,
                 int32_t head_dim, const qvg_config *cfg /* host */, const double *pp_draws,
                 const double *warm_init, uint8_t *payload, uint8_t *scales, uint16_t *centroids,
                 uint8_t *assign, double *centroids_f64, int32_t *iters, int32_t *status,
                 void *workspace, size_t workspace_bytes, void *stream);

/* Replaces quantize_matrix(final_residual(...)) given the stage metadata
 * (Q/smoothing.py:40 residual chain + Q/quant.py:40-55,78-100,134-148):
 * the quantize half of the codec, with centroids/assignments already
 * known (S = 0 is plain RTN quantize_plane, Q/quant.py:124).  x_dtype may
 * also be QVG_DTYPE_F64 (quantize_matrix on a float64 matrix, S = 0). */
QVG_API int qvg_quantize(const void *x, int32_t x_dtype, int64_t n_planes, int64_t n_tokens,
                 int32_t head_dim, const qvg_config *cfg /* host */, const uint16_t *centroids,
                 const uint8_t *assign, uint8_t *payload, uint8_t *scales, int32_t *status,
                 void *stream);

/* Replaces prq_decompress_onepass(chunk) (Q/prq.py:113-132, bit-identical
 * to prq_decompress :92-101) and, for S = 0, dequantize_plane
 * (Q/quant.py:151-168).  out [P][N][d]: QVG_DTYPE_F32 is the reference's
 * float32 bit for bit; QVG_DTYPE_BF16 is that float32 rounded to bf16. */
QVG_API int qvg_dequantize(const uint8_t *payload, const uint8_t *scales, const uint16_t *centroids,
                   const uint8_t *assign, int64_t n_planes, int64_t n_tokens, int32_t head_dim,
                   const qvg_config *cfg /* host */, void *out, int32_t out_dtype,
                   int32_t *status, void *stream);

/* pack_payload(q, bits) (Q/quant.py:78-100): n int8 codes -> ceil(n*bits/8)
 * bytes; a code outside +-(2^(b-1)-1) sets QVG_STATUS_RANGE (RangeOverflow). */
QVG_API int qvg_pack_codes(const int8_t *q, int64_t n, int32_t bits, uint8_t *out, int32_t *status,
                           void *stream);
/* unpack_payload(data, count, bits) (Q/quant.py:103-116): sign-extended int8. */
QVG_API int qvg_unpack_codes(const uint8_t *in, int64_t n, int32_t bits, int8_t *out, void *stream);

/* ---- clustering / smoothing (Q/clustering.py, Q/smoothing.py) ----------
 * rows are float64 [P][N][d] with 1 <= d <= 128; one independent problem per
 * plane.  draws [P][K] are one plane's k-means++ rng.random() draws. */
QVG_API size_t qvg_kmeans_workspace_size(int64_t n_planes, int64_t n_rows, int32_t d, int32_t k);

/* kmeans_pp_init(rows, k, seed) (Q/clustering.py:47-63): centroids [P][K][d]. */
QVG_API int qvg_kmeanspp(const double *rows, int64_t n_planes, int64_t n_rows, int32_t d, int32_t k,
                 const double *draws, double *centroids, void *workspace,
                 size_t workspace_bytes, void *stream);

/* _assign(rows, centroids) (Q/clustering.py:66-71): assign [P][N] i32. */
QVG_API int qvg_assign(const double *rows, const double *centroids, int64_t n_planes, int64_t n_rows,
               int32_t d, int32_t k, int32_t *assign, void *stream);

/* lloyd_step(rows, centroids) (Q/clustering.py:74-107): centroids updated
 * in place; assign [P][N] u8; objective [P] f64. */
QVG_API int qvg_lloyd_step(const double *rows, double *centroids, int64_t n_planes, int64_t n_rows,
                   int32_t d, int32_t k, uint8_t *assign, double *objective, void *workspace,
                   size_t workspace_bytes, void *stream);

/* kmeans(rows, k, max_iters, tol, seed, init) (Q/clustering.py:110-160):
 * init [P][K][d] or NULL (then draws); outputs centroids [P][K][d] f64,
 * assign [P][N] u8, objective [P] f64, iters [P] i32 (each may be NULL
 * except centroids). */
QVG_API int qvg_kmeans(const double *rows, int64_t n_planes, int64_t n_rows, int32_t d, int32_t k,
               int32_t max_iters, double tol, const double *draws, const double *init,
               double *centroids, uint8_t *assign, double *objective, int32_t *iters,
               void *workspace, size_t workspace_bytes, void *stream);

/* sa_smoothing(x, k, seed, warm_init, max_iters, tol) (Q/smoothing.py:23-41):
 * residual [P][N][d] f64 = x - C_bf16[pi]; centroids [P][K][d] bf16 bits,
 * assign [P][N] u8, centroids_f64 / iters optional. */
QVG_API size_t qvg_sa_smoothing_workspace_size(int64_t n_planes, int64_t n_rows, int32_t d, int32_t k);
QVG_API int qvg_sa_smoothing(const double *x, int64_t n_planes, int64_t n_rows, int32_t d, int32_t k,
                     int32_t max_iters, double tol, const double *draws,
                     const double *warm_init, double *residual, uint16_t *centroids,
                     uint8_t *assign, double *centroids_f64, int32_t *iters, void *workspace,
                     size_t workspace_bytes, void *stream);

/* add_back(residual, meta) (Q/smoothing.py:44-54): out = residual + C[pi]. */
QVG_API int qvg_add_back(const double *residual, const uint16_t *centroids, const uint8_t *assign,
                 int64_t n_planes, int64_t n_rows, int32_t d, int32_t k, double *out,
                 void *stream);

/* Attention over the quantized cache (no reference symbol: SURVEY §8(a)
 * A24; the paper's fused dequant-attention).
 * For each head h: O = softmax(q K^T * scale) V over the keys
 * [Khat_cache(h) ; k_cur(h)] and values [Vhat_cache(h) ; v_cur(h)], where
 * Khat/Vhat are the prq_decompress_onepass reconstructions of the head's
 * K and V planes (plane index 2h and 2h+1 in the cache buffers, i.e. the
 * cache holds P = 2H planes of n_cache tokens).  No mask: the current
 * chunk attends to all cached tokens and to itself.
 *   q       [nq][H][d] bf16      k_cur, v_cur [n_cur][H][d] bf16
 *   out     [nq][H][d] bf16
 * With payload == NULL the cache is taken as plain bf16 planes
 * kv_bf16 [2H][n_cache][d] (the bf16 comparator of the same kernel).
 * status (device int32, may be NULL): OR-ed with QVG_STATUS_NAN_SCALE /
 * QVG_STATUS_BAD_ASSIGN when the cache holds an E4M3 NaN-pattern scale or an
 * assignment >= K (that element decodes with centroid 0; read the word after
 * the stream synchronises, as for qvg_dequantize). */
QVG_API size_t qvg_attention_workspace_size(int64_t nq, int64_t n_cache, int64_t n_cur, int32_t n_heads,
                                    int32_t head_dim, const qvg_config *cfg /* host */);
QVG_API int qvg_attention(const uint16_t *q, const uint8_t *payload, const uint8_t *scales,
                  const uint16_t *centroids, const uint8_t *assign, const uint16_t *kv_bf16,
                  const uint16_t *k_cur, const uint16_t *v_cur, int64_t nq, int64_t n_cache,
                  int64_t n_cur, int32_t n_heads, int32_t head_dim,
                  const qvg_config *cfg /* host */, float softmax_scale, uint16_t *out,
                  void *workspace, size_t workspace_bytes, int32_t *status, void *stream);

/* qvg_attention with PRE-RoPE cached keys: the
 * cache holds keys before the rotary embedding; after the reconstruction
 * each cached key row t is rotated with rope_cos / rope_sin [n_cache][d/2]
 * (f32, the caller's positions / frequencies — any 1-D or 3-D RoPE layout):
 * rope_mode 1 = rotate-half pairs (i, i + d/2), 2 = interleaved (2i, 2i+1);
 * 0 = none (== qvg_attention).  q and k_cur are expected post-RoPE.  Needs
 * the reconstruction workspace (also for the bf16 comparator, kv_bf16). */
QVG_API int qvg_attention_rope(const uint16_t *q, const uint8_t *payload, const uint8_t *scales,
                               const uint16_t *centroids, const uint8_t *assign, const uint16_t *kv_bf16,
                               const uint16_t *k_cur, const uint16_t *v_cur, int64_t nq, int64_t n_cache,
                               int64_t n_cur, int32_t n_heads, int32_t head_dim, const qvg_config *cfg,
                               float softmax_scale, const float *rope_cos, const float *rope_sin,
                               int32_t rope_mode, uint16_t *out, void *workspace, size_t workspace_bytes,
                               int32_t *status, void *stream);

/* Baseline competitors (Q/baselines.py), composed with qvg_quantize /
 * qvg_dequantize at S = 0 (= RTN, Q/baselines.py:20-42):
 *  - qvg_hadamard replaces hadamard_transform / inverse_hadamard
 *    (Q/baselines.py:148-164) for n_rows rows of d (power of two, 32..1024):
 *    out = fwht(x * signs) / sqrt_d (inverse = 0) or fwht(x) / sqrt_d * signs
 *    (inverse = 1), float64 butterflies in numpy's order, stored as f64
 *    (the reference's return value) or rounded to f32 (out_dtype); signs [d]
 *    f32 +-1 (random_signs, host), sqrt_d = np.sqrt(d).
 *  - qvg_token_transpose builds the KIVI key path's transposed plane
 *    (Q/baselines.py:60-73): [P][N][d] -> [P][d][n_padded] f32 with zero
 *    pad rows (inverse = 1: [P][d][n_padded] f32 -> [P][N][d] f32). */
QVG_API int qvg_hadamard(const void *x, int32_t x_dtype, int64_t n_rows, int32_t d, const float *signs,
                         double sqrt_d, int32_t inverse, void *out, int32_t out_dtype, void *stream);
QVG_API int qvg_token_transpose(const void *x, int32_t x_dtype, int64_t n_planes, int64_t n_tokens,
                                int64_t n_padded, int32_t d, int32_t inverse, float *out, void *stream);

/* ---- QVGC records from / into device buffers (Q/container.py:158-218, 230-343) ----
 * A batch of P planes in the DeviceChunks layout ([P] payload, [P] scales,
 * [P][S][K][d] bf16 centroids, [P][S][N] assignments) <-> P back-to-back QVGC
 * records (u32 chunk_index, n_tokens, payload_len, scales_len, body_len | body =
 * payload | scales | per stage centroids (bf16 LE) + assignments | u32 crc32),
 * byte-identical to the reference ChunkWriter.append_chunk output; record p gets
 * chunk_index first_index + p.  qvg_record_bytes = 24 + body bytes (0: bad config).
 * qvg_unpack_records verifies every record on the device: ok[p] = 1 intact,
 * 2 CRC mismatch (Q/container.py:297-299), 3 header fields disagree with the
 * config (the reader's structural check, Q/container.py:258-270). */
QVG_API size_t qvg_record_bytes(int64_t n_tokens, int32_t head_dim, const qvg_config *cfg);
QVG_API int qvg_pack_records(const uint8_t *payload, const uint8_t *scales, const uint16_t *centroids,
                             const uint8_t *assign, int64_t n_planes, int64_t n_tokens, int32_t head_dim,
                             const qvg_config *cfg, uint32_t first_index, uint8_t *out, void *stream);
QVG_API int qvg_unpack_records(const uint8_t *records, int64_t n_planes, int64_t n_tokens, int32_t head_dim,
                               const qvg_config *cfg, uint8_t *payload, uint8_t *scales, uint16_t *centroids,
                               uint8_t *assign, uint32_t *ok, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* QVG_B200_H */
