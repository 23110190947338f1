// qvg_internal.h — declarations shared by the .cu files of libqvg_b200.so.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/qvg.h"

namespace qvg {

int set_err(int code, const char *fmt, ...);

struct PlaneState {
    double prev;
    double obj;
    int32_t done;
    int32_t iters;
};

struct KMeansBuffers {
    double *rows, *cent, *d2, *nodes;
    int32_t *assign, *counts, *offsets, *members;
    PlaneState *st;
    int64_t *pk_off;
    int32_t *pk_len;
    int pk_leaves;
    int32_t *pk_l, *pk_r, *pk_hstart;   // numpy recursion tree over the N-long pick weights
    int pk_heights;
    int64_t *ob_off;
    int32_t *ob_len, *nd_l, *nd_r, *h_start;
    int ob_leaves, ob_heights;
    // tensor-core assignment (qvg_assign_tc.cu); rsplit == nullptr: exact kernel only
    uint16_t *rsplit;      // [P][T][3][128x128] bf16 row splits (UMMA layout)
    float *xnorm;          // [P][N] row norms
    double *c2;            // [P][K] exact centroid squared norms
    int32_t *recheck, *n_recheck;
    float *rows32;         // [P][N][d] float32 copy of the stage rows (k_split_rows)
    int32_t *rows32_ok;    // [P] nonzero: the copy is exact for the whole plane
    int rows32_valid;      // set once k_split_rows has filled rows32 for the current rows
    const uint16_t *src16; // the bf16 input when the current rows are exactly it (stage 1 of a bf16 chunk)
    // stage 2 of a bf16 chunk: the rows are x - C1_bf16[pi1] (k-means++ rebuilds them)
    const uint16_t *res_x16, *res_c1;
    const uint8_t *res_a1;
    int64_t res_c1_stride, res_a1_stride;
};

// qvg_codec.cu
int launch_quantize(const void *x, int xdtype, int64_t P, int64_t N, int d, int bits, int B, int S,
                    int K, const uint16_t *cent, const uint8_t *asg, uint8_t *payload,
                    uint8_t *scales, int32_t *status, cudaStream_t st);
int launch_dequantize(const uint8_t *payload, const uint8_t *scales, const uint16_t *cent,
                      const uint8_t *asg, int64_t P, int64_t N, int d, int bits, int B, int S, int K,
                      void *out, int odtype, int32_t *status, cudaStream_t st);

int launch_pack(const int8_t *q, int64_t n, int bits, uint8_t *out, int32_t *status, cudaStream_t st);
int launch_unpack(const uint8_t *in, int64_t n, int bits, int8_t *out, cudaStream_t st);

// qvg_kmeans.cu
int launch_widen(const void *x, int xbf16, double *rows, int64_t n, int32_t *status, cudaStream_t st);
int run_kmeanspp(const KMeansBuffers &b, int64_t P, int64_t N, int d, int K, const double *draws,
                 int64_t draws_stride, cudaStream_t st);
int run_kmeans_stage(KMeansBuffers &b, int64_t P, int64_t N, int d, int K, int max_iters,
                     double tol, const double *draws_stage, int64_t draws_stride, bool warm,
                     cudaStream_t st);
int kmeans_outputs(const KMeansBuffers &b, int64_t P, int64_t N, int d, int K, uint8_t *assign,
                   double *objective, int32_t *iters, cudaStream_t st);
int lloyd_once(KMeansBuffers &b, int64_t P, int64_t N, int d, int K, uint8_t *assign,
               double *objective, cudaStream_t st);
int run_assign(const double *rows, const double *cent, int32_t *assign, int64_t P, int64_t N, int d,
               int K, cudaStream_t st);
int finalize_stage(const KMeansBuffers &b, int64_t P, int64_t N, int d, int K, int S, int t,
                   uint16_t *cent_out, double *cent64_out, uint8_t *assign_out, int32_t *iters_out,
                   cudaStream_t st, bool update_rows = true);
int run_add_back(const double *residual, const uint16_t *cent, const uint8_t *assign, int64_t P,
                 int64_t N, int d, int K, double *out, cudaStream_t st);

// qvg_assign_tc.cu
size_t assign_tc_split_elems(int64_t P, int64_t N);
bool assign_tc_ok(int d, int K);
int launch_split_rows(const double *rows, const uint16_t *x16, uint16_t *split, float *xnorm, float *rows32,
                      int32_t *rows32_ok, int64_t P, int64_t N, cudaStream_t st);
int launch_assign_tc(const uint16_t *split, const float *xnorm, const double *rows, const double *cent,
                     const double *c2, int32_t *assign, int32_t *recheck, int32_t *n_recheck,
                     const PlaneState *st_planes, int skip_done, int64_t P, int64_t N, int K, int a_one,
                     cudaStream_t st);

// qvg_attn.cu
size_t attention_workspace_size(int64_t nq, int64_t n_cache, int64_t n_cur, int H, int d,
                                const qvg_config *cfg);
int run_attention(const uint16_t *q, const uint8_t *payload, const uint8_t *scales,
                  const uint16_t *cent, const uint8_t *assign, const uint16_t *kv_bf16,
                  const uint16_t *k_cur, const uint16_t *v_cur, int64_t nq, int64_t n_cache,
                  int64_t n_cur, int H, int d, const qvg_config *cfg, float scale, uint16_t *out,
                  void *workspace, size_t wbytes, int32_t *status, cudaStream_t st, const float *rope_cos = nullptr,
                  const float *rope_sin = nullptr, int rope_mode = 0);

}  // namespace qvg
