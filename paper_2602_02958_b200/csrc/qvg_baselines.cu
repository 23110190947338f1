// qvg_baselines.cu — the reference's competitor quantizers on the device
// (Q/baselines.py): the seeded randomized Hadamard rotation of QuaRot and
// the token-axis regrouping of KIVI.  Both feed / follow the shared group
// quantizer (k_quantize / k_dequant with S = 0 = RTN, Q/baselines.py:20-42).
//
// Hadamard (Q/baselines.py:132-164): y = fwht(x * signs) / sqrt(d) (forward)
// or fwht(x) / sqrt(d) * signs (inverse), in float64 with numpy's butterfly
// order — level h = 1, 2, 4, ...: (a, b) = (y[i] + y[i+h], y[i] - y[i+h]) —
// then rounded to float32 (the reference's .astype(np.float32)), so the
// rotated plane is bit-identical.  One warp per row, d/32 elements per lane:
// levels h < d/32 in registers, the others by xor shuffles.
#include "qvg_common.cuh"
#include "qvg_internal.h"

namespace qvg {
namespace base {

template <int M, bool XBF16, bool OUT64>
__global__ void k_hadamard_rows(const void *x, int64_t rows, const float *signs, double sqrt_d,
                                int inverse, void *out) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    constexpr int D = 32 * M;
    float sg[M];
#pragma unroll
    for (int m = 0; m < M; m++) sg[m] = signs[lane * M + m];
    for (int64_t r = w0; r < rows; r += nw) {
        double y[M];
#pragma unroll
        for (int m = 0; m < M; m++) {
            const int64_t e = r * D + lane * M + m;
            const double v = XBF16 ? double(bf16_to_f32(static_cast<const uint16_t *>(x)[e]))
                                   : double(static_cast<const float *>(x)[e]);
            y[m] = inverse ? v : v * double(sg[m]);          // x * signs (exact: +-1)
        }
        // in-register levels
#pragma unroll
        for (int h = 1; h < M; h *= 2) {
#pragma unroll
            for (int m = 0; m < M; m++) {
                if (m & h) continue;
                const double a = y[m], b = y[m + h];
                y[m] = __dadd_rn(a, b);
                y[m + h] = __dsub_rn(a, b);
            }
        }
        // cross-lane levels: partner lane = lane ^ (h / M)
#pragma unroll
        for (int hl = 1; hl < 32; hl *= 2) {
            const bool upper = lane & hl;
#pragma unroll
            for (int m = 0; m < M; m++) {
                const double p = __shfl_xor_sync(0xffffffffu, y[m], hl);
                y[m] = upper ? __dsub_rn(p, y[m]) : __dadd_rn(y[m], p);
            }
        }
#pragma unroll
        for (int m = 0; m < M; m++) {
            double v = __ddiv_rn(y[m], sqrt_d);                   // / np.sqrt(d)
            if (inverse) v = v * double(sg[m]);
            if constexpr (OUT64) static_cast<double *>(out)[r * D + lane * M + m] = v;
            else static_cast<float *>(out)[r * D + lane * M + m] = __double2float_rn(v);
        }
    }
}

// [P][N][d] -> [P][d][Np] (Np = N + pad, zero rows appended), the
// KIVI key path's transposed plane (Q/baselines.py:60-73), and back
template <bool XBF16>
__global__ void k_token_transpose(const void *x, int64_t P, int64_t N, int64_t Np, int d, float *out) {
    __shared__ float tile[32][33];
    const int64_t p = blockIdx.z;
    const int64_t n0 = int64_t(blockIdx.x) * 32, c0 = int64_t(blockIdx.y) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t n = n0 + i, c = c0 + threadIdx.x;
        float v = 0.f;
        if (n < N && c < d) {
            const int64_t e = (p * N + n) * d + c;
            v = XBF16 ? bf16_to_f32(static_cast<const uint16_t *>(x)[e]) : static_cast<const float *>(x)[e];
        }
        tile[i][threadIdx.x] = v;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, n = n0 + threadIdx.x;
        if (c < d && n < Np) out[(p * d + c) * Np + n] = tile[threadIdx.x][i];
    }
}

__global__ void k_token_untranspose(const float *in, int64_t P, int64_t N, int64_t Np, int d, float *out) {
    __shared__ float tile[32][33];
    const int64_t p = blockIdx.z;
    const int64_t c0 = int64_t(blockIdx.x) * 32, n0 = int64_t(blockIdx.y) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, n = n0 + threadIdx.x;
        tile[i][threadIdx.x] = (c < d && n < Np) ? in[(p * d + c) * Np + n] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t n = n0 + i, c = c0 + threadIdx.x;
        if (n < N && c < d) out[(p * N + n) * d + c] = tile[threadIdx.x][i];
    }
}

}  // namespace base
}  // namespace qvg

using namespace qvg;

extern "C" {

QVG_API int qvg_hadamard(const void *x, int32_t x_dtype, int64_t n_rows, int32_t d, const float *signs,
                         double sqrt_d, int32_t inverse, void *out, int32_t out_dtype, void *stream) {
    if (out_dtype != QVG_DTYPE_F32 && out_dtype != QVG_DTYPE_F64)
        return set_err(QVG_ERR_BAD_CONFIG, "out_dtype must be f32 or f64");
    if (x_dtype != QVG_DTYPE_F32 && x_dtype != QVG_DTYPE_BF16)
        return set_err(QVG_ERR_BAD_CONFIG, "x_dtype must be f32 or bf16");
    if (d < 32 || d > 1024 || (d & (d - 1)))
        return set_err(QVG_ERR_UNSUPPORTED, "hadamard kernel supports power-of-two head_dim in [32, 1024], got %d", d);
    if (n_rows <= 0) return QVG_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int64_t g = (n_rows * 32 + 255) / 256;
    if (g > 148 * 32) g = 148 * 32;
    const bool bf = x_dtype == QVG_DTYPE_BF16, o64 = out_dtype == QVG_DTYPE_F64;
#define HD(MM)                                                                                              \
    if (bf && o64) base::k_hadamard_rows<MM, true, true><<<unsigned(g), 256, 0, st>>>(x, n_rows, signs, sqrt_d, inverse, out); \
    else if (bf) base::k_hadamard_rows<MM, true, false><<<unsigned(g), 256, 0, st>>>(x, n_rows, signs, sqrt_d, inverse, out); \
    else if (o64) base::k_hadamard_rows<MM, false, true><<<unsigned(g), 256, 0, st>>>(x, n_rows, signs, sqrt_d, inverse, out); \
    else base::k_hadamard_rows<MM, false, false><<<unsigned(g), 256, 0, st>>>(x, n_rows, signs, sqrt_d, inverse, out);
    switch (d) {
        case 32: HD(1) break;
        case 64: HD(2) break;
        case 128: HD(4) break;
        case 256: HD(8) break;
        case 512: HD(16) break;
        default: HD(32) break;
    }
#undef HD
    return cudaGetLastError() == cudaSuccess ? QVG_OK : set_err(QVG_ERR_CUDA, "hadamard launch failed");
}

QVG_API int qvg_token_transpose(const void *x, int32_t x_dtype, int64_t n_planes, int64_t n_tokens,
                                int64_t n_padded, int32_t d, int32_t inverse, float *out, void *stream) {
    if (n_padded < n_tokens || d < 1) return set_err(QVG_ERR_BAD_CONFIG, "bad transpose shape");
    if (n_planes <= 0 || n_tokens <= 0) return QVG_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    dim3 blk(32, 8);
    if (!inverse) {
        if (x_dtype != QVG_DTYPE_F32 && x_dtype != QVG_DTYPE_BF16)
            return set_err(QVG_ERR_BAD_CONFIG, "x_dtype must be f32 or bf16");
        dim3 grid(unsigned((n_padded + 31) / 32), unsigned((d + 31) / 32), unsigned(n_planes));
        if (x_dtype == QVG_DTYPE_BF16)
            base::k_token_transpose<true><<<grid, blk, 0, st>>>(x, n_planes, n_tokens, n_padded, d, out);
        else
            base::k_token_transpose<false><<<grid, blk, 0, st>>>(x, n_planes, n_tokens, n_padded, d, out);
    } else {
        dim3 grid(unsigned((d + 31) / 32), unsigned((n_padded + 31) / 32), unsigned(n_planes));
        base::k_token_untranspose<<<grid, blk, 0, st>>>(static_cast<const float *>(x), n_planes, n_tokens,
                                                        n_padded, d, out);
    }
    return cudaGetLastError() == cudaSuccess ? QVG_OK : set_err(QVG_ERR_CUDA, "transpose launch failed");
}

}  // extern "C"
