// qvg_container.cu — QVGC records assembled from / scattered into device
// buffers (format: Q/container.py:3-36).
//
// A batch of P planes held as DeviceChunks ([P] payload, [P] scales,
// [P][S][K][d] bf16 centroids, [P][S][N] assignments) becomes P back-to-back
// records in one device buffer:
//
//   u32 chunk_index | u32 n_tokens | u32 payload_len | u32 scales_len |
//   u32 body_len | body = payload | scales | per stage (K*d bf16 LE, N u8) |
//   u32 crc32(body)   (IEEE 802.3 reflected, == zlib.crc32)
//
// so a writer needs ONE device->host copy per batch and the file bytes are
// identical to the reference writer's.  The reader does the inverse: one
// host->device copy of a run of records, CRC verification and field scatter
// on the device, straight into the buffers the decoder reads.
//
// CRC on the device: one CTA per record; each thread runs the byte-wise
// table CRC (init 0) over a contiguous segment of length L; warp 0 builds
// the GF(2) operator Z_L ("append L zero bytes", 32x32 bit matrix, squared
// and multiplied column-parallel) and thread 0 folds the segment CRCs in
// order: s <- Z_L(s) ^ c_i, starting from the standard ~0 preset; the short
// tail segment is fed byte-wise.  crc = ~s.
#include <cstdint>

#include "qvg_common.cuh"
#include "qvg_internal.h"

namespace qvg {
namespace qvgc {

constexpr uint32_t kPoly = 0xEDB88320u;     // reflected IEEE polynomial
constexpr int kThreads = 256;
constexpr uint32_t kHdr = 20, kCrc = 4;

struct Layout {
    uint32_t pb, ng, S, kd2, N, body, rec;   // byte counts of one record
};

__host__ __device__ inline Layout layout(int64_t N, int d, int bits, int B, int S, int K) {
    Layout L;
    L.pb = uint32_t((N * d * bits + 7) / 8);
    L.ng = uint32_t(N * d / B);
    L.S = uint32_t(S);
    L.kd2 = uint32_t(K) * uint32_t(d) * 2u;
    L.N = uint32_t(N);
    L.body = L.pb + L.ng + L.S * (L.kd2 + L.N);
    L.rec = kHdr + L.body + kCrc;
    return L;
}

__device__ inline void build_table(uint32_t *tab) {
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = i;
        for (int k = 0; k < 8; k++) c = (c >> 1) ^ ((c & 1u) ? kPoly : 0u);
        tab[i] = c;
    }
}

__device__ inline uint32_t crc_bytes(const uint8_t *p, uint32_t n, uint32_t s, const uint32_t *tab) {
    for (uint32_t i = 0; i < n; i++) s = tab[(s ^ p[i]) & 0xFFu] ^ (s >> 8);
    return s;
}

// columns of a GF(2) operator: M(v) = XOR of col[b] over the set bits b of v
__device__ inline uint32_t apply(const uint32_t *col, uint32_t v) {
    uint32_t r = 0;
    for (int b = 0; b < 32; b++)
        if ((v >> b) & 1u) r ^= col[b];
    return r;
}

// CRC32 of body[0, n) by the CTA; valid in thread 0
__device__ uint32_t crc_cta(const uint8_t *body, uint32_t n, const uint32_t *tab, uint32_t *seg,
                            uint32_t *zl, uint32_t *zp) {
    const uint32_t L = (n + kThreads - 1) / kThreads;
    const uint32_t full = L ? n / L : 0, tail = n - full * L;
    const uint32_t t = threadIdx.x;
    seg[t] = t < full ? crc_bytes(body + size_t(t) * L, L, 0u, tab) : 0u;
    if (t < 32) {
        // zp = Z_1 (one zero byte), zl = identity; zl <- zl * zp^L by square-and-multiply
        uint32_t c = 1u << t;
        for (int k = 0; k < 8; k++) c = (c >> 1) ^ ((c & 1u) ? kPoly : 0u);
        zp[t] = c;
        zl[t] = 1u << t;
        __syncwarp();
        for (uint32_t e = L; e; e >>= 1) {
            if (e & 1u) {
                const uint32_t v = apply(zp, zl[t]);     // column t of zp * zl
                __syncwarp();
                zl[t] = v;
                __syncwarp();
            }
            const uint32_t sq = apply(zp, zp[t]);        // column t of zp * zp
            __syncwarp();
            zp[t] = sq;
            __syncwarp();
        }
    }
    __syncthreads();
    uint32_t s = 0xFFFFFFFFu;
    if (t == 0) {
        for (uint32_t i = 0; i < full; i++) s = apply(zl, s) ^ seg[i];
        s = crc_bytes(body + size_t(full) * L, tail, s, tab);
        s = ~s;
    }
    return s;
}

__device__ inline void put_u32(uint8_t *p, uint32_t v) {
    p[0] = uint8_t(v);
    p[1] = uint8_t(v >> 8);
    p[2] = uint8_t(v >> 16);
    p[3] = uint8_t(v >> 24);
}
__device__ inline uint32_t get_u32(const uint8_t *p) {
    return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}

// copy n bytes with 4-byte words when both ends share alignment, else bytes
__device__ inline void copy_bytes(uint8_t *dst, const uint8_t *src, uint32_t n) {
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 3u) == 0) {
        const uint32_t nw = n >> 2;
        for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x)
            reinterpret_cast<uint32_t *>(dst)[i] = reinterpret_cast<const uint32_t *>(src)[i];
        for (uint32_t i = (nw << 2) + threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    } else {
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    }
}

__global__ void __launch_bounds__(kThreads) k_pack(const uint8_t *payload, const uint8_t *scales,
                                                    const uint16_t *cent, const uint8_t *asg, Layout L,
                                                    uint32_t first_index, uint8_t *out) {
    __shared__ uint32_t tab[256], seg[kThreads], zl[32], zp[32];
    const uint32_t p = blockIdx.x;
    uint8_t *rec = out + size_t(p) * L.rec;
    uint8_t *body = rec + kHdr;
    build_table(tab);
    if (threadIdx.x == 0) {
        put_u32(rec, first_index + p);
        put_u32(rec + 4, L.N);
        put_u32(rec + 8, L.pb);
        put_u32(rec + 12, L.ng);
        put_u32(rec + 16, L.body);
    }
    copy_bytes(body, payload + size_t(p) * L.pb, L.pb);
    copy_bytes(body + L.pb, scales + size_t(p) * L.ng, L.ng);
    uint32_t at = L.pb + L.ng;
    for (uint32_t s = 0; s < L.S; s++) {
        // bf16 centroids are stored as little-endian u16 (the device layout already is)
        copy_bytes(body + at, reinterpret_cast<const uint8_t *>(cent) + (size_t(p) * L.S + s) * L.kd2, L.kd2);
        at += L.kd2;
        copy_bytes(body + at, asg + (size_t(p) * L.S + s) * L.N, L.N);
        at += L.N;
    }
    __syncthreads();
    const uint32_t crc = crc_cta(body, L.body, tab, seg, zl, zp);
    if (threadIdx.x == 0) put_u32(body + L.body, crc);
}

// verify header fields + CRC of every record, scatter the fields; ok[p] = 1
// when record p is intact (2: bad CRC, 3: header/length mismatch)
__global__ void __launch_bounds__(kThreads) k_unpack(const uint8_t *in, Layout L, uint8_t *payload,
                                                      uint8_t *scales, uint16_t *cent, uint8_t *asg,
                                                      uint32_t *ok) {
    __shared__ uint32_t tab[256], seg[kThreads], zl[32], zp[32];
    const uint32_t p = blockIdx.x;
    const uint8_t *rec = in + size_t(p) * L.rec;
    const uint8_t *body = rec + kHdr;
    build_table(tab);
    const bool hdr_ok = get_u32(rec + 4) == L.N && get_u32(rec + 8) == L.pb && get_u32(rec + 12) == L.ng &&
                        get_u32(rec + 16) == L.body;
    copy_bytes(payload + size_t(p) * L.pb, body, L.pb);
    copy_bytes(scales + size_t(p) * L.ng, body + L.pb, L.ng);
    uint32_t at = L.pb + L.ng;
    for (uint32_t s = 0; s < L.S; s++) {
        copy_bytes(reinterpret_cast<uint8_t *>(cent) + (size_t(p) * L.S + s) * L.kd2, body + at, L.kd2);
        at += L.kd2;
        copy_bytes(asg + (size_t(p) * L.S + s) * L.N, body + at, L.N);
        at += L.N;
    }
    __syncthreads();
    const uint32_t crc = crc_cta(body, L.body, tab, seg, zl, zp);
    if (threadIdx.x == 0) ok[p] = !hdr_ok ? 3u : (crc == get_u32(body + L.body) ? 1u : 2u);
}

static int check_cfg(int64_t n_planes, int64_t n_tokens, int d, const qvg_config *cfg) {
    if (!cfg) return set_err(QVG_ERR_BAD_CONFIG, "config is NULL");
    if (n_planes < 0 || n_tokens < 1 || d < 1) return set_err(QVG_ERR_DIMENSION_MISMATCH, "bad record shape");
    if (cfg->bits != 2 && cfg->bits != 4 && cfg->bits != 8) return set_err(QVG_ERR_BAD_CONFIG, "bits must be 2, 4 or 8");
    if (cfg->group_size < 1 || d % cfg->group_size) return set_err(QVG_ERR_DIMENSION_MISMATCH, "group_size must divide head_dim");
    if (cfg->stages < 0 || cfg->centroids < 1) return set_err(QVG_ERR_BAD_CONFIG, "bad stages / centroids");
    const Layout L = layout(n_tokens, d, cfg->bits, cfg->group_size, cfg->stages, cfg->centroids);
    const int64_t body = (n_tokens * d * cfg->bits + 7) / 8 + n_tokens * d / cfg->group_size +
                         int64_t(cfg->stages) * (int64_t(cfg->centroids) * d * 2 + n_tokens);
    if (body + 24 > int64_t(0xFFFFFFFFu) || n_planes > int64_t(0x7FFFFFFF) || int64_t(L.body) != body)
        return set_err(QVG_ERR_DIMENSION_MISMATCH, "record larger than the u32 length fields");
    return QVG_OK;
}

}  // namespace qvgc
}  // namespace qvg

using namespace qvg;

QVG_API size_t qvg_record_bytes(int64_t n_tokens, int32_t head_dim, const qvg_config *cfg) {
    if (qvgc::check_cfg(0, n_tokens, head_dim, cfg)) return 0;
    return qvgc::layout(n_tokens, head_dim, cfg->bits, cfg->group_size, cfg->stages, cfg->centroids).rec;
}

QVG_API int qvg_pack_records(const uint8_t *payload, const uint8_t *scales, const uint16_t *centroids,
                             const uint8_t *assign, int64_t n_planes, int64_t n_tokens, int32_t head_dim,
                             const qvg_config *cfg, uint32_t first_index, uint8_t *out, void *stream) {
    if (int rc = qvgc::check_cfg(n_planes, n_tokens, head_dim, cfg)) return rc;
    if (n_planes == 0) return QVG_OK;
    if (!payload || !scales || !out || (cfg->stages && (!centroids || !assign)))
        return set_err(QVG_ERR_BAD_CONFIG, "NULL buffer");
    const qvgc::Layout L = qvgc::layout(n_tokens, head_dim, cfg->bits, cfg->group_size, cfg->stages, cfg->centroids);
    qvgc::k_pack<<<unsigned(n_planes), qvgc::kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        payload, scales, centroids, assign, L, first_index, out);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : set_err(QVG_ERR_CUDA, "record pack launch failed");
}

QVG_API int qvg_unpack_records(const uint8_t *records, int64_t n_planes, int64_t n_tokens, int32_t head_dim,
                               const qvg_config *cfg, uint8_t *payload, uint8_t *scales, uint16_t *centroids,
                               uint8_t *assign, uint32_t *ok, void *stream) {
    if (int rc = qvgc::check_cfg(n_planes, n_tokens, head_dim, cfg)) return rc;
    if (n_planes == 0) return QVG_OK;
    if (!records || !payload || !scales || !ok || (cfg->stages && (!centroids || !assign)))
        return set_err(QVG_ERR_BAD_CONFIG, "NULL buffer");
    const qvgc::Layout L = qvgc::layout(n_tokens, head_dim, cfg->bits, cfg->group_size, cfg->stages, cfg->centroids);
    qvgc::k_unpack<<<unsigned(n_planes), qvgc::kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        records, L, payload, scales, centroids, assign, ok);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : set_err(QVG_ERR_CUDA, "record unpack launch failed");
}
