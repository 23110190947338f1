// qvg_attn.cu — attention over the QVG-quantized KV cache on sm_100a.
//
// O = softmax(q [Khat ; k_cur]^T * scale) [Vhat ; v_cur] per head, where
// Khat/Vhat are the one-pass reconstructions (Q/prq.py:113-132) of the head's
// K and V planes.  No mask: the current chunk attends to every cached token
// and to itself (block-causal video diffusion).
//
// Structure (one CTA = 128 query rows of one head, 128 threads; thread t
// owns query row t = TMEM lane t):
//   * the Q tile is staged once in shared memory (UMMA K-major, no swizzle);
//   * for every 128-token KV block the threads build the K and V operand tiles
//     in shared memory — dequantizing the packed codes, E4M3 scales and the
//     per-token centroid add-back in-tile for cached blocks, copying bf16 for
//     the current chunk (and for the bf16 comparator mode);
//   * one thread issues tcgen05.mma (kind::f16, M=128, N=128, K=16 steps):
//     S = Q K^T into TMEM columns [0,128), completion via tcgen05.commit on
//     an mbarrier;
//   * softmax (online, exp2 domain, lazy rescale when the running max grows
//     by more than 2^8) reads S with tcgen05.ld, writes P (bf16) to shared
//     memory; O (TMEM columns [128,256)) is rescaled in place with
//     tcgen05.ld/st when needed;
//   * tcgen05.mma: O += P V, then the next block.
// Epilogue: O / l -> bf16.
#include <cstdio>
#include <type_traits>
#include <cstdlib>
#include <cstring>
#include <cuda.h>

#include "qvg_common.cuh"
#include "qvg_internal.h"

namespace qvg {
namespace attn {

constexpr int kTile = 128;                  // query rows per CTA = KV tokens per block
constexpr int kD = 128;                     // head_dim supported by the tcgen05 path
constexpr int kTileBytes = kTile * kD * 2;  // one bf16 operand tile (32 KB)
constexpr uint32_t kSbo = 2048;             // byte stride between 8-row core groups
constexpr uint32_t kLbo = 128;              // byte stride between 8-column core chunks

// ---- PTX wrappers ----------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }

// UMMA shared-memory matrix descriptor (SWIZZLE_NONE, version 1 for sm_100)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFFu);
    d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;                      // version
    return d;                                    // base_offset 0, lbo_mode 0, layout 0
}

// instruction descriptor: kind::f16, A=B=bf16, D=f32, M=128, N=128
__host__ __device__ constexpr uint32_t umma_idesc(bool b_mn_major) {
    return (1u << 4)                 // c_format F32
           | (1u << 7)               // a_format BF16
           | (1u << 10)              // b_format BF16
           | (0u << 15)              // a K-major
           | (uint32_t(b_mn_major) << 16)
           | (uint32_t(kTile >> 3) << 17)   // N
           | (uint32_t(kTile >> 4) << 24);  // M
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
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

// wait with nanosleep back-off: a warp that finds the phase incomplete sleeps
// instead of re-issuing try_wait, leaving the issue slots of its SMSP to the
// working softmax warps (ns = 0: plain spin)
__device__ __forceinline__ bool bar_try(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}"
        : "=r"(ok)
        : "r"(su32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void bar_wait_nap(uint64_t *bar, uint32_t parity, uint32_t ns) {
    while (!bar_try(bar, parity))
        if (ns) __nanosleep(ns);
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 32 consecutive 32-bit TMEM columns of this thread's lane
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

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float v[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
        "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
        "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
        "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
        "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
        "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// ---- operand-tile layout (UMMA canonical, no swizzle) ----------------------
// K-major tile, row r (M or N index), 16-byte chunk c of the K dimension.
__device__ __forceinline__ uint32_t kmaj_off(uint32_t r, uint32_t c) {
    return (r >> 3) * kSbo + c * kLbo + (r & 7u) * 16u;
}
// MN-major tile (B operand of P.V): token k (K index), 8-wide chunk c of the
// N (= head_dim) index.
__device__ __forceinline__ uint32_t mnmaj_off(uint32_t k, uint32_t c) {
    return c * kSbo + (k >> 3) * kLbo + (k & 7u) * 16u;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

struct AttnArgs {
    const uint16_t *q, *k_cur, *v_cur, *kv_bf16;
    const uint8_t *payload, *scales, *asg;
    const uint16_t *cent;
    uint16_t *out;
    int64_t nq, n_cache, n_cur;
    int H, bits, B, S, K;
    float scale_log2;
    int32_t *status;        // NaN-pattern scale / assignment >= K flags (may be NULL)
};

// One token row (128 channels) of plane `pl` of the quantized cache,
// reconstructed (f32 add-back in the reference's order, then bf16 RNE) and
// written chunk by chunk into an operand tile via `put(c, uint4)`.
template <int BITS, int S, typename Put>
__device__ __forceinline__ void dequant_row(const AttnArgs &a, int64_t pl, int64_t tok, Put put) {
    const int64_t N = a.n_cache;
    const uint8_t *pp = a.payload + pl * ((N * kD * BITS) >> 3) + ((tok * kD * BITS) >> 3);
    const uint8_t *sp = a.scales + pl * (N * kD / a.B) + tok * (kD / a.B);
    const uint16_t *crow[S > 0 ? S : 1];
#pragma unroll
    for (int t = 0; t < S; t++) {
        int ai = __ldg(a.asg + (pl * S + t) * N + tok);
        if (ai >= a.K) {                   // corrupt cache: flag it, decode with centroid 0
            if (a.status) atomicOr(a.status, int(QVG_STATUS_BAD_ASSIGN));
            ai = 0;
        }
        crow[t] = a.cent + ((pl * S + t) * a.K + ai) * kD;
    }
    constexpr uint32_t mask = (1u << BITS) - 1u, sign = 1u << (BITS - 1);
#pragma unroll 4
    for (int c = 0; c < kD / 8; c++) {
        // 8 fields = BITS bytes of payload
        uint64_t w;
        if constexpr (BITS == 2) w = __ldg(reinterpret_cast<const uint16_t *>(pp) + c);
        else if constexpr (BITS == 4) w = __ldg(reinterpret_cast<const uint32_t *>(pp) + c);
        else { const uint2 v = __ldg(reinterpret_cast<const uint2 *>(pp) + c); w = uint64_t(v.x) | (uint64_t(v.y) << 32); }
        const uint32_t sb = __ldg(sp + (c * 8) / a.B);
        if ((sb & 0x7Fu) == 0x7Fu && a.status) atomicOr(a.status, int(QVG_STATUS_NAN_SCALE));
        const float s = e4m3_to_f32(sb);
        float y[8];
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const uint32_t u = uint32_t(w >> (k * BITS)) & mask;
            y[k] = float(int(u ^ sign) - int(sign)) * s;
        }
#pragma unroll
        for (int t = S - 1; t >= 0; t--) {
            const uint4 cv = __ldg(reinterpret_cast<const uint4 *>(crow[t]) + c);
            y[0] += bf16_lo(cv.x); y[1] += bf16_hi(cv.x); y[2] += bf16_lo(cv.y); y[3] += bf16_hi(cv.y);
            y[4] += bf16_lo(cv.z); y[5] += bf16_hi(cv.z); y[6] += bf16_lo(cv.w); y[7] += bf16_hi(cv.w);
        }
        put(c, make_uint4(pack_bf16(y[0], y[1]), pack_bf16(y[2], y[3]), pack_bf16(y[4], y[5]), pack_bf16(y[6], y[7])));
    }
}

template <typename Put>
__device__ __forceinline__ void copy_row_bf16(const uint16_t *src, Put put) {
#pragma unroll 4
    for (int c = 0; c < 16; c++) put(c, __ldg(reinterpret_cast<const uint4 *>(src) + c));
}

template <int BITS, int S, bool QUANT>
__global__ void __launch_bounds__(128, 1) k_attention(AttnArgs a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *sQ = smem;
    uint8_t *sK = smem + kTileBytes;
    uint8_t *sV = smem + 2 * kTileBytes;
    uint8_t *sP = smem + 3 * kTileBytes;
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base_sh;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int h = blockIdx.y;
    const int64_t q0 = int64_t(blockIdx.x) * kTile;
    const int64_t H = a.H;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tmem_base_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        bar_init(&mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // Q tile: row tid = query q0 + tid of head h (zeros past nq)
    {
        const int64_t qi = q0 + tid;
        auto putq = [&](int c, uint4 v) { *reinterpret_cast<uint4 *>(sQ + kmaj_off(tid, c)) = v; };
        if (qi < a.nq) copy_row_bf16(a.q + (qi * H + h) * kD, putq);
        else
            for (int c = 0; c < 16; c++) putq(c, make_uint4(0, 0, 0, 0));
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base_sh;
    const uint32_t t_lane = uint32_t(warp * 32) << 16;
    const uint32_t tS = tmem, tO = tmem + 128;

    const uint64_t dQ = umma_desc(su32(sQ), kLbo, kSbo);
    const uint64_t dK = umma_desc(su32(sK), kLbo, kSbo);
    const uint64_t dP = umma_desc(su32(sP), kLbo, kSbo);
    const uint64_t dV = umma_desc(su32(sV), kLbo, kSbo);
    constexpr uint32_t idK = umma_idesc(false), idV = umma_idesc(true);

    float m_run = -INFINITY, l_run = 0.f;
    uint32_t phase = 0;
    const int64_t n_tot = a.n_cache + a.n_cur;
    const int64_t n_blocks = (a.n_cache + kTile - 1) / kTile + (a.n_cur + kTile - 1) / kTile;
    const int64_t cache_blocks = (a.n_cache + kTile - 1) / kTile;
    (void)n_tot;

    for (int64_t jb = 0; jb < n_blocks; jb++) {
        // ---- build K / V operand tiles for this block (thread tid = token row)
        const bool in_cache = jb < cache_blocks;
        const int64_t base = in_cache ? jb * kTile : (jb - cache_blocks) * kTile;
        const int64_t cnt = in_cache ? a.n_cache : a.n_cur;
        const int64_t tok = base + tid;
        const bool valid = tok < cnt;
        auto putk = [&](int c, uint4 v) { *reinterpret_cast<uint4 *>(sK + kmaj_off(tid, c)) = v; };
        auto putv = [&](int c, uint4 v) { *reinterpret_cast<uint4 *>(sV + mnmaj_off(tid, c)) = v; };
        if (!valid) {
            for (int c = 0; c < 16; c++) { putk(c, make_uint4(0, 0, 0, 0)); putv(c, make_uint4(0, 0, 0, 0)); }
        } else if (in_cache) {
            if constexpr (QUANT) {
                dequant_row<BITS, S>(a, 2 * h, tok, putk);
                dequant_row<BITS, S>(a, 2 * h + 1, tok, putv);
            } else {
                copy_row_bf16(a.kv_bf16 + ((2 * h) * a.n_cache + tok) * kD, putk);
                copy_row_bf16(a.kv_bf16 + ((2 * h + 1) * a.n_cache + tok) * kD, putv);
            }
        } else {
            copy_row_bf16(a.k_cur + (tok * H + h) * kD, putk);
            copy_row_bf16(a.v_cur + (tok * H + h) * kD, putv);
        }
        fence_proxy_async();
        fence_before();
        __syncthreads();
        // ---- S = Q K^T
        if (tid == 0) {
            fence_after();
#pragma unroll
            for (int k = 0; k < kD / 16; k++)
                mma_f16(tS, dQ + uint64_t((k * 2 * kLbo) >> 4), dK + uint64_t((k * 2 * kLbo) >> 4), idK, k > 0);
            mma_commit(&mbar);
        }
        bar_wait(&mbar, phase);
        phase ^= 1u;
        fence_after();
        // ---- online softmax on row tid (exp2 domain); lazy rescale of O
        const int nvalid = int(cnt - base < kTile ? cnt - base : kTile);
        float mx = -INFINITY;
#pragma unroll
        for (int ch = 0; ch < 4; ch++) {
            float sv[32];
            tmem_ld32(tS + t_lane + ch * 32, sv);
#pragma unroll
            for (int i = 0; i < 32; i++)
                if (ch * 32 + i < nvalid) mx = fmaxf(mx, sv[i] * a.scale_log2);
        }
        const bool grow = mx > m_run + 8.f;       // rescale only when the max grows by > 2^8
        const float m_new = grow ? mx : m_run;
        const float alpha = grow ? exp2f(m_run - m_new) : 1.f;
        if (__any_sync(0xffffffffu, grow) && jb > 0) {
#pragma unroll
            for (int ch = 0; ch < 4; ch++) {
                float ov[32];
                tmem_ld32(tO + t_lane + ch * 32, ov);
#pragma unroll
                for (int i = 0; i < 32; i++) ov[i] *= alpha;
                tmem_st32(tO + t_lane + ch * 32, ov);
            }
        }
        l_run *= alpha;
        m_run = m_new;
        float lsum = 0.f;
#pragma unroll
        for (int ch = 0; ch < 4; ch++) {
            float sv[32];
            tmem_ld32(tS + t_lane + ch * 32, sv);
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const float p0 = ch * 32 + i < nvalid ? exp2f(sv[i] * a.scale_log2 - m_run) : 0.f;
                const float p1 = ch * 32 + i + 1 < nvalid ? exp2f(sv[i + 1] * a.scale_log2 - m_run) : 0.f;
                lsum += p0 + p1;
                pk[i >> 1] = pack_bf16(p0, p1);
            }
#pragma unroll
            for (int c = 0; c < 4; c++)
                *reinterpret_cast<uint4 *>(sP + kmaj_off(tid, ch * 4 + c)) =
                    make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
        }
        l_run += lsum;
        fence_proxy_async();
        fence_before();
        __syncthreads();
        // ---- O += P V
        if (tid == 0) {
            fence_after();
#pragma unroll
            for (int k = 0; k < kTile / 16; k++)
                mma_f16(tO, dP + uint64_t((k * 2 * kLbo) >> 4), dV + uint64_t((k * 2 * kLbo) >> 4), idV,
                        (jb > 0 || k > 0) ? 1u : 0u);
            mma_commit(&mbar);
        }
        bar_wait(&mbar, phase);
        phase ^= 1u;
        fence_after();
    }
    // ---- epilogue: O / l -> bf16
    const float inv_l = 1.f / l_run;
    const int64_t qi = q0 + tid;
#pragma unroll
    for (int ch = 0; ch < 4; ch++) {
        float ov[32];
        tmem_ld32(tO + t_lane + ch * 32, ov);
        if (qi < a.nq) {
            uint4 *dst = reinterpret_cast<uint4 *>(a.out + (qi * H + h) * kD + ch * 32);
#pragma unroll
            for (int c = 0; c < 4; c++)
                dst[c] = make_uint4(pack_bf16(ov[8 * c] * inv_l, ov[8 * c + 1] * inv_l),
                                    pack_bf16(ov[8 * c + 2] * inv_l, ov[8 * c + 3] * inv_l),
                                    pack_bf16(ov[8 * c + 4] * inv_l, ov[8 * c + 5] * inv_l),
                                    pack_bf16(ov[8 * c + 6] * inv_l, ov[8 * c + 7] * inv_l));
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int BITS, int S, bool QUANT>
static int launch(const AttnArgs &a, cudaStream_t st) {
    const size_t smem = 4 * size_t(kTileBytes) + 1024;
    auto kern = k_attention<BITS, S, QUANT>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    dim3 grid(unsigned((a.nq + kTile - 1) / kTile), unsigned(a.H));
    kern<<<grid, 128, smem, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

template <int BITS>
static int dispatch_s(const AttnArgs &a, cudaStream_t st) {
    switch (a.S) {
        case 0: return launch<BITS, 0, true>(a, st);
        case 1: return launch<BITS, 1, true>(a, st);
        case 2: return launch<BITS, 2, true>(a, st);
        case 3: return launch<BITS, 3, true>(a, st);
        case 4: return launch<BITS, 4, true>(a, st);
        default: return set_err(QVG_ERR_UNSUPPORTED, "attention supports stages <= 4");
    }
}

}  // namespace attn

// ============================================================================
// v2: warp-specialised, pipelined tcgen05 attention over bf16 operands.
//   warps 0-3  softmax (thread t = query row t = TMEM lane t) + epilogue
//   warp  4    TMA producer: Q once, then K/V tiles into a 2-stage ring
//   warp  5    TMEM allocator + single-thread MMA issuer
// S_j = Q K_j^T goes to TMEM buffer j%2 while softmax works on S_{j-1};
// O += P_{j-1} V_{j-1} is issued as soon as softmax publishes P_{j-1}.
// Q/K/V tiles: TMA boxes [128 rows][64 cols] with 128B swizzle (UMMA
// K-major SW128 for Q/K, MN-major SW128 for V); P: no-swizzle K-major.
// The quantized cache is first reconstructed to bf16 by the K6 kernel into
// the workspace (an HBM-bound pass), then attended here.
// ============================================================================
namespace attn2 {
using attn::kTile;
using attn::kD;

constexpr uint32_t kBox = kTile * 64 * 2;          // one TMA box (16 KB)
constexpr uint32_t kOpTile = 2 * kBox;             // a 128x128 bf16 operand (32 KB)
constexpr uint32_t kSmem = kOpTile /*Q*/ + 2 * 2 * kOpTile /*K,V x 2 stages*/ + kOpTile /*P*/;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFFu);
    d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;                        // version (sm_100)
    d |= uint64_t(2) << 61;                        // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *tm, int x, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            attn::su32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(attn::su32(bar))
        : "memory");
}

__device__ __forceinline__ void expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(attn::su32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(attn::su32(bar)) : "memory");
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct Args {
    int64_t nq, n_cache, n_cur;
    int H;
    float scale_log2;
    uint16_t *out;
    uint32_t nap_sm = 0, nap_mma = 0, nap_tma = 0;   // nanosleep back-off of the softmax / MMA / TMA waits
};

struct Bars {
    uint64_t q_full, kv_full[2], kv_empty[2], s_full[2], s_free[2], p_full, o_done;
    uint32_t tmem;
};

// (the v2 single-tile kernel is gone; these helpers serve the pp4 / in-tile kernels)

// ---- host: tensor maps via the driver entry point (no -lcuda needed) -------
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;      // immutable once resolved
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 2-D bf16 tensor [rows][cols] (row pitch `pitch` elements), box [128][64], SW128
static bool make_map(CUtensorMap *m, const void *base, uint64_t rows, uint64_t cols, uint64_t pitch) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {pitch * 2};
    cuuint32_t box[2] = {64, uint32_t(kTile)};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace attn2


// ============================================================================
// helpers shared by the two-tile (ping-pong) kernel below: TMEM-A MMA, TMEM
// stores of P, the barrier set
// ============================================================================
namespace attn3 {
using attn::kTile;
using attn::kD;
using attn2::kBox;
using attn2::kOpTile;
constexpr uint32_t kSmem = 2 * kOpTile /*Q_A,Q_B*/ + 2 * 2 * kOpTile /*K,V x 2 stages*/;

__device__ __forceinline__ void mma_f16_tmem_a(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st32u(uint32_t taddr, const uint32_t v[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}

struct Bars {
    uint64_t q_full, kv_full[2], kv_empty[2], s_full[2], p_full[2], o_final;
    uint32_t tmem;
};

}  // namespace attn3

// ============================================================================
// v4: the v3 ping-pong with (1) the MMA order PV_A(j) S_A(j+1) PV_B(j)
// S_B(j+1), so that each softmax phase overlaps two MMAs of the other tile,
// (2) the S row loaded from TMEM once (128 registers, one wait::ld), (3) packed
// f32x2 arithmetic for scale/shift and row sums, and (4) 3/8 of the exp2 on
// the FMA pipe (degree-3 polynomial on the rounded-off fraction, exponent
// added in the integer domain) to relieve the 16/clk/SM MUFU.
// ============================================================================
// QVG_ATTN_NAP="sm,mma,tma": nanosleep back-off (ns) of the softmax, MMA-issuer
// and TMA-producer waits.  Default 0 (plain spin): on the LongCat layer no
// setting changed pp4 (5.46 ms); pp5 needs sm >= 16 (6.05 -> 5.54 ms)
static void nap_args(attn2::Args &a) {
    static const uint32_t v[3] = {[] {
                                      const char *e = getenv("QVG_ATTN_NAP");
                                      return e ? uint32_t(atoi(e)) : 0u;
                                  }(),
                                  [] {
                                      const char *e = getenv("QVG_ATTN_NAP");
                                      const char *c = e ? strchr(e, ',') : nullptr;
                                      return c ? uint32_t(atoi(c + 1)) : 0u;
                                  }(),
                                  [] {
                                      const char *e = getenv("QVG_ATTN_NAP");
                                      const char *c = e ? strchr(e, ',') : nullptr;
                                      c = c ? strchr(c + 1, ',') : nullptr;
                                      return c ? uint32_t(atoi(c + 1)) : 0u;
                                  }()};
    a.nap_sm = v[0];
    a.nap_mma = v[1];
    a.nap_tma = v[2];
}

namespace attn4 {
using attn::kTile;
using attn::kD;
using attn2::kBox;
using attn2::kOpTile;
using attn3::Bars;
constexpr uint32_t kSmem = attn3::kSmem;

__device__ __forceinline__ void tmem_ld128(uint32_t taddr, float v[128]) {
    uint32_t *r = reinterpret_cast<uint32_t *>(v);
#pragma unroll
    for (int c = 0; c < 4; c++) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[32 * c + 0]), "=r"(r[32 * c + 1]), "=r"(r[32 * c + 2]), "=r"(r[32 * c + 3]),
              "=r"(r[32 * c + 4]), "=r"(r[32 * c + 5]), "=r"(r[32 * c + 6]), "=r"(r[32 * c + 7]),
              "=r"(r[32 * c + 8]), "=r"(r[32 * c + 9]), "=r"(r[32 * c + 10]), "=r"(r[32 * c + 11]),
              "=r"(r[32 * c + 12]), "=r"(r[32 * c + 13]), "=r"(r[32 * c + 14]), "=r"(r[32 * c + 15]),
              "=r"(r[32 * c + 16]), "=r"(r[32 * c + 17]), "=r"(r[32 * c + 18]), "=r"(r[32 * c + 19]),
              "=r"(r[32 * c + 20]), "=r"(r[32 * c + 21]), "=r"(r[32 * c + 22]), "=r"(r[32 * c + 23]),
              "=r"(r[32 * c + 24]), "=r"(r[32 * c + 25]), "=r"(r[32 * c + 26]), "=r"(r[32 * c + 27]),
              "=r"(r[32 * c + 28]), "=r"(r[32 * c + 29]), "=r"(r[32 * c + 30]), "=r"(r[32 * c + 31])
            : "r"(taddr + 32 * c));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float ex2_mufu(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 2^x for a pair, x >= -126: x = j + f, j = rint(x) (magic-number add),
// 2^f by a degree-3 polynomial on [-1/2, 1/2] (max rel. error 7.5e-5, far
// below the bf16 rounding of P), 2^j added to the exponent field
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
    const float2 M = make_float2(12582912.f, 12582912.f);
    const float2 xm = __fadd2_rn(x, M);
    const float2 jf = __fadd2_rn(xm, make_float2(-12582912.f, -12582912.f));
    const float2 f = __fadd2_rn(x, make_float2(-jf.x, -jf.y));
    float2 p = __ffma2_rn(make_float2(0.05517162f, 0.05517162f), f, make_float2(0.24261117f, 0.24261117f));
    p = __ffma2_rn(p, f, make_float2(0.693261f, 0.693261f));
    p = __ffma2_rn(p, f, make_float2(0.99992806f, 0.99992806f));
    uint32_t r0, r1;   // bits(p) + (bits(xm) << 23) on the FMA pipe (IMAD)
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r0) : "r"(__float_as_uint(xm.x)), "r"(1u << 23), "r"(__float_as_uint(p.x)));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r1) : "r"(__float_as_uint(xm.y)), "r"(1u << 23), "r"(__float_as_uint(p.y)));
    return make_float2(__uint_as_float(r0), __uint_as_float(r1));
}

// columns [POLY_FROM, 128) of each S row use the polynomial exp2
template <int POLY_FROM, bool TR = false>
__global__ void __launch_bounds__(320, 1)
k_attention_pp4(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                const __grid_constant__ CUtensorMap tmKc, const __grid_constant__ CUtensorMap tmVc, attn2::Args a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sQ = smem;
    uint8_t *sKV = smem + 2 * kOpTile;
    __shared__ Bars bars;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int h = blockIdx.y;
    const int64_t q0 = int64_t(blockIdx.x) * 2 * kTile;
    const int64_t cb = (a.n_cache + kTile - 1) / kTile;
    const int64_t nb = cb + (a.n_cur + kTile - 1) / kTile;

    if (tid == 0) {
        attn::bar_init(&bars.q_full, 1);
        for (int i = 0; i < 2; i++) {
            attn::bar_init(&bars.kv_full[i], 1);
            attn::bar_init(&bars.kv_empty[i], 1);
            attn::bar_init(&bars.s_full[i], 1);
            attn::bar_init(&bars.p_full[i], 128);
        }
        attn::bar_init(&bars.o_final, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 9) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(attn::su32(&bars.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    attn::fence_before();
    __syncthreads();
    attn::fence_after();
    const uint32_t tmem = bars.tmem;

    if (warp == 8) {
        if (lane == 0) {                              // ---- TMA producer (as v3)
            attn2::expect_tx(&bars.q_full, 2 * kOpTile);
            for (int t = 0; t < 2; t++) {
                attn2::tma_load_2d(sQ + t * kOpTile, &tmQ, h * kD, int(q0 + t * kTile), &bars.q_full);
                attn2::tma_load_2d(sQ + t * kOpTile + kBox, &tmQ, h * kD + 64, int(q0 + t * kTile), &bars.q_full);
            }
            for (int64_t j = 0; j < nb; j++) {
                const int st = int(j & 1);
                if (j >= 2) attn::bar_wait_nap(&bars.kv_empty[st], uint32_t(((j - 2) >> 1) & 1), a.nap_tma);
                uint8_t *sK = sKV + st * 2 * kOpTile, *sV = sK + kOpTile;
                attn2::expect_tx(&bars.kv_full[st], 2 * kOpTile);
                if (j < cb) {
                    const int yk = int(2 * h * a.n_cache + j * kTile), yv = int((2 * h + 1) * a.n_cache + j * kTile);
                    attn2::tma_load_2d(sK, &tmKV, 0, yk, &bars.kv_full[st]);
                    attn2::tma_load_2d(sK + kBox, &tmKV, 64, yk, &bars.kv_full[st]);
                    attn2::tma_load_2d(sV, &tmKV, 0, yv, &bars.kv_full[st]);
                    attn2::tma_load_2d(sV + kBox, &tmKV, 64, yv, &bars.kv_full[st]);
                } else {
                    const int y = int((j - cb) * kTile);
                    attn2::tma_load_2d(sK, &tmKc, h * kD, y, &bars.kv_full[st]);
                    attn2::tma_load_2d(sK + kBox, &tmKc, h * kD + 64, y, &bars.kv_full[st]);
                    attn2::tma_load_2d(sV, &tmVc, h * kD, y, &bars.kv_full[st]);
                    attn2::tma_load_2d(sV + kBox, &tmVc, h * kD + 64, y, &bars.kv_full[st]);
                }
            }
        }
    } else if (warp == 9) {
        if (lane == 0) {                              // ---- MMA issuer
            constexpr uint32_t idK = attn::umma_idesc(false), idV = attn::umma_idesc(true);
            auto issue_s = [&](int t, int64_t j) {    // S_t = Q_t K_j^T
                const int st = int(j & 1);
                const uint32_t sk = attn::su32(sKV + st * 2 * kOpTile);
                const uint32_t sq = attn::su32(sQ + t * kOpTile);
#pragma unroll
                for (int k = 0; k < kD / 16; k++) {
                    const uint32_t off = (k >> 2) * kBox + (k & 3) * 32;
                    attn::mma_f16(tmem + t * 128, attn2::desc_sw128(sq + off, 16, 1024),
                                  attn2::desc_sw128(sk + off, 16, 1024), idK, k > 0);
                }
                attn::mma_commit(&bars.s_full[t]);
            };
            auto issue_pv = [&](int t, int64_t j) {   // O_t += P_t V_j  (P in TMEM over S_t)
                const int st = int(j & 1);
                const uint32_t sv = attn::su32(sKV + st * 2 * kOpTile) + kOpTile;
#pragma unroll
                for (int k = 0; k < kTile / 16; k++)
                    attn3::mma_f16_tmem_a(tmem + 256 + t * 128, tmem + t * 128 + k * 8,
                                          attn2::desc_sw128(sv + k * 2048, kBox, 1024), idV,
                                          (j > 0 || k > 0) ? 1u : 0u);
            };
            attn::bar_wait(&bars.q_full, 0);
            attn::bar_wait(&bars.kv_full[0], 0);
            attn::fence_after();
            issue_s(0, 0);
            issue_s(1, 0);
            long long tr[4][4];
            const long long t0c = clock64();
            for (int64_t j = 0; j < nb; j++) {
                attn::bar_wait_nap(&bars.p_full[0], uint32_t(j & 1), a.nap_mma);
                if (TR && j >= 8 && j < 12) tr[j - 8][0] = clock64() - t0c;
                attn::fence_after();
                issue_pv(0, j);
                if (j + 1 < nb) {
                    attn::bar_wait_nap(&bars.kv_full[(j + 1) & 1], uint32_t(((j + 1) >> 1) & 1), a.nap_mma);
                    if (TR && j >= 8 && j < 12) tr[j - 8][1] = clock64() - t0c;
                    attn::fence_after();
                    issue_s(0, j + 1);                // overwrites P_A(j): MMAs execute in order
                }
                attn::bar_wait_nap(&bars.p_full[1], uint32_t(j & 1), a.nap_mma);
                if (TR && j >= 8 && j < 12) tr[j - 8][2] = clock64() - t0c;
                attn::fence_after();
                issue_pv(1, j);
                attn::mma_commit(&bars.kv_empty[j & 1]);
                if (j + 1 < nb) issue_s(1, j + 1);
                if (TR && j >= 8 && j < 12) tr[j - 8][3] = clock64() - t0c;
            }
            if (TR && blockIdx.x == 0 && blockIdx.y == 0)
                for (int q = 0; q < 4; q++)
                    printf("MMA j=%d pA_ready=%lld kv_ready=%lld pB_ready=%lld issued=%lld\n", q + 8, tr[q][0], tr[q][1],
                           tr[q][2], tr[q][3]);
            attn::mma_commit(&bars.o_final);
        }
    } else {
        // ---- softmax (tile t = warp / 4), thread = query row = TMEM lane ----
        const int t = warp >> 2;
        const uint32_t t_lane = uint32_t((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + t * 128 + t_lane, tO = tmem + 256 + t * 128 + t_lane;
        const float sl2 = a.scale_log2;
        float m_run = -INFINITY, l_run = 0.f;
        long long tr[4][8];
        const long long t0c = clock64();
        for (int64_t j = 0; j < nb; j++) {
            const int64_t cnt = j < cb ? a.n_cache - j * kTile : a.n_cur - (j - cb) * kTile;
            const int nvalid = int(cnt < kTile ? cnt : kTile);
            if (TR && j >= 8 && j < 12) tr[j - 8][0] = clock64() - t0c;
            attn::bar_wait_nap(&bars.s_full[t], uint32_t(j & 1), a.nap_sm);
            if (TR && j >= 8 && j < 12) tr[j - 8][1] = clock64() - t0c;
            attn::fence_after();
            float s[128];
            tmem_ld128(tS, s);
            if (TR && j >= 8 && j < 12) tr[j - 8][2] = clock64() - t0c;
            float m_new, alpha;
            bool grow;
            float2 acc4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                              make_float2(0.f, 0.f)};     // independent partial row sums
            auto phase = [&](auto mask_tag) {
                constexpr bool MASK = decltype(mask_tag)::value;
                if constexpr (MASK) {
#pragma unroll
                    for (int i = 0; i < 128; i++) s[i] = i < nvalid ? s[i] : -INFINITY;
                }
                // 3-input max tree: 128 -> 43 -> 15 -> 5 -> 2 -> 1
                float m43[43];
#pragma unroll
                for (int i = 0; i < 42; i++) m43[i] = fmaxf(fmaxf(s[3 * i], s[3 * i + 1]), s[3 * i + 2]);
                m43[42] = fmaxf(s[126], s[127]);
                float m15[15];
#pragma unroll
                for (int i = 0; i < 14; i++) m15[i] = fmaxf(fmaxf(m43[3 * i], m43[3 * i + 1]), m43[3 * i + 2]);
                m15[14] = m43[42];
                float m5[5];
#pragma unroll
                for (int i = 0; i < 5; i++) m5[i] = fmaxf(fmaxf(m15[3 * i], m15[3 * i + 1]), m15[3 * i + 2]);
                const float mx = fmaxf(fmaxf(m5[0], m5[1]), fmaxf(fmaxf(m5[2], m5[3]), m5[4])) * sl2;
                if (TR && j >= 8 && j < 12) tr[j - 8][4] = clock64() - t0c;
                grow = mx > m_run + 16.f;     // lazy rescale: only when the max grows by > 2^16 (P <= 2^16: fp32/bf16-safe)
                m_new = grow ? mx : m_run;
                alpha = grow ? ex2_mufu(m_run - m_new) : 1.f;
                const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m_new, -m_new);
                // P = exp2(S scale - m) in two halves of 64 columns, each packed to bf16
                // pairs and written back over S columns already consumed
#pragma unroll
                for (int hf = 0; hf < 2; hf++) {
                    uint32_t pk[32];
#pragma unroll
                    for (int i2 = 0; i2 < 32; i2++) {
                        const int i = hf * 32 + i2;
                        const float2 x = __ffma2_rn(make_float2(s[2 * i], s[2 * i + 1]), sc2, nm2);
                        float2 e;
                        if (2 * i < POLY_FROM) e = make_float2(ex2_mufu(x.x), ex2_mufu(x.y));
                        else e = ex2_poly2(make_float2(fmaxf(x.x, -126.f), fmaxf(x.y, -126.f)));
                        if constexpr (MASK) {      // the poly path has no -inf
                            e.x = 2 * i < nvalid ? e.x : 0.f;
                            e.y = 2 * i + 1 < nvalid ? e.y : 0.f;
                        }
                        acc4[i2 & 3] = __fadd2_rn(acc4[i2 & 3], e);
                        pk[i2] = attn::pack_bf16(e.x, e.y);
                    }
                    attn3::tmem_st32u(tS + hf * 32, pk);
                    if (TR && j >= 8 && j < 12) tr[j - 8][5 + hf] = clock64() - t0c;
                }
            };
            if (nvalid == kTile) phase(std::false_type{});
            else phase(std::true_type{});
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            if (TR && j >= 8 && j < 12) tr[j - 8][7] = clock64() - t0c;
            // S_t(j) arrived => PV_t(j-1) has completed and PV_t(j) waits for this
            // thread's p_full arrival: O_t is quiescent for the lazy rescale
            if (j > 0 && __any_sync(0xffffffffu, grow)) {
#pragma unroll
                for (int ch = 0; ch < 4; ch++) {
                    float ov[32];
                    attn::tmem_ld32(tO + ch * 32, ov);
#pragma unroll
                    for (int i = 0; i < 32; i++) ov[i] *= alpha;
                    attn::tmem_st32(tO + ch * 32, ov);
                }
            }
            const float2 acc = __fadd2_rn(__fadd2_rn(acc4[0], acc4[1]), __fadd2_rn(acc4[2], acc4[3]));
            l_run = l_run * alpha + (acc.x + acc.y);
            m_run = m_new;
            attn::fence_before();
            attn2::arrive(&bars.p_full[t]);
            if (TR && j >= 8 && j < 12) tr[j - 8][3] = clock64() - t0c;
        }
        if (TR && blockIdx.x == 0 && blockIdx.y == 0 && (tid & 127) == 0)
            for (int q = 0; q < 4; q++)
                printf("SM%d j=%d start=%lld s_ready=%lld s_loaded=%lld max=%lld half0=%lld half1=%lld st_done=%lld p_arrived=%lld\n",
                       t, q + 8, tr[q][0], tr[q][1], tr[q][2], tr[q][4], tr[q][5], tr[q][6], tr[q][7], tr[q][3]);
        // ---- epilogue ----
        attn::bar_wait(&bars.o_final, 0);
        attn::fence_after();
        const float inv_l = 1.f / l_run;
        const int64_t qi = q0 + t * kTile + (tid & 127);
#pragma unroll
        for (int ch = 0; ch < 4; ch++) {
            float ov[32];
            attn::tmem_ld32(tO + ch * 32, ov);
            if (qi < a.nq) {
                uint4 *dst = reinterpret_cast<uint4 *>(a.out + (qi * a.H + h) * kD + ch * 32);
#pragma unroll
                for (int c = 0; c < 4; c++)
                    dst[c] = make_uint4(attn::pack_bf16(ov[8 * c] * inv_l, ov[8 * c + 1] * inv_l),
                                        attn::pack_bf16(ov[8 * c + 2] * inv_l, ov[8 * c + 3] * inv_l),
                                        attn::pack_bf16(ov[8 * c + 4] * inv_l, ov[8 * c + 5] * inv_l),
                                        attn::pack_bf16(ov[8 * c + 6] * inv_l, ov[8 * c + 7] * inv_l));
            }
        }
    }
    attn::fence_before();
    __syncthreads();
    if (warp == 9) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

static int run(const uint16_t *q, const uint16_t *kv, const uint16_t *kc, const uint16_t *vc, int64_t nq,
               int64_t nc, int64_t ncur, int H, float scale_log2, uint16_t *out, cudaStream_t st) {
    CUtensorMap mQ, mKV, mKc, mVc;
    const bool okq = attn2::make_map(&mQ, q, uint64_t(nq), uint64_t(H) * kD, uint64_t(H) * kD);
    const bool okkv = nc > 0 ? attn2::make_map(&mKV, kv, uint64_t(2 * H) * nc, kD, kD)
                             : attn2::make_map(&mKV, q, 1, kD, kD);
    const bool okk = ncur > 0 ? attn2::make_map(&mKc, kc, uint64_t(ncur), uint64_t(H) * kD, uint64_t(H) * kD)
                              : attn2::make_map(&mKc, q, 1, kD, kD);
    const bool okv = ncur > 0 ? attn2::make_map(&mVc, vc, uint64_t(ncur), uint64_t(H) * kD, uint64_t(H) * kD)
                              : attn2::make_map(&mVc, q, 1, kD, kD);
    if (!(okq && okkv && okk && okv)) return set_err(QVG_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    const size_t smem = kSmem + 1024;
    dim3 grid(unsigned((nq + 2 * kTile - 1) / (2 * kTile)), unsigned(H));
    attn2::Args args{nq, nc, ncur, H, scale_log2, out};
    nap_args(args);
    static const int poly = [] { const char *e = getenv("QVG_ATTN_POLY"); return e ? atoi(e) : 96; }();
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        kern<<<grid, 320, smem, st>>>(mQ, mKV, mKc, mVc, args);
    };
    static const bool trace = getenv("QVG_ATTN_TRACE") != nullptr;
    if (trace) {
        if (poly >= 96) go(k_attention_pp4<96, true>);
        else if (poly >= 80) go(k_attention_pp4<80, true>);
        else if (poly >= 64) go(k_attention_pp4<64, true>);
        else go(k_attention_pp4<48, true>);
        return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
    }
    if (poly >= 128) go(k_attention_pp4<128>);
    else if (poly >= 96) go(k_attention_pp4<96>);
    else if (poly >= 80) go(k_attention_pp4<80>);
    else if (poly >= 64) go(k_attention_pp4<64>);
    else go(k_attention_pp4<48>);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}
}  // namespace attn4


// ============================================================================
// pre-RoPE key caching: the cache stores keys BEFORE the
// rotary embedding; after the K6 reconstruction the K planes are rotated in
// place with the caller's per-position tables (any 1-D / 3-D RoPE layout
// reduces to cos/sin [n_cache][d/2]): mode 1 = rotate-half pairs (i, i+d/2),
// mode 2 = interleaved pairs (2i, 2i+1).  fp32 math, bf16 RNE store.
// ============================================================================
__global__ void k_rope_kplanes(uint16_t *kv, int64_t H, int64_t n, int d, const float *cosv, const float *sinv,
                               int mode, const uint16_t *src) {
    const int half = d / 2;
    const int64_t total = H * n * half;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e % half);
        const int64_t hn = e / half;
        const int64_t h = hn / n, t = hn - h * n;
        const int64_t base = ((2 * h) * n + t) * d;           // K plane of head h, token t
        const int i0 = mode == 1 ? i : 2 * i, i1 = mode == 1 ? i + half : 2 * i + 1;
        const uint16_t *in = src ? src : kv;
        const float a = bf16_to_f32(in[base + i0]), b = bf16_to_f32(in[base + i1]);
        const float c = cosv[t * half + i], sn = sinv[t * half + i];
        kv[base + i0] = f32_to_bf16_bits_rne(__fsub_rn(__fmul_rn(a, c), __fmul_rn(b, sn)));
        kv[base + i1] = f32_to_bf16_bits_rne(__fadd_rn(__fmul_rn(a, sn), __fmul_rn(b, c)));
    }
}

// copy of the V planes of a bf16 cache into the workspace (the comparator
// path with RoPE: K is rotated out of place, V copied beside it)
__global__ void k_copy_vplanes(const uint16_t *src, uint16_t *dst, int64_t H, int64_t n, int d) {
    const int64_t per = n * d, total = H * per;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t h = e / per, r = e - h * per;
        dst[(2 * h + 1) * per + r] = src[(2 * h + 1) * per + r];
    }
}

int run_rope_cache(uint16_t *ws_kv, const uint16_t *src_kv, int64_t H, int64_t n, int d, const float *cosv,
                   const float *sinv, int mode, cudaStream_t st) {
    const int64_t total = H * n * (d / 2);
    int64_t g = (total + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    if (src_kv) {
        k_copy_vplanes<<<unsigned(g), 256, 0, st>>>(src_kv, ws_kv, H, n, d);
    }
    k_rope_kplanes<<<unsigned(g), 256, 0, st>>>(ws_kv, H, n, d, cosv, sinv, mode, src_kv);
    return cudaGetLastError() == cudaSuccess ? QVG_OK : QVG_ERR_CUDA;
}

size_t attention_workspace_size(int64_t, int64_t n_cache, int64_t, int H, int d, const qvg_config *) {
    // bf16 reconstruction of the quantized cache (2H planes) for the TMA kernel
    return n_cache > 0 ? size_t(2) * H * n_cache * d * 2 + 256 : 0;
}

int run_attention(const uint16_t *q, const uint8_t *payload, const uint8_t *scales,
                  const uint16_t *cent, const uint8_t *assign, const uint16_t *kv_bf16,
                  const uint16_t *k_cur, const uint16_t *v_cur, int64_t nq, int64_t n_cache,
                  int64_t n_cur, int H, int d, const qvg_config *cfg, float scale, uint16_t *out,
                  void *workspace, size_t wbytes, int32_t *status, cudaStream_t st, const float *rope_cos,
                  const float *rope_sin, int rope_mode) {
    using namespace attn;
    if (d != kD) return set_err(QVG_ERR_UNSUPPORTED, "attention kernel supports head_dim 128, got %d", d);
    if (n_cur > 0 && (!k_cur || !v_cur)) return set_err(QVG_ERR_BAD_CONFIG, "k_cur/v_cur are NULL");
    const float sl2 = scale * 1.4426950408889634f;
    const uint16_t *kv = kv_bf16;
    if (rope_mode && (!rope_cos || !rope_sin || d % 2 || rope_mode > 2))
        return set_err(QVG_ERR_BAD_CONFIG, "rope needs cos/sin tables [n_cache][d/2] and mode 1 or 2");
    if (rope_mode && n_cache > 0 && payload && !workspace)
        return set_err(QVG_ERR_WORKSPACE, "pre-RoPE keys need the reconstruction workspace");
    if (n_cache > 0 && payload && !workspace) {
        // no workspace: the fused kernel dequantizes codes/scales/centroids in-tile
        if (cfg->group_size % 8 != 0 || kD % cfg->group_size != 0)
            return set_err(QVG_ERR_UNSUPPORTED, "attention needs group_size | 128 and 8 | group_size");
        AttnArgs ia{q, k_cur, v_cur, nullptr, payload, scales, assign, cent, out, nq, n_cache, n_cur, H,
                    cfg->bits, cfg->group_size, cfg->stages, cfg->centroids, sl2, status};
        int rc = cfg->bits == 2 ? dispatch_s<2>(ia, st) : cfg->bits == 4 ? dispatch_s<4>(ia, st) : dispatch_s<8>(ia, st);
        return rc ? set_err(rc, "attention launch failed: %s", cudaGetErrorString(cudaGetLastError())) : QVG_OK;
    }
    if (n_cache > 0 && payload) {
        // K6: reconstruct the 2H cache planes to bf16 (HBM-bound), then attend
        const size_t need = attention_workspace_size(nq, n_cache, n_cur, H, d, cfg);
        if (wbytes < need) return set_err(QVG_ERR_WORKSPACE, "attention workspace needs %zu bytes", need);
        uint16_t *rec = static_cast<uint16_t *>(workspace);
        int32_t *stw = status;
        if (!stw) {                        // no caller word: a scratch one at the end of the workspace
            stw = reinterpret_cast<int32_t *>(static_cast<uint8_t *>(workspace) + need - 256);
            cudaMemsetAsync(stw, 0, sizeof(int32_t), st);
        }
        int rc = launch_dequantize(payload, scales, cent, assign, 2 * int64_t(H), n_cache, d, cfg->bits,
                                   cfg->group_size, cfg->stages, cfg->centroids, rec, QVG_DTYPE_BF16,
                                   stw, st);
        if (rc) return set_err(rc, "cache reconstruction failed");
        kv = rec;
        if (rope_mode && run_rope_cache(rec, nullptr, H, n_cache, d, rope_cos, rope_sin, rope_mode, st))
            return set_err(QVG_ERR_CUDA, "rope launch failed");
    } else if (n_cache > 0 && kv && rope_mode) {
        // bf16 comparator with pre-RoPE keys: rotated copy in the workspace
        const size_t need = attention_workspace_size(nq, n_cache, n_cur, H, d, cfg);
        if (!workspace || wbytes < need) return set_err(QVG_ERR_WORKSPACE, "rope needs %zu workspace bytes", need);
        uint16_t *rec = static_cast<uint16_t *>(workspace);
        if (run_rope_cache(rec, kv, H, n_cache, d, rope_cos, rope_sin, rope_mode, st))
            return set_err(QVG_ERR_CUDA, "rope launch failed");
        kv = rec;
    } else if (n_cache > 0 && !kv) {
        return set_err(QVG_ERR_BAD_CONFIG, "cache is NULL");
    }
    const int rc = attn4::run(q, kv, k_cur, v_cur, nq, n_cache, n_cur, H, sl2, out, st);
    return rc ? set_err(rc, "attention launch failed: %s", cudaGetErrorString(cudaGetLastError())) : QVG_OK;
}

}  // namespace qvg
