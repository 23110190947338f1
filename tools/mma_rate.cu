// Microbenchmark: steady-state rate of the attention kernel's tcgen05 MMA
// groups (bf16 -> f32, M = 128, cta_group::1) issued back to back by one
// thread, one CTA per SM.  mode 0: S-type 128x128x128 (A, B from SW128 shared
// memory, both K-major); 1: PV-type (A from TMEM, B MN-major SW128);
// 2: alternating S / PV (the pp4 issue order); 3: S-type with N = 256;
// 4: two S-type groups with N = 64; 5: two PV-type groups with K = 64;
// 6: PV64 S64 PV64 S64 (64-token blocks).  The second argument runs 8 more
// warps that load 32-column chunks of TMEM and store one back in a loop (the
// softmax's TMEM traffic) while the MMAs run.
// Prints cycles per group (clock64 of the issuing thread, commit -> mbarrier).
// Results: profiles/r02/mma_rate_r02g.txt.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_rate tools/mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFFu);
    d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc(bool b_mn_major, uint32_t n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(b_mn_major) << 16) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                 "r"(a), "l"(b), "r"(id), "r"(acc));
}

__global__ void __launch_bounds__(288, 1) k_rate(int mode, int groups, long long *out, int ldst) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tmem_base;
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    if (threadIdx.x >= 32 && ldst) {
        // 8 softmax-like warps: load 64 S columns of their lane quadrant, store 32 P columns, repeat
        const int w = threadIdx.x >> 5;
        const uint32_t ta = tm + 256 + ((w >> 2) & 1) * 128 + (uint32_t((w & 3) * 32) << 16);
        uint32_t acc = 0;
        while (!done) {
            uint32_t r[32];
            for (int c = 0; c < ldst; c++) {
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                             "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                             : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                               "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                               "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                               "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                               "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                             : "r"(ta + 32 * (c & 1)));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                for (int i = 0; i < 32; i++) acc += r[i];
            }
            for (int i = 0; i < 32; i++) r[i] += acc;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                         "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta + 64),
                         "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
                         "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
                         "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
                         "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
                         : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        if (acc == 0x12345678u) out[200] = acc;
    }
    if (threadIdx.x == 0) {
        const uint32_t sq = su32(sm), sk = su32(sm + 32768), sv = su32(sm + 65536), sk2 = su32(sm + 98304);
        auto S = [&](int t) {
            for (int k = 0; k < 8; k++) {
                const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
                mma_ss(tm + t * 128, desc_sw128(sq + off, 16, 1024), desc_sw128(sk + off, 16, 1024), idesc(false, 128), k > 0);
            }
        };
        auto PV = [&](int t) {
            for (int k = 0; k < 8; k++)
                mma_ts(tm + 256 + t * 128, tm + t * 128 + k * 8, desc_sw128(sv + k * 2048, 16384, 1024), idesc(true, 128), 1);
        };
        auto S256 = [&]() {
            for (int k = 0; k < 8; k++) {
                const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
                mma_ss(tm, desc_sw128(sq + off, 16, 1024), desc_sw128(sk + off, 16, 1024), idesc(false, 256), k > 0);
            }
            (void)sk2;
        };
        auto S64 = [&](int t) {            // 128 x 64 x 128 (N = 64)
            for (int k = 0; k < 8; k++) {
                const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
                mma_ss(tm + 256 + t * 64, desc_sw128(sq + off, 16, 1024), desc_sw128(sk + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024),
                       idesc(false, 64), k > 0);
            }
        };
        auto PV64 = [&](int t) {           // 128 x 128 x 64 (K = 64 tokens, A from TMEM)
            for (int k = 0; k < 4; k++)
                mma_ts(tm + t * 128, tm + 256 + t * 64 + k * 8, desc_sw128(sv + k * 2048, 8192, 1024), idesc(true, 128), 1);
        };
        const long long t0 = clock64();
        for (int g = 0; g < groups; g++) {
            if (mode == 0) S(g & 1);
            else if (mode == 1) PV(g & 1);
            else if (mode == 2) { if (g & 1) PV((g >> 1) & 1); else S((g >> 1) & 1); }
            else if (mode == 3) S256();
            else if (mode == 4) { S64(g & 1); S64((g & 1) + 2); }
            else if (mode == 5) { PV64(g & 1); PV64((g & 1) ^ 1); }
            else { PV64(0); S64(2); PV64(1); S64(3); }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}" ::"r"(su32(&bar))
                     : "memory");
        const long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
        done = 1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
    long long *d, h[148];
    cudaMalloc(&d, 256 * sizeof(long long));
    const int smem = 160 * 1024 + 1024;
    cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char *names[7] = {"S  (SS, K-major B)", "PV (TS, MN-major B)", "S/PV alternating", "S N=256 (SS)",
                            "2x S N=64", "2x PV K=64", "PV64 S64 PV64 S64"};
    for (int ldst : {0, 1, 2, 4})
    for (int grid : {148})
        for (int mode = 0; mode < 7; mode++) {
            const int groups = 400;
            if (ldst) printf("[8 warps: %d x tcgen05.ld.x32 + 1 x st.x32 in a loop] ", ldst);
            k_rate<<<grid, 288, smem>>>(mode, groups, d, ldst);
            k_rate<<<grid, 288, smem>>>(mode, groups, d, ldst);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < grid; i++) mx = h[i] > mx ? h[i] : mx;
            printf("grid %3d  %-22s %7.1f cycles/group (floor %d)\n", grid, names[mode], double(mx) / groups,
                   mode == 3 ? 1024 : mode == 6 ? 1024 : 512);
        }
    return 0;
}
