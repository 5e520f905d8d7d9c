// Probe: tcgen05.mma.cta_group::2 with M = 128 (64 A rows per CTA).  Where does D land in
// each CTA's TMEM (which lanes / columns), may the D address carry a lane offset (a second
// accumulator in the other lane half), and what does one MMA cost vs M = 256?
// D[m][n] = (m+1) + 256 (n+1) (A[m] = {m+1, 256, 0..}, B[n] = {1, n+1, 0..}): exact in fp32,
// so every written TMEM word names its (m, n).  Unwritten words keep the sentinel -1.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/umma_m128_probe tools/umma_m128_probe.cu
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2206_05506_b200/csrc/sm100_ptx.cuh"

using namespace pnce;

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

// smem: A (64 rows x 128 B = 8 KB, padded to 16 KB) | B (N/2 rows x 128 B <= 16 KB) | bars
template <int M, int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
k_m128(const __half* __restrict__ a_full, const __half* __restrict__ b_full, uint32_t d_off, int iters,
       long long* cycles, float* d_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + 16384;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768);
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 32768 + 64);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_ctarank();
    constexpr int kRows = M / 2;  // A rows per CTA
    for (int idx = tid; idx < kRows * 64; idx += 128) {
        int r = idx / 64, k = idx % 64;
        *reinterpret_cast<__half*>(sA + r * 128 + (((k >> 3) ^ (r & 7)) << 4) + (k & 7) * 2) =
            a_full[(rank * kRows + r) * 64 + k];
    }
    for (int idx = tid; idx < (N / 2) * 64; idx += 128) {
        int n = idx / 64, k = idx % 64;
        *reinterpret_cast<__half*>(sB + n * 128 + (((k >> 3) ^ (n & 7)) << 4) + (k & 7) * 2) =
            b_full[(rank * (N / 2) + n) * 64 + k];
    }
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 2);
        fence_mbar_init();
    }
    fence_proxy_async_smem();
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *slot;
    {  // sentinel everywhere
        uint32_t s[32];
        for (int i = 0; i < 32; ++i) s[i] = __float_as_uint(-1.f);
        for (int c = 0; c < 512; c += 32) tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + c, s);
        tmem_wait_st();
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    if (tid == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&bar[1]), 0));
    const uint32_t idesc = make_idesc_f16(M, N, 0);
    if (rank == 0 && warp == 1 && lane == 0) {
        mbar_wait(&bar[1], 0);
        const uint64_t ad = make_sdesc(smem_u32(sA), 16, 1024, 2);
        const uint64_t bd = make_sdesc(smem_u32(sB), 16, 1024, 2);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it)
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                ::"r"(tmem + d_off), "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(it > 0 && iters > 1 ? 0 : 0))
                : "memory");
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
            ::"r"(smem_u32(&bar[0])), "h"((uint16_t)3) : "memory");
        mbar_wait(&bar[0], 0);
        cycles[blockIdx.x / 2] = clock64() - t0;
    }
    mbar_wait(&bar[0], 0);
    tc_fence_after();
    if (blockIdx.x < 2) {
        const int row = warp * 32 + lane;
        for (int c0 = 0; c0 < 512; c0 += 16) {
            float v[16];
            tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
            for (int i = 0; i < 16; ++i) d_out[((size_t)rank * 128 + row) * 512 + c0 + i] = v[i];
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

template <int M, int N>
void run(uint32_t d_off, int nsm, const char* tag) {
    std::vector<__half> a(M * 64, __float2half(0.f)), b(N * 64, __float2half(0.f));
    for (int m = 0; m < M; ++m) { a[m * 64] = __float2half((float)(m + 1)); a[m * 64 + 1] = __float2half(256.f); }
    for (int n = 0; n < N; ++n) { b[n * 64] = __float2half(1.f); b[n * 64 + 1] = __float2half((float)(n + 1)); }
    __half *da, *db;
    float* dd;
    long long* dc;
    CK(cudaMalloc(&da, a.size() * 2));
    CK(cudaMalloc(&db, b.size() * 2));
    CK(cudaMalloc(&dd, 2 * 128 * 512 * 4));
    CK(cudaMalloc(&dc, nsm * 8));
    CK(cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice));
    const int smem = 32768 + 128 + 1024 + 160000;
    CK(cudaFuncSetAttribute(k_m128<M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_m128<M, N><<<2, 128, smem>>>(da, db, d_off, 1, dc, dd);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("%s M=%d N=%d d_off=0x%x: launch error %s\n", tag, M, N, d_off, cudaGetErrorString(e));
        exit(0);
    }
    std::vector<float> d(2 * 128 * 512);
    CK(cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost));
    printf("== %s M=%d N=%d d_off=0x%x\n", tag, M, N, d_off);
    for (int r = 0; r < 2; ++r) {
        int bad = 0, written = 0;
        for (int lane = 0; lane < 128; ++lane) {
            int c_lo = -1, c_hi = -1, m_lo = 1 << 30, m_hi = -1, n_lo = 1 << 30, n_hi = -1;
            for (int c = 0; c < 512; ++c) {
                const float v = d[((size_t)r * 128 + lane) * 512 + c];
                if (v == -1.f) continue;
                const int iv = (int)v;
                const int m = iv % 256 - 1, n = iv / 256 - 1;
                if ((float)iv != v || m < 0 || m >= M || n < 0 || n >= N) { ++bad; continue; }
                ++written;
                if (c_lo < 0) c_lo = c;
                c_hi = c;
                m_lo = m < m_lo ? m : m_lo; m_hi = m > m_hi ? m : m_hi;
                n_lo = n < n_lo ? n : n_lo; n_hi = n > n_hi ? n : n_hi;
            }
            if (c_lo >= 0 && (lane % 16 == 0 || lane % 16 == 15))
                printf("  cta%d lane %3d: cols %3d-%3d  m %3d-%3d  n %3d-%3d\n", r, lane, c_lo, c_hi, m_lo, m_hi, n_lo,
                       n_hi);
        }
        printf("  cta%d: %d words written, %d undecodable\n", r, written, bad);
    }
    // throughput: 4096 MMAs per pair on every SM pair
    k_m128<M, N><<<nsm, 128, smem>>>(da, db, d_off, 4096, dc, dd);
    CK(cudaDeviceSynchronize());
    std::vector<long long> c(nsm / 2);
    CK(cudaMemcpy(c.data(), dc, c.size() * 8, cudaMemcpyDeviceToHost));
    long long cm = 0;
    for (auto x : c) cm = x > cm ? x : cm;
    printf("  cycles per MMA (max over pairs): %.1f  (MACs/cycle/pair %.0f)\n", (double)cm / 4096,
           (double)M * N * 16 * 4096 / cm);
    cudaFree(da); cudaFree(db); cudaFree(dd); cudaFree(dc);
}

int main(int argc, char** argv) {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    const int v = argc > 1 ? atoi(argv[1]) : 0;
    if (v == 0) run<256, 256>(0, nsm, "ref M=256");
    if (v == 1) run<128, 256>(0, nsm, "M=128");
    if (v == 2) run<128, 256>(256, nsm, "M=128 col 256");
    if (v == 3) run<128, 256>(64u << 16, nsm, "M=128 lane 64");
    if (v == 4) run<128, 256>(32u << 16, nsm, "M=128 lane 32");
    if (v == 5) run<128, 256>(16u << 16, nsm, "M=128 lane 16");
    return 0;
}
