// Probe for tcgen05 cta_group::2 (CTA pair, M=256): numerical check of the operand
// split conventions (A rows 0-127 from CTA rank 0, 128-255 from rank 1; B rows
// [0,N/2) from rank 0, [N/2,N) from rank 1; D rows 128r.. in rank r's TMEM) and
// cycles per MMA.  Also exercises: 2-SM TMEM alloc, multicast commit, remote
// mbarrier arrive (mapa), cluster barrier teardown.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma2_probe tools/umma2_probe.cu
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
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

__device__ __forceinline__ uint32_t cluster_rank() { return cluster_ctarank(); }
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) { return mapa_shared(addr, rank); }
__device__ __forceinline__ void mbar_arrive_remote_rel(uint32_t a) { mbar_arrive_cluster(a); }

constexpr int NMAX = 256;
// smem: A 16 KB | B (NMAX/2 rows x 128 B) 16 KB | bars
template <int N, int VAR = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
k_probe2(const __half* __restrict__ a_full, const __half* __restrict__ b_full, int iters, long long* cycles,
         float* d_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + 16384;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768);   // [0] mma done, [1] remote-arrive test
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 32768 + 64);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();

    for (int idx = tid; idx < 128 * 64; idx += 128) {
        int r = idx / 64, k = idx % 64;
        *reinterpret_cast<__half*>(sA + r * 128 + (((k >> 3) ^ (r & 7)) << 4) + (k & 7) * 2) =
            a_full[(rank * 128 + r) * 64 + k];
    }
    for (int idx = tid; idx < (N / 2) * 64; idx += 128) {
        int n = idx / 64, k = idx % 64;
        *reinterpret_cast<__half*>(sB + n * 128 + (((k >> 3) ^ (n & 7)) << 4) + (k & 7) * 2) =
            b_full[(rank * (N / 2) + n) * 64 + k];
    }
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 2);
        mbar_init(&bar[2], 1 << 20);
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

    // remote arrive test: both CTAs arrive on rank 0's bar[1]
    if (tid == 0) mbar_arrive_remote_rel(mapa(smem_u32(&bar[1]), 0));

    const uint32_t idesc = make_idesc_f16(256, N, 0);
    if (rank == 0 && warp == 1 && lane == 0) {
        mbar_wait(&bar[1], 0);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            int ks = it & 3;
            uint32_t dcol = 0;
            if (VAR == 1) { ks = (it >> 1) & 3; dcol = (it & 1) * 256; }          // alternate accumulators
            if (VAR == 2) { ks = it & 3; dcol = ((it >> 2) & 1) * 256; }          // 4 then switch
            const uint64_t ad = make_sdesc(smem_u32(sA) + ks * 32, 16, 1024, 2);
            uint64_t bd = make_sdesc(smem_u32(sB) + ks * 32, 16, 1024, 2);
            if (VAR == 3) bd = make_sdesc(smem_u32(sB) + ((it * 16) % 1024) * 16 % 8192, 128, 128, 0);
            if (VAR == 4) bd = make_sdesc(smem_u32(sB) + ks * 256, 128, 256, 0);
            if (VAR == 5) bd = make_sdesc(smem_u32(sB) + ((it * 16 + 3) % 256) * 16, 128, 128, 0);
            if (VAR == 6) {  // kernel pattern: 4 units (mu = 63 + 254u), k-step s = it / 4
                const int u = it & 3, st = it >> 2;
                const int rho = ((16 * st - (63 + 254 * u)) % 1023 + 1023) % 1023;
                bd = make_sdesc(smem_u32(sB) + (rho % 960) * 16, 128, 128, 0);
            }
            if (VAR == 7) {  // 4 units, same start (no jumps)
                const int st = it >> 2;
                bd = make_sdesc(smem_u32(sB) + ((16 * st) % 960) * 16, 128, 128, 0);
            }
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                ::"r"(tmem + dcol), "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(it > 1)) : "memory");
            if (VAR >= 1 && (it & 7) == 7)
                asm volatile(
                    "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                    ::"r"(smem_u32(&bar[2])), "h"((uint16_t)3) : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
            ::"r"(smem_u32(&bar[0])), "h"((uint16_t)3) : "memory");
        mbar_wait(&bar[0], 0);
        cycles[blockIdx.x / 2] = clock64() - t0;
    }
    // both CTAs: wait for the multicast commit, read own TMEM rows
    mbar_wait(&bar[0], 0);
    tc_fence_after();
    if (blockIdx.x < 2) {
        const int m = rank * 128 + warp * 32 + lane;
        for (int c0 = 0; c0 < N; c0 += 16) {
            float v[16];
            tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
            for (int i = 0; i < 16; ++i) d_out[m * NMAX + c0 + i] = v[i];
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

template <int N, int VAR = 0>
void run(int nsm) {
    const int M = 256, K = 64;
    std::vector<__half> a(M * K), b(N * K);
    std::vector<float> af(M * K), bf(N * K);
    srand(11 + N);
    for (int i = 0; i < M * K; ++i) { a[i] = __float2half((rand() % 2001 - 1000) / 1000.f); af[i] = __half2float(a[i]); }
    for (int i = 0; i < N * K; ++i) { b[i] = __float2half((rand() & 1) ? 1.f : -1.f); bf[i] = __half2float(b[i]); }
    __half *da, *db;
    float* dd;
    long long* dc;
    CK(cudaMalloc(&da, a.size() * 2));
    CK(cudaMalloc(&db, b.size() * 2));
    CK(cudaMalloc(&dd, 256 * NMAX * 4));
    CK(cudaMalloc(&dc, nsm * 8));
    CK(cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice));
    const int smem = 32768 + 128 + 1024;
    CK(cudaFuncSetAttribute(k_probe2<N, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem + 160000));
    k_probe2<N, VAR><<<2, 128, smem + 160000>>>(da, db, 4, dc, dd);   // big smem -> 1 CTA per SM
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> d(256 * NMAX);
    CK(cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost));
    double err = 0, mx = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double ref = 0;
            for (int k = 0; k < K; ++k) ref += (double)af[m * K + k] * bf[n * K + k];
            err = fmax(err, fabs(ref - d[m * NMAX + n]));
            mx = fmax(mx, fabs(ref));
        }
    const int iters = 8192;
    k_probe2<N, VAR><<<nsm, 128, smem + 160000>>>(da, db, iters, dc, dd);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<long long> c(nsm / 2);
    CK(cudaMemcpy(c.data(), dc, c.size() * 8, cudaMemcpyDeviceToHost));
    long long cm = 0;
    for (auto x : c) cm = x > cm ? x : cm;
    const double floor_c = 256.0 * N / 512.0;
    printf("var%d 2CTA M=256 N=%3d  err=%.2e (ref max %.1f)  cyc/mma=%.1f floor=%.0f eff=%.1f%%\n", VAR, N, err, mx,
           (double)cm / iters, floor_c, 100.0 * floor_c * iters / cm);
    cudaFree(da); cudaFree(db); cudaFree(dd); cudaFree(dc);
}

int main() {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    run<128, 3>(nsm);
    run<128, 6>(nsm);
    run<128, 7>(nsm);
    run<256, 6>(nsm);
    return 0;
}
