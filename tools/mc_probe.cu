// Ingress probe for the K3 main loop: per K-block every CTA receives a 32 KB "raw" chunk
// (streamed from HBM, distinct per CTA) and a 32 KB "circulant" chunk (L2-resident, the
// same for all CTAs).  Compares the circulant fetched per CTA (unicast) against a cluster
// multicast where each of the `csz` CTAs fetches 1/csz of it for all of them
// (cp.async.bulk ... .multicast::cluster), with a cluster-wide empty barrier per stage.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/mc_probe tools/mc_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../paper_2206_05506_b200/csrc/sm100_ptx.cuh"

using namespace pnce;

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e = (x);                                                                      \
        if (e != cudaSuccess) {                                                                   \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));     \
            exit(1);                                                                              \
        }                                                                                         \
    } while (0)

constexpr int kRaw = 32768, kCirc = 32768, kStages = 3, kStage = kRaw + kCirc;

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_load_mc(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar,
                                             uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}

// flags: 1 = raw stream, 2 = circulant stream; mc = multicast the circulant over the cluster.
__global__ void __launch_bounds__(64, 1) k_probe(const uint8_t* raw, size_t raw_per_cta, const uint8_t* circ,
                                                 size_t circ_bytes, int iters, int flags, int mc, int csz,
                                                 unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t full[kStages], empty[kStages];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const uint32_t rank = csz > 1 ? cluster_ctarank() : 0;
    if (t == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], csz);  // one arrive per consumer CTA of the cluster
        }
        fence_mbar_init();
    }
    if (csz > 1) cluster_sync_all(); else __syncthreads();
    const uint32_t per_stage = ((flags & 1) ? kRaw : 0) + ((flags & 2) ? kCirc : 0);
    if (warp == 0 && lane == 0) {  // producer
        const uint8_t* rb = raw + (size_t)blockIdx.x * raw_per_cta;
        const uint64_t pol = policy_evict_last();
        (void)pol;
        for (int i = 0; i < iters; ++i) {
            const int s = i % kStages;
            if (i >= kStages) mbar_wait_cluster(&empty[s], ((i / kStages) - 1) & 1);
            mbar_arrive_expect_tx(&full[s], per_stage);
            uint8_t* st = smem + s * kStage;
            if (flags & 1) {
                const size_t off = ((size_t)i * kRaw) % raw_per_cta;
                bulk_load(smem_u32(st), rb + off, kRaw / 2, &full[s]);
                bulk_load(smem_u32(st) + kRaw / 2, rb + off + kRaw / 2, kRaw / 2, &full[s]);
            }
            if (flags & 2) {
                const size_t off = ((size_t)i * kCirc) % circ_bytes;
                if (mc && csz > 1) {
                    const uint32_t part = kCirc / csz;
                    bulk_load_mc(smem_u32(st + kRaw) + rank * part, circ + off + rank * part, part, &full[s],
                                 (uint16_t)((1u << csz) - 1));
                } else {
                    bulk_load(smem_u32(st + kRaw), circ + off, kCirc / 2, &full[s]);
                    bulk_load(smem_u32(st + kRaw) + kCirc / 2, circ + off + kCirc / 2, kCirc / 2, &full[s]);
                }
            }
        }
    } else if (warp == 1 && lane == 0) {  // consumer: releases the stage in every CTA of the cluster
        for (int i = 0; i < iters; ++i) {
            const int s = i % kStages;
            mbar_wait(&full[s], (i / kStages) & 1);
            for (int r = 0; r < csz; ++r) {
                if (csz > 1)
                    mbar_arrive_remote(mapa_shared(smem_u32(&empty[s]), r));
                else
                    mbar_arrive(&empty[s]);
            }
        }
        sink[blockIdx.x] = smem[7];
    }
    if (csz > 1) cluster_sync_all();
}

double run(int grid, int csz, const uint8_t* raw, size_t raw_per_cta, const uint8_t* circ, size_t circ_bytes,
           int iters, int flags, int mc, unsigned long long* sink) {
    const int smem = kStages * kStage;
    CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csz;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_probe, raw, raw_per_cta, circ, circ_bytes, iters, flags, mc, csz, sink));
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    const int reps = 5;
    for (int i = 0; i < reps; ++i)
        CK(cudaLaunchKernelEx(&cfg, k_probe, raw, raw_per_cta, circ, circ_bytes, iters, flags, mc, csz, sink));
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e-3 / reps;
}

int main() {
    const int iters = 512;                                // 16 MB raw + 16 MB circulant per CTA
    const size_t raw_per_cta = (size_t)iters * kRaw;      // streamed once (HBM)
    const size_t circ_bytes = 2u << 20;                   // 2 MB L2-resident circulant
    uint8_t *raw, *circ;
    unsigned long long* sink;
    CK(cudaMalloc(&raw, raw_per_cta * 148));
    CK(cudaMemset(raw, 1, raw_per_cta * 148));
    CK(cudaMalloc(&circ, circ_bytes));
    CK(cudaMemset(circ, 2, circ_bytes));
    CK(cudaMalloc(&sink, 148 * 8));
    struct Case {
        const char* name;
        int flags, mc, csz;
    } cases[] = {{"raw only          ", 1, 0, 1}, {"circ only         ", 2, 0, 1}, {"raw+circ unicast  ", 3, 0, 1},
                 {"raw+circ uc  csz2 ", 3, 0, 2}, {"raw+circ mc  csz2 ", 3, 1, 2}, {"raw+circ uc  csz4 ", 3, 0, 4},
                 {"raw+circ mc  csz4 ", 3, 1, 4}, {"circ mc csz2      ", 2, 1, 2}, {"circ mc csz4      ", 2, 1, 4}};
    for (int grid : {148, 144}) {
        for (const Case& c : cases) {
            if (grid % c.csz) continue;
            const double t = run(grid, c.csz, raw, raw_per_cta, circ, circ_bytes, iters, c.flags, c.mc, sink);
            const double per_cta = (double)iters * (((c.flags & 1) ? kRaw : 0) + ((c.flags & 2) ? kCirc : 0));
            printf("grid %3d %s  %8.1f us  %6.2f us/K-block  received %6.1f GB/s per SM (%7.1f total)\n", grid, c.name,
                   t * 1e6, t * 1e6 / iters, per_cta / t / 1e9, grid * per_cta / t / 1e9);
        }
    }
    return 0;
}
