// Ingress probe: per-SM and aggregate bulk-copy (TMA engine) read bandwidth into shared
// memory, from HBM (streaming) and from an L2-resident buffer (like the circulant rows),
// alone and while the same CTA stores (egress) -- the K3 mainloop's raw/circulant loads
// overlapped with an epilogue drain.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/load_probe tools/load_probe.cu
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

constexpr int kChunk = 16384, kSlots = 8;  // 128 KB in flight

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void stg256(float* p, float a) {
    asm volatile("st.global.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "f"(a) : "memory");
}

// mode 0: loads only; mode 1: loads + stores by warps 1..3 (stores sized to `store_bytes` per CTA)
__global__ void __launch_bounds__(128, 1) k_load(const uint8_t* src, size_t cta_stride, size_t wrap, int chunks,
                                                 float* out, size_t store_bytes, int mode, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bars[kSlots];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    if (t == 0) {
        for (int s = 0; s < kSlots; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint8_t* base = src + (size_t)blockIdx.x * cta_stride;
    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < chunks; ++i) {
                const int s = i % kSlots;
                if (i >= kSlots) mbar_wait(&bars[s], ((i / kSlots) - 1) & 1);
                mbar_arrive_expect_tx(&bars[s], kChunk);
                const size_t off = ((size_t)i * kChunk) % wrap;
                bulk_load(smem_u32(smem + s * kChunk), base + off, kChunk, &bars[s]);
            }
            for (int i = chunks; i < chunks + kSlots; ++i) {
                const int s = i % kSlots;
                if (i >= kSlots) mbar_wait(&bars[s], ((i / kSlots) - 1) & 1);
            }
            sink[blockIdx.x] = smem[5];
        }
    } else if (mode == 1) {
        float* o = out + (size_t)blockIdx.x * (store_bytes / 4) + (size_t)(warp - 1) * (store_bytes / 12);
        const int n = (int)(store_bytes / 3 / 1024);
        for (int i = 0; i < n; ++i) stg256(o + (size_t)i * 256 + lane * 8, 1.f);
    }
}

double timeit(int grid, const uint8_t* src, size_t per_cta, int chunks, float* out, size_t store_bytes, int mode,
              unsigned long long* sink) {
    const size_t wrap = per_cta ? per_cta : kChunk;
    const int smem = kChunk * kSlots;
    CK(cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_load<<<grid, 128, smem>>>(src, per_cta, wrap, chunks, out, store_bytes, mode, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    const int iters = 5;
    for (int i = 0; i < iters; ++i) k_load<<<grid, 128, smem>>>(src, per_cta, wrap, chunks, out, store_bytes, mode, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e-3 / iters;
}


// LDG ingress: `warps` warps stream 16-byte loads (8 in flight per thread) from a per-CTA
// region; optional concurrent bulk loads by warp 0 (mode 2).
__global__ void __launch_bounds__(512, 1) k_ldg(const float4* src, size_t per_cta_f4, int iters,
                                                unsigned long long* sink, int ldg_warps, int bulk_chunks,
                                                const uint8_t* bsrc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bars[kSlots];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    if (t == 0) {
        for (int s = 0; s < kSlots; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0 && bulk_chunks > 0) {
            const uint8_t* base = bsrc + (size_t)blockIdx.x * (64 << 10);
            for (int i = 0; i < bulk_chunks; ++i) {
                const int s = i % kSlots;
                if (i >= kSlots) mbar_wait(&bars[s], ((i / kSlots) - 1) & 1);
                mbar_arrive_expect_tx(&bars[s], kChunk);
                bulk_load(smem_u32(smem + s * kChunk), base + ((size_t)i * kChunk) % (64 << 10), kChunk, &bars[s]);
            }
            for (int i = bulk_chunks; i < bulk_chunks + kSlots; ++i) {
                const int s = i % kSlots;
                if (i >= kSlots) mbar_wait(&bars[s], ((i / kSlots) - 1) & 1);
            }
        }
        return;
    }
    if (warp > ldg_warps) return;
    const float4* b = src + (size_t)blockIdx.x * per_cta_f4;
    const int nthr = ldg_warps * 32, me = (warp - 1) * 32 + lane;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(b + (((size_t)it * 8 + u) * nthr + me) % per_cta_f4);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
    if (acc == 1234.5f) sink[blockIdx.x] = 1;
}

double time_ldg(int grid, const float4* src, size_t per_cta_f4, int iters, unsigned long long* sink, int warps,
                int bulk_chunks, const uint8_t* bsrc) {
    const int smem = kChunk * kSlots;
    CK(cudaFuncSetAttribute(k_ldg, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_ldg<<<grid, 512, smem>>>(src, per_cta_f4, iters, sink, warps, bulk_chunks, bsrc);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) k_ldg<<<grid, 512, smem>>>(src, per_cta_f4, iters, sink, warps, bulk_chunks, bsrc);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e-3 / 5;
}

int main() {
    const size_t big = (size_t)148 * 4 * 1024 * 1024;  // 4 MB per CTA stream, 592 MB total
    uint8_t* src;
    float* out;
    unsigned long long* sink;
    CK(cudaMalloc(&src, big));
    CK(cudaMemset(src, 1, big));
    CK(cudaMalloc(&out, (size_t)148 * 2 * 1024 * 1024));
    CK(cudaMalloc(&sink, 148 * 8));
    const int chunks = 256;  // 4 MB per CTA
    const double bytes = (double)chunks * kChunk;
    for (int grid : {1, 148}) {
        double t_hbm = timeit(grid, src, 4 << 20, chunks, out, 0, 0, sink);
        double t_l2 = timeit(grid, src, 64 << 10, chunks, out, 0, 0, sink);  // each CTA re-reads its own 64 KB
        double t_l2_shared = timeit(grid, src, 0, chunks, out, 0, 0, sink);  // every CTA reads the same 16 KB
        printf("grid %3d  load HBM %7.1f GB/s per CTA (%8.1f total) | L2-resident 64KB/CTA %7.1f | same 16KB all CTAs %7.1f\n",
               grid, bytes / t_hbm / 1e9, grid * bytes / t_hbm / 1e9, bytes / t_l2 / 1e9, bytes / t_l2_shared / 1e9);
        // loads (L2-resident) overlapped with 1 MB of stores per CTA
        const size_t sb = (size_t)3 * 1024 * 1024 / 2;  // 1.5 MB
        double t_both = timeit(grid, src, 64 << 10, chunks, out, sb, 1, sink);
        double t_st = timeit(grid, src, 64 << 10, 1, out, sb, 1, sink);
        printf("grid %3d  L2 loads 4 MB + stores 1.5 MB: %.1f us (stores alone %.1f us, loads alone %.1f us)\n", grid,
               t_both * 1e6, t_st * 1e6, t_l2 * 1e6);
    }
    // LDG path: 4 MB per CTA streamed from HBM (per-CTA region) and from a 64 KB L2-resident region
    for (int grid : {1, 148}) {
        for (int warps : {4, 8, 15}) {
            const int nthr = warps * 32;
            const int iters = (int)((4u << 20) / 16 / 8 / nthr);
            const double by = (double)iters * 8 * nthr * 16;
            double th = time_ldg(grid, (const float4*)src, (4u << 20) / 16, iters, sink, warps, 0, src);
            double tl = time_ldg(grid, (const float4*)src, (64u << 10) / 16, iters, sink, warps, 0, src);
            double tb = time_ldg(grid, (const float4*)src, (64u << 10) / 16, iters, sink, warps, chunks, src);
            printf("grid %3d LDG %2d warps: HBM %6.1f GB/s/CTA | L2 %6.1f GB/s/CTA | L2 LDG + 4 MB bulk: %.1f us (LDG alone %.1f us, bulk alone %.1f us)\n",
                   grid, warps, by / th / 1e9, by / tl / 1e9, tb * 1e6, tl * 1e6,
                   timeit(grid, src, 64 << 10, chunks, out, 0, 0, sink) * 1e6);
        }
    }
    return 0;
}
