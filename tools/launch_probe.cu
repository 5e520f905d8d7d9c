// Fixed-cost probe for the single frame-set latency: back-to-back launches of near-empty
// kernels with the correlator's launch shape (512 threads, 2-CTA cluster, 227 KB dynamic
// shared memory, TMEM alloc/dealloc), each variant timed with CUDA events over 200 launches.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__global__ void __cluster_dims__(2, 1, 1) k_empty_cluster(int* p) { if (p && threadIdx.x == 9999) p[0] = 1; }
__global__ void k_empty(int* p) { if (p && threadIdx.x == 9999) p[0] = 1; }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) k_tmem(int* p) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)), "r"(512) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512) : "memory");
    if (p && threadIdx.x == 9999) p[0] = 1;
}

template <typename F>
float time_it(F launch, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 20; ++i) launch();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1000.f / reps;
}

int main() {
    const int smem = 227 * 1024;
    cudaFuncSetAttribute(k_empty_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int reps = 200;
    printf("empty 32 thr, grid 2, no smem         : %6.2f us/launch\n", time_it([&] { k_empty<<<2, 32>>>(nullptr); }, reps));
    printf("empty 512 thr, cluster 2, no smem     : %6.2f us/launch\n", time_it([&] { k_empty_cluster<<<2, 512>>>(nullptr); }, reps));
    printf("empty 512 thr, cluster 2, 227 KB smem : %6.2f us/launch\n", time_it([&] { k_empty_cluster<<<2, 512, smem>>>(nullptr); }, reps));
    printf("empty 512 thr, cluster 2, 227 KB, g32 : %6.2f us/launch\n", time_it([&] { k_empty_cluster<<<32, 512, smem>>>(nullptr); }, reps));
    printf("tmem alloc/dealloc, 227 KB            : %6.2f us/launch\n", time_it([&] { k_tmem<<<2, 512, smem>>>(nullptr); }, reps));
    printf("tmem alloc/dealloc, 227 KB, grid 148  : %6.2f us/launch\n", time_it([&] { k_tmem<<<148, 512, smem>>>(nullptr); }, reps));
    // single launch latency (event around ONE launch, after an idle gap)
    float tot = 0;
    for (int i = 0; i < 50; ++i) {
        cudaDeviceSynchronize();
        tot += time_it([&] { k_tmem<<<2, 512, smem>>>(nullptr); }, 1);
    }
    printf("tmem kernel, single launch (idle gap) : %6.2f us\n", tot / 50);
    return 0;
}
