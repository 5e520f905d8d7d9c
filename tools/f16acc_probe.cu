// Probe: tcgen05.mma kind::f16 with an F16 accumulator (c_format = 0) -- TMEM layout of D,
// rounding/saturation behaviour, and speed relative to the F32 accumulator.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/f16acc_probe tools/f16acc_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

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

constexpr int N = 128;

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
    tmem_ld32_nowait(taddr, r);
    tmem_wait_ld();
}

// A[m][k], B[n][k] given in global (128 x 64 and N x 64 fp16); D = sum over K=64 (4 MMAs),
// repeated `reps` times with accumulate (D grows by reps).  Output: raw 32-bit TMEM words
// of columns [0, 128) for every lane.
__global__ void __launch_bounds__(128, 1) k_probe(const __half* a, const __half* b, int f16acc, int reps,
                                                  uint32_t* out, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = smem;
    uint8_t* sb = smem + 16384;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + N * 128);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int idx = tid; idx < 128 * 64; idx += 128) {
        const int r = idx / 64, k = idx % 64;
        *reinterpret_cast<__half*>(sa + r * 128 + (((k >> 3) ^ (r & 7)) << 4) + (k & 7) * 2) = a[idx];
    }
    for (int idx = tid; idx < N * 64; idx += 128) {
        const int r = idx / 64, k = idx % 64;
        *reinterpret_cast<__half*>(sb + r * 128 + (((k >> 3) ^ (r & 7)) << 4) + (k & 7) * 2) = b[idx];
    }
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) tmem_alloc(slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    uint32_t idesc = make_idesc_f16(128, N, 0);
    if (f16acc) idesc &= ~(3u << 4);  // c_format = F16
    if (warp == 1 && lane == 0) {
        const long long t0 = clock64();
        for (int it = 0; it < reps * 4; ++it) {
            const int ks = it & 3;
            umma_f16_ss(tmem, make_sdesc(smem_u32(sa) + ks * 32, 16, 1024, 2), make_sdesc(smem_u32(sb) + ks * 32, 16, 1024, 2),
                        idesc, it > 0);
        }
        umma_commit(bar);
        mbar_wait(bar, 0);
        cyc[0] = clock64() - t0;
    }
    __syncthreads();
    tc_fence_after();
    const int m = warp * 32 + lane;
    for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t r[32];
        ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, r);
        for (int i = 0; i < 32; ++i) out[m * 128 + c0 + i] = r[i];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

int main() {
    std::vector<__half> a(128 * 64), b(N * 64);
    // D[m][n] = sum_k A[m][k] B[n][k] with A[m][0] = m/4, A[m][1] = 1, B[n][0] = 1, B[n][1] = n
    for (int m = 0; m < 128; ++m)
        for (int k = 0; k < 64; ++k) a[m * 64 + k] = __float2half(k == 0 ? m * 0.25f : (k == 1 ? 1.f : 0.f));
    for (int n = 0; n < N; ++n)
        for (int k = 0; k < 64; ++k) b[n * 64 + k] = __float2half(k == 0 ? 1.f : (k == 1 ? (float)n : 0.f));
    __half *da, *db;
    uint32_t* dout;
    long long* dc;
    CK(cudaMalloc(&da, a.size() * 2));
    CK(cudaMalloc(&db, b.size() * 2));
    CK(cudaMalloc(&dout, 128 * 128 * 4));
    CK(cudaMalloc(&dc, 8));
    CK(cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice));
    const int smem = 16384 + N * 128 + 64 + 1024;
    CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    std::vector<uint32_t> out(128 * 128);
    for (int f16 = 0; f16 < 2; ++f16) {
        for (int reps : {1, 1000}) {
            k_probe<<<1, 128, smem>>>(da, db, f16, reps, dout, dc);
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
            long long cyc;
            CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
            printf("== accumulator %s, reps %d: %lld cycles (%.1f per MMA)\n", f16 ? "F16" : "F32", reps, cyc,
                   (double)cyc / (reps * 4));
            for (int m : {0, 1, 5, 127}) {
                printf("  lane %3d:", m);
                for (int c = 0; c < 6; ++c) {
                    const uint32_t w = out[m * 128 + c];
                    if (f16) {
                        __half_raw lo, hi;
                        lo.x = (unsigned short)(w & 0xffff);
                        hi.x = (unsigned short)(w >> 16);
                        printf(" [%g|%g]", __half2float(__half(lo)), __half2float(__half(hi)));
                    } else {
                        float f;
                        memcpy(&f, &w, 4);
                        printf(" %g", f);
                    }
                }
                printf("  ... col 63/64/127: %08x %08x %08x\n", out[m * 128 + 63], out[m * 128 + 64], out[m * 128 + 127]);
            }
        }
    }
    return 0;
}
