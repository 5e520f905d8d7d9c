// Store-egress probe: how fast can one SM (and all SMs together) push the correlator's
// epilogue output to HBM with different store patterns?
//
// Each CTA (128 threads = the 4 epilogue warps) writes 256 KB = one K3 tile's taps for
// one CTA (64 links x 512 complex lags, 4 KB per link).  Patterns:
//   0 "k3"      : current K3 epilogue -- lane = TMEM row; even/odd lanes of a link write
//                 64 B each per 16-column slice (2 x STG.256), 16 links per instruction
//   1 "coal256" : warp writes 1 KB contiguous per STG.256 instruction
//   2 "coal128" : warp writes 512 B contiguous per STG.128 instruction
//   3 "bulk"    : cp.async.bulk.global.shared::cta of 4 KB per link from a 32 KB smem tile
//   4 "k3x2"    : 16x256b-style: lane quad of a link writes 64 B contiguous (STG.128 x4 lanes)
// Grids: 1 CTA (per-SM egress) and 148 CTAs (aggregate).  Reports GB/s.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/store_probe tools/store_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e = (x);                                                                      \
        if (e != cudaSuccess) {                                                                   \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));     \
            exit(1);                                                                              \
        }                                                                                         \
    } while (0)

constexpr int kLinks = 64, kLags = 512;                       // per CTA tile
constexpr size_t kTileBytes = (size_t)kLinks * kLags * 8;     // 256 KB

__device__ __forceinline__ void stg256(float* p, float a) {
    asm volatile("st.global.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "f"(a) : "memory");
}
__device__ __forceinline__ void stg128(float* p, float a) {
    asm volatile("st.global.v4.f32 [%0], {%1,%1,%1,%1};" ::"l"(p), "f"(a) : "memory");
}

template <int P>
__global__ void __launch_bounds__(128, 1) k_store(float* out, int reps, float val) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int r = 0; r < reps; ++r) {
        float* base = out + ((size_t)blockIdx.x * reps + r) * (kTileBytes / 4);
        if (P == 0) {
            // warp w owns TMEM rows 32w..32w+31 = links 16w..16w+15
            const int link = warp * 16 + (lane >> 1), odd = lane & 1;
            float* row = base + (size_t)link * kLags * 2;
#pragma unroll 4
            for (int s = 0; s < kLags / 16; ++s) {
                float* d = row + 2 * (s * 16 + odd * 8);
                stg256(d, val);
                stg256(d + 8, val);
            }
        } else if (P == 1) {
            float* w = base + (size_t)warp * (kTileBytes / 16);      // 64 KB per warp
#pragma unroll 4
            for (int i = 0; i < (int)(kTileBytes / 4 / 1024); ++i) stg256(w + i * 256 + lane * 8, val);
        } else if (P == 2) {
            float* w = base + (size_t)warp * (kTileBytes / 16);
#pragma unroll 4
            for (int i = 0; i < (int)(kTileBytes / 4 / 512); ++i) stg128(w + i * 128 + lane * 4, val);
        } else if (P == 3) {
            // 8 passes of 32 KB: one thread issues 8 bulk copies of 4 KB (one link row each)
            if (t == 0) {
                const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
                for (int pass = 0; pass < 8; ++pass) {
                    for (int l = 0; l < 8; ++l) {
                        float* d = base + (size_t)(pass * 8 + l) * kLags * 2;
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d),
                                     "r"(s + l * 4096), "r"(4096)
                                     : "memory");
                    }
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                }
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            }
        } else {
            // 16x256b layout: a warp covers 16 links; thread t -> link t/4 (+8), 2 complex at
            // lag 8*rep + 2*(t%4): 4 lanes of a link write 64 B contiguous per instruction
            for (int half = 0; half < 2; ++half) {
                const int link = warp * 16 + half * 8 + (lane >> 2);
                float* row = base + (size_t)link * kLags * 2;
#pragma unroll 4
                for (int rep = 0; rep < kLags / 8; ++rep) stg128(row + 2 * (rep * 8 + 2 * (lane & 3)), val);
            }
        }
    }
}

template <int P>
double run(float* out, int grid, int reps) {
    const int smem = P == 3 ? 32768 : 0;
    if (smem) CK(cudaFuncSetAttribute(k_store<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_store<P><<<grid, 128, smem>>>(out, reps, 1.f);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    const int iters = 5;
    for (int i = 0; i < iters; ++i) k_store<P><<<grid, 128, smem>>>(out, reps, 1.f);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return (double)grid * reps * kTileBytes * iters / (ms * 1e-3) / 1e9;
}

int main() {
    const int reps = 16;
    float* out;
    CK(cudaMalloc(&out, (size_t)148 * reps * kTileBytes));  // 620 MB >> L2
    const char* names[] = {"k3", "coal256", "coal128", "bulk", "k3x2"};
    for (int grid : {1, 148, 296}) {
        const int rp = grid == 1 ? reps : (grid == 296 ? reps / 2 : reps);
        double g[5] = {run<0>(out, grid, rp), run<1>(out, grid, rp), run<2>(out, grid, rp), run<3>(out, grid, rp),
                       run<4>(out, grid, rp)};
        for (int p = 0; p < 5; ++p)
            printf("grid %3d  %-8s %8.1f GB/s total  %6.1f GB/s per CTA\n", grid, names[p], g[p], g[p] / grid);
    }
    CK(cudaFree(out));
    return 0;
}
