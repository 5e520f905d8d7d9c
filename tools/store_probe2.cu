// Per-SM store egress vs the number of storing warps (one CTA on one SM, and one CTA per SM on
// all SMs): can the drain go faster with the idle converter warps helping?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/store_probe2 tools/store_probe2.cu
#include <cuda_runtime.h>

#include <cstdio>

constexpr size_t kTileBytes = 256 * 1024;  // one CTA's taps per K3 tile

__global__ void k_store(float* out, int reps, int pattern) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
    for (int r = 0; r < reps; ++r) {
        float* base = out + ((size_t)blockIdx.x * reps + r) * (kTileBytes / 4);
        if (pattern == 0) {  // coalesced: warp w writes its contiguous slice, 512 B per instruction
            const size_t per = kTileBytes / 4 / nw;
            float* w = base + (size_t)warp * per;
            for (size_t i = 0; i + 128 <= per; i += 128)
                asm volatile("st.global.v4.f32 [%0], {%1,%1,%1,%1};" ::"l"(w + i + lane * 4), "f"(1.f) : "memory");
        } else {  // epilogue-like: 64 links x 4 KB runs, 4 lanes per link write 64 B per instruction
            for (int link = warp * 8 + (lane >> 2); link < 64; link += nw * 8) {
                float* row = base + (size_t)link * 1024;
                for (int rep = 0; rep < 64; ++rep)
                    asm volatile("st.global.v4.f32 [%0], {%1,%1,%1,%1};" ::"l"(row + 16 * rep + 4 * (lane & 3)),
                                 "f"(1.f)
                                 : "memory");
            }
        }
    }
}

int main() {
    const int reps = 16;
    float* out;
    if (cudaMalloc(&out, (size_t)148 * reps * kTileBytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    setvbuf(stdout, nullptr, _IONBF, 0);
    for (int pattern = 0; pattern < 2; ++pattern)
        for (int grid : {1, 74, 148})
            for (int warps : {4, 8, 16}) {
                k_store<<<grid, warps * 32>>>(out, reps, pattern);
                if (cudaDeviceSynchronize() != cudaSuccess) { printf("kernel error\n"); return 1; }
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                cudaEventRecord(a);
                for (int i = 0; i < 5; ++i) k_store<<<grid, warps * 32>>>(out, reps, pattern);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                const double gbs = (double)grid * reps * kTileBytes * 5 / (ms * 1e-3) / 1e9;
                printf("%s grid %3d warps %2d: %7.1f GB/s total, %6.1f per SM\n", pattern ? "epi " : "coal", grid, warps,
                       gbs, gbs / grid);
            }
    return 0;
}
