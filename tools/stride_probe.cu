// DRAM access-pattern probe with TMA 2-D boxes (the fused kernel's raw-chunk load): every CTA
// streams its own slab of a row-major f32 tensor into an 8-slot shared-memory ring, one box
// per slot, and the aggregate read bandwidth is reported for (a) the fused kernel's box
// [64 rows x 64 floats] over rows of 2300 floats (9200 B), (b) the same box over a tensor
// whose rows are exactly 64 floats (contiguous 16 KB boxes), (c) [16 rows x 256 floats].
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#ifndef SLOTS
#define SLOTS 8
#endif
constexpr int kSlots = SLOTS;

__global__ void __launch_bounds__(32, 1) k_stream(const __grid_constant__ CUtensorMap tm, int box_bytes, int cols_boxes,
                                                   int rows_per_cta, int box_rows, int chunks, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t full[kSlots];
    if (threadIdx.x == 0) {
        for (int s = 0; s < kSlots; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    if (threadIdx.x != 0) return;
    unsigned long long acc = 0;
    const int row0 = blockIdx.x * rows_per_cta;
    for (int c = 0; c < chunks + kSlots; ++c) {
        if (c >= kSlots) {
            const int s = (c - kSlots) % kSlots;
            const uint32_t par = ((c - kSlots) / kSlots) & 1;
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.b32 %0,1,0,p;}"
                             : "=r"(ok) : "r"(su32(&full[s])), "r"(par));
            acc += sm[s * box_bytes];
        }
        if (c < chunks) {
            const int s = c % kSlots;
            // chunk c: column box c % cols_boxes of row block c / cols_boxes (row-block-major walk,
            // like a CTA walking its tile's K-blocks, then the next tile)
            const int cb = c % cols_boxes, rb = c / cols_boxes;
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(box_bytes));
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(su32(sm + s * box_bytes)), "l"(&tm), "r"(cb * (box_bytes / box_rows / 4)),
                           "r"(row0 + (rb * box_rows) % rows_per_cta), "r"(su32(&full[s])) : "memory");
        }
    }
    if (acc == 12345) sink[0] = acc;
}

int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    const int grid = 148;
    const size_t total = 36ull << 30;
    float* buf;
    CK(cudaMalloc(&buf, total));
    CK(cudaMemset(buf, 1, total));
    unsigned long long* sink;
    CK(cudaMalloc(&sink, 8));
    struct Case { const char* name; int row_floats, box_cols, box_rows; } cases[] = {
        {"box 64 rows x 64 f32, row 9200 B (fused raw chunk)", 2300, 64, 64},
        {"box 64 rows x 64 f32, row 256 B (contiguous 16 KB)", 64, 64, 64},
        {"box 16 rows x 256 f32, row 9200 B                  ", 2300, 256, 16},
        {"box 32 rows x 128 f32, row 9200 B                  ", 2300, 128, 32},
    };
    for (auto& c : cases) {
        const uint64_t rows = total / 4 / c.row_floats;
        const int rows_per_cta = (int)(rows / grid) / c.box_rows * c.box_rows;
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)c.row_floats, rows};
        cuuint64_t strides[1] = {(cuuint64_t)c.row_floats * 4};
        cuuint32_t box[2] = {(cuuint32_t)c.box_cols, (cuuint32_t)c.box_rows};
        cuuint32_t es[2] = {1, 1};
        if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("encode failed\n");
            return 1;
        }
        const int box_bytes = c.box_cols * c.box_rows * 4;
        const int cols_boxes = (c.row_floats - 8) / c.box_cols > 0 ? (c.row_floats - 8) / c.box_cols : 1;
        const int chunks = (int)((size_t)rows_per_cta * c.row_floats * 4 / box_bytes * 0.9);
        cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlots * box_bytes);
        k_stream<<<grid, 32, kSlots * box_bytes>>>(tm, box_bytes, cols_boxes, rows_per_cta, c.box_rows, 256, sink);
        CK(cudaDeviceSynchronize());
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k_stream<<<grid, 32, kSlots * box_bytes>>>(tm, box_bytes, cols_boxes, rows_per_cta, c.box_rows, chunks, sink);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)chunks * box_bytes * grid;
        printf("%s: %6.0f GB/s (%.1f GB in %.2f ms)\n", c.name, bytes / ms / 1e6, bytes / 1e9, ms);
    }
    return 0;
}
