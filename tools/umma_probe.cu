// Microbenchmark + correctness probe for tcgen05 operand paths on sm_100a.
//
// Measures cycles per tcgen05.mma (kind::f16, M=128, cta_group::1) for
//   SS  : A and B from shared memory (128B-swizzled K-major tiles)
//   SSH : B from a "Hankel table" (no-swizzle K-major, LBO = SBO = 128 B, so
//         core matrix (g, c) = table row 8(g+c) + i: one table of 16-byte chip
//         windows serves every lag row and every K block of the circulant)
//   TS  : A from tensor memory
// and checks numerically (one CTA) that the SSH and TS descriptors compute
// D[m, n] = sum_k A[m, k] * chip[(k - (mu - n)) mod M].
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_probe tools/umma_probe.cu
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2206_05506_b200/csrc/sm100_ptx.cuh"

using namespace pnce;

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e = (x);                                                            \
        if (e != cudaSuccess) {                                                         \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                    \
        }                                                                               \
    } while (0)

constexpr int M_PN = 1023;
constexpr int TABLE_ROWS = M_PN + 256 + 32;

__device__ __forceinline__ void umma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
        ::"r"(d_tmem), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
          "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),
          "r"(r[14]), "r"(r[15])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// smem: [A 16 KB SW128 128x64][B 32 KB SW128 256x64][table TABLE_ROWS x 16 B][bar][slot]
struct Smem {
    static constexpr int A = 0;
    static constexpr int B = 16384;
    static constexpr int T = 16384 + 32768;
    static constexpr int BAR = T + ((TABLE_ROWS * 16 + 1023) / 1024) * 1024;
    static constexpr int TOTAL = BAR + 64;
};

// MODE: 0 SS N=256, 1 SS N=128, 2 SS N=64, 3 SSH N=64 (8 windows), 4 SSH N=256,
//       5 TS N=256, 6 TS N=64 SSH, 7 TS N=128 SSH
template <int MODE>
__global__ void __launch_bounds__(128, 1)
k_probe(const __half* __restrict__ a_in, const float* __restrict__ chips, int iters,
        long long* cycles, float* d_out, int mu) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Smem::BAR);
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + Smem::BAR + 16);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // A tile 128 x 64 fp16, SW128: element (r, k) at r*128 + ((k/8) ^ (r%8))*16 + (k%8)*2
    for (int idx = tid; idx < 128 * 64; idx += 128) {
        int r = idx / 64, k = idx % 64;
        __half v = a_in[idx];
        *reinterpret_cast<__half*>(smem + Smem::A + r * 128 + (((k >> 3) ^ (r & 7)) << 4) + (k & 7) * 2) = v;
    }
    // B tile 256 x 64 SW128: B[n, k] = chip[(k - (mu - n)) mod M]
    for (int idx = tid; idx < 256 * 64; idx += 128) {
        int n = idx / 64, k = idx % 64;
        int ci = ((k - (mu - n)) % M_PN + M_PN) % M_PN;
        *reinterpret_cast<__half*>(smem + Smem::B + n * 128 + (((k >> 3) ^ (n & 7)) << 4) + (k & 7) * 2) =
            __float2half(chips[ci]);
    }
    // Hankel table: row rho = chip[(rho + jj) mod M], jj = 0..7
    for (int idx = tid; idx < TABLE_ROWS * 8; idx += 128) {
        int rho = idx / 8, jj = idx % 8;
        *reinterpret_cast<__half*>(smem + Smem::T + rho * 16 + jj * 2) = __float2half(chips[(rho + jj) % M_PN]);
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

    constexpr bool TS = MODE >= 5;
    // A into TMEM columns [256, 288): lane = row m, column c holds k = 2c, 2c+1
    if (TS) {
        for (int kb = 0; kb < 4; ++kb) {   // 4 k-steps of 16 -> 8 cols each
            uint32_t r[16];
            const int m = warp * 32 + lane;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                __half2 h = __halves2half2(a_in[m * 64 + kb * 16 + 2 * c], a_in[m * 64 + kb * 16 + 2 * c + 1]);
                r[c] = *reinterpret_cast<uint32_t*>(&h);
            }
#pragma unroll
            for (int c = 8; c < 16; ++c) r[c] = 0;
            if (kb < 4) {
                // write 8 real columns (x16 store writes 16; the upper 8 are overwritten by next kb)
                tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + 256 + kb * 8, r);
            }
        }
        tc_fence_before();
    }
    __syncthreads();
    tc_fence_after();

    constexpr int N = (MODE == 0 || MODE == 4 || MODE == 5) ? 256 : (MODE == 1 || MODE == 7) ? 128 : 64;
    const uint32_t idesc = make_idesc_f16(128, N, 0);
    const uint32_t sa = smem_u32(smem + Smem::A);
    const uint32_t sb = smem_u32(smem + Smem::B);
    const uint32_t st = smem_u32(smem + Smem::T);

    long long t0 = 0, t1 = 0;
    if (warp == 1 && lane == 0) {
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int ks = it & 3;                   // k-step within the 64-wide tile
            const uint32_t acc = (it > 0) ? 1u : 0u;
            uint64_t bd;
            if (MODE <= 2 || MODE == 5) {
                bd = make_sdesc(sb + ks * 32, 16, 1024, 2);
            } else {
                // window w (for timing: cycle through 8 start rows)
                int w = (MODE == 3 || MODE == 6) ? ((it >> 2) & 7) : 0;
                int rho = ((16 * ks - mu - 127 * w) % M_PN + M_PN) % M_PN;
                bd = make_sdesc(st + rho * 16, 128, 128, 0);
            }
            if (TS) {
                umma_f16_ts(tmem, tmem + 256 + ks * 8, bd, idesc, acc);
            } else {
                const uint64_t ad = make_sdesc(sa + ks * 32, 16, 1024, 2);
                umma_f16_ss(tmem, ad, bd, idesc, acc);
            }
        }
        umma_commit(bar);
        mbar_wait(bar, 0);
        t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    __syncthreads();
    tc_fence_after();
    // D -> global (block 0) for the correctness check (valid for iters == 4)
    if (blockIdx.x == 0) {
        const int m = warp * 32 + lane;
        for (int c0 = 0; c0 < N; c0 += 16) {
            float v[16];
            tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
            for (int i = 0; i < 16; ++i) d_out[m * 256 + c0 + i] = v[i];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int MODE>
void run(const char* name, const __half* d_a, const float* d_chips, const std::vector<float>& chips,
         const std::vector<float>& a_host, int nsm) {
    long long* d_cyc;
    float* d_out;
    CK(cudaMalloc(&d_cyc, sizeof(long long) * nsm));
    CK(cudaMalloc(&d_out, sizeof(float) * 128 * 256));
    const int mu = 300;
    CK(cudaFuncSetAttribute(k_probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem::TOTAL + 1024));
    // correctness: one CTA, one 64-wide K tile (4 MMAs), window 0
    k_probe<MODE><<<1, 128, Smem::TOTAL + 1024>>>(d_a, d_chips, 4, d_cyc, d_out, mu);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> out(128 * 256);
    CK(cudaMemcpy(out.data(), d_out, out.size() * 4, cudaMemcpyDeviceToHost));
    constexpr int N = (MODE == 0 || MODE == 4 || MODE == 5) ? 256 : (MODE == 1 || MODE == 7) ? 128 : 64;
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
            double ref = 0;
            for (int k = 0; k < 64; ++k) {
                int ci = ((k - (mu - n)) % M_PN + M_PN) % M_PN;
                ref += (double)a_host[m * 64 + k] * chips[ci];
            }
            maxerr = fmax(maxerr, fabs(ref - out[m * 256 + n]));
            maxref = fmax(maxref, fabs(ref));
        }
    // timing: all SMs
    const int iters = 8192;
    k_probe<MODE><<<nsm, 128, Smem::TOTAL + 1024>>>(d_a, d_chips, iters, d_cyc, d_out, mu);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<long long> cyc(nsm);
    CK(cudaMemcpy(cyc.data(), d_cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
    long long mx = 0, mn = 1LL << 62;
    for (auto c : cyc) {
        mx = c > mx ? c : mx;
        mn = c < mn ? c : mn;
    }
    const double floor_cyc = 128.0 * N / 256.0;
    printf("%-34s N=%3d  err=%.2e (ref max %.1f)  cyc/mma max=%.1f min=%.1f  floor=%.0f  eff=%.1f%%\n", name, N,
           maxerr, maxref, (double)mx / iters, (double)mn / iters, floor_cyc, 100.0 * floor_cyc * iters / mx);
    cudaFree(d_cyc);
    cudaFree(d_out);
}

int main() {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    // chips: degree-10 m-sequence (taps 10,3) via the reference LFSR
    std::vector<float> chips(M_PN);
    unsigned s = 1, mask = 1023, tapm = (1u << 9) | (1u << 2);
    for (int i = 0; i < M_PN; ++i) {
        chips[i] = ((s >> 9) & 1) ? -1.f : 1.f;
        unsigned fb = __builtin_popcount(s & tapm) & 1;
        s = ((s << 1) | fb) & mask;
    }
    std::vector<float> a_host(128 * 64);
    std::vector<__half> a_h(128 * 64);
    srand(7);
    for (int i = 0; i < 128 * 64; ++i) {
        float v = (float)(rand() % 2001 - 1000) / 1000.f;
        a_h[i] = __float2half(v);
        a_host[i] = __half2float(a_h[i]);
    }
    __half* d_a;
    float* d_chips;
    CK(cudaMalloc(&d_a, sizeof(__half) * a_h.size()));
    CK(cudaMalloc(&d_chips, sizeof(float) * M_PN));
    CK(cudaMemcpy(d_a, a_h.data(), sizeof(__half) * a_h.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_chips, chips.data(), sizeof(float) * M_PN, cudaMemcpyHostToDevice));
    printf("SMs=%d\n", nsm);
    run<0>("SS  sw128 A, sw128 B", d_a, d_chips, chips, a_host, nsm);
    run<1>("SS  sw128 A, sw128 B", d_a, d_chips, chips, a_host, nsm);
    run<2>("SS  sw128 A, sw128 B", d_a, d_chips, chips, a_host, nsm);
    run<3>("SSH sw128 A, Hankel B (8 windows)", d_a, d_chips, chips, a_host, nsm);
    run<4>("SSH sw128 A, Hankel B", d_a, d_chips, chips, a_host, nsm);
    run<5>("TS  tmem A, sw128 B", d_a, d_chips, chips, a_host, nsm);
    run<6>("TSH tmem A, Hankel B (8 windows)", d_a, d_chips, chips, a_host, nsm);
    run<7>("TSH tmem A, Hankel B (8 windows)", d_a, d_chips, chips, a_host, nsm);
    return 0;
}
