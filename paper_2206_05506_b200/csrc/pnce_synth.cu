// Device-side frame synthesis: channel draw + pilot sweep + AWGN.
//
// Reference semantics (pnce/channel.py):
//   draw_channel (96-108): per (r, t) link, L_nz distinct tap positions, amplitude
//       uniform on (0, A_max], A_max^2 = 1 / (N_t sqrt(L_nz)), phase uniform [0, 2pi).
//   simulate_frame (186-214) per batch b of the plan: every transmitter t of the batch
//       sends its pilot [CP | PN rolled by s_t] (pilots.py:103-110), the receiver sees
//       the LINEAR convolution with h[r, t, :] (apply_channel, 111-142; P + L - 1 samples),
//       plus circular complex AWGN of variance sigma^2 = ref / 10^(SNR/10) on every sample,
//       ref = mean_{r, k in body} |clean|^2 / (n_tx L) (noise_reference_power, 175-183).
// The pilot of t at sample n' in [0, P) is chip[(n' - C - s_t) mod M]; so
//   clean[r, n] = sum_{t in batch} sum_{l : 0 <= n - l < P} h[r, t, l] chip[(n - l - C - s_t) mod M].
// Random streams are Philox (curand), keyed by (seed, link) / (seed, sample group):
// statistically equivalent to the reference's numpy PCG64 streams, not the same draws.
//
// The body n in [C, C+M) is the circular convolution, i.e. the GEMM
//   Y[(plane, f, r), k] = H[(plane, f, r), (j, l)] . A[(j, l), k],  A = chip[(k - s_j - l) mod M]
// (the same lag-window rows the correlator uses; +-1 exact), done with cuBLAS SGEMM (a plain
// library GEMM, fp32).  The cyclic prefix is the body's tail and the convolution tail its
// head, minus the few terms that fall outside the pilot: y[n < C] = Y[n + M - C] -
// sum_{l > n} ..., y[P + q] = Y[q] - sum_{l <= q} ... (at most L - 1 terms each).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <curand_kernel.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <string>

#include "../../include/pnce_b200.h"
#include "pnce_internal.h"

namespace {

using pnce_internal::PlanView;

constexpr float kTwoPi = 6.283185307179586f;

__global__ void k_draw_channel(float2* __restrict__ h, int64_t n_links, int L, int l_nz, float amax,
                               unsigned long long seed) {
    for (int64_t link = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; link < n_links;
         link += (int64_t)gridDim.x * blockDim.x) {
        curandStatePhilox4_32_10_t st;
        curand_init(seed, (unsigned long long)link, 0ull, &st);
        float2* out = h + link * L;
        if (l_nz >= L) {
            for (int l = 0; l < L; ++l) {
                const float u = curand_uniform(&st);           // (0, 1]: amplitude law (0, A_max]
                const float v = 1.f - curand_uniform(&st);     // [0, 1): phase
                float s, c;
                sincosf(kTwoPi * v, &s, &c);
                out[l] = make_float2(amax * u * c, amax * u * s);
            }
        } else {
            // L_nz distinct positions = the L_nz smallest of L random keys (ties impossible
            // in practice; broken by index)
            float keys[256];
            for (int l = 0; l < L; ++l) keys[l] = curand_uniform(&st);
            for (int l = 0; l < L; ++l) {
                int rank = 0;
                for (int q = 0; q < L; ++q) rank += (keys[q] < keys[l]) || (keys[q] == keys[l] && q < l);
                if (rank < l_nz) {
                    const float u = curand_uniform(&st);
                    const float v = 1.f - curand_uniform(&st);
                    float s, c;
                    sincosf(kTwoPi * v, &s, &c);
                    out[l] = make_float2(amax * u * c, amax * u * s);
                } else {
                    out[l] = make_float2(0.f, 0.f);
                }
            }
        }
    }
}

constexpr int kSynThreads = 256;

// A[(j, l), k] = chip[(k - s_j - l) mod M] as fp32, rows = n_batch * L
__global__ void k_build_a32(const float* __restrict__ chips, float* __restrict__ a, int m, int l, int rows,
                            int spacing) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)rows * m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int row = (int)(i / m), k = (int)(i - (int64_t)row * m);
        const int j = row / l, lag = row - j * l;
        int idx = (k - spacing * j - lag) % m;
        if (idx < 0) idx += m;
        a[i] = chips[idx];
    }
}

// h complex64 [F][n_r][n_t][L] -> planes [2][F][n_r][n_t][L] (re, im)
__global__ void k_h_planes(const float2* __restrict__ h, float* __restrict__ hp, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 v = h[i];
        hp[i] = v.x;
        hp[n + i] = v.y;
    }
}

// Frame assembly for batch b from the GEMM body Y [2][F][n_r][M]: body copy, cyclic prefix
// and convolution tail with their edge corrections, body power per frame-set.
// Block = (frame-set, receiver); threads over the P + L - 1 samples.
__global__ void __launch_bounds__(kSynThreads) k_synth_assemble(const float* __restrict__ chips,
                                                                const float2* __restrict__ h,
                                                                const float* __restrict__ y, float2* __restrict__ iq,
                                                                double* __restrict__ power, int b, int m, int c, int l,
                                                                int n_t, int n_r, int n_batch, int n_batches,
                                                                int spacing, int64_t plane) {
    extern __shared__ float ch[];  // [m]
    const int r = blockIdx.x % n_r;
    const int64_t f = blockIdx.x / n_r;
    const int n_tx = min(n_batch, n_t - b * n_batch);
    const int p = c + m;
    const int S = p + l - 1;
    for (int i = threadIdx.x; i < m; i += kSynThreads) ch[i] = chips[i];
    __syncthreads();
    const float* yr = y + (f * n_r + r) * (int64_t)m;
    const float* yi = yr + plane;
    const float2* hr = h + ((f * n_r + r) * n_t + (int64_t)b * n_batch) * l;
    float2* out = iq + ((f * n_batches + b) * n_r + r) * (int64_t)S;
    float pw = 0.f;
    for (int n = threadIdx.x; n < S; n += kSynThreads) {
        int k;          // body column of the circular value
        int l_lo, l_hi; // lags to subtract (outside the pilot)
        if (n < c) {
            k = n + m - c;
            l_lo = n + 1;
            l_hi = l - 1;
        } else if (n < p) {
            k = n - c;
            l_lo = 1;
            l_hi = 0;
        } else {
            k = n - p;
            l_lo = 0;
            l_hi = n - p;
        }
        float ax = yr[k], ay = yi[k];
        for (int j = 0; j < n_tx; ++j) {
            int idx = (n - l_lo - c - spacing * j) % m;
            if (idx < 0) idx += m;
            const float2* hj = hr + j * l;
            for (int lag = l_lo; lag <= l_hi; ++lag) {
                const float chip = ch[idx];
                ax = fmaf(-hj[lag].x, chip, ax);
                ay = fmaf(-hj[lag].y, chip, ay);
                idx = idx == 0 ? m - 1 : idx - 1;
            }
        }
        out[n] = make_float2(ax, ay);
        if (n >= c && n < p) pw += ax * ax + ay * ay;
    }
    for (int o = 16; o > 0; o >>= 1) pw += __shfl_xor_sync(0xffffffffu, pw, o);
    __shared__ float red[kSynThreads / 32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = pw;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < kSynThreads / 32; ++i) s += red[i];
        atomicAdd(power + f * n_batches + b, s);
    }
}

// AWGN: sigma^2 = body_power / (n_r M) / (n_tx L) / 10^(snr/10), per component sigma^2 / 2.
// Thread g adds one curand_normal4 draw (Philox subsequence g) to complex samples 2g, 2g+1.
__global__ void k_synth_noise(float2* __restrict__ iq, const double* __restrict__ power, int64_t n_samples,
                              int64_t per_batch, int n_r, int m, int l, int n_t, int n_batch, int n_batches,
                              double snr_lin, unsigned long long seed) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; 2 * g < n_samples;
         g += (int64_t)gridDim.x * blockDim.x) {
        curandStatePhilox4_32_10_t st;
        curand_init(seed, (unsigned long long)g, 0ull, &st);
        const float4 z = curand_normal4(&st);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int64_t s = 2 * g + q;
            if (s >= n_samples) break;
            const int64_t fb = s / per_batch;
            const int b = (int)(fb % n_batches);
            const int n_tx = min(n_batch, n_t - b * n_batch);
            const double ref = power[fb] / ((double)n_r * m) / ((double)n_tx * l);
            const float sig = (float)sqrt(ref / snr_lin / 2.0);
            float2 v = iq[s];
            v.x = fmaf(sig, q == 0 ? z.x : z.z, v.x);
            v.y = fmaf(sig, q == 0 ? z.y : z.w, v.y);
            iq[s] = v;
        }
    }
}

int grid_for(int64_t work, int threads) {
    int64_t b = (work + threads - 1) / threads;
    return (int)(b < 148 * 32 ? (b > 0 ? b : 1) : 148 * 32);
}

// Per-plan synthesiser state: the fp32 lag-window rows and a cuBLAS handle.
struct SynthCache {
    float* a32 = nullptr;  // [n_batch * L][M]
    cublasHandle_t blas = nullptr;
    std::mutex mu;
};

pnce_status_t synth_cache(const PlanView& v, cudaStream_t st, SynthCache*& out) {
    using pnce_internal::set_error;
    static std::mutex create_mu;
    std::lock_guard<std::mutex> lock(create_mu);
    if (*v.synth_cache) {
        out = static_cast<SynthCache*>(*v.synth_cache);
        return PNCE_OK;
    }
    auto* sc = new SynthCache();
    const int rows = v.cfg.n_batch * v.cfg.l;
    cudaError_t e = cudaMalloc(&sc->a32, sizeof(float) * rows * (size_t)v.cfg.m);
    if (e != cudaSuccess) {
        delete sc;
        return set_error(PNCE_ERR_CUDA, std::string("synth rows: ") + cudaGetErrorString(e));
    }
    k_build_a32<<<grid_for((int64_t)rows * v.cfg.m, 256), 256, 0, st>>>(v.chips, sc->a32, v.cfg.m, v.cfg.l, rows,
                                                                        v.cfg.m / v.cfg.n_batch);
    pnce_internal::count_launch();
    if (cublasCreate(&sc->blas) != CUBLAS_STATUS_SUCCESS) {
        cudaFree(sc->a32);
        delete sc;
        return set_error(PNCE_ERR_CUDA, "cublasCreate failed");
    }
    cublasSetMathMode(sc->blas, CUBLAS_PEDANTIC_MATH);  // true fp32 (no TF32): the body feeds parity tests
    *v.synth_cache = sc;
    out = sc;
    return PNCE_OK;
}

}  // namespace

namespace pnce_internal {
void synth_cache_free(void* cache) {
    auto* sc = static_cast<SynthCache*>(cache);
    if (sc->blas) cublasDestroy(sc->blas);
    if (sc->a32) cudaFree(sc->a32);
    delete sc;
}
}  // namespace pnce_internal

extern "C" {

pnce_status_t pnce_draw_channel(const pnce_plan_t* plan, int32_t l_nz, uint64_t seed, float* h, int64_t n_frames,
                                void* stream) {
    using pnce_internal::set_error;
    if (!plan) return set_error(PNCE_ERR_INVALID_CONFIG, "null plan");
    const PlanView v = pnce_internal::plan_view(plan);
    if (n_frames < 0) return set_error(PNCE_ERR_DIMENSION, "n_frames < 0");
    if (l_nz < 1 || l_nz > v.cfg.l) return set_error(PNCE_ERR_INVALID_SPEC, "l_nz must be in [1, L]");
    if (v.cfg.l > 256 && l_nz < v.cfg.l) return set_error(PNCE_ERR_INVALID_SPEC, "sparse draws need L <= 256");
    if (n_frames == 0) return PNCE_OK;
    if (!h || (reinterpret_cast<uintptr_t>(h) & 7)) return set_error(PNCE_ERR_DIMENSION, "h must be 8-byte aligned");
    const int64_t links = n_frames * v.cfg.n_r * (int64_t)v.cfg.n_t;
    const float amax = (float)std::sqrt(1.0 / (v.cfg.n_t * std::sqrt((double)l_nz)));   // channel.py:91-93
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_draw_channel<<<grid_for(links, 128), 128, 0, st>>>(reinterpret_cast<float2*>(h), links, v.cfg.l, l_nz, amax,
                                                          (unsigned long long)seed);
    pnce_internal::count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(PNCE_ERR_CUDA, std::string("k_draw_channel: ") + cudaGetErrorString(e));
    return PNCE_OK;
}

pnce_status_t pnce_simulate_frames(const pnce_plan_t* plan, const float* h, double snr_db, uint64_t seed, float* iq,
                                   int64_t n_frames, void* stream) {
    using pnce_internal::set_error;
    if (!plan) return set_error(PNCE_ERR_INVALID_CONFIG, "null plan");
    const PlanView v = pnce_internal::plan_view(plan);
    if (!v.chips) return set_error(PNCE_ERR_INVALID_CONFIG, "synthesis needs a PN plan (pnce_plan_create)");
    if (n_frames < 0) return set_error(PNCE_ERR_DIMENSION, "n_frames < 0");
    if (n_frames == 0) return PNCE_OK;
    if (!h || !iq || (reinterpret_cast<uintptr_t>(h) & 7) || (reinterpret_cast<uintptr_t>(iq) & 7))
        return set_error(PNCE_ERR_DIMENSION, "h and iq must be 8-byte aligned device buffers");
    if (std::isnan(snr_db)) return set_error(PNCE_ERR_INVALID_SPEC, "snr_db is NaN");
    const pnce_cfg_t& c = v.cfg;
    const int spacing = c.m / c.n_batch;
    const int S = c.c + c.m + c.l - 1;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    SynthCache* sc = nullptr;
    pnce_status_t s = synth_cache(v, st, sc);
    if (s != PNCE_OK) return s;
    // frame chunks so the fp32 body (2 F n_r M floats) and H planes stay bounded (~512 MB)
    const int64_t per_frame = 2LL * c.n_r * c.m + 2LL * c.n_r * c.n_t * c.l;
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n_frames, (int64_t)(128ll << 20) / per_frame));
    const int64_t n_fb = n_frames * v.n_batches;
    double* power = nullptr;
    float* work = nullptr;
    cudaError_t e = cudaMallocAsync(&power, sizeof(double) * n_fb, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(power, 0, sizeof(double) * n_fb, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&work, sizeof(float) * per_frame * chunk, st);
    if (e != cudaSuccess) {
        if (power) cudaFreeAsync(power, st);
        return set_error(PNCE_ERR_CUDA, std::string("synth scratch: ") + cudaGetErrorString(e));
    }
    std::lock_guard<std::mutex> lock(sc->mu);
    cublasSetStream(sc->blas, st);
    const size_t smem = sizeof(float) * c.m;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_synth_assemble, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cublasStatus_t bs = CUBLAS_STATUS_SUCCESS;
    for (int64_t f0 = 0; f0 < n_frames && bs == CUBLAS_STATUS_SUCCESS; f0 += chunk) {
        const int64_t fc = std::min(chunk, n_frames - f0);
        const int64_t nh = fc * c.n_r * (int64_t)c.n_t * c.l;
        float* hp = work;                    // [2][fc][n_r][n_t][L]
        float* y = work + 2 * nh;            // [2][fc][n_r][M]
        const float2* hf = reinterpret_cast<const float2*>(h) + f0 * c.n_r * (int64_t)c.n_t * c.l;
        k_h_planes<<<grid_for(nh, 256), 256, 0, st>>>(hf, hp, nh);
        pnce_internal::count_launch();
        const int rows = (int)(2 * fc * c.n_r);  // both planes: H row stride n_t*L is uniform
        for (int b = 0; b < v.n_batches && bs == CUBLAS_STATUS_SUCCESS; ++b) {
            const int n_tx = std::min(c.n_batch, c.n_t - b * c.n_batch);
            const float one = 1.f, zero = 0.f;
            // column-major: Y^T [M x rows] = A^T [M x K] . H_b^T [K x rows]
            bs = cublasSgemm(sc->blas, CUBLAS_OP_N, CUBLAS_OP_N, c.m, rows, n_tx * c.l, &one, sc->a32, c.m,
                             hp + (int64_t)b * c.n_batch * c.l, c.n_t * c.l, &zero, y, c.m);
            if (bs != CUBLAS_STATUS_SUCCESS) break;
            k_synth_assemble<<<(unsigned)(fc * c.n_r), kSynThreads, smem, st>>>(
                v.chips, hf, y, reinterpret_cast<float2*>(iq) + f0 * v.n_batches * c.n_r * (int64_t)S,
                power + f0 * v.n_batches, b, c.m, c.c, c.l, c.n_t, c.n_r, c.n_batch, v.n_batches, spacing,
                fc * c.n_r * (int64_t)c.m);
            pnce_internal::count_launch();
        }
    }
    e = cudaGetLastError();
    if (e == cudaSuccess && bs == CUBLAS_STATUS_SUCCESS && std::isfinite(snr_db)) {
        const int64_t n_samples = n_fb * c.n_r * (int64_t)S;
        k_synth_noise<<<grid_for((n_samples + 1) / 2, 256), 256, 0, st>>>(
            reinterpret_cast<float2*>(iq), power, n_samples, (int64_t)c.n_r * S, c.n_r, c.m, c.l, c.n_t, c.n_batch,
            v.n_batches, std::pow(10.0, snr_db / 10.0), (unsigned long long)seed);
        pnce_internal::count_launch();
        e = cudaGetLastError();
    }
    cudaFreeAsync(work, st);
    cudaFreeAsync(power, st);
    if (bs != CUBLAS_STATUS_SUCCESS) return set_error(PNCE_ERR_CUDA, "cublasSgemm failed: " + std::to_string((int)bs));
    if (e != cudaSuccess) return set_error(PNCE_ERR_CUDA, std::string("k_synth: ") + cudaGetErrorString(e));
    return PNCE_OK;
}

}  // extern "C"
