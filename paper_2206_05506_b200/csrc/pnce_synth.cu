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
#include <cuda_runtime.h>
#include <curand_kernel.h>

#include <cmath>
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
constexpr int kSynRx = 4;  // receivers per block

// clean frames + per-(frame-set, batch) body power.  Block = (frame-set, batch, 4 receivers).
__global__ void __launch_bounds__(kSynThreads) k_synth_clean(const float* __restrict__ chips, const float2* __restrict__ h,
                                                              float2* __restrict__ iq, double* __restrict__ power, int m,
                                                              int c, int l, int n_t, int n_r, int n_batch, int n_batches,
                                                              int spacing) {
    extern __shared__ float sm[];
    float* ch = sm;                                         // [m]
    float2* hs = reinterpret_cast<float2*>(sm + ((m + 1) & ~1));  // [kSynRx][n_batch * l]
    const int r_tiles = (n_r + kSynRx - 1) / kSynRx;
    const int64_t blk = blockIdx.x;
    const int rt = (int)(blk % r_tiles);
    const int64_t fb = blk / r_tiles;
    const int b = (int)(fb % n_batches);
    const int64_t f = fb / n_batches;
    const int n_tx = min(n_batch, n_t - b * n_batch);
    const int R = n_tx * l;
    const int p = c + m;
    const int S = p + l - 1;
    for (int i = threadIdx.x; i < m; i += kSynThreads) ch[i] = chips[i];
    for (int i = threadIdx.x; i < kSynRx * R; i += kSynThreads) {
        const int rr = i / R, q = i - rr * R;
        const int r = rt * kSynRx + rr;
        const int t = b * n_batch + q / l;
        hs[rr * (n_batch * l) + q] = r < n_r ? h[((f * n_r + r) * n_t + t) * l + (q % l)] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    // all kSynRx receivers of the block per output sample: one chip load feeds 4 complex FMAs
    float pw = 0.f;
    const int n_rx = min(kSynRx, n_r - rt * kSynRx);
    for (int n = threadIdx.x; n < S; n += kSynThreads) {
        const int l_lo = max(0, n - p + 1), l_hi = min(l - 1, n);
        float2 acc[kSynRx];
#pragma unroll
        for (int rr = 0; rr < kSynRx; ++rr) acc[rr] = make_float2(0.f, 0.f);
        for (int j = 0; j < n_tx; ++j) {
            // chip index (n - lag - C - s_j) mod M, walking down with the lag
            int idx = (n - l_lo - c - spacing * j) % m;
            if (idx < 0) idx += m;
            const float2* hj = hs + j * l;
            for (int lag = l_lo; lag <= l_hi; ++lag) {
                const float chip = ch[idx];
#pragma unroll
                for (int rr = 0; rr < kSynRx; ++rr) {
                    const float2 hv = hj[rr * (n_batch * l) + lag];
                    acc[rr].x = fmaf(hv.x, chip, acc[rr].x);
                    acc[rr].y = fmaf(hv.y, chip, acc[rr].y);
                }
                idx = idx == 0 ? m - 1 : idx - 1;
            }
        }
        const bool body = n >= c && n < c + m;
#pragma unroll
        for (int rr = 0; rr < kSynRx; ++rr) {
            if (rr < n_rx) {
                const int r = rt * kSynRx + rr;
                iq[((f * n_batches + b) * n_r + r) * (int64_t)S + n] = acc[rr];
                if (body) pw += acc[rr].x * acc[rr].x + acc[rr].y * acc[rr].y;
            }
        }
    }
    // block reduction of the body power -> one float64 atomic per block
    for (int o = 16; o > 0; o >>= 1) pw += __shfl_xor_sync(0xffffffffu, pw, o);
    __shared__ float red[kSynThreads / 32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = pw;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < kSynThreads / 32; ++i) s += red[i];
        atomicAdd(power + fb, s);
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

}  // namespace

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
    if (n_frames < 0) return set_error(PNCE_ERR_DIMENSION, "n_frames < 0");
    if (n_frames == 0) return PNCE_OK;
    if (!h || !iq || (reinterpret_cast<uintptr_t>(h) & 7) || (reinterpret_cast<uintptr_t>(iq) & 7))
        return set_error(PNCE_ERR_DIMENSION, "h and iq must be 8-byte aligned device buffers");
    if (std::isnan(snr_db)) return set_error(PNCE_ERR_INVALID_SPEC, "snr_db is NaN");
    const pnce_cfg_t& c = v.cfg;
    const int spacing = c.m / c.n_batch;
    const int S = c.c + c.m + c.l - 1;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double* power = nullptr;
    const int64_t n_fb = n_frames * v.n_batches;
    cudaError_t e = cudaMallocAsync(&power, sizeof(double) * n_fb, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(power, 0, sizeof(double) * n_fb, st);
    if (e != cudaSuccess) return set_error(PNCE_ERR_CUDA, std::string("synth scratch: ") + cudaGetErrorString(e));
    const int r_tiles = (c.n_r + kSynRx - 1) / kSynRx;
    const size_t smem = sizeof(float) * ((c.m + 1) & ~1) + sizeof(float2) * kSynRx * c.n_batch * c.l;
    if (smem > 200 * 1024) {
        cudaFreeAsync(power, st);
        return set_error(PNCE_ERR_INVALID_CONFIG, "synthesis tile does not fit in shared memory");
    }
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_synth_clean, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_synth_clean<<<(unsigned)(n_fb * r_tiles), kSynThreads, smem, st>>>(
        v.chips, reinterpret_cast<const float2*>(h), reinterpret_cast<float2*>(iq), power, c.m, c.c, c.l, c.n_t, c.n_r,
        c.n_batch, v.n_batches, spacing);
    pnce_internal::count_launch();
    e = cudaGetLastError();
    if (e == cudaSuccess && std::isfinite(snr_db)) {
        const int64_t n_samples = n_fb * c.n_r * (int64_t)S;
        k_synth_noise<<<grid_for((n_samples + 1) / 2, 256), 256, 0, st>>>(
            reinterpret_cast<float2*>(iq), power, n_samples, (int64_t)c.n_r * S, c.n_r, c.m, c.l, c.n_t, c.n_batch,
            v.n_batches, std::pow(10.0, snr_db / 10.0), (unsigned long long)seed);
        pnce_internal::count_launch();
        e = cudaGetLastError();
    }
    cudaFreeAsync(power, st);
    if (e != cudaSuccess) return set_error(PNCE_ERR_CUDA, std::string("k_synth: ") + cudaGetErrorString(e));
    return PNCE_OK;
}

}  // extern "C"
