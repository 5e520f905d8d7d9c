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
// (the same lag-window rows the correlator uses; +-1 exact), done on the tensor cores by
// k_synth_gemm (tcgen05 kind::f16 with bf16 operands, fp32 accumulator in TMEM): H is split
// into three bf16 terms h = b0 + b1 + b2 (24 mantissa bits, fp32's exponent range, so no
// scaling), A is +-1 (exact in bf16), the products are exact and the sums fp32 -- the
// accuracy of an fp32 SGEMM.  The cyclic prefix is the body's tail and the convolution tail
// its head, minus the few terms that fall outside the pilot: y[n < C] = Y[n + M - C] -
// sum_{l > n} ..., y[P + q] = Y[q] - sum_{l <= q} ... (at most L - 1 terms each).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <curand_kernel.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pnce_b200.h"
#include "pnce_internal.h"
#include "sm100_ptx.cuh"

namespace {

using namespace pnce;

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

// ---------------------------------------------------------------- tensor-core body GEMM
// Y[row, k] = sum_q Hs[row, q] Bs[k, q] with K' = 3 * Rp (Rp = roundup(n_batch L, 64)):
//   Hs[row][t * Rp + (j L + l)] = b_t(h[f, r, b*n_batch + j, l]) (plane re/im by row half),
//   Bs[k][t * Rp + (j L + l)]  = chip[(k - s_j - l) mod M]       (t = 0, 1, 2)
// so the three bf16 terms of h meet the same +-1 entry.  One CTA per 128 x 256 tile of Y:
// warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer (one thread), warps 2-5 epilogue.
constexpr int kSgM = 128, kSgN = 256, kSgK = 64, kSgStages = 4;
constexpr uint32_t kSgABytes = kSgM * kSgK * 2, kSgBBytes = kSgN * kSgK * 2;
constexpr uint32_t kSgStageBytes = kSgABytes + kSgBBytes;
constexpr int kSgThreads = 192;

// Bs [Np][3 Rp] bf16 (Np = roundup(M, 256)), zero outside k < M, q < n_batch L
__global__ void k_build_bsyn(const float* __restrict__ chips, __nv_bfloat16* __restrict__ bs, int m, int l, int nbl,
                             int rp, int np, int spacing) {
    const int64_t total = (int64_t)np * 3 * rp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(i / (3 * rp));
        const int q = (int)(i - (int64_t)k * 3 * rp) % rp;
        float v = 0.f;
        if (k < m && q < nbl) {
            const int j = q / l, lag = q - j * l;
            int idx = (k - spacing * j - lag) % m;
            if (idx < 0) idx += m;
            v = chips[idx];
        }
        bs[i] = __float2bfloat16_rn(v);
    }
}

// Hs rows (plane, f, r) of batch b: the three bf16 terms of each tap, zero beyond n_tx L
__global__ void k_h_split(const float2* __restrict__ h, __nv_bfloat16* __restrict__ hs, int64_t fr, int n_t, int l,
                          int b, int n_batch, int n_tx, int rp) {
    const int64_t total = 2 * fr * rp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / rp;
        const int q = (int)(i - row * rp);
        const int plane = row >= fr;
        const int64_t link = plane ? row - fr : row;   // f * n_r + r
        float x = 0.f;
        if (q < n_tx * l) {
            const float2 v = h[(link * n_t + (int64_t)b * n_batch) * l + q];
            x = plane ? v.y : v.x;
        }
        const __nv_bfloat16 b0 = __float2bfloat16_rn(x);
        const float r0 = x - __bfloat162float(b0);
        const __nv_bfloat16 b1 = __float2bfloat16_rn(r0);
        const __nv_bfloat16 b2 = __float2bfloat16_rn(r0 - __bfloat162float(b1));
        __nv_bfloat16* dst = hs + row * 3 * rp + q;
        dst[0] = b0;
        dst[rp] = b1;
        dst[2 * rp] = b2;
    }
}

__global__ void __launch_bounds__(kSgThreads, 1)
k_synth_gemm(const __grid_constant__ CUtensorMap tm_h, const __grid_constant__ CUtensorMap tm_b,
             float* __restrict__ y, int64_t rows, int m, int k_blocks) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSgStages * kSgStageBytes);
    uint64_t* empty = full + kSgStages;
    uint64_t* done = empty + kSgStages;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row0 = (int64_t)blockIdx.x * kSgM;
    const int col0 = blockIdx.y * kSgN;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kSgStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tslot, kSgN);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tm_h);
        tma_prefetch(&tm_b);
        for (int kb = 0; kb < k_blocks; ++kb) {
            const int s = kb % kSgStages;
            mbar_wait(&empty[s], ((kb / kSgStages) & 1) ^ 1);
            mbar_arrive_expect_tx(&full[s], kSgStageBytes);
            uint8_t* sa = smem + s * kSgStageBytes;
            tma_load_2d(sa, &tm_h, &full[s], kb * kSgK, (int)row0, policy_evict_first());
            tma_load_2d(sa + kSgABytes, &tm_b, &full[s], kb * kSgK, col0, policy_evict_last());
        }
    } else if (warp == 1 && lane == 0) {
        const uint32_t idesc = make_idesc_f16(kSgM, kSgN, 1);
        for (int kb = 0; kb < k_blocks; ++kb) {
            const int s = kb % kSgStages;
            mbar_wait(&full[s], (kb / kSgStages) & 1);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + s * kSgStageBytes);
#pragma unroll
            for (int ks = 0; ks < kSgK / 16; ++ks)
                umma_f16_ss(tmem, make_sdesc(sa + ks * 32, 16, 1024, 2),
                            make_sdesc(sa + kSgABytes + ks * 32, 16, 1024, 2), idesc, (kb | ks) != 0);
            umma_commit(&empty[s]);
        }
        umma_commit(done);
    } else if (warp >= 2) {
        // warp w drains TMEM lanes 32 (w % 4) .. +31 (its sub-partition): one Y row per thread
        const int q = warp & 3;
        mbar_wait(done, 0);
        tc_fence_after();
        const int64_t row = row0 + q * 32 + lane;
        float* dst = y + row * (int64_t)m + col0;
        const bool vec = (m & 3) == 0;
        for (int c = 0; c < kSgN; c += 32) {
            uint32_t v[32];
            tmem_ld32_nowait(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
            tmem_wait_ld();
            if (row >= rows) continue;
            if (vec && col0 + c + 32 <= m) {
#pragma unroll
                for (int i = 0; i < 32; i += 4)
                    st_global_v4(dst + c + i, __uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                 __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
            } else {
                for (int i = 0; i < 32; ++i)
                    if (col0 + c + i < m) dst[c + i] = __uint_as_float(v[i]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, kSgN);
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

// Per-plan synthesiser state: the transposed lag-window operand Bs and its tensor map.
struct SynthCache {
    __nv_bfloat16* bs = nullptr;  // [np][3 rp]
    int rp = 0, np = 0;
    CUtensorMap tm_b;
    std::mutex mu;
};

size_t sg_smem() { return 1024 + (size_t)kSgStages * kSgStageBytes + 256; }

// Once per device: the GEMM's dynamic shared-memory opt-in (function attributes are per device).
pnce_status_t synth_device_setup() {
    static std::mutex mu;
    static std::vector<int> done;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return pnce_internal::set_error(PNCE_ERR_CUDA, "cudaGetDevice failed");
    std::lock_guard<std::mutex> lock(mu);
    if (std::find(done.begin(), done.end(), dev) != done.end()) return PNCE_OK;
    cudaError_t e = cudaFuncSetAttribute(k_synth_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sg_smem());
    if (e != cudaSuccess) return pnce_internal::set_error(PNCE_ERR_CUDA, std::string("synth attr: ") + cudaGetErrorString(e));
    done.push_back(dev);
    return PNCE_OK;
}

pnce_status_t synth_cache(const PlanView& v, cudaStream_t st, SynthCache*& out) {
    using pnce_internal::set_error;
    static std::mutex create_mu;
    std::lock_guard<std::mutex> lock(create_mu);
    if (*v.synth_cache) {
        out = static_cast<SynthCache*>(*v.synth_cache);
        return PNCE_OK;
    }
    pnce_status_t s = synth_device_setup();
    if (s != PNCE_OK) return s;
    auto* sc = new SynthCache();
    const int nbl = v.cfg.n_batch * v.cfg.l;
    sc->rp = (nbl + kSgK - 1) / kSgK * kSgK;
    sc->np = (v.cfg.m + kSgN - 1) / kSgN * kSgN;
    const size_t n = (size_t)sc->np * 3 * sc->rp;
    cudaError_t e = cudaMalloc(&sc->bs, sizeof(__nv_bfloat16) * n);
    if (e != cudaSuccess) {
        delete sc;
        return set_error(PNCE_ERR_CUDA, std::string("synth operand: ") + cudaGetErrorString(e));
    }
    k_build_bsyn<<<grid_for((int64_t)n, 256), 256, 0, st>>>(v.chips, sc->bs, v.cfg.m, v.cfg.l, nbl, sc->rp, sc->np,
                                                            v.cfg.m / v.cfg.n_batch);
    pnce_internal::count_launch();
    s = pnce_internal::encode_tmap_k16(&sc->tm_b, sc->bs, 3 * sc->rp, sc->np, kSgN, 1);
    if (s != PNCE_OK) {
        cudaFree(sc->bs);
        delete sc;
        return s;
    }
    *v.synth_cache = sc;
    out = sc;
    return PNCE_OK;
}

}  // namespace

namespace pnce_internal {
void synth_cache_free(void* cache) {
    auto* sc = static_cast<SynthCache*>(cache);
    if (sc->bs) cudaFree(sc->bs);
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
    // frame chunks so the fp32 body (2 F n_r M floats) and the split H stay bounded (~512 MB)
    const int64_t per_frame = 2LL * c.n_r * c.m * 4 + 2LL * c.n_r * 3 * sc->rp * 2;
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n_frames, (int64_t)(512ll << 20) / per_frame));
    // the split H starts 256-byte aligned after the body (TMA global addresses: 16 B)
    const size_t y_bytes = ((size_t)2 * chunk * c.n_r * c.m * 4 + 255) & ~(size_t)255;
    const int64_t n_fb = n_frames * v.n_batches;
    double* power = nullptr;
    uint8_t* work = nullptr;
    cudaError_t e = cudaMallocAsync(&power, sizeof(double) * n_fb, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(power, 0, sizeof(double) * n_fb, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&work, y_bytes + (size_t)2 * chunk * c.n_r * 3 * sc->rp * 2, st);
    if (e != cudaSuccess) {
        if (power) cudaFreeAsync(power, st);
        return set_error(PNCE_ERR_CUDA, std::string("synth scratch: ") + cudaGetErrorString(e));
    }
    std::lock_guard<std::mutex> lock(sc->mu);
    const size_t smem = sizeof(float) * c.m;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_synth_assemble, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    pnce_status_t ms = PNCE_OK;
    for (int64_t f0 = 0; f0 < n_frames && ms == PNCE_OK; f0 += chunk) {
        const int64_t fc = std::min(chunk, n_frames - f0);
        const int64_t fr = fc * c.n_r;
        const int64_t rows = 2 * fr;                                   // (plane, f, r)
        float* y = reinterpret_cast<float*>(work);                     // [2][fc][n_r][M]
        __nv_bfloat16* hs = reinterpret_cast<__nv_bfloat16*>(work + y_bytes);  // [rows][3 rp]
        const float2* hf = reinterpret_cast<const float2*>(h) + f0 * c.n_r * (int64_t)c.n_t * c.l;
        CUtensorMap tm_h;
        ms = pnce_internal::encode_tmap_k16(&tm_h, hs, 3 * sc->rp, rows, kSgM, 1);
        for (int b = 0; b < v.n_batches && ms == PNCE_OK; ++b) {
            const int n_tx = std::min(c.n_batch, c.n_t - b * c.n_batch);
            k_h_split<<<grid_for(rows * sc->rp, 256), 256, 0, st>>>(hf, hs, fr, c.n_t, c.l, b, c.n_batch, n_tx, sc->rp);
            pnce_internal::count_launch();
            const dim3 grid((unsigned)((rows + kSgM - 1) / kSgM), (unsigned)(sc->np / kSgN));
            k_synth_gemm<<<grid, kSgThreads, sg_smem(), st>>>(tm_h, sc->tm_b, y, rows, c.m, 3 * sc->rp / kSgK);
            pnce_internal::count_launch();
            k_synth_assemble<<<(unsigned)fr, kSynThreads, smem, st>>>(
                v.chips, hf, y, reinterpret_cast<float2*>(iq) + f0 * v.n_batches * c.n_r * (int64_t)S,
                power + f0 * v.n_batches, b, c.m, c.c, c.l, c.n_t, c.n_r, c.n_batch, v.n_batches, spacing,
                fr * (int64_t)c.m);
            pnce_internal::count_launch();
        }
    }
    e = cudaGetLastError();
    if (e == cudaSuccess && ms == PNCE_OK && std::isfinite(snr_db)) {
        const int64_t n_samples = n_fb * c.n_r * (int64_t)S;
        k_synth_noise<<<grid_for((n_samples + 1) / 2, 256), 256, 0, st>>>(
            reinterpret_cast<float2*>(iq), power, n_samples, (int64_t)c.n_r * S, c.n_r, c.m, c.l, c.n_t, c.n_batch,
            v.n_batches, std::pow(10.0, snr_db / 10.0), (unsigned long long)seed);
        pnce_internal::count_launch();
        e = cudaGetLastError();
    }
    cudaFreeAsync(work, st);
    cudaFreeAsync(power, st);
    if (ms != PNCE_OK) return ms;
    if (e != cudaSuccess) return set_error(PNCE_ERR_CUDA, std::string("k_synth: ") + cudaGetErrorString(e));
    return PNCE_OK;
}

}  // extern "C"
