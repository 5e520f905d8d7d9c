// B200-native PN-correlation channel estimator: device kernels + C ABI.
//
// Hot path (reference: pnce/experiments.py:176-208 process_frames ->
// pnce/estimator.py:68-86 correlate_rows):
//   K1  k_lfsr / k_build_circulant : generate_mseq (pn.py:109-138) on device and
//       the stacked lag-window rows A[j*L+l, k] = chip[(k - s_j - l) mod M]
//       (estimator.py:62-65,114-117) as an fp16/bf16 K-major operand.
//   K2  k_pack_iq : remove_cp (estimator.py:40-47) + de-interleave + quantise the
//       received f32 (I,Q) samples into rows (frame, batch, rx, re|im) x K (two-pass path).
//   K3  k_correlate<MODE, SCORED, EPI8, T16> : tcgen05 CTA-pair UMMA
//       D[rows, lags] = X[rows, K] . C[lags, K]^T (both real GEMMs of estimator.py:77-80 in
//       one contraction; the frame x batch x rx x re/im axis is the UMMA M dimension);
//       MODE 2 converts the f32 rows itself (TMA-staged chunks -> fp16/bf16 A stages), so
//       K2 is fused away; warp-specialised, persistent, mbarrier pipelines, accumulators
//       in TMEM (512 columns at cfg3, single-buffered, with the first N half released to
//       the next tile's MMAs as soon as it is drained: "split drain").  With several
//       lag-row groups (R > 512, or the 256-column scored / tensor16 tilings) a cluster
//       converts a row tile once and re-reads its fp16 A stages from an L2 scratch for the
//       other groups ("A-stage reuse").
//   K4  (K3's epilogue) x 1/M, per-transmitter window demux into taps[f, r, t, l]
//       (experiments.py:206-207), optional sum|e|, sum|e|^2, non-finite count and per-link
//       MSE vs. truth (metrics.py:19-25 + MSE), or the tensor16 chunk fold (halfprec.py).
// DESIGN.md §5 has the layouts, rooflines and measurements.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pnce_b200.h"
#include "pnce_internal.h"
#include "sm100_ptx.cuh"

using namespace pnce;

namespace {

constexpr int kBM = 128;       // UMMA M (input rows per tile)
constexpr int kMaxPeers = 7;   // peer CSI buffers of a gather launch (8 GPUs per node)
constexpr int kBK = 64;        // K per pipeline stage (one 128B swizzle atom of 16-bit)
constexpr int kUmmaK = 16;     // K per tcgen05.mma kind::f16
constexpr int kSmemLimit = 227 * 1024;

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

#define s_ok_or_return(expr)              \
    do {                                  \
        pnce_status_t s_ = (expr);        \
        if (s_ != PNCE_OK) return s_;     \
    } while (0)

// Tuning knobs (diagnostics): read from the environment ONCE per process, so
// no launch pays a getenv.  -1 = unset where the default depends on the launch.
struct Knobs {
    int epi8, group_fused, group_packed, group_packed_ldg, t16_g, narrow_g;
    int store_hint, raw_pol, split_drain, packed_mode, scored_g, narrow, mid, fused_mode, narrow_ldg;
    int a_reuse, scr_pol, scr_slots, truth_slots, ab_stages, raw_stages, scored_epi, t16_epi, wide_ldg;
};
int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}
const Knobs& knobs() {
    static const Knobs k = [] {
        Knobs r;
        r.epi8 = env_int("PNCE_TUNE_EPI8", -1);
        r.group_fused = env_int("PNCE_TUNE_GROUP_FUSED", 512);
        r.group_packed = env_int("PNCE_TUNE_GROUP_PACKED", 512);
        r.group_packed_ldg = env_int("PNCE_TUNE_GROUP_PACKED_LDG", 256);
        r.t16_g = env_int("PNCE_TUNE_T16_G", 256);
        const int ng = env_int("PNCE_TUNE_NARROW_G", 128);
        r.narrow_g = (ng == 64 || ng == 96 || ng == 192 || ng == 256) ? ng : 128;
        r.store_hint = env_int("PNCE_TUNE_STORE_HINT", 1);
        r.raw_pol = env_int("PNCE_TUNE_RAW_POL", -1);
        r.split_drain = env_int("PNCE_TUNE_SPLIT_DRAIN", 1);
        r.packed_mode = env_int("PNCE_TUNE_PACKED_MODE", 0);
        r.scored_g = env_int("PNCE_TUNE_SCORED_G", 512);
        r.narrow = env_int("PNCE_TUNE_NARROW", 1);
        r.mid = env_int("PNCE_TUNE_MID", 1);
        r.fused_mode = env_int("PNCE_TUNE_FUSED_MODE", -1);
        r.narrow_ldg = env_int("PNCE_TUNE_NARROW_LDG", 1);
        r.a_reuse = env_int("PNCE_TUNE_A_REUSE", 1);
        r.scr_pol = env_int("PNCE_TUNE_SCR_POL", 1);
        r.scr_slots = env_int("PNCE_TUNE_SCR_SLOTS", -1);
        r.truth_slots = env_int("PNCE_TUNE_TRUTH_SLOTS", 2);
        r.ab_stages = env_int("PNCE_TUNE_AB_STAGES", -1);
        r.raw_stages = env_int("PNCE_TUNE_RAW_STAGES", -1);
        r.scored_epi = env_int("PNCE_TUNE_SCORED_EPI", 8);
        r.t16_epi = env_int("PNCE_TUNE_T16_EPI", 8);
        r.wide_ldg = env_int("PNCE_TUNE_WIDE_LDG", 1);
        return r;
    }();
    return k;
}

pnce_status_t fail(pnce_status_t code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                 \
    do {                                                                               \
        cudaError_t e_ = (expr);                                                       \
        if (e_ != cudaSuccess)                                                         \
            return fail(PNCE_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
    } while (0)

// ------------------------------------------------------------------ K1: LFSR
// One thread runs the Fibonacci LFSR for one period (pn.py:115-137):
// out = MSB, fb = parity(state & tap_mask), state = ((state << 1) | fb) & mask.
__global__ void k_lfsr(int degree, uint32_t tap_mask, uint32_t state0, float* chips, int m,
                       int* period_out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const uint32_t mask = (1u << degree) - 1u;
    uint32_t s = state0;
    int n = 0;
    const int limit = 1 << degree;
    for (int i = 0; i < limit; ++i) {
        uint32_t bit = (s >> (degree - 1)) & 1u;
        if (n < m) chips[n] = bit ? -1.0f : 1.0f;
        ++n;
        uint32_t fb = __popc(s & tap_mask) & 1u;
        s = ((s << 1) | fb) & mask;
        if (s == state0) break;
    }
    *period_out = n;
}

// Stacked lag-window rows, K-major, zero padded: A[n, k] for n < rows_alloc, k < k_pad.
template <typename T>
__global__ void k_build_circulant(const float* __restrict__ chips, T* __restrict__ a, int m,
                                  int k_pad, int r_total, int rows_alloc, int l, int spacing) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t total = (int64_t)rows_alloc * k_pad;
    for (; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        int n = (int)(idx / k_pad);
        int k = (int)(idx % k_pad);
        float v = 0.0f;
        if (n < r_total && k < m) {
            int lag = (spacing * (n / l) + (n % l)) % m;  // shift_for_transmitter + window lag
            int ci = k - lag;
            if (ci < 0) ci += m;
            v = chips[ci];
        }
        if constexpr (sizeof(T) == 2 && std::is_same<T, __half>::value)
            a[idx] = __float2half_rn(v);
        else
            a[idx] = __float2bfloat16_rn(v);
    }
}

// Caller-supplied correlation rows (correlate_rows' `rows`, estimator.py:68-86) as the
// K-major operand: rows [n_rows][m] f32 -> [rows_alloc][k_pad] fp16/bf16 (RN), zero padded.
template <typename T>
__global__ void k_rows_to_operand(const float* __restrict__ rows, T* __restrict__ a, int m, int k_pad, int n_rows,
                                  int rows_alloc) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)rows_alloc * k_pad;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int n = (int)(idx / k_pad), k = (int)(idx % k_pad);
        const float v = (n < n_rows && k < m) ? rows[(int64_t)n * m + k] : 0.f;
        if constexpr (std::is_same<T, __half>::value)
            a[idx] = __float2half_rn(v);
        else
            a[idx] = __float2bfloat16_rn(v);
    }
}

// ------------------------------------------------------------------ K2: pack
// Packed-operand row order (shared with the fused converters): links are grouped by 8 and
// each 16-row block holds the 8 Re rows then the 8 Im rows, so that the 16x256b TMEM load
// of the epilogue hands one thread Re and Im of the same link (see k_correlate).
__host__ __device__ __forceinline__ int64_t a_row(int64_t link, int im) {
    return ((link >> 3) << 4) | ((int64_t)im << 3) | (link & 7);
}

// One thread per (link q, 8-sample chunk c): read samples [C+8c, C+8c+8) of link q
// (q = (f*nb + b)*n_r + r), write 8 quantised Re to row a_row(q, 0) and 8 Im to
// a_row(q, 1) (16 B each); zero beyond M and for the padding links up to a multiple of 8.
template <typename T>
__global__ void k_pack_iq(const float* __restrict__ iq, T* __restrict__ out, int64_t n_links,
                          int samples, int c, int m, int k_pad) {
    const int chunks = k_pad >> 3;
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t padded = (n_links + 7) & ~int64_t(7);
    const int64_t total = padded * chunks;
    for (; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = idx / chunks;
        const int ch = (int)(idx - q * chunks);
        const int k0 = ch << 3;
        float re[8], im[8];
        if (q < n_links && k0 + 8 <= m) {
            const float2* src = reinterpret_cast<const float2*>(iq) + q * samples + c + k0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                float2 v = __ldg(src + j);
                re[j] = v.x;
                im[j] = v.y;
            }
        } else {
            const float2* src = reinterpret_cast<const float2*>(iq) + (q < n_links ? q : 0) * samples + c + k0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                float2 v = (q < n_links && k0 + j < m) ? __ldg(src + j) : make_float2(0.f, 0.f);
                re[j] = v.x;
                im[j] = v.y;
            }
        }
        uint4 pr, pi;
        T* hr = reinterpret_cast<T*>(&pr);
        T* hi = reinterpret_cast<T*>(&pi);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if constexpr (std::is_same<T, __half>::value) {
                hr[j] = __float2half_rn(re[j]);
                hi[j] = __float2half_rn(im[j]);
            } else {
                hr[j] = __float2bfloat16_rn(re[j]);
                hi[j] = __float2bfloat16_rn(im[j]);
            }
        }
        *reinterpret_cast<uint4*>(out + a_row(q, 0) * k_pad + k0) = pr;
        *reinterpret_cast<uint4*>(out + a_row(q, 1) * k_pad + k0) = pi;
    }
}

// ------------------------------------------------------------------ K3+K4
// Correlation kernel, one CTA pair (cluster 2x1, tcgen05 cta_group::2) per 256 input
// rows (128 links; each CTA owns 64 links = 128 A rows in the a_row order above).
// Variants (template MODE):
//   kModePacked   : rows = the packed 16-bit operand of K2, TMA-loaded;
//   kModeFusedTma : rows = raw f32 (I,Q) frames, TMA-staged in shared memory in
//                   half-K-block chunks (32 samples x 64 links) and converted (remove_cp +
//                   de-interleave + fp16/bf16) by converter warps straight into the
//                   128B-swizzled UMMA A stage -- K2 fused away;
//   kModeFusedLdg : as above but converters LDG the f32 rows (row strides that are not
//                   16-byte multiples).
//   kModePackedLdg: packed 16-bit rows LDG'd by the converter warps into the A stage (a
//                   separate ingress path from the TMA engine, which then only carries the
//                   circulant), so a 256-column double-buffered accumulator can hide the
//                   epilogue drain without exceeding the TMA ingress rate.
// Warp roles (16 warps, both CTAs unless noted):
//   0 TMA producer (circulant rows; + packed rows)   1 MMA issuer (leader CTA only)
//   2 raw-chunk TMA producer (FusedTma)              3 idle
//   4-11 converters (fused)                          12-15 epilogue (one per TMEM lane quarter)
enum { kModePacked = 0, kModeFusedLdg = 1, kModeFusedTma = 2, kModePackedLdg = 3 };

#ifdef PNCE_DIAG_CHECKS
// Diagnostic build: device-side bounds checks on every global / shared access of the kernels
// (compute-sanitizer is not available on the GPU pool); a violation prints and traps.
#define PNCE_CHECK(cond)                                                                               \
    do {                                                                                               \
        if (!(cond)) {                                                                                 \
            printf("PNCE_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,     \
                   (int)blockIdx.x, (int)threadIdx.x);                                                 \
            __trap();                                                                                  \
        }                                                                                              \
    } while (0)
#else
#define PNCE_CHECK(cond) \
    do {                 \
    } while (0)
#endif
#ifdef PNCE_DIAG_TRACE
// Diagnostic timeline (globaltimer ns) for the first CTA pair: [cta][slot][index].
constexpr int kTraceSlots = 16, kTraceMax = 512;
__device__ long long g_trace[2 * kTraceSlots * kTraceMax];
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TRACE(slot, idx)                                                                   \
    do {                                                                                   \
        if (blockIdx.x < 2 && (idx) < kTraceMax)                                           \
            g_trace[(blockIdx.x * kTraceSlots + (slot)) * kTraceMax + (idx)] = gtimer();  \
    } while (0)
#else
#define TRACE(slot, idx) \
    do {                 \
    } while (0)
#endif
#ifdef PNCE_DIAG_PROF
// Cycle accounting (clock64, kept in registers, written once per role at the end):
// per CTA 16 slots, see kProf* below.
constexpr int kProfSlots = 16;
__device__ unsigned long long g_prof[1024 * kProfSlots];
#define PROF_BEGIN(n) uint64_t _pacc[n] = {}; uint64_t _pt = clock64()
#define PROF_MARK(i) do { const uint64_t _n = clock64(); _pacc[i] += _n - _pt; _pt = _n; } while (0)
#define PROF_END(base, n) do { for (int _i = 0; _i < (n); ++_i) g_prof[blockIdx.x * kProfSlots + (base) + _i] = _pacc[_i]; } while (0)
#else
#define PROF_BEGIN(n) do { } while (0)
#define PROF_MARK(i) do { } while (0)
#define PROF_END(base, n) do { } while (0)
#endif
// slots: B producer {wait empty, issue} 0-1; MMA {wait tempty, wait full, issue} 2-4;
// raw producer {wait raw_empty, issue} 5-6; converter {wait empty, wait raw, convert} 7-9;
// epilogue {wait tfull, drain} 10-11; MMA total 12
constexpr int kWarps = 16;
constexpr int kThreadsK3 = kWarps * 32;
constexpr int kConvWarp0 = 4;
constexpr int kConvWarps = 8;
constexpr int kLinksPerTile = kBM / 2;                                        // 64 links per CTA
constexpr int kRawChunk = kBK / 2;  // samples per raw staging chunk (half a K-block)

struct CorrParams {
    int64_t total_links;  // n_frames * n_batches * n_r
    int32_t m_tiles;      // 128-link tiles (one per CTA pair)
    int32_t n_groups;     // lag-row groups
    int32_t g_cols;       // accumulator columns per group (= sum of the MMAs' N)
    int32_t n_mma;        // MMAs per k-step (1 or 2), each N = nm
    int32_t nm;
    int32_t acc_stages;   // TMEM accumulator buffers (2 if 2*g_cols <= 512)
    int32_t k_blocks;
    int32_t stages;
    int32_t raw_stages;      // FusedTma: f32 staging ring depth (half-K-block chunks)
    int32_t raw_row_floats;  // floats per staged link row: 64, +4 slack when C is odd
    uint32_t raw_stage_bytes;
    // antenna-split all-gather fused into the epilogue (pnce_process_frames_gather): taps are
    // laid out as the FULL [F][out_nr][n_t][L] CSI with this launch's receivers at rows
    // out_r0.., written to `taps` and to every peer buffer in gather_dst (NVLink stores)
    int32_t out_nr;       // receiver rows of the output layout (= n_r outside gather launches)
    int32_t out_r0;       // first receiver row of this launch's slice (0 outside gather launches)
    int32_t gather_n;     // peer buffers (0: none)
    float* gather_dst[kMaxPeers];
    int32_t store_hint;   // L2 policy of the taps stores: 1 evict_first (default), 2 evict_last, 3 normal, 0 none
    int32_t raw_pol;      // L2 policy of the raw f32 row loads: 0 evict_first, 1 normal, 2 evict_last
    int32_t a_reuse;      // FusedTma, n_groups > 1: group 0 converts once and stores the fp16 A
                          // stages to `scratch`; the other groups of the row tile TMA them back
    uint32_t bar_bytes;   // barrier block bytes (1 KB; 2 KB with a_reuse: + scratch barriers)
    int32_t scr_pol;      // a_reuse: 1 = evict_last L2 policy on the scratch stores / reloads
    int32_t scr_slots;    // a_reuse: scratch slots (row tiles) per cluster: 1 when k_blocks >= stages
    uint8_t* scratch;     // a_reuse: [2 slots][clusters][2 CTAs][k_blocks][128 rows][128 B]
    int32_t split_drain;  // release the first N half of a single accumulator early (see k_correlate)
    int32_t truth_slots;  // scored drain: per-thread LDGSTS ring depth for the truth (0: register path)
    uint32_t truth_off;   // byte offset of the truth ring in dynamic shared memory (after the raw ring)
    uint32_t stage_bytes;
    uint32_t tx_bytes;    // transaction bytes per stage for BOTH CTAs of the pair
    uint32_t idesc;
    uint32_t tmem_cols;
    int32_t n_r, n_t, n_batches, n_batch, l;
    int32_t m, c, samples;  // PN length, CP length, samples per received row
    int32_t bf16;
    float inv_m;
    const float* iq;
    const uint16_t* packed;  // kModePackedLdg: packed operand, packed_rows x K_pad
    int64_t packed_rows;
    int32_t k_pad;
    float* taps;
    const float* truth;
    double* stats;
    float* link_err;  // optional [F][n_r][n_t]: mean_l |h_est - h_true|^2 per link (needs truth)
    float inv_l;
    // tensor16 emulation on real tensor cores (halfprec.py:93-125): accumulation units of
    // chunk_kb K-blocks, each folded x fp32(1/M) into an fp32 running total kept in TMEM
    int32_t chunk_kb;    // K-blocks per accumulation unit (= k_blocks outside tensor16 mode)
    int32_t acc16;       // 1: binary16 partials (F16 TMEM accumulator), 0: binary32
    uint32_t* sat_flags; // tensor16: [F][n_batches] set when a partial / total is non-finite
    // bounds of the caller's buffers (PNCE_DIAG_CHECKS builds)
    int64_t n_taps;      // complex taps in `taps` (and `truth`): F n_r n_t L
    int64_t n_frames;    // F
    int64_t scr_rows;    // rows of the a_reuse scratch
};

__device__ __forceinline__ uint32_t pack2(float a, float b, int bf16) {
    if (bf16) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

// 128B swizzle of the UMMA K-major A stage: 16-byte chunk c of row r lives at chunk c ^ (r % 8).
__device__ __forceinline__ uint32_t swz(uint32_t base, int row, int byte_in_row) {
    return base + row * 128 + ((((byte_in_row >> 4) ^ (row & 7))) << 4) + (byte_in_row & 15);
}

// Output window of one link (f, b, r) for the epilogue.
struct EpiLink {
    int64_t out;      // complex index of lag 0 of the link's run in taps[f, r, t, l]; -1 = padding link
    int64_t lbase;    // (f, r, first transmitter of the batch) index into link_err
    int64_t f;        // frame-set
    int n_valid;      // valid lags in the run (n_tx * L)
    bool vec;         // taps + 2*out is 16-byte aligned (pairs of lags as one 16-byte store)
    bool tvec;        // same for truth
};

__device__ __forceinline__ EpiLink make_link(const CorrParams& p, int64_t link) {
    EpiLink e;
    if (link >= p.total_links) {
        e.out = -1;
        e.lbase = -1;
        e.f = -1;
        e.n_valid = 0;
        e.vec = e.tvec = false;
        return e;
    }
    // links < 2^31 (checked on the host): 32-bit divisions
    const uint32_t l32 = (uint32_t)link;
    const uint32_t fb = l32 / (uint32_t)p.n_r;
    const int r = (int)(l32 - fb * (uint32_t)p.n_r);
    const uint32_t f32 = fb / (uint32_t)p.n_batches;
    const int b = (int)(fb - f32 * (uint32_t)p.n_batches);
    e.f = f32;
    const int n_tx = min(p.n_batch, p.n_t - b * p.n_batch);
    e.n_valid = n_tx * p.l;
    e.lbase = (e.f * p.out_nr + p.out_r0 + r) * p.n_t + (int64_t)b * p.n_batch;
    e.out = e.lbase * p.l;
    e.vec = (reinterpret_cast<uintptr_t>(p.taps + 2 * e.out) & 15) == 0;
    e.tvec = p.truth != nullptr && (reinterpret_cast<uintptr_t>(p.truth + 2 * e.out) & 15) == 0;
    return e;
}

__device__ __forceinline__ float err_acc(float re, float im, float hr, float hi, float& s_abs, float& s_sq) {
    const float dx = re - hr, dy = im - hi;
    const float sq = dx * dx + dy * dy;
    s_sq += sq;
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(sq));  // MAE term: ~1 ulp is plenty
    s_abs += r;
    return sq;
}

// Per-link (per transmitter window) squared-error partial of one thread.  A thread's lags
// increase monotonically, so windows are visited in order: flush when a lag crosses the
// next window boundary.  `quad`: L % 8 == 0, so the four lanes of a link cross together
// (warp-uniform) and reduce with two shuffles before one atomic; otherwise each lane
// flushes on its own.
struct LinkAcc {
    int w;       // current window (transmitter within the batch)
    int next;    // first lag of window w + 1
    float part;
};

__device__ __forceinline__ void link_flush(const CorrParams& p, const EpiLink& e, LinkAcc& a, bool quad) {
    float v = a.part;
    if (quad) {
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
    }
    if ((!quad || (threadIdx.x & 3) == 0) && e.out >= 0 && a.w >= 0 && v != 0.f) {
        PNCE_CHECK(e.lbase + a.w < p.n_taps / p.l && a.w < p.n_batch);
        atomicAdd(p.link_err + e.lbase + a.w, v * p.inv_l);
    }
    a.part = 0.f;
}

__device__ __forceinline__ void link_add(const CorrParams& p, const EpiLink& e, LinkAcc& a, int lag, float sq) {
    if (lag >= a.next) {
        link_flush(p, e, a, false);
        a.w = lag / p.l;
        a.next = (a.w + 1) * p.l;
    }
    a.part += sq;
}

// K4 for R repetitions of a 16x256b TMEM load: repetition i holds, for this thread's link,
// Re (v[4i], v[4i+1]) and Im (v[4i+2], v[4i+3]) of lags n + 8i and n + 8i + 1.
template <int R, bool SC, bool GA = false>
__device__ __forceinline__ void epi_reps(const CorrParams& p, const uint32_t* v, const EpiLink& e, int n,
                                         float& s_abs, float& s_sq, float& nf, LinkAcc& la) {
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int lag = n + 8 * i;
        const float re0 = __uint_as_float(v[4 * i + 0]) * p.inv_m;
        const float re1 = __uint_as_float(v[4 * i + 1]) * p.inv_m;
        const float im0 = __uint_as_float(v[4 * i + 2]) * p.inv_m;
        const float im1 = __uint_as_float(v[4 * i + 3]) * p.inv_m;
        if (e.out < 0 || lag >= e.n_valid) continue;
        if (SC && p.stats != nullptr) {
            // sticky non-finite detector (inf * 0 = NaN); exact count only when it fires
            nf = fmaf(re0, 0.f, nf);
            nf = fmaf(im0, 0.f, nf);
        }
#ifdef PNCE_DIAG_NO_STORE
        if (re0 == 12345.678f) p.taps[0] = re1 + im0 + im1;  // keep the work, drop the stores
        continue;
#endif
        float* dst = p.taps + 2 * (e.out + lag);
        const float* tr = p.truth + 2 * (e.out + lag);
        PNCE_CHECK(e.out + lag >= 0 && e.out + lag + (lag + 1 < e.n_valid ? 1 : 0) < p.n_taps);
        if (lag + 1 < e.n_valid) {
            if (SC && p.stats != nullptr) {
                nf = fmaf(re1, 0.f, nf);
                nf = fmaf(im1, 0.f, nf);
            }
            if (e.vec) {
                st_global_v4(dst, re0, im0, re1, im1);
            } else {
                *reinterpret_cast<float2*>(dst) = make_float2(re0, im0);
                *reinterpret_cast<float2*>(dst + 2) = make_float2(re1, im1);
            }
            if (GA) {
                for (int d = 0; d < p.gather_n; ++d) {  // the same taps into every peer's CSI
                    float* pd = p.gather_dst[d] + 2 * (e.out + lag);
                    if (e.vec) {
                        st_global_v4(pd, re0, im0, re1, im1);
                    } else {
                        *reinterpret_cast<float2*>(pd) = make_float2(re0, im0);
                        *reinterpret_cast<float2*>(pd + 2) = make_float2(re1, im1);
                    }
                }
            }
            if (SC && p.truth != nullptr) {
                float4 h;
                if (e.tvec) {
                    h = ld_global_nc_v4(tr);
                } else {
                    const float2 a = __ldg(reinterpret_cast<const float2*>(tr));
                    const float2 b = __ldg(reinterpret_cast<const float2*>(tr) + 1);
                    h = make_float4(a.x, a.y, b.x, b.y);
                }
                const float q0 = err_acc(re0, im0, h.x, h.y, s_abs, s_sq);
                const float q1 = err_acc(re1, im1, h.z, h.w, s_abs, s_sq);
                if (p.link_err != nullptr) {
                    link_add(p, e, la, lag, q0);
                    link_add(p, e, la, lag + 1, q1);
                }
            }
        } else {
            *reinterpret_cast<float2*>(dst) = make_float2(re0, im0);
            if (GA)
                for (int d = 0; d < p.gather_n; ++d)
                    *reinterpret_cast<float2*>(p.gather_dst[d] + 2 * (e.out + lag)) = make_float2(re0, im0);
            if (SC && p.truth != nullptr) {
                const float2 a = __ldg(reinterpret_cast<const float2*>(tr));
                const float q0 = err_acc(re0, im0, a.x, a.y, s_abs, s_sq);
                if (p.link_err != nullptr) link_add(p, e, la, lag, q0);
            }
        }
    }
}

// Drain one 16-lane block (8 links) of the accumulator: TMEM -> x 1/M -> taps (+ scoring).
// 64-column chunks double-buffered (the next chunk's TMEM load is in flight while the
// current one is scaled and stored), then 16-column remainder pieces.
template <bool SC, bool GA = false>
__device__ __forceinline__ void epi_block(const CorrParams& p, uint32_t taddr, const EpiLink& e, int n0,
                                          float& s_abs, float& s_sq, float& nf, int cols) {
    int c = 0;
    LinkAcc la{-1, 0, 0.f};
    uint32_t va[32], vb[32];
    if (cols >= 64) {
        tmem_ld_16x256b_x8(taddr, va);
        tmem_wait_ld();
        while (true) {
            const bool more = c + 128 <= cols;
            if (more) tmem_ld_16x256b_x8(taddr + c + 64, vb);
            epi_reps<8, SC, GA>(p, va, e, n0 + c, s_abs, s_sq, nf, la);
            c += 64;
            if (!more) break;
            tmem_wait_ld();
            const bool more2 = c + 128 <= cols;
            if (more2) tmem_ld_16x256b_x8(taddr + c + 64, va);
            epi_reps<8, SC, GA>(p, vb, e, n0 + c, s_abs, s_sq, nf, la);
            c += 64;
            if (!more2) break;
            tmem_wait_ld();
        }
    }
    for (; c < cols; c += 16) {
        uint32_t v[8];
        tmem_ld_16x256b_x2(taddr + c, v);
        tmem_wait_ld();
        epi_reps<2, SC, GA>(p, v, e, n0 + c, s_abs, s_sq, nf, la);
    }
    if (SC && p.link_err != nullptr) link_flush(p, e, la, false);
}

// Scored drain (truth present, g_cols % 32 == 0): 32-column chunks; the truth of chunk k+1
// is loaded while chunk k is processed (two register buffers), after the whole tile's
// truth was pulled into L2 during the main loop.  Per-link errors reduce over the lane quad.
__device__ __forceinline__ void load_truth4(const CorrParams& p, const EpiLink& e, int lag0, float4 (&h)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int lag = lag0 + 8 * i;
        const float* tr = p.truth + 2 * (e.out + lag);
        if (e.out >= 0 && lag + 1 < e.n_valid && e.tvec) {
            h[i] = ld_global_nc_v4(tr);
        } else if (e.out >= 0 && lag < e.n_valid) {
            const float2 a = __ldg(reinterpret_cast<const float2*>(tr));
            const float2 b = lag + 1 < e.n_valid ? __ldg(reinterpret_cast<const float2*>(tr) + 1) : make_float2(0.f, 0.f);
            h[i] = make_float4(a.x, a.y, b.x, b.y);
        } else {
            h[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
}

__device__ __forceinline__ void epi_reps_scored(const CorrParams& p, const uint32_t (&v)[16], const float4 (&h)[4],
                                                const EpiLink& e, int n, float& s_abs, float& s_sq, float& nf,
                                                LinkAcc& la, bool quad) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int lag = n + 8 * i;
        if (p.link_err != nullptr && quad && lag >= la.next) {  // warp-uniform when quad
            link_flush(p, e, la, true);
            la.w = lag / p.l;
            la.next = (la.w + 1) * p.l;
        }
        const float re0 = __uint_as_float(v[4 * i + 0]) * p.inv_m;
        const float re1 = __uint_as_float(v[4 * i + 1]) * p.inv_m;
        const float im0 = __uint_as_float(v[4 * i + 2]) * p.inv_m;
        const float im1 = __uint_as_float(v[4 * i + 3]) * p.inv_m;
        if (e.out < 0 || lag >= e.n_valid) continue;
        // (non-finite taps show up in s_sq: the caller flags a recount from it, see below)
        float* dst = p.taps + 2 * (e.out + lag);
        PNCE_CHECK(e.out + lag >= 0 && e.out + lag + (lag + 1 < e.n_valid ? 1 : 0) < p.n_taps);
        const float q0 = err_acc(re0, im0, h[i].x, h[i].y, s_abs, s_sq);
        if (lag + 1 < e.n_valid) {
            if (e.vec) {
                st_global_v4(dst, re0, im0, re1, im1);
            } else {
                *reinterpret_cast<float2*>(dst) = make_float2(re0, im0);
                *reinterpret_cast<float2*>(dst + 2) = make_float2(re1, im1);
            }
            const float q1 = err_acc(re1, im1, h[i].z, h[i].w, s_abs, s_sq);
            if (p.link_err != nullptr) {
                if (quad) {
                    la.part += q0 + q1;
                } else {
                    link_add(p, e, la, lag, q0);
                    link_add(p, e, la, lag + 1, q1);
                }
            }
        } else {
            *reinterpret_cast<float2*>(dst) = make_float2(re0, im0);
            if (p.link_err != nullptr) {
                if (quad) la.part += q0;
                else link_add(p, e, la, lag, q0);
            }
        }
    }
}

__device__ __forceinline__ void epi_block_scored(const CorrParams& p, uint32_t taddr, const EpiLink& e, int n0,
                                                 float& s_abs, float& s_sq, float& nf, int cols) {
    // cols: multiple of 32 here
    const bool quad = (p.l & 7) == 0;
    LinkAcc la{-1, 0, 0.f};
    float4 h0[4], h1[4];
    uint32_t v[16];
    int c = 0;
    load_truth4(p, e, n0, h0);
    auto step = [&](float4 (&hc)[4], float4 (&hn)[4]) -> bool {
        tmem_ld_16x256b_x4(taddr + c, v);
        if (c + 32 < cols) load_truth4(p, e, n0 + c + 32, hn);
        tmem_wait_ld();
        epi_reps_scored(p, v, hc, e, n0 + c, s_abs, s_sq, nf, la, quad);
        c += 32;
        return c < cols;
    };
    while (step(h0, h1) && step(h1, h0)) {
    }
    if (p.link_err != nullptr) link_flush(p, e, la, quad);
    // a non-finite tap (or truth) makes the squared-error sum non-finite; overflow of finite
    // errors also lands here, which only costs the exact recount
    if (!isfinite(s_sq)) nf = 1.f;
}

// Scored drain with the truth staged through shared memory: each thread keeps a private
// ring of D 32-column chunks (4 x 16 B per chunk: its two lags of every 8-lag repetition)
// filled by LDGSTS, so D chunks of truth are in flight without holding registers -- the
// register path above keeps one chunk in flight and is L2-latency bound.  Layout per warp:
// [slot][rep][lane] x 16 B (conflict-free LDS.128).  Needs 16-byte aligned truth runs (even L).
template <int D>
__device__ __forceinline__ void epi_block_scored_smem(const CorrParams& p, uint32_t taddr, const EpiLink& e, int n0,
                                                      uint32_t ring, float& s_abs, float& s_sq, float& nf,
                                                      int cols) {
    // cols: multiple of 32 here
    const bool quad = (p.l & 7) == 0;
    const int lane = threadIdx.x & 31;
    LinkAcc la{-1, 0, 0.f};
    auto issue = [&](int c, int slot) {
        if (c < cols) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int lag = n0 + c + 8 * i;
                const bool ok = e.out >= 0 && lag < e.n_valid;
                const uint32_t bytes = ok ? (lag + 1 < e.n_valid ? 16u : 8u) : 0u;
                const float* src = ok ? p.truth + 2 * (e.out + lag) : p.truth;
                PNCE_CHECK(!ok || (e.out + lag + (bytes == 16u ? 1 : 0) < p.n_taps));
                cp_async_16(ring + (uint32_t)(((slot * 4 + i) * 32 + lane) * 16), src, bytes);
            }
        }
        cp_async_commit();  // (empty groups keep the in-order group count uniform)
    };
#pragma unroll
    for (int d = 0; d < D; ++d) issue(32 * d, d);
    uint32_t v[16];
    float4 h[4];
    int slot = 0;
    for (int c = 0; c < cols; c += 32) {
        tmem_ld_16x256b_x4(taddr + c, v);
        cp_async_wait<D - 1>();  // chunk c's group has landed (groups retire in order)
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = ld_shared_v4f(ring + (uint32_t)(((slot * 4 + i) * 32 + lane) * 16));
        tmem_wait_ld();
        epi_reps_scored(p, v, h, e, n0 + c, s_abs, s_sq, nf, la, quad);
        issue(c + 32 * D, slot);  // refill the slot just consumed (its values are in registers)
        if (++slot == D) slot = 0;
    }
    cp_async_wait<0>();
    if (p.link_err != nullptr) link_flush(p, e, la, quad);
    if (!isfinite(s_sq)) nf = 1.f;  // (as epi_block_scored)
}

// Fast drain of one 16-lane block when every lag this thread owns is valid, the run is
// 16-byte aligned and nothing is scored: no per-lag predicates, one pointer per block,
// 4 FMUL + one 16-byte store per repetition.
__device__ __forceinline__ void epi_reps_fast(const uint32_t* v, float* dst, float s, int reps, uint64_t pol) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (i < reps) {
#ifdef PNCE_DIAG_NO_STORE
            const float x = __uint_as_float(v[4 * i]) * s;
            if (x == 12345.678f) dst[0] = x;
#else
            if (pol)
                st_global_v4_hint(dst + 16 * i, __uint_as_float(v[4 * i + 0]) * s, __uint_as_float(v[4 * i + 2]) * s,
                                  __uint_as_float(v[4 * i + 1]) * s, __uint_as_float(v[4 * i + 3]) * s, pol);
            else
                st_global_v4(dst + 16 * i, __uint_as_float(v[4 * i + 0]) * s, __uint_as_float(v[4 * i + 2]) * s,
                             __uint_as_float(v[4 * i + 1]) * s, __uint_as_float(v[4 * i + 3]) * s);
#endif
        }
    }
}

template <bool GA = false>
__device__ __forceinline__ void epi_block_fast(const CorrParams& p, uint32_t taddr, float* dst, int cols) {
    const float s = p.inv_m;
    // GA: the same registers also go to every peer's CSI (same offset in each buffer)
    const int64_t off = dst - p.taps;
    auto emit = [&](const uint32_t* v, int c, int reps, uint64_t pol) {
        epi_reps_fast(v, dst + 2 * c, s, reps, pol);
        if constexpr (GA)
            for (int d = 0; d < p.gather_n; ++d) epi_reps_fast(v, p.gather_dst[d] + off + 2 * c, s, reps, pol);
    };
    PNCE_CHECK(dst >= p.taps && dst + 2 * cols - 12 <= p.taps + 2 * p.n_taps);  // last 16-byte store of the thread
    const uint64_t pol = p.store_hint == 1   ? policy_evict_first()
                         : p.store_hint == 2 ? policy_evict_last()
                         : p.store_hint == 3 ? policy_evict_normal()
                                             : 0ull;
    int c = 0;
    uint32_t va[32], vb[32];
    if (cols >= 64) {
        tmem_ld_16x256b_x8(taddr, va);
        tmem_wait_ld();
        while (true) {
            const bool more = c + 128 <= cols;
            if (more) tmem_ld_16x256b_x8(taddr + c + 64, vb);
            emit(va, c, 8, pol);
            c += 64;
            if (!more) break;
            tmem_wait_ld();
            const bool more2 = c + 128 <= cols;
            if (more2) tmem_ld_16x256b_x8(taddr + c + 64, va);
            emit(vb, c, 8, pol);
            c += 64;
            if (!more2) break;
            tmem_wait_ld();
        }
    }
    for (; c < cols; c += 16) {
        uint32_t v[8];
        tmem_ld_16x256b_x2(taddr + c, v);
        tmem_wait_ld();
        emit(v, c, 2, pol);
    }
}

// Exact non-finite count of the taps this thread wrote for one link (rare path: only
// when the sticky detector fired).  Reads back this thread's own stores.
__device__ __noinline__ float recount_nonfinite(const CorrParams& p, const EpiLink& e, int n0) {
    float bad = 0.f;
    for (int c = 0; c < p.g_cols; c += 8)
        for (int t = 0; t < 2; ++t) {
            const int lag = n0 + c + t;
            if (lag < e.n_valid) {
                const volatile float* v = p.taps + 2 * (e.out + lag);
                const float x = v[0], y = v[1];
                if (!(isfinite(x) && isfinite(y))) bad += 1.f;
            }
        }
    return bad;
}

// tensor16 fold (halfprec.py:104-125 on real tensor cores): the accumulation unit just
// finished in TMEM (binary16 or binary32 partial of one chunk) is widened to fp32, scaled
// by fp32(1/M) and added to the fp32 running total in TMEM (two roundings, as the
// reference's `total + acc * scale`); the last unit writes the demuxed taps.  Any
// non-finite partial or total raises the (frame-set, batch) saturation flag.
__device__ __forceinline__ void t16_fold(const CorrParams& p, uint32_t t_part, uint32_t t_tot, const EpiLink& e,
                                         int n0, bool first, bool last, bool& sat) {
    for (int c = 0; c < p.g_cols; c += 32) {
        uint32_t d[16], t[16];
        tmem_ld_16x256b_x4(t_part + c, d);
        if (!first) tmem_ld_16x256b_x4(t_tot + c, t);
        tmem_wait_ld();
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const float x = p.acc16 ? __half2float(__ushort_as_half((unsigned short)(d[i] & 0xffffu)))
                                    : __uint_as_float(d[i]);
            if (!isfinite(x)) sat = true;
            const float y = __fmul_rn(x, p.inv_m);
            v[i] = first ? y : __fadd_rn(__uint_as_float(t[i]), y);
        }
        if (!last) {
            uint32_t w[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) w[i] = __float_as_uint(v[i]);
            tmem_st_16x256b_x4(t_tot + c, w);
        } else if (e.out >= 0) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int lag = n0 + c + 8 * r;
                const float re0 = v[4 * r], re1 = v[4 * r + 1], im0 = v[4 * r + 2], im1 = v[4 * r + 3];
                if (lag >= e.n_valid) continue;
                if (!(isfinite(re0) && isfinite(im0))) sat = true;
                float* dst = p.taps + 2 * (e.out + lag);
                PNCE_CHECK(e.out + lag >= 0 && e.out + lag + (lag + 1 < e.n_valid ? 1 : 0) < p.n_taps);
                if (lag + 1 < e.n_valid) {
                    if (!(isfinite(re1) && isfinite(im1))) sat = true;
                    if (e.vec) {
                        st_global_v4(dst, re0, im0, re1, im1);
                    } else {
                        *reinterpret_cast<float2*>(dst) = make_float2(re0, im0);
                        *reinterpret_cast<float2*>(dst + 2) = make_float2(re1, im1);
                    }
                } else {
                    *reinterpret_cast<float2*>(dst) = make_float2(re0, im0);
                }
            }
        }
    }
    if (!last) tmem_wait_st();
}

// Intermediate tensor16 fold (every accumulation unit but the last): elementwise on the
// warp's 32 TMEM lanes, layout-agnostic, so the 32x32b.x32 shape (32 columns per thread per
// load) halves the instruction count of the 16x256b path; the next 32 columns are in flight
// while this block is folded.  total = fl32(total + fl32(fl32(partial) * fl32(1/M))), two
// roundings as halprec.py:104-117; a non-finite partial or total leaves `nf` non-finite.
__device__ __forceinline__ void t16_fold_mid(const CorrParams& p, uint32_t t_part, uint32_t t_tot, bool first,
                                             float& nf, int c0, int c1) {
    uint32_t pa[32], ta[32];
    for (int c = c0; c < c1; c += 32) {
        tmem_ld32_nowait(t_part + c, pa);
        if (!first) tmem_ld32_nowait(t_tot + c, ta);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const float x = p.acc16 ? __half2float(__ushort_as_half((unsigned short)(pa[i] & 0xffffu)))
                                    : __uint_as_float(pa[i]);
            const float y = __fmul_rn(x, p.inv_m);
            const float t = first ? y : __fadd_rn(__uint_as_float(ta[i]), y);
            nf = fmaf(t, 0.f, nf);   // inf / NaN anywhere -> NaN (sticky)
            ta[i] = __float_as_uint(t);
        }
        tmem_st32(t_tot + c, ta);
    }
    tmem_wait_st();
}

// GATHER: plain launches whose epilogue also stores every tap into the peers' CSI buffers
// (pnce_process_frames_gather; a separate instantiation so the other drains keep their registers)
template <int MODE, bool SCORED, bool EPI8 = false, bool T16 = false, bool GATHER = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsK3, 1)
k_correlate(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_circ,
            const __grid_constant__ CUtensorMap tm_scr, const CorrParams p) {
    constexpr bool A_TMA = MODE == kModePacked;     // A via TMA with the circulant
    constexpr bool RAW = MODE == kModeFusedTma;     // f32 rows TMA-staged, converted
    constexpr bool FLDG = MODE == kModeFusedLdg;    // f32 rows LDG'd, converted
    constexpr bool PLDG = MODE == kModePackedLdg;   // packed 16-bit rows LDG'd
    // Warp layout: EPI8 trades 4 converter warps for epilogue warps (the scored variant's
    // default: its drain does ~4x the work; packed/TMA mode has no converter work)
    constexpr int kCW = (EPI8 && (RAW || A_TMA)) ? 4 : kConvWarps;
    constexpr int kEW0 = kConvWarp0 + kCW;
    constexpr int kEW = kWarps - kEW0;
    // converter warps arriving per stage (both CTAs): all 8 (RAW), one 4-warp group (FLDG),
    // one 2-warp group (PLDG)
    constexpr int kConvArrivals = RAW ? 2 * kCW : (FLDG ? kConvWarps : (PLDG ? kConvWarps / 2 : 0));
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    // [A/B stages][1 KB barrier block][raw f32 stages]
    const int S = p.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * p.stage_bytes);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint64_t* raw_full = tempty + 2;
    uint64_t* raw_empty = raw_full + (RAW ? p.raw_stages : 0);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(raw_empty + (RAW ? p.raw_stages : 0));
    uint8_t* raw_base = smem + (size_t)S * p.stage_bytes + p.bar_bytes;
    // a_reuse: per (slot, K-block) "A stage stored" barriers in the second KB of the block
    uint64_t* scr_full = reinterpret_cast<uint64_t*>(smem + (size_t)S * p.stage_bytes + 1024);
    const bool reuse = RAW && p.a_reuse;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    if (threadIdx.x == 0) TRACE(13, 0);  // kernel entry

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            // Leader: producer expect_tx + the converter warps of BOTH CTAs (the peer's TMA
            // bytes and converter arrives land on the leader's barrier).
            // (LDG mode: only one 4-warp group converts a given stage)
            mbar_init(&full[s], 1 + kConvArrivals);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * kEW);
        }
        if (RAW) {
            for (int s = 0; s < p.raw_stages; ++s) {
                mbar_init(&raw_full[s], 1);
                mbar_init(&raw_empty[s], kCW);
            }
        }
        if (reuse)
            for (int s = 0; s < 2 * p.k_blocks; ++s) mbar_init(&scr_full[s], 1);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        if (A_TMA || RAW) tma_prefetch(&tm_in);
        tma_prefetch(&tm_circ);
        if (reuse) tma_prefetch(&tm_scr);
    }
    if (warp == 1) tmem_alloc_pair(tmem_slot, p.tmem_cols);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) TRACE(14, 0);  // prologue done

    const int n_clusters = gridDim.x >> 1;
    const int cid = blockIdx.x >> 1;
    const int total_tiles = p.m_tiles * p.n_groups;
    // Tile order: tile = cid + ti * n_clusters, (row tile, group) = divmod(tile, n_groups);
    // with a_reuse a cluster takes whole row tiles (all groups back to back, group 0 first).
    const int my_rows = cid < p.m_tiles ? (p.m_tiles - 1 - cid) / n_clusters + 1 : 0;
    const int my_tiles = reuse ? my_rows * p.n_groups
                               : (cid < total_tiles ? (total_tiles - 1 - cid) / n_clusters + 1 : 0);
    auto coords = [&](int ti) -> int2 {  // (row tile, group)
        if (reuse) {
            const int r = ti / p.n_groups;
            return make_int2(cid + r * n_clusters, ti - r * p.n_groups);
        }
        const int tile = cid + ti * n_clusters;
        const int mt = tile / p.n_groups;
        return make_int2(mt, tile - mt * p.n_groups);
    };
    // scratch row of (row-tile iteration r, this CTA, K-block kb); slots alternate per row tile
    auto scr_row = [&](int r, int kb) -> int {
        const int row = ((((r % p.scr_slots) * n_clusters + cid) * 2 + (int)rank) * p.k_blocks + kb) * kBM;
        PNCE_CHECK(row >= 0 && row + kBM <= p.scr_rows);
        return row;
    };
    const int jobs = my_tiles * p.k_blocks;  // one job = one K-block of one tile
    const uint32_t a_bytes = kBM * kBK * 2;
    const uint32_t b_half_bytes = (uint32_t)(p.nm / 2) * kBK * 2;
    // split drain (single accumulator of two N halves): the epilogue releases the first half
    // early on tempty[1] and the MMA warp starts the next tile's first-half MMAs on it
    const bool split = !T16 && p.split_drain && p.acc_stages == 1 && p.n_mma == 2;


    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer: circulant rows (+ packed sample rows); bytes land on the leader
            const uint64_t pol_in = p.raw_pol == 0 ? policy_evict_first()
                                                   : (p.raw_pol == 2 ? policy_evict_last() : policy_evict_normal());
            const uint64_t pol_circ = policy_evict_last();
            int kb = 0, ti = 0, stage = 0, mt = 0, g = 0;
            { const int2 _c = coords(0); mt = _c.x; g = _c.y; }
            uint32_t phase = 0;
#ifdef PNCE_DIAG_PROF
            uint64_t prof_scr_wait = 0;
#endif
            PROF_BEGIN(2);
            for (int j = 0; j < jobs; ++j) {
                mbar_wait(&empty[stage], phase ^ 1u);
                PROF_MARK(0);
                TRACE(0, j);
                uint8_t* sa = smem + (size_t)stage * p.stage_bytes;
                uint8_t* sb = sa + a_bytes;
                const uint32_t fb_leader = mapa_shared(smem_u32(&full[stage]), 0);
                const bool from_scr = reuse && g > 0;
                const int r = ti / p.n_groups;
                if (from_scr) {
                    // group 0 of this row tile stored the converted A stage of K-block kb
#ifdef PNCE_DIAG_PROF
                    const uint64_t w0 = clock64();
#endif
                    mbar_wait(&scr_full[(r % p.scr_slots) * p.k_blocks + kb], (uint32_t)(r / p.scr_slots) & 1u);
#ifdef PNCE_DIAG_PROF
                    prof_scr_wait += clock64() - w0;
#endif
                    fence_proxy_async_global();
                }
#ifdef PNCE_DIAG_NO_B
                // diagnostic: no circulant loads (B stage left as is; results are garbage)
                if (leader) mbar_arrive_expect_tx(&full[stage], (A_TMA ? 2 * a_bytes : 0u) + (from_scr ? 2 * a_bytes : 0u));
                (void)sb;
#else
                if (leader) mbar_arrive_expect_tx(&full[stage], p.tx_bytes + (from_scr ? 2 * a_bytes : 0u));
#endif
                if (A_TMA)
                    tma_load_2d_pair(sa, &tm_in, fb_leader, kb * kBK, mt * 2 * kBM + (int)rank * kBM, pol_in);
                if (from_scr)  // keep the stage in L2 for the row tile's later groups
                    tma_load_2d_pair(sa, &tm_scr, fb_leader, 0, scr_row(r, kb),
                                     g == p.n_groups - 1 ? policy_evict_first()
                                                         : (p.scr_pol ? policy_evict_last() : policy_evict_normal()));
#ifndef PNCE_DIAG_NO_B
                for (int jj = 0; jj < p.n_mma; ++jj)
                    tma_load_2d_pair(sb + jj * b_half_bytes, &tm_circ, fb_leader, kb * kBK,
                                     g * p.g_cols + jj * p.nm + (int)rank * (p.nm / 2), pol_circ);
#endif
                if (++stage == S) { stage = 0; phase ^= 1u; }
                if (++kb == p.k_blocks) {
                    kb = 0;
                    { const int2 _c = coords(++ti); mt = _c.x; g = _c.y; }
                }
                PROF_MARK(1);
            }
            PROF_END(0, 2);
#ifdef PNCE_DIAG_PROF
            g_prof[blockIdx.x * kProfSlots + 15] = prof_scr_wait;
#endif
        }
    } else if (warp == 1) {
        if (leader && lane == 0 && split) {
            // ===== MMA issuer, split-drain variant: per K-block the first-half MMAs (columns
            // [0, nm)) go as soon as the epilogue released that half; second-half MMAs of the
            // stages held meanwhile are issued once the whole accumulator is drained.
            int stage = 0;
            uint32_t phase = 0, tphase = 0;
            int pend_stage0 = 0, pend_kb0 = 0;  // held stages are consecutive (ring order, kb order)
            auto issue_half = [&](int st, int kb, int jj) {
                const uint32_t sa = smem_u32(smem + (size_t)st * p.stage_bytes);
                const uint32_t sb = sa + a_bytes;
#pragma unroll
                for (int ks = 0; ks < kBK / kUmmaK; ++ks) {
                    const uint64_t ad = make_sdesc(sa + ks * 32, 16, 1024, 2);
                    const uint64_t bd = make_sdesc(sb + jj * b_half_bytes + ks * 32, 16, 1024, 2);
                    umma_f16_ss_pair(tmem_base + (uint32_t)(jj * p.nm), ad, bd, p.idesc, (kb | ks) != 0);
                }
            };
            PROF_BEGIN(3);
            for (int ti = 0; ti < my_tiles; ++ti) {
                mbar_wait(&tempty[1], tphase ^ 1);
                PROF_MARK(0);
                TRACE(1, ti);
                tc_fence_after();
                bool hi_ok = false;
                int np = 0;
                auto flush = [&]() {
                    tc_fence_after();
                    hi_ok = true;
                    int st = pend_stage0;
                    for (int i = 0; i < np; ++i) {
                        issue_half(st, pend_kb0 + i, 1);
                        umma_commit_pair(&empty[st]);
                        if (++st == S) st = 0;
                    }
                    np = 0;
                };
                for (int kb = 0; kb < p.k_blocks; ++kb) {
                    if (!hi_ok && np == S) {  // every stage held: wait for the whole drain
                        mbar_wait(&tempty[0], tphase ^ 1);
                        flush();
                    }
                    mbar_wait(&full[stage], phase);
                    PROF_MARK(1);
                    TRACE(2, ti * p.k_blocks + kb);
                    tc_fence_after();
                    if (!hi_ok && mbar_test_wait(&tempty[0], tphase ^ 1)) flush();
                    issue_half(stage, kb, 0);
                    if (hi_ok) {
                        issue_half(stage, kb, 1);
                        umma_commit_pair(&empty[stage]);
                    } else {
                        if (np++ == 0) {
                            pend_stage0 = stage;
                            pend_kb0 = kb;
                        }
                    }
                    if (++stage == S) { stage = 0; phase ^= 1u; }
                    PROF_MARK(2);
                }
                if (!hi_ok) {
                    mbar_wait(&tempty[0], tphase ^ 1);
                    flush();
                }
                umma_commit_pair(&tfull[0]);
                tphase ^= 1;
            }
            PROF_END(2, 3);
        } else if (leader && lane == 0) {
            // ===== MMA issuer (leader CTA, single thread) for the whole pair
            int acc = 0, stage = 0;
            uint32_t acc_phase = 0, phase = 0;
#ifdef PNCE_DIAG_PROF
            const uint64_t t_start = clock64();
#endif
            PROF_BEGIN(3);
            for (int ti = 0; ti < my_tiles; ++ti) {
                uint32_t d_tmem = 0;
                int kc = 0;  // K-block within the accumulation unit (the whole K outside tensor16)
                for (int kb = 0; kb < p.k_blocks; ++kb) {
                    const int j = ti * p.k_blocks + kb;
                    if (kc == 0) {
                        mbar_wait(&tempty[acc], acc_phase ^ 1);
                        PROF_MARK(0);
                        TRACE(1, ti);
                        tc_fence_after();
                        d_tmem = tmem_base + (uint32_t)(acc * p.g_cols);
                    }
#ifndef PNCE_DIAG_NO_FULLWAIT
                    mbar_wait(&full[stage], phase);
#else
                    (void)phase;
#endif
                    PROF_MARK(1);
                    TRACE(2, j);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + (size_t)stage * p.stage_bytes);
                    const uint32_t sb = sa + a_bytes;
#pragma unroll
                    for (int ks = 0; ks < kBK / kUmmaK; ++ks) {
                        const uint64_t ad = make_sdesc(sa + ks * 32, 16, 1024, 2);
                        for (int jj = 0; jj < p.n_mma; ++jj) {
                            const uint64_t bd = make_sdesc(sb + jj * b_half_bytes + ks * 32, 16, 1024, 2);
                            umma_f16_ss_pair(d_tmem + (uint32_t)(jj * p.nm), ad, bd, p.idesc, (kc | ks) != 0);
                        }
                    }
                    umma_commit_pair(&empty[stage]);
                    TRACE(3, j);
                    (void)j;
                    if (++stage == S) { stage = 0; phase ^= 1u; }
                    PROF_MARK(2);
                    if (++kc == p.chunk_kb || kb == p.k_blocks - 1) {
                        umma_commit_pair(&tfull[acc]);
                        if (++acc == p.acc_stages) { acc = 0; acc_phase ^= 1; }
                        kc = 0;
                    }
                }
            }
            PROF_END(2, 3);
#ifdef PNCE_DIAG_PROF
            g_prof[blockIdx.x * kProfSlots + 12] = clock64() - t_start;
#endif
        }
    } else if (warp == 2) {
        if (RAW && lane == 0) {
            // ===== raw-chunk producer: TMA the f32 (I,Q) rows of this CTA's 64 links for half a
            // K-block (64 links x 32 samples x 8 B = 16 KB, +16 B per row when C is odd) into the
            // staging ring.  Finer chunks = more loads in flight for the same shared memory.
            // evict_first when a row tile is read once; with several lag-row groups the
            // neighbouring cluster reads the same rows for the next group (tiles are g-minor)
            const uint64_t pol = p.raw_pol == 0 ? policy_evict_first()
                                                : (p.raw_pol == 2 ? policy_evict_last() : policy_evict_normal());
            int kb = 0, ti = 0, rs = 0, mt = 0, g = 0;
            { const int2 _c = coords(0); mt = _c.x; g = _c.y; }
            uint32_t rphase = 0;
            PROF_BEGIN(2);
            for (int j = 0; j < jobs; ++j) {
                // a_reuse: only group 0 reads the raw rows
#pragma unroll
                for (int h = 0; h < 2 && !(reuse && g > 0); ++h) {
                    mbar_wait(&raw_empty[rs], rphase ^ 1u);
                    PROF_MARK(0);
                    if (h == 0) TRACE(6, j);
#ifdef PNCE_DIAG_NO_RAW
                    mbar_arrive(&raw_full[rs]);
                    (void)pol; (void)mt; (void)kb;
#else
                    mbar_arrive_expect_tx(&raw_full[rs], p.raw_stage_bytes);
                    // box start rounded down to a 16-byte boundary; converters skip the slack
                    tma_load_2d(raw_base + (size_t)rs * p.raw_stage_bytes, &tm_in, &raw_full[rs],
                                (2 * (p.c + kb * kBK + h * kRawChunk)) & ~3, (mt * 2 + (int)rank) * kLinksPerTile,
                                pol);
#endif
                    if (++rs == p.raw_stages) { rs = 0; rphase ^= 1u; }
                    PROF_MARK(1);
                }
                if (++kb == p.k_blocks) {
                    kb = 0;
                    { const int2 _c = coords(++ti); mt = _c.x; g = _c.y; }
                }
            }
            PROF_END(5, 2);
        }
    } else if (warp >= kConvWarp0 && warp < kEW0) {
        if (RAW) {
            const int cw = warp - kConvWarp0;
            int kb = 0, stage = 0, rs = 0, ti = 0, mt = 0, g = 0;
            { const int2 _c = coords(0); mt = _c.x; g = _c.y; }
            uint32_t phase = 0, rphase = 0;
#ifdef PNCE_DIAG_PROF
            uint64_t prof_read_wait = 0, prof_bar_wait = 0, prof_done_wait = 0;
#endif
            PROF_BEGIN(3);
            for (int j = 0; j < jobs; ++j) {
                const uint32_t sa = smem_u32(smem + (size_t)stage * p.stage_bytes);
                if (reuse && g > 0) {
                    // the A stage comes from the scratch by TMA: only keep the arrival count
                    mbar_wait(&empty[stage], phase ^ 1u);
                    __syncwarp();
                    if (lane == 0) mbar_arrive_remote(mapa_shared(smem_u32(&full[stage]), 0));
                } else {
                    // staged f32 chunks -> A stage.  Per chunk a warp converts 8 links: lanes
                    // 0-15 link a, lanes 16-31 link a+4 (so the two Re rows fall in different
                    // swizzle halves: conflict-free STS); lane l handles samples 2(l%16), +1
                    // (one LDS.128 of the link's 256 B row, two STS.32 into its Re / Im rows).
                    mbar_wait(&empty[stage], phase ^ 1u);
                    PROF_MARK(0);
                    if (cw == 0 && lane == 0) TRACE(8, j);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        mbar_wait(&raw_full[rs], rphase);
                        PROF_MARK(1);
                        if (h == 0 && cw == 0 && lane == 0) TRACE(7, j);
                        const int slack = (2 * (p.c + kb * kBK + h * kRawChunk)) & 3;  // 0 or 2 floats
                        const uint32_t raw =
                            smem_u32(raw_base + (size_t)rs * p.raw_stage_bytes) + slack * 4 + (lane & 15) * 16;
                        const int k = kb * kBK + h * kRawChunk + 2 * (lane & 15);
                        const bool ok0 = k < p.m, ok1 = k + 1 < p.m;
                        const int col_byte = h * 64 + (lane & 15) * 4;
#ifndef PNCE_DIAG_NO_CONV
                        // all of the chunk's LDS first, then the conversions and STS: the loads
                        // overlap instead of one LDS -> F2FP -> STS round trip per link pair
                        constexpr int kIt = kLinksPerTile / (2 * kCW);
                        float4 v[kIt];
#pragma unroll
                        for (int it = 0; it < kIt; ++it) {
                            const int idx = cw + kCW * it;  // 0..31
                            const int link = (idx & 3) | ((lane >> 4) << 2) | ((idx >> 2) << 3);
                            const uint32_t src = raw + link * (p.raw_row_floats * 4);
                            PNCE_CHECK(src + 16 <= smem_u32(raw_base + (size_t)(rs + 1) * p.raw_stage_bytes));
                            if (slack == 0) {
                                v[it] = ld_shared_v4f(src);
                            } else {
                                const float2 a = ld_shared_v2f(src);
                                const float2 b = ld_shared_v2f(src + 8);
                                v[it] = make_float4(a.x, a.y, b.x, b.y);
                            }
                        }
#pragma unroll
                        for (int it = 0; it < kIt; ++it) {
                            const int idx = cw + kCW * it;
                            const int link = (idx & 3) | ((lane >> 4) << 2) | ((idx >> 2) << 3);
                            PNCE_CHECK(swz(sa, (int)a_row(link, 1), col_byte) + 4 <= sa + kBM * kBK * 2);
                            if (!ok0) { v[it].x = 0.f; v[it].y = 0.f; }
                            if (!ok1) { v[it].z = 0.f; v[it].w = 0.f; }
                            st_shared_u32(swz(sa, (int)a_row(link, 0), col_byte), pack2(v[it].x, v[it].z, p.bf16));
                            st_shared_u32(swz(sa, (int)a_row(link, 1), col_byte), pack2(v[it].y, v[it].w, p.bf16));
                        }
#else
                        (void)raw; (void)ok0; (void)ok1; (void)col_byte;
#endif
                        // the chunk's values are consumed (the STS above depend on them)
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&raw_empty[rs]);
                        if (++rs == p.raw_stages) { rs = 0; rphase ^= 1u; }
                        PROF_MARK(2);
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        // proxy fence above completed this warp's STS; plain (CTA-scope
                        // release) arrive on the leader's barrier, no GPU-scope membar
                        mbar_arrive_remote(mapa_shared(smem_u32(&full[stage]), 0));
                        if (cw == 0) TRACE(9, j);
                    }
                    if (reuse) {
                        // group 0: store the converted A stage (16 KB, swizzled image) to the
                        // scratch for the row tile's other groups once every converter warp has
                        // fenced its STS.  The issuer first waits for the previous store's smem
                        // reads (issued a job ago: that stage is rewritten after this barrier
                        // when S = 2); a K-block's barrier fires once its store has completed,
                        // kScrLag stores later (all of them at the row tile's last K-block).
                        constexpr int kScrLag = 4;
#ifdef PNCE_DIAG_PROF
                        const uint64_t w0 = clock64();
#endif
                        if (cw == 0 && lane == 0) bulk_wait_read<0>();
#ifdef PNCE_DIAG_PROF
                        const uint64_t w1 = clock64();
#endif
                        named_bar_sync(1, kCW * 32);
#ifdef PNCE_DIAG_PROF
                        const uint64_t w2 = clock64();
                        prof_read_wait += w1 - w0;
                        prof_bar_wait += w2 - w1;
#endif
                        if (cw == 0 && lane == 0) {
                            const int r = ti / p.n_groups;
                            if (p.scr_pol)
                                bulk_store_s2g_hint(p.scratch + (size_t)scr_row(r, kb) * 128, sa, a_bytes,
                                                    policy_evict_last());
                            else
                                bulk_store_s2g(p.scratch + (size_t)scr_row(r, kb) * 128, sa, a_bytes);
                            bulk_commit();
                            uint64_t* sf = &scr_full[(r % p.scr_slots) * p.k_blocks];
#ifdef PNCE_DIAG_PROF
                            const uint64_t w3 = clock64();
#endif
                            if (kb == p.k_blocks - 1) {
                                bulk_wait<0>();
                                for (int q = max(0, kb - kScrLag); q <= kb; ++q) mbar_arrive(&sf[q]);
                            } else if (kb >= kScrLag) {
                                bulk_wait<kScrLag>();
                                mbar_arrive(&sf[kb - kScrLag]);
                            }
#ifdef PNCE_DIAG_PROF
                            prof_done_wait += clock64() - w3;
#endif
                        }
                    }
                }
                PROF_MARK(2);
                if (++stage == S) { stage = 0; phase ^= 1u; }
                if (++kb == p.k_blocks) {
                    kb = 0;
                    { const int2 _c = coords(++ti); mt = _c.x; g = _c.y; }
                }
            }
            if (reuse && cw == 0 && lane == 0) bulk_wait<0>();  // shared memory must outlive the stores
            if (cw == 0 && lane == 0) PROF_END(7, 3);
#ifdef PNCE_DIAG_PROF
            if (cw == 0 && lane == 0) {
                g_prof[blockIdx.x * kProfSlots + 13] = prof_read_wait + prof_bar_wait;
                g_prof[blockIdx.x * kProfSlots + 14] = prof_done_wait;
            }
#endif
        } else if (FLDG) {
            // ===== pipelined LDG converters.  Group gsel (warps 4-7 / 8-11) converts the jobs
            // j = gsel (mod 2); each thread holds one K-block of its 16 links' samples in
            // registers (64 links x 64 samples per group = 32 KB in flight per group), issued
            // right AFTER the previous job's proxy fence -- fence.proxy.async waits for the
            // thread's outstanding loads, so loads must never straddle it.  Loads go through
            // L1 (LDG), a separate ingress path from the TMA engine that feeds the circulant.
            const int cw = warp - kConvWarp0;
            const int gsel = cw >> 2, gw = cw & 3;
            const bool vec = ((p.samples | p.c) & 1) == 0 && (reinterpret_cast<uintptr_t>(p.iq) & 15) == 0;
            float4 v[kLinksPerTile / 4];
            int kb = gsel % p.k_blocks, ti = gsel / p.k_blocks;
            int stage = gsel % S;
            uint32_t phase = (uint32_t)(gsel / S) & 1u;
            auto load_job = [&](int lti, int lkb) {
                const int mt = (cid + lti * n_clusters) / p.n_groups;
                const int64_t link0 = ((int64_t)mt * 2 + rank) * kLinksPerTile + gw;
                const int k = lkb * kBK + 2 * lane;
                const bool ok0 = k < p.m, ok1 = k + 1 < p.m;
#pragma unroll
                for (int q = 0; q < kLinksPerTile / 4; ++q) {
                    const int64_t link = link0 + 4 * q;
                    const float* src = p.iq + 2 * (link * p.samples + p.c + k);
                    if (link < p.total_links && ok1 && vec) {
                        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                                     : "=f"(v[q].x), "=f"(v[q].y), "=f"(v[q].z), "=f"(v[q].w)
                                     : "l"(src));
                    } else {
                        const bool l_ok = link < p.total_links;
                        const float2 a = (l_ok && ok0) ? __ldg(reinterpret_cast<const float2*>(src)) : make_float2(0.f, 0.f);
                        const float2 b = (l_ok && ok1) ? __ldg(reinterpret_cast<const float2*>(src) + 1) : make_float2(0.f, 0.f);
                        v[q] = make_float4(a.x, a.y, b.x, b.y);
                    }
                }
            };
            if (gsel < jobs) load_job(ti, kb);
            PROF_BEGIN(3);
            for (int j = gsel; j < jobs; j += 2) {
                const uint32_t sa = smem_u32(smem + (size_t)stage * p.stage_bytes);
                mbar_wait(&empty[stage], phase ^ 1u);
                PROF_MARK(0);
                if (cw == 0 && lane == 0) TRACE(8, j);
#pragma unroll
                for (int q = 0; q < kLinksPerTile / 4; ++q) {
                    // link 4q + gw of the tile; lane -> samples 2*lane, 2*lane+1 (one 128 B row)
                    const int link_local = 4 * q + gw;
                    PNCE_CHECK(swz(sa, (int)a_row(link_local, 1), lane * 4) + 4 <= sa + kBM * kBK * 2);
                    st_shared_u32(swz(sa, (int)a_row(link_local, 0), lane * 4), pack2(v[q].x, v[q].z, p.bf16));
                    st_shared_u32(swz(sa, (int)a_row(link_local, 1), lane * 4), pack2(v[q].y, v[q].w, p.bf16));
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive_remote(mapa_shared(smem_u32(&full[stage]), 0));
                    if (cw == 0) TRACE(9, j);
                }
                // advance two jobs and prefetch the next one (after the fence)
                stage += 2;
                while (stage >= S) { stage -= S; phase ^= 1u; }
                kb += 2;
                while (kb >= p.k_blocks) { kb -= p.k_blocks; ++ti; }
                if (j + 2 < jobs) load_job(ti, kb);
                PROF_MARK(2);
            }
            if (cw == 0 && lane == 0) PROF_END(7, 3);
        }
        if (PLDG) {
            // ===== packed rows via LDG: 4 groups of 2 warps; group g copies the A tiles of
            // jobs j = g (mod 4).  Thread t of a group holds 16 of the stage's 128 rows x 8
            // 16-byte chunks in registers (64 KB in flight per CTA), loaded after the
            // previous job's proxy fence, and stores them into the 128B-swizzled stage.
            const int cw = warp - kConvWarp0;
            constexpr int kGroups = 4;
            const int gsel = cw >> 1;
            const int tid = (cw & 1) * 32 + lane;  // 0..63
            uint4 v[16];
            int kb = gsel % p.k_blocks, ti = gsel / p.k_blocks;
            int stage = gsel % S;
            uint32_t phase = (uint32_t)(gsel / S) & 1u;
            auto load_job = [&](int lti, int lkb) {
                const int mt = (cid + lti * n_clusters) / p.n_groups;
                const int64_t row0 = ((int64_t)mt * 2 + rank) * kBM;
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const int idx = tid + 64 * q;  // (row, chunk) = (idx / 8, idx % 8)
                    const int64_t row = row0 + (idx >> 3);
                    if (row < p.packed_rows) {
                        const uint16_t* src = p.packed + row * p.k_pad + lkb * kBK + (idx & 7) * 8;
                        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(v[q].x), "=r"(v[q].y), "=r"(v[q].z), "=r"(v[q].w)
                                     : "l"(src));
                    } else {
                        v[q] = make_uint4(0u, 0u, 0u, 0u);
                    }
                }
            };
            if (gsel < jobs) load_job(ti, kb);
            PROF_BEGIN(3);
            for (int j = gsel; j < jobs; j += kGroups) {
                const uint32_t sa = smem_u32(smem + (size_t)stage * p.stage_bytes);
                mbar_wait(&empty[stage], phase ^ 1u);
                PROF_MARK(0);
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const int idx = tid + 64 * q;
                    st_shared_v4(swz(sa, idx >> 3, (idx & 7) * 16), v[q]);
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(mapa_shared(smem_u32(&full[stage]), 0));
                stage += kGroups;
                while (stage >= S) { stage -= S; phase ^= 1u; }
                kb += kGroups;
                while (kb >= p.k_blocks) { kb -= p.k_blocks; ++ti; }
                if (j + kGroups < jobs) load_job(ti, kb);
                PROF_MARK(2);
            }
            if (cw == 0 && lane == 0) PROF_END(7, 3);
        }
    } else if (warp >= kEW0) {
        // ===== epilogue (both CTAs): warp q = warp % 4 owns TMEM lanes 32q..32q+31 = two
        // 16-row blocks = links 16q..16q+15 of this CTA's 64; thread t handles link
        // 8*block + t/4 of its quarter and lags 2(t%4), 2(t%4)+1 of every 8-lag repetition.
        const int quarter = warp & 3;
        // 4 epilogue warps: each drains both 16-lane blocks of its quarter; 8 (scored): one
        constexpr int kBlocksPerWarp = kEW == 4 ? 2 : 1;
        const int bb0 = kEW == 4 ? 0 : (warp - kEW0) >> 2;
        const int colp = 2 * (lane & 3);
        const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        PROF_BEGIN(2);
        if constexpr (T16) {
            // accumulation units of chunk_kb K-blocks; partials at columns [acc*G, (acc+1)*G)
            // (double-buffered when 3G <= 512: the MMA fills one while this folds the other),
            // running total at [acc_stages*G, (acc_stages+1)*G)
            const int n_units = (p.k_blocks + p.chunk_kb - 1) / p.chunk_kb;
            for (int ti = 0; ti < my_tiles; ++ti) {
                int mt, g;
                { const int2 _c = coords(ti); mt = _c.x; g = _c.y; }
                const int64_t link0 = ((int64_t)mt * 2 + rank) * kLinksPerTile + quarter * 16 + (lane >> 2);
                const int n0 = g * p.g_cols + colp;
                bool sat[2] = {false, false};
                float nf_mid = 0.f;
                for (int u = 0; u < n_units; ++u) {
                    mbar_wait(&tfull[acc], acc_phase);
                    tc_fence_after();
                    if (u < n_units - 1) {
                        // intermediate unit: elementwise over the warp's 32 lanes (both 16-lane
                        // blocks); with 8 epilogue warps the two warps of a quarter split the columns
                        const uint32_t lanes = (uint32_t)(quarter * 32) << 16;
                        const int half_cols = (p.g_cols / 64) * 32;   // a multiple of 32
                        const int c0 = kBlocksPerWarp == 2 ? 0 : bb0 * half_cols;
                        const int c1 = kBlocksPerWarp == 2 ? p.g_cols : (bb0 ? p.g_cols : half_cols);
                        t16_fold_mid(p, tmem_base + lanes + (uint32_t)(acc * p.g_cols),
                                     tmem_base + lanes + (uint32_t)(p.acc_stages * p.g_cols), u == 0, nf_mid, c0, c1);
                    } else {
#pragma unroll
                        for (int k = 0; k < kBlocksPerWarp; ++k) {
                            const int bb = bb0 + k;
                            const EpiLink e = make_link(p, link0 + 8 * bb);
                            const uint32_t lanes = (uint32_t)(quarter * 32 + 16 * bb) << 16;
                            t16_fold(p, tmem_base + lanes + (uint32_t)(acc * p.g_cols),
                                     tmem_base + lanes + (uint32_t)(p.acc_stages * p.g_cols), e, n0, u == 0,
                                     u == n_units - 1, sat[k]);
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster_relaxed(tempty_leader0 + (uint32_t)(acc * 8));
                    if (++acc == p.acc_stages) { acc = 0; acc_phase ^= 1; }
                }
                if (nf_mid != 0.f) {
                    // thread = TMEM lane = A row 32q + lane of this CTA: link (r / 16) * 8 + r % 8
                    const int r = quarter * 32 + lane;
                    const int64_t link = ((int64_t)mt * 2 + rank) * kLinksPerTile + ((r >> 4) << 3) + (r & 7);
                    if (link < p.total_links) atomicOr(p.sat_flags + (uint32_t)link / (uint32_t)p.n_r, 1u);
                }
#pragma unroll
                for (int k = 0; k < kBlocksPerWarp; ++k) {
                    const int64_t link = link0 + 8 * (bb0 + k);
                    if (sat[k] && link < p.total_links) atomicOr(p.sat_flags + (uint32_t)link / (uint32_t)p.n_r, 1u);
                }
            }
        } else
        for (int ti = 0; ti < my_tiles; ++ti) {
            int mt, g;
            { const int2 _c = coords(ti); mt = _c.x; g = _c.y; }
            const int64_t link0 = ((int64_t)mt * 2 + rank) * kLinksPerTile + quarter * 16 + (lane >> 2);
            // (links are re-derived where needed instead of kept live: register pressure)
            const int n0 = g * p.g_cols + colp;
#ifndef PNCE_DIAG_NO_TRUTH_PF
            // (not with the LDGSTS truth ring: its loads are in flight early enough, and the bulk
            // prefetches compete with the TMA loads for the copy engine: -5 % scored)
            if (SCORED && p.truth != nullptr && p.truth_slots == 0 && (lane & 3) == 0) {
#else
            if (false) {
#endif
                // pull this tile's truth windows into L2 while the MMAs run
                for (int k = 0; k < kBlocksPerWarp; ++k) {
                    const EpiLink e = make_link(p, link0 + 8 * (bb0 + k));
                    const int lag0 = g * p.g_cols;
                    const int n = min(p.g_cols, e.n_valid - lag0);
                    if (e.out >= 0 && n > 0) {
                        const uintptr_t a0 = reinterpret_cast<uintptr_t>(p.truth + 2 * (e.out + lag0)) & ~uintptr_t(15);
                        const uintptr_t a1 =
                            (reinterpret_cast<uintptr_t>(p.truth + 2 * (e.out + lag0 + n)) + 15) & ~uintptr_t(15);
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0))
                                     : "memory");
                    }
                }
            }
            // plain drain: decide the fast path and its output pointer before the wait
            float* fast_dst[2] = {nullptr, nullptr};
            if constexpr (!SCORED) {
#pragma unroll
                for (int k = 0; k < kBlocksPerWarp; ++k) {
                    const EpiLink e = make_link(p, link0 + 8 * (bb0 + k));
                    const bool ok = __all_sync(0xffffffffu, e.out >= 0 && e.vec && g * p.g_cols + p.g_cols <= e.n_valid);
                    fast_dst[k] = ok ? p.taps + 2 * (e.out + n0) : nullptr;
                }
            }
            mbar_wait(&tfull[acc], acc_phase);
            PROF_MARK(0);
            if (lane == 0 && warp == kEW0) TRACE(10, ti);
            tc_fence_after();

            float s_abs[2] = {0.f, 0.f}, s_sq[2] = {0.f, 0.f}, nf[2] = {0.f, 0.f};
            const uint32_t t_acc = tmem_base + (uint32_t)(acc * p.g_cols);
            if constexpr (SCORED) {
                // split: as the plain drain below (per-link partials flush at the half boundary)
                const int nh = split ? 2 : 1;
                for (int h = 0; h < nh; ++h) {
                    const int c0 = h ? p.nm : 0;
                    const int nc = split ? (h ? p.g_cols - p.nm : p.nm) : p.g_cols;
#pragma unroll
                    for (int k = 0; k < kBlocksPerWarp; ++k) {
                        const int bb = bb0 + k;
                        const uint32_t taddr = t_acc + ((uint32_t)(quarter * 32 + 16 * bb) << 16) + (uint32_t)c0;
                        const EpiLink e = make_link(p, link0 + 8 * bb);
                        const uint32_t ring =
                            smem_u32(smem) + p.truth_off + (uint32_t)((warp - kEW0) * p.truth_slots * 2048);
                        const bool c32 = p.truth != nullptr && (nc & 31) == 0;
                        if (p.truth_slots == 2 && c32)
                            epi_block_scored_smem<2>(p, taddr, e, n0 + c0, ring, s_abs[k], s_sq[k], nf[k], nc);
                        else if (p.truth_slots == 3 && c32)
                            epi_block_scored_smem<3>(p, taddr, e, n0 + c0, ring, s_abs[k], s_sq[k], nf[k], nc);
                        else if (p.truth_slots == 4 && c32)
                            epi_block_scored_smem<4>(p, taddr, e, n0 + c0, ring, s_abs[k], s_sq[k], nf[k], nc);
                        else if (c32)
                            epi_block_scored(p, taddr, e, n0 + c0, s_abs[k], s_sq[k], nf[k], nc);
                        else
                            epi_block<true>(p, taddr, e, n0 + c0, s_abs[k], s_sq[k], nf[k], nc);
                    }
                    if (split && h == 0) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster_relaxed(tempty_leader0 + 8u);
                    }
                }
            } else {
                // plain drain; split: columns [0, nm) of every block first, released to the MMA
                // warp (the next tile's first-half MMAs) before [nm, g_cols) is drained
                const int nh = split ? 2 : 1;
                for (int h = 0; h < nh; ++h) {
                    const int c0 = h ? p.nm : 0;
                    const int nc = split ? (h ? p.g_cols - p.nm : p.nm) : p.g_cols;
#pragma unroll
                    for (int k = 0; k < kBlocksPerWarp; ++k) {
                        const int bb = bb0 + k;
                        const uint32_t taddr = t_acc + ((uint32_t)(quarter * 32 + 16 * bb) << 16) + (uint32_t)c0;
                        // warp-uniform choice (tcgen05.ld is .sync.aligned): every lane's run covers the tile
                        if (fast_dst[k] != nullptr) {
                            epi_block_fast<GATHER>(p, taddr, fast_dst[k] + 2 * c0, nc);
                        } else {
                            const EpiLink e = make_link(p, link0 + 8 * bb);
                            epi_block<false, GATHER>(p, taddr, e, n0 + c0, s_abs[k], s_sq[k], nf[k], nc);
                        }
                    }
                    if (split && h == 0) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster_relaxed(tempty_leader0 + 8u);
                    }
                }
            }
            // this warp's share of the accumulator is drained -> tell the leader's MMA warp
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster_relaxed(tempty_leader0 + (uint32_t)(acc * 8));
            if (lane == 0 && warp == kEW0) TRACE(11, ti);
            if (lane == 0 && warp == kWarps - 1) TRACE(12, ti);
            if (++acc == p.acc_stages) { acc = 0; acc_phase ^= 1; }
            PROF_MARK(1);

            if (SCORED && p.stats != nullptr) {
#pragma unroll
                for (int k = 0; k < kBlocksPerWarp; ++k) {
                    const EpiLink e = make_link(p, link0 + 8 * (bb0 + k));
                    float bad = 0.f;
                    if (e.out >= 0 && nf[k] != 0.f) {
                        bad = recount_nonfinite(p, e, n0);
                        // saturated (frame-set, batch): zeroed, counted and rescored by k_sat_finish
                        if (bad != 0.f && p.sat_flags != nullptr)
                            atomicOr(p.sat_flags + (uint32_t)(link0 + 8 * (bb0 + k)) / (uint32_t)p.n_r, 1u);
                    }
                    float sa = s_abs[k], sq = s_sq[k];
                    // per-frame reduction: warp-uniform frame -> one atomic per warp.  Links
                    // ascend with the lane, so lane 0 holds the block's first (valid) link.
                    const bool lead_ok = __shfl_sync(0xffffffffu, e.out >= 0, 0);
                    const int64_t f0 = __shfl_sync(0xffffffffu, e.f, 0);
                    const bool uniform = __all_sync(0xffffffffu, e.f == f0 || e.out < 0);
                    if (uniform) {
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            sa += __shfl_xor_sync(0xffffffffu, sa, o);
                            sq += __shfl_xor_sync(0xffffffffu, sq, o);
                            bad += __shfl_xor_sync(0xffffffffu, bad, o);
                        }
                        if (lane == 0 && lead_ok) {
                            PNCE_CHECK(f0 >= 0 && f0 < p.n_frames);
                            if (p.truth != nullptr) {
                                atomicAdd(&p.stats[f0 * 4 + 0], (double)sa);
                                atomicAdd(&p.stats[f0 * 4 + 1], (double)sq);
                            }
                            if (bad != 0.f) atomicAdd(&p.stats[f0 * 4 + 2], (double)bad);
                        }
                    } else if (e.out >= 0) {
                        PNCE_CHECK(e.f >= 0 && e.f < p.n_frames);
                        if (p.truth != nullptr) {
                            atomicAdd(&p.stats[e.f * 4 + 0], (double)sa);
                            atomicAdd(&p.stats[e.f * 4 + 1], (double)sq);
                        }
                        if (bad != 0.f) atomicAdd(&p.stats[e.f * 4 + 2], (double)bad);
                    }
                }
            }
        }
        if (warp == kEW0 && lane == 0) PROF_END(10, 2);
    }

    __syncwarp();
    tc_fence_before();
    cluster_sync_all();
    if (threadIdx.x == 0) TRACE(15, 0);  // all roles done
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair(tmem_base, p.tmem_cols);
    }
}

// tensor16 finish (experiments.py:201-205): a (frame-set, batch) whose partial or total
// went non-finite is scored as all-zero taps and counted as n_r * n_tx saturations
// (stats[:, 3]); then the per-frame error sums against the truth (stats[:, 0..2]).
__global__ void k_t16_finish(float* __restrict__ taps, const float* __restrict__ truth, double* __restrict__ stats,
                             const uint32_t* __restrict__ flags, int n_r, int n_t, int n_batch, int n_batches, int l) {
    const int64_t fb = blockIdx.x;
    const int b = (int)(fb % n_batches);
    const int64_t f = fb / n_batches;
    const int n_tx = min(n_batch, n_t - b * n_batch);
    const bool sat = flags[fb] != 0;
    const int per_r = n_tx * l;
    float s_abs = 0.f, s_sq = 0.f, bad = 0.f;
    for (int idx = threadIdx.x; idx < n_r * per_r; idx += blockDim.x) {
        const int r = idx / per_r, q = idx - r * per_r;
        const int64_t pos = ((f * n_r + r) * n_t + (int64_t)b * n_batch) * l + q;
        float2* tp = reinterpret_cast<float2*>(taps) + pos;
        float2 v = *tp;
        if (sat) {
            v = make_float2(0.f, 0.f);
            *tp = v;
        }
        if (!(isfinite(v.x) && isfinite(v.y))) bad += 1.f;
        if (truth != nullptr) {
            const float2 h = reinterpret_cast<const float2*>(truth)[pos];
            const float dx = v.x - h.x, dy = v.y - h.y;
            s_sq += dx * dx + dy * dy;
            s_abs += sqrtf(dx * dx + dy * dy);
        }
    }
    if (stats == nullptr) return;
    for (int o = 16; o > 0; o >>= 1) {
        s_abs += __shfl_xor_sync(0xffffffffu, s_abs, o);
        s_sq += __shfl_xor_sync(0xffffffffu, s_sq, o);
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (truth != nullptr) {
            atomicAdd(&stats[f * 4 + 0], (double)s_abs);
            atomicAdd(&stats[f * 4 + 1], (double)s_sq);
        }
        if (bad != 0.f) atomicAdd(&stats[f * 4 + 2], (double)bad);
    }
    if (threadIdx.x == 0 && sat) atomicAdd(&stats[f * 4 + 3], (double)n_r * n_tx);
}


// Saturation finish of a scored launch (experiments.py:201-205 for the fp16/bf16 path): one
// warp per frame-set.  A frame-set none of whose batches was flagged just adds the launch's
// fused sums to the caller's stats; a flagged (frame-set, batch) -- one of its taps came out
// non-finite, e.g. an input beyond the fp16 range -- is scored as all-zero taps, counted as
// n_r * n_tx saturations (stats[:, 3]), and the frame-set's sums and the flagged links'
// per-link MSE are recomputed from the taps.
__global__ void k_sat_finish(float* __restrict__ taps, const float* __restrict__ truth, const double* __restrict__ part,
                             double* __restrict__ stats, float* __restrict__ link_err,
                             const uint32_t* __restrict__ flags, int64_t n_frames, int n_r, int n_t, int n_batch,
                             int n_batches, int l) {
    const int lane = threadIdx.x & 31;
    const int64_t f = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (f >= n_frames) return;
    const uint32_t* fl = flags + f * n_batches;
    bool any = false;
    for (int b = lane; b < n_batches; b += 32) any |= fl[b] != 0;
    any = __any_sync(0xffffffffu, any);
    if (!any) {
        if (lane < 4) stats[f * 4 + lane] += part[f * 4 + lane];
        return;
    }
    const int64_t per_f = (int64_t)n_r * n_t * l;
    float2* tp = reinterpret_cast<float2*>(taps) + f * per_f;
    const float2* hp = truth ? reinterpret_cast<const float2*>(truth) + f * per_f : nullptr;
    double s_abs = 0.0, s_sq = 0.0, bad = 0.0;
    for (int64_t i = lane; i < per_f; i += 32) {
        const int t = (int)((i / l) % n_t);
        float2 v = tp[i];
        if (fl[t / n_batch]) {
            v = make_float2(0.f, 0.f);
            tp[i] = v;
        }
        if (!(isfinite(v.x) && isfinite(v.y))) bad += 1.0;
        if (hp) {
            const double dx = (double)v.x - hp[i].x, dy = (double)v.y - hp[i].y;
            s_sq += dx * dx + dy * dy;
            s_abs += sqrt(dx * dx + dy * dy);
        }
    }
    if (link_err && hp) {
        for (int64_t q = lane; q < (int64_t)n_r * n_t; q += 32) {
            const int t = (int)(q % n_t);
            if (!fl[t / n_batch]) continue;
            float acc = 0.f;
            for (int k = 0; k < l; ++k) {
                const float2 h = hp[q * l + k];
                acc += h.x * h.x + h.y * h.y;
            }
            link_err[f * (int64_t)n_r * n_t + q] = acc / (float)l;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        s_abs += __shfl_xor_sync(0xffffffffu, s_abs, o);
        s_sq += __shfl_xor_sync(0xffffffffu, s_sq, o);
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if (lane == 0) {
        double sat = 0.0;
        for (int b = 0; b < n_batches; ++b)
            if (fl[b]) sat += (double)n_r * min(n_batch, n_t - b * n_batch);
        if (hp) {
            stats[f * 4 + 0] += s_abs;
            stats[f * 4 + 1] += s_sq;
        }
        stats[f * 4 + 2] += bad;
        stats[f * 4 + 3] += sat;
    }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

// 2-D row-major [rows][cols] 16-bit tensor, box [box_rows][64], 128B swizzle.
pnce_status_t make_tmap(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                        uint32_t box_rows, int bf16) {
    auto enc = get_encode();
    if (!enc) return fail(PNCE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)kBK, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                     2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PNCE_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return PNCE_OK;
}

// Received f32 rows as a 2-D tensor [links][2*samples] floats, box [64 links][box_floats]
// (half a K-block = 32 (I,Q) samples for 64 links, + 16 B slack when C is odd so the box
// start can be rounded down to a 16-byte boundary), no swizzle.
pnce_status_t make_tmap_raw(CUtensorMap* map, const float* base, uint64_t row_floats, uint64_t rows,
                            uint32_t box_floats, uint32_t box_rows = kLinksPerTile) {
    auto enc = get_encode();
    if (!enc) return fail(PNCE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {row_floats, rows};
    cuuint64_t strides[1] = {row_floats * 4};
    cuuint32_t box[2] = {(cuuint32_t)box_floats, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PNCE_ERR_CUDA, "cuTensorMapEncodeTiled(raw) failed: " + std::to_string((int)r));
    return PNCE_OK;
}

// A-stage scratch (a_reuse) as a 2-D tensor [rows][128 B] of 16-bit words, box [128 rows][64],
// no swizzle: the stored bytes are already the 128B-swizzled shared-memory image of a stage.
pnce_status_t make_tmap_scr(CUtensorMap* map, const void* base, uint64_t rows) {
    auto enc = get_encode();
    if (!enc) return fail(PNCE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)kBK, rows};
    cuuint64_t strides[1] = {(cuuint64_t)kBK * 2};
    cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)kBM};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PNCE_ERR_CUDA, "cuTensorMapEncodeTiled(scratch) failed: " + std::to_string((int)r));
    return PNCE_OK;
}

}  // namespace

// Lag-row tiling of one K3 variant.
struct Tiling {
    int n_groups;    // lag-row groups per 256-row tile
    int g_cols;      // accumulator columns per group
    int n_mma;       // pair MMAs per k-step (N = nm each)
    int nm;
    int acc_stages;  // TMEM accumulator buffers
    int stages;      // smem pipeline depth
    uint32_t stage_bytes;
    uint32_t tmem_cols;
    CUtensorMap tm_circ;  // circulant rows, box = nm/2 rows x 64 K
};

// Per-(plan, stream) launch resources, created on first use and reused by every later launch
// on that stream (stream order serialises their users; launches on different streams get
// different entries, so the library stays reentrant): the A-stage scratch of a_reuse, the
// saturation flags and per-launch stats of the scored / tensor16 finish, and the last-built
// tensor maps of the caller's input (rebuilt only when the pointer or extent changes).
struct StreamRes {
    cudaStream_t stream = nullptr;
    uint64_t last_use = 0;
    uint8_t* scratch = nullptr;
    size_t scratch_bytes = 0;
    CUtensorMap tm_scr;
    uint64_t tm_scr_rows = 0;
    uint32_t* flags = nullptr;  // [F][n_batches] saturation flags
    size_t flags_n = 0;
    double* stats = nullptr;    // [F][4] this launch's sums before the saturation finish
    size_t stats_n = 0;
    CUtensorMap tm_in;          // raw f32 rows or the packed operand
    const void* tm_in_ptr = nullptr;
    uint64_t tm_in_key[3] = {0, 0, 0};
};

struct pnce_plan {
    pnce_cfg_t cfg;
    int device = 0;  // the device the plan's operand lives on; launches must run there
    std::mutex res_mu;
    std::vector<StreamRes*> res;
    uint64_t res_clock = 0;
    int n_batches;
    int r_total;     // N_b * L
    int k_pad;       // roundup(M, 64)
    int rows_alloc;  // circulant rows (>= every tiling's coverage)
    int num_sms;
    Tiling fused;    // f32 IQ in: prefer one group (<= 512 cols) so samples are converted once
    Tiling packed;   // packed operand via TMA: same grouping (TMA ingress, not the drain, bounds G=256)
    Tiling packed_ldg;  // <= 256 columns, double-buffered accumulator (packed LDG mode, scored launches)
    Tiling t16;      // tensor16 emulation: <= 256 columns (multiple of 32), partial + running total
    Tiling narrow;   // plain launches with few tiles: <= 128 columns, groups spread over clusters
    Tiling mid;      // plain launches with a few more tiles: <= 256 columns
    float* chips;    // device [m]
    void* circ;      // device [rows_alloc][k_pad] 16-bit
    void* synth = nullptr;  // synthesiser state (pnce_synth.cu)
    float inv_norm = 0.f;   // 1 / norm_len (correlate_rows' norm_len; M for PN plans)
};

namespace pnce_internal {
PlanView plan_view(const pnce_plan_t* p) {
    return PlanView{p->cfg, p->n_batches, p->chips, const_cast<void**>(&p->synth)};
}
pnce_status_t set_error(pnce_status_t code, const std::string& msg) { return fail(code, msg); }
void count_launch() { g_launches++; }
pnce_status_t encode_tmap_k16(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows,
                              int bf16) {
    return make_tmap(map, base, cols, rows, box_rows, bf16);
}
}  // namespace pnce_internal

static pnce_status_t device_setup(int dev);

// The plan's resource entry for `st` (created on first use; at most kMaxStreamRes entries, the
// least recently used one is released -- cudaFree waits for the device, so its last launch
// has finished).
constexpr int kMaxStreamRes = 16;
static StreamRes* stream_res(pnce_plan* p, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(p->res_mu);
    for (StreamRes* r : p->res)
        if (r->stream == st) {
            r->last_use = ++p->res_clock;
            return r;
        }
    if ((int)p->res.size() >= kMaxStreamRes) {
        auto it = std::min_element(p->res.begin(), p->res.end(),
                                   [](const StreamRes* a, const StreamRes* b) { return a->last_use < b->last_use; });
        StreamRes* old = *it;
        if (old->scratch) cudaFree(old->scratch);
        if (old->flags) cudaFree(old->flags);
        if (old->stats) cudaFree(old->stats);
        delete old;
        p->res.erase(it);
    }
    StreamRes* r = new StreamRes();
    r->stream = st;
    r->last_use = ++p->res_clock;
    p->res.push_back(r);
    return r;
}

// Grow-only device buffer of a StreamRes; a reallocation first waits for the stream (the old
// buffer may still be read by an earlier launch on it).  Rare: the first launch and growth.
template <typename T>
static pnce_status_t ensure_buf(T*& buf, size_t& have, size_t need, cudaStream_t st, const char* what) {
    if (need <= have && buf) return PNCE_OK;
    if (buf) {
        cudaStreamSynchronize(st);
        cudaFree(buf);
        buf = nullptr;
        have = 0;
    }
    cudaError_t e = cudaMalloc(&buf, need * sizeof(T));
    if (e != cudaSuccess) return fail(PNCE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    have = need;
    return PNCE_OK;
}

// Launch preconditions shared by the compute entry points: the plan's device is current.
static pnce_status_t check_device(const pnce_plan* p) {
    int dev = -1;
    CUDA_TRY(cudaGetDevice(&dev));
    if (dev != p->device)
        return fail(PNCE_ERR_DIMENSION, "plan lives on device " + std::to_string(p->device) +
                                            " but the current device is " + std::to_string(dev));
    return PNCE_OK;
}

static void make_tiling(Tiling& t, int r_total, int max_group, int align = 16) {
    const int r16 = (r_total + align - 1) / align * align;
    t.n_groups = (r16 + max_group - 1) / max_group;
    int g = ((r16 + t.n_groups - 1) / t.n_groups + align - 1) / align * align;
    if (g > 256) {
        g = (g + 31) / 32 * 32;
        t.n_mma = 2;
    } else {
        t.n_mma = 1;
    }
    t.g_cols = g;
    t.nm = g / t.n_mma;
    t.acc_stages = (2 * g <= 512) ? 2 : 1;
    t.stage_bytes = (uint32_t)(kBM * kBK * 2 + (g / 2) * kBK * 2);
    int stages = (int)((kSmemLimit - 2048) / t.stage_bytes);
    t.stages = stages > 8 ? 8 : stages;
    uint32_t cols = 32;
    while (cols < (uint32_t)(t.acc_stages * g)) cols <<= 1;
    t.tmem_cols = cols;
}

template <int MODE>
static cudaError_t set_smem_attrs() {
    cudaError_t e = cudaFuncSetAttribute(k_correlate<MODE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_correlate<MODE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
    if (e == cudaSuccess && (MODE == kModeFusedTma || MODE == kModePacked))
        e = cudaFuncSetAttribute(k_correlate<MODE, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemLimit);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_correlate<MODE, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemLimit);
    if (e == cudaSuccess && MODE == kModeFusedTma)
        e = cudaFuncSetAttribute(k_correlate<kModeFusedTma, false, false, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
    if (e == cudaSuccess && MODE == kModeFusedTma)
        e = cudaFuncSetAttribute(k_correlate<kModeFusedTma, false, true, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
    if constexpr (MODE == kModeFusedTma || MODE == kModeFusedLdg)
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_correlate<MODE, false, false, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
    return e;
}

// Scored variants (truth / stats / per-link errors) are separate instantiations so the
// plain drain keeps its registers.
template <int MODE>
static void launch_k3(bool scored, int grid, size_t smem, cudaStream_t st, const CUtensorMap& a,
                      const CUtensorMap& b, const CorrParams& prm, const CUtensorMap* scr = nullptr) {
    const CUtensorMap& c = scr ? *scr : b;  // scratch map (a_reuse) or an unused placeholder
    // 8 epilogue warps: +1 % for the packed operand (its converter warps are idle anyway),
    // -5 % for the fused path (converters become the bottleneck); PNCE_TUNE_EPI8 overrides
    const int epi8_env = knobs().epi8;
    const bool epi8 = epi8_env < 0 ? MODE == kModePacked : epi8_env == 1;
    if constexpr (MODE == kModeFusedTma || MODE == kModeFusedLdg) {
        if (prm.gather_n > 0) {  // antenna-split gather (plain launches only)
            k_correlate<MODE, false, false, false, true><<<grid, kThreadsK3, smem, st>>>(a, b, c, prm);
            return;
        }
    }
    if (scored && knobs().scored_epi == 4)
        k_correlate<MODE, true, false><<<grid, kThreadsK3, smem, st>>>(a, b, c, prm);
    else if (scored)
        k_correlate<MODE, true, true><<<grid, kThreadsK3, smem, st>>>(a, b, c, prm);
    else if ((MODE == kModeFusedTma || MODE == kModePacked) && epi8)
        k_correlate<MODE, false, true><<<grid, kThreadsK3, smem, st>>>(a, b, c, prm);
    else
        k_correlate<MODE, false><<<grid, kThreadsK3, smem, st>>>(a, b, c, prm);
}

// Tilings, operand rows and tensor maps of a plan: the PN lag-window rows built from the
// plan's chips (rows == nullptr) or caller-supplied rows [r_total][m] f32 (device).
static pnce_status_t plan_build(pnce_plan* p, const float* rows, cudaStream_t st) {
    const pnce_cfg_t& cfg = p->cfg;
    p->k_pad = (cfg.m + kBK - 1) / kBK * kBK;
    // Tuning knobs (diagnostics): maximum accumulator columns per lag-row group.
    const Knobs& kn = knobs();
    make_tiling(p->fused, p->r_total, kn.group_fused);
    make_tiling(p->packed, p->r_total, kn.group_packed);
    make_tiling(p->packed_ldg, p->r_total, kn.group_packed_ldg);
    // tensor16: partial(s) + running total in TMEM.  Default: one partial of <= 256 columns
    // (the MMA waits for every fold).  PNCE_TUNE_T16_G=160: two partial buffers of <= 160
    // columns (3 x G <= 512), the MMA filling one while the epilogue folds the other --
    // measured slower at cfg3 (4.05 vs 3.76 us/frame-set: twice the groups at N=128).
    make_tiling(p->t16, p->r_total, kn.t16_g >= 256 ? 256 : 160, 32);  // 32-column fold chunks
    make_tiling(p->narrow, p->r_total, kn.narrow_g);
    make_tiling(p->mid, p->r_total, 256);
    p->t16.acc_stages = 3 * p->t16.g_cols <= 512 ? 2 : 1;
    p->t16.tmem_cols = 512;
    p->rows_alloc = std::max({p->fused.n_groups * p->fused.g_cols, p->packed.n_groups * p->packed.g_cols,
                              p->packed_ldg.n_groups * p->packed_ldg.g_cols, p->t16.n_groups * p->t16.g_cols,
                              p->narrow.n_groups * p->narrow.g_cols, p->mid.n_groups * p->mid.g_cols});
    cudaError_t e = cudaMalloc(&p->circ, (size_t)p->rows_alloc * p->k_pad * 2);
    if (e != cudaSuccess) return fail(PNCE_ERR_CUDA, std::string("plan alloc: ") + cudaGetErrorString(e));
    const int64_t total = (int64_t)p->rows_alloc * p->k_pad;
    const int blocks = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    const bool bf16 = cfg.dtype == PNCE_DTYPE_BF16;
    if (rows) {
        if (bf16)
            k_rows_to_operand<__nv_bfloat16><<<blocks, 256, 0, st>>>(rows, (__nv_bfloat16*)p->circ, cfg.m, p->k_pad,
                                                                      p->r_total, p->rows_alloc);
        else
            k_rows_to_operand<__half><<<blocks, 256, 0, st>>>(rows, (__half*)p->circ, cfg.m, p->k_pad, p->r_total,
                                                               p->rows_alloc);
    } else {
        const int spacing = cfg.m / cfg.n_batch;
        if (bf16)
            k_build_circulant<__nv_bfloat16><<<blocks, 256, 0, st>>>(
                p->chips, (__nv_bfloat16*)p->circ, cfg.m, p->k_pad, p->r_total, p->rows_alloc, cfg.l, spacing);
        else
            k_build_circulant<__half><<<blocks, 256, 0, st>>>(p->chips, (__half*)p->circ, cfg.m, p->k_pad,
                                                               p->r_total, p->rows_alloc, cfg.l, spacing);
    }
    g_launches++;
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(PNCE_ERR_CUDA, std::string("operand rows: ") + cudaGetErrorString(e));
    const uint64_t circ_rows = (uint64_t)p->rows_alloc;
    pnce_status_t s = make_tmap(&p->fused.tm_circ, p->circ, p->k_pad, circ_rows, p->fused.nm / 2, bf16);
    if (s == PNCE_OK) s = make_tmap(&p->packed.tm_circ, p->circ, p->k_pad, circ_rows, p->packed.nm / 2, bf16);
    if (s == PNCE_OK) s = make_tmap(&p->t16.tm_circ, p->circ, p->k_pad, circ_rows, p->t16.nm / 2, bf16);
    if (s == PNCE_OK) s = make_tmap(&p->narrow.tm_circ, p->circ, p->k_pad, circ_rows, p->narrow.nm / 2, bf16);
    if (s == PNCE_OK) s = make_tmap(&p->mid.tm_circ, p->circ, p->k_pad, circ_rows, p->mid.nm / 2, bf16);
    if (s == PNCE_OK)
        s = make_tmap(&p->packed_ldg.tm_circ, p->circ, p->k_pad, circ_rows, p->packed_ldg.nm / 2, bf16);
    if (s != PNCE_OK) return s;
    return device_setup(p->device);
}

// Once per DEVICE (function attributes are per device): the 227 KB dynamic shared-memory
// opt-in of every k_correlate instantiation.  Called with `dev` current.
static pnce_status_t device_setup(int dev) {
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> lock(mu);
    if (std::find(done.begin(), done.end(), dev) != done.end()) return PNCE_OK;
    cudaError_t e = set_smem_attrs<kModePacked>();
    if (e == cudaSuccess) e = set_smem_attrs<kModeFusedLdg>();
    if (e == cudaSuccess) e = set_smem_attrs<kModeFusedTma>();
    if (e == cudaSuccess) e = set_smem_attrs<kModePackedLdg>();
    if (e != cudaSuccess)
        return fail(PNCE_ERR_CUDA, "cudaFuncSetAttribute on device " + std::to_string(dev) + ": " + cudaGetErrorString(e));
    done.push_back(dev);
    return PNCE_OK;
}

extern "C" {

int32_t pnce_version(void) { return 100; }

const char* pnce_last_error(void) { return g_err.c_str(); }

int64_t pnce_kernel_launches(void) { return g_launches.load(); }

pnce_status_t pnce_config_check(const pnce_cfg_t* cfg) {
    if (!cfg) return fail(PNCE_ERR_INVALID_CONFIG, "null config");
    if (cfg->degree < 2 || cfg->degree > 16)
        return fail(PNCE_ERR_INVALID_SPEC, "degree must be in [2, 16]");
    const uint32_t full = (1u << cfg->degree) - 1u;
    if (cfg->state == 0) return fail(PNCE_ERR_ZERO_STATE, "initial LFSR state must be nonzero");
    if (cfg->state > full) return fail(PNCE_ERR_INVALID_SPEC, "state wider than degree bits");
    if (!(cfg->tap_mask & (1u << (cfg->degree - 1))))
        return fail(PNCE_ERR_INVALID_SPEC, "tap set must include the degree");
    if (cfg->tap_mask & ~full) return fail(PNCE_ERR_INVALID_SPEC, "tap outside [1, degree]");
    if ((int64_t)cfg->m != (int64_t)full)
        return fail(PNCE_ERR_INVALID_CONFIG, "m must equal 2^degree - 1");
    if (cfg->n_t < 1 || cfg->n_r < 1) return fail(PNCE_ERR_INVALID_CONFIG, "n_t, n_r must be >= 1");
    if (!(1 <= cfg->l && cfg->l <= cfg->c && cfg->c <= cfg->m))
        return fail(PNCE_ERR_INVALID_CONFIG, "need 1 <= L <= C <= M");
    if (!(1 <= cfg->n_batch && cfg->n_batch <= cfg->m / cfg->c))
        return fail(PNCE_ERR_INVALID_CONFIG, "n_batch outside [1, floor(M/C)]");
    if (cfg->dtype != PNCE_DTYPE_FP16 && cfg->dtype != PNCE_DTYPE_BF16)
        return fail(PNCE_ERR_INVALID_CONFIG, "dtype must be fp16 or bf16");
    // build_batch_plan separation check (pilots.py:134-142)
    const int spacing = cfg->m / cfg->n_batch;
    for (int i = 0; i < cfg->n_batch; ++i)
        for (int j = i + 1; j < cfg->n_batch; ++j) {
            int d = (spacing * (j - i)) % cfg->m;
            d = d < cfg->m - d ? d : cfg->m - d;
            if (d < cfg->l) return fail(PNCE_ERR_INVALID_CONFIG, "shift separation < L");
        }
    return PNCE_OK;
}

pnce_status_t pnce_generate_mseq(int32_t degree, uint32_t tap_mask, uint32_t state, float* chips_dev,
                                 int32_t m, void* stream) {
    if (degree < 2 || degree > 16) return fail(PNCE_ERR_INVALID_SPEC, "degree must be in [2, 16]");
    if (state == 0) return fail(PNCE_ERR_ZERO_STATE, "initial LFSR state must be nonzero");
    if (state >= (1u << degree)) return fail(PNCE_ERR_INVALID_SPEC, "state wider than degree bits");
    if (m != (int32_t)((1u << degree) - 1u)) return fail(PNCE_ERR_DIMENSION, "m must be 2^degree - 1");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int* d_period = nullptr;
    CUDA_TRY(cudaMallocAsync(&d_period, sizeof(int), st));
    k_lfsr<<<1, 1, 0, st>>>(degree, tap_mask, state, chips_dev, m, d_period);
    g_launches++;
    int period = 0;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(&period, d_period, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFreeAsync(d_period, st);
    if (e != cudaSuccess) return fail(PNCE_ERR_CUDA, std::string("k_lfsr: ") + cudaGetErrorString(e));
    if (period != m)
        return fail(PNCE_ERR_NOT_MAXIMAL, "LFSR period " + std::to_string(period) + " != " +
                                              std::to_string(m) + "; feedback polynomial is not primitive");
    return PNCE_OK;
}

pnce_status_t pnce_plan_create(const pnce_cfg_t* cfg, pnce_plan_t** out, void* stream) {
    if (!out) return fail(PNCE_ERR_INVALID_CONFIG, "null plan out-pointer");
    *out = nullptr;
    pnce_status_t s = pnce_config_check(cfg);
    if (s != PNCE_OK) return s;
    int dev = 0, major = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major != 10) return fail(PNCE_ERR_UNSUPPORTED_DEVICE, "pnce_b200 needs an sm_100 (B200) device");
    int sms = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));

    pnce_plan* p = new pnce_plan();
    p->cfg = *cfg;
    p->device = dev;
    p->n_batches = (cfg->n_t + cfg->n_batch - 1) / cfg->n_batch;
    p->r_total = cfg->n_batch * cfg->l;
    p->num_sms = sms;
    p->inv_norm = 1.0f / (float)cfg->m;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMalloc(&p->chips, sizeof(float) * cfg->m);
    if (e != cudaSuccess) {
        pnce_plan_destroy(p);
        return fail(PNCE_ERR_CUDA, std::string("plan alloc: ") + cudaGetErrorString(e));
    }
    s = pnce_generate_mseq(cfg->degree, cfg->tap_mask, cfg->state, p->chips, cfg->m, stream);
    if (s == PNCE_OK) s = plan_build(p, nullptr, st);
    if (s != PNCE_OK) {
        pnce_plan_destroy(p);
        return s;
    }
    *out = p;
    return PNCE_OK;
}

pnce_status_t pnce_plan_create_rows(const pnce_cfg_t* cfg, const float* rows, int32_t n_rows, int32_t norm_len,
                                    pnce_plan_t** out, void* stream) {
    if (!out) return fail(PNCE_ERR_INVALID_CONFIG, "null plan out-pointer");
    *out = nullptr;
    if (!cfg || !rows) return fail(PNCE_ERR_INVALID_CONFIG, "null config or rows");
    if (cfg->m < 1 || cfg->n_r < 1) return fail(PNCE_ERR_DIMENSION, "m and n_r must be >= 1");
    if (n_rows < 1 || n_rows > cfg->m) return fail(PNCE_ERR_ROWS_OUT_OF_RANGE, "row count outside [1, M]");
    if (norm_len < 1) return fail(PNCE_ERR_INVALID_CONFIG, "norm_len must be >= 1");
    if (cfg->dtype != PNCE_DTYPE_FP16 && cfg->dtype != PNCE_DTYPE_BF16)
        return fail(PNCE_ERR_INVALID_CONFIG, "dtype must be fp16 or bf16");
    int dev = 0, major = 0, sms = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major != 10) return fail(PNCE_ERR_UNSUPPORTED_DEVICE, "pnce_b200 needs an sm_100 (B200) device");
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // one "batch" of one "transmitter" whose window is the whole row set: taps[f][r][0][q] = row q
    pnce_plan* p = new pnce_plan();
    p->cfg = *cfg;
    p->device = dev;
    p->cfg.c = 0;
    p->cfg.l = n_rows;
    p->cfg.n_t = 1;
    p->cfg.n_batch = 1;
    p->n_batches = 1;
    p->r_total = n_rows;
    p->num_sms = sms;
    p->inv_norm = 1.0f / (float)norm_len;
    pnce_status_t s = plan_build(p, rows, static_cast<cudaStream_t>(stream));
    if (s != PNCE_OK) {
        pnce_plan_destroy(p);
        return s;
    }
    *out = p;
    return PNCE_OK;
}

pnce_status_t pnce_plan_destroy(pnce_plan_t* p) {
    if (!p) return PNCE_OK;
    if (p->chips) cudaFree(p->chips);
    if (p->circ) cudaFree(p->circ);
    if (p->synth) pnce_internal::synth_cache_free(p->synth);
    for (StreamRes* r : p->res) {
        if (r->scratch) cudaFree(r->scratch);
        if (r->flags) cudaFree(r->flags);
        if (r->stats) cudaFree(r->stats);
        delete r;
    }
    delete p;
    return PNCE_OK;
}

pnce_status_t pnce_plan_chips(const pnce_plan_t* p, float* dst, void* stream) {
    if (!p || !dst) return fail(PNCE_ERR_INVALID_CONFIG, "null plan or destination");
    if (!p->chips) return fail(PNCE_ERR_INVALID_CONFIG, "plan was built from caller rows (no PN chips)");
    CUDA_TRY(cudaMemcpyAsync(dst, p->chips, sizeof(float) * p->cfg.m, cudaMemcpyDeviceToDevice,
                             static_cast<cudaStream_t>(stream)));
    return PNCE_OK;
}

pnce_status_t pnce_plan_operand(const pnce_plan_t* p, void* dst, int32_t* n_rows, int32_t* k_pad, void* stream) {
    if (!p) return fail(PNCE_ERR_INVALID_CONFIG, "null plan");
    if (n_rows) *n_rows = p->rows_alloc;
    if (k_pad) *k_pad = p->k_pad;
    if (!dst) return PNCE_OK;
    CUDA_TRY(cudaMemcpyAsync(dst, p->circ, (size_t)p->rows_alloc * p->k_pad * 2, cudaMemcpyDeviceToDevice,
                             static_cast<cudaStream_t>(stream)));
    return PNCE_OK;
}

size_t pnce_workspace_bytes(const pnce_plan_t* p, int64_t n_frames) {
    if (!p || n_frames < 0) return 0;
    const int64_t links = n_frames * p->n_batches * (int64_t)p->cfg.n_r;
    const int64_t rows = (links + 7) / 8 * 16;  // a_row order: whole 8-link blocks
    return (size_t)rows * p->k_pad * 2;
}

pnce_status_t pnce_pack_iq(const pnce_plan_t* p, const float* iq, void* packed, int64_t n_frames,
                           void* stream) {
    if (!p) return fail(PNCE_ERR_INVALID_CONFIG, "null plan");
    if (n_frames < 0) return fail(PNCE_ERR_DIMENSION, "n_frames < 0");
    if (n_frames == 0) return PNCE_OK;
    if (!iq || !packed) return fail(PNCE_ERR_DIMENSION, "null buffer");
    if (reinterpret_cast<uintptr_t>(packed) & 15) return fail(PNCE_ERR_DIMENSION, "packed buffer must be 16-byte aligned");
    if (reinterpret_cast<uintptr_t>(iq) & 7) return fail(PNCE_ERR_DIMENSION, "iq buffer must be 8-byte aligned");
    s_ok_or_return(check_device(p));
    const pnce_cfg_t& c = p->cfg;
    const int samples = c.c + c.m + c.l - 1;
    const int64_t links = n_frames * p->n_batches * (int64_t)c.n_r;
    const int64_t work = (links + 7) / 8 * 8 * (p->k_pad / 8);
    const int64_t want = (work + 255) / 256;
    const int blocks = (int)(want < (int64_t)p->num_sms * 16 ? want : (int64_t)p->num_sms * 16);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (c.dtype == PNCE_DTYPE_BF16)
        k_pack_iq<__nv_bfloat16><<<blocks, 256, 0, st>>>(iq, (__nv_bfloat16*)packed, links, samples, c.c, c.m, p->k_pad);
    else
        k_pack_iq<__half><<<blocks, 256, 0, st>>>(iq, (__half*)packed, links, samples, c.c, c.m, p->k_pad);
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    return PNCE_OK;
}

// Diagnostic builds only: dump the cycle accounting / trace buffers after a launch.
static void diag_dump(cudaStream_t st) {
    (void)st;
#ifdef PNCE_DIAG_PROF
    if (const char* pf = std::getenv("PNCE_PROF_FILE")) {
        static std::vector<unsigned long long> host(1024 * kProfSlots);
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(host.data(), g_prof, host.size() * sizeof(unsigned long long));
        if (FILE* fh = std::fopen(pf, "wb")) {
            std::fwrite(host.data(), sizeof(unsigned long long), host.size(), fh);
            std::fclose(fh);
        }
    }
#endif
#ifdef PNCE_DIAG_TRACE
    if (const char* tf = std::getenv("PNCE_TRACE_FILE")) {
        static std::vector<long long> host(2 * kTraceSlots * kTraceMax);
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(host.data(), g_trace, host.size() * sizeof(long long));
        if (FILE* fh = std::fopen(tf, "wb")) {
            std::fwrite(host.data(), sizeof(long long), host.size(), fh);
            std::fclose(fh);
        }
    }
#endif
}


// Shared launch setup for both K3 variants.
static pnce_status_t fill_params(const pnce_plan_t* p, const Tiling& t, bool fused, float* taps, const float* truth,
                                 double* stats, int64_t n_frames, CorrParams& prm) {
    if ((reinterpret_cast<uintptr_t>(taps) & 7) || (truth && (reinterpret_cast<uintptr_t>(truth) & 7)))
        return fail(PNCE_ERR_DIMENSION, "taps/truth must be 8-byte aligned");
    const pnce_cfg_t& c = p->cfg;
    prm = CorrParams{};
    prm.total_links = n_frames * p->n_batches * (int64_t)c.n_r;
    const int64_t m_tiles = (prm.total_links + kBM - 1) / kBM;
    if (m_tiles * t.n_groups > INT32_MAX || 2 * prm.total_links > INT32_MAX)
        return fail(PNCE_ERR_DIMENSION, "too many frames for one call");
    prm.m_tiles = (int32_t)m_tiles;
    const Knobs& kn = knobs();
    prm.store_hint = kn.store_hint;  // evict_first taps: +1.5 % (keeps L2 for the circulant)
    prm.n_groups = t.n_groups;
    prm.bar_bytes = 1024;
    prm.raw_pol = kn.raw_pol >= 0 ? kn.raw_pol : (t.n_groups > 1 ? 1 : 0);
    prm.split_drain = kn.split_drain;
    prm.g_cols = t.g_cols;
    prm.n_mma = t.n_mma;
    prm.nm = t.nm;
    prm.acc_stages = t.acc_stages;
    prm.k_blocks = p->k_pad / kBK;
    prm.stages = t.stages;
    prm.stage_bytes = t.stage_bytes;
    const uint32_t b_half = (uint32_t)(t.g_cols / 2) * kBK * 2;
    prm.tx_bytes = 2 * (b_half + (fused ? 0u : (uint32_t)(kBM * kBK * 2)));
    prm.idesc = make_idesc_f16(2 * kBM, t.nm, c.dtype == PNCE_DTYPE_BF16);
    prm.tmem_cols = t.tmem_cols;
    prm.n_r = c.n_r;
    prm.n_t = c.n_t;
    prm.n_batches = p->n_batches;
    prm.n_batch = c.n_batch;
    prm.l = c.l;
    prm.m = c.m;
    prm.c = c.c;
    prm.samples = c.c + c.m + c.l - 1;
    prm.bf16 = c.dtype == PNCE_DTYPE_BF16;
    prm.inv_m = p->inv_norm;
    prm.inv_l = 1.0f / (float)c.l;
    prm.k_pad = p->k_pad;
    prm.chunk_kb = prm.k_blocks;
    prm.taps = taps;
    prm.truth = truth;
    prm.stats = stats;
    prm.n_frames = n_frames;
    prm.n_taps = n_frames * (int64_t)c.n_r * c.n_t * c.l;
    prm.out_nr = c.n_r;
    prm.out_r0 = 0;
    prm.gather_n = 0;
    return PNCE_OK;
}

static int pair_grid(const pnce_plan_t* p, const CorrParams& prm) {
    const int64_t tiles = (int64_t)prm.m_tiles * prm.n_groups;
    const int64_t pairs = std::min<int64_t>(tiles, p->num_sms / 2);
    return (int)(2 * std::max<int64_t>(pairs, 1));
}


// Scored launches with stats: the kernel accumulates into a per-launch stats buffer and
// raises per-(frame-set, batch) saturation flags; scored_finish then folds them into the
// caller's stats (k_sat_finish).
static pnce_status_t scored_prepare(const pnce_plan_t* p, StreamRes* res, int64_t n_frames, cudaStream_t st,
                                    CorrParams& prm) {
    const size_t n_fb = (size_t)n_frames * p->n_batches;
    s_ok_or_return(ensure_buf(res->flags, res->flags_n, n_fb, st, "saturation flags"));
    s_ok_or_return(ensure_buf(res->stats, res->stats_n, (size_t)n_frames * 4, st, "launch stats"));
    CUDA_TRY(cudaMemsetAsync(res->flags, 0, n_fb * sizeof(uint32_t), st));
    CUDA_TRY(cudaMemsetAsync(res->stats, 0, (size_t)n_frames * 4 * sizeof(double), st));
    prm.sat_flags = res->flags;
    prm.stats = res->stats;
    return PNCE_OK;
}

static pnce_status_t scored_finish(const pnce_plan_t* p, StreamRes* res, float* taps, const float* truth,
                                   double* stats, float* link_err, int64_t n_frames, cudaStream_t st) {
    const pnce_cfg_t& c = p->cfg;
    const unsigned blocks = (unsigned)((n_frames + 7) / 8);
    k_sat_finish<<<blocks, 256, 0, st>>>(taps, truth, res->stats, stats, link_err, res->flags, n_frames, c.n_r,
                                         c.n_t, c.n_batch, p->n_batches, c.l);
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    return PNCE_OK;
}

pnce_status_t pnce_correlate(const pnce_plan_t* p, const void* packed, float* taps, const float* truth,
                             double* stats, int64_t n_frames, void* stream) {
    if (!p) return fail(PNCE_ERR_INVALID_CONFIG, "null plan");
    if (n_frames < 0) return fail(PNCE_ERR_DIMENSION, "n_frames < 0");
    if (n_frames == 0) return PNCE_OK;
    if (!packed || !taps) return fail(PNCE_ERR_DIMENSION, "null buffer");
    if (reinterpret_cast<uintptr_t>(packed) & 15) return fail(PNCE_ERR_DIMENSION, "packed buffer must be 16-byte aligned");
    // packed operand: A with the circulant through TMA, one 512-column group (default), or
    // LDG-fed A + double-buffered 256-column accumulators (PNCE_TUNE_PACKED_MODE=3; parity-
    // green but 1.3x slower: one N=256 MMA per K-step cannot share A reads and the extra
    // A stores push shared-memory bandwidth past the tensor rate)
    s_ok_or_return(check_device(p));
    const bool ldg = knobs().packed_mode == kModePackedLdg;
    const Tiling& t = ldg ? p->packed_ldg : p->packed;
    CorrParams prm;
    pnce_status_t s = fill_params(p, t, false, taps, truth, stats, n_frames, prm);
    if (s != PNCE_OK) return s;
    // packed rows: 2 per link, padded to whole 8-link blocks (a_row order)
    const uint64_t packed_rows = (uint64_t)((prm.total_links + 7) / 8) * 16;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamRes* res = stream_res(const_cast<pnce_plan*>(p), st);
    const bool scored = truth || stats;
    if (stats) {
        s = scored_prepare(p, res, n_frames, st, prm);
        if (s != PNCE_OK) return s;
    }
    if (ldg) {
        prm.packed = static_cast<const uint16_t*>(packed);
        prm.packed_rows = (int64_t)packed_rows;
        prm.tx_bytes = 2 * (uint32_t)(t.g_cols / 2) * kBK * 2;  // circulant only
        const size_t smem = 1024 + (size_t)prm.stages * prm.stage_bytes + 1024;
        launch_k3<kModePackedLdg>(scored, pair_grid(p, prm), smem, st, t.tm_circ, t.tm_circ, prm);
    } else {
        const uint64_t key[3] = {packed_rows, (uint64_t)p->k_pad, 1};
        if (res->tm_in_ptr != packed || std::memcmp(res->tm_in_key, key, sizeof(key)) != 0) {
            s = make_tmap(&res->tm_in, packed, p->k_pad, packed_rows, kBM, p->cfg.dtype == PNCE_DTYPE_BF16);
            if (s != PNCE_OK) {
                res->tm_in_ptr = nullptr;
                return s;
            }
            res->tm_in_ptr = packed;
            std::memcpy(res->tm_in_key, key, sizeof(key));
        }
        const size_t smem = 1024 + (size_t)prm.stages * prm.stage_bytes + 1024;
        launch_k3<kModePacked>(scored, pair_grid(p, prm), smem, st, res->tm_in, t.tm_circ, prm);
    }
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    if (stats) {
        s = scored_finish(p, res, taps, truth, stats, nullptr, n_frames, st);
        if (s != PNCE_OK) return s;
    }
    diag_dump(st);
    return PNCE_OK;
}

struct T16Opts {
    int chunk_kb;
    int acc16;
};
// Input row layout override: compact CP-stripped bodies (row stride in samples, no offset)
struct BodyLayout {
    int stride;
};
// Antenna-split gather: the launch's receivers are rows [r0, r0 + n_r) of an n_r_total-row CSI
struct GatherOpts {
    float* const* peers;
    int n_peers;
    int n_r_total;
    int r0;
};
static pnce_status_t process_frames_impl(const pnce_plan_t* p, const float* iq, float* taps, const float* truth,
                                         double* stats, float* link_err, int64_t n_frames, void* stream,
                                         const T16Opts* t16 = nullptr, const BodyLayout* bodies = nullptr,
                                         const GatherOpts* gather = nullptr);

pnce_status_t pnce_process_frames(const pnce_plan_t* p, const float* iq, float* taps, const float* truth,
                                  double* stats, void* workspace, size_t workspace_bytes, int64_t n_frames,
                                  void* stream) {
    (void)workspace;
    (void)workspace_bytes;
    return process_frames_impl(p, iq, taps, truth, stats, nullptr, n_frames, stream);
}

pnce_status_t pnce_process_frames_gather(const pnce_plan_t* p, const float* iq, float* csi, float* const* peers,
                                         int32_t n_peers, int32_t n_r_total, int32_t r0, int64_t n_frames,
                                         void* stream) {
    if (!p) return fail(PNCE_ERR_INVALID_CONFIG, "null plan");
    if (n_peers < 0 || n_peers > kMaxPeers) return fail(PNCE_ERR_INVALID_CONFIG, "0..7 peer buffers");
    if (n_peers > 0 && !peers) return fail(PNCE_ERR_DIMENSION, "null peer list");
    for (int d = 0; d < n_peers; ++d)
        if (!peers[d] || ((reinterpret_cast<uintptr_t>(peers[d]) ^ reinterpret_cast<uintptr_t>(csi)) & 15))
            return fail(PNCE_ERR_DIMENSION, "peer CSI buffers must share the local buffer's 16-byte alignment");
    if (r0 < 0 || n_r_total < p->cfg.n_r || r0 + p->cfg.n_r > n_r_total)
        return fail(PNCE_ERR_DIMENSION, "receiver slice [r0, r0 + n_r) outside [0, n_r_total)");
    GatherOpts g{peers, n_peers, n_r_total, r0};
    return process_frames_impl(p, iq, csi, nullptr, nullptr, nullptr, n_frames, stream, nullptr, nullptr, &g);
}

pnce_status_t pnce_process_frames_scored(const pnce_plan_t* p, const float* iq, float* taps, const float* truth,
                                         double* stats, float* link_err, int64_t n_frames, void* stream) {
    if (link_err && !truth) return fail(PNCE_ERR_INVALID_CONFIG, "per-link errors need the ground truth");
    if (reinterpret_cast<uintptr_t>(link_err) & 3) return fail(PNCE_ERR_DIMENSION, "link_err must be 4-byte aligned");
    return process_frames_impl(p, iq, taps, truth, stats, link_err, n_frames, stream);
}

pnce_status_t pnce_process_bodies(const pnce_plan_t* p, const float* bodies, int32_t body_stride, float* taps,
                                  const float* truth, double* stats, float* link_err, int64_t n_frames, void* stream) {
    if (!p) return fail(PNCE_ERR_INVALID_CONFIG, "null plan");
    if (body_stride < p->cfg.m) return fail(PNCE_ERR_DIMENSION, "body_stride must be >= m");
    if (link_err && !truth) return fail(PNCE_ERR_INVALID_CONFIG, "per-link errors need the ground truth");
    BodyLayout b{body_stride};
    return process_frames_impl(p, bodies, taps, truth, stats, link_err, n_frames, stream, nullptr, &b);
}

pnce_status_t pnce_copy_bodies_h2d(const pnce_plan_t* p, const float* iq_host, float* bodies_dev, int32_t body_stride,
                                   int64_t n_frames, void* stream) {
    if (!p) return fail(PNCE_ERR_INVALID_CONFIG, "null plan");
    if (n_frames < 0) return fail(PNCE_ERR_DIMENSION, "n_frames < 0");
    if (n_frames == 0) return PNCE_OK;
    if (!iq_host || !bodies_dev) return fail(PNCE_ERR_DIMENSION, "null buffer");
    if (body_stride < p->cfg.m) return fail(PNCE_ERR_DIMENSION, "body_stride must be >= m");
    const pnce_cfg_t& c = p->cfg;
    const int64_t rows = n_frames * p->n_batches * (int64_t)c.n_r;
    const size_t samples = (size_t)c.c + c.m + c.l - 1;
    // remove_cp (estimator.py:40-47) as a pitched DMA: only the M body samples cross PCIe
    CUDA_TRY(cudaMemcpy2DAsync(bodies_dev, (size_t)body_stride * 8, iq_host + 2 * (size_t)c.c, samples * 8,
                               (size_t)c.m * 8, (size_t)rows, cudaMemcpyHostToDevice,
                               static_cast<cudaStream_t>(stream)));
    return PNCE_OK;
}

// tensor16 options of a plan (halfprec.py:44-55, 135-146 checks; device chunks are whole K-blocks)
static pnce_status_t t16_opts(const pnce_plan_t* p, int32_t chunk_len, int32_t binary16_accumulator, T16Opts& o) {
    if (!p) return fail(PNCE_ERR_INVALID_CONFIG, "null plan");
    const int kp4 = (p->cfg.m + 3) / 4 * 4;  // the reference pads K to its 4-wide tile (halfprec.py:80-81)
    if (chunk_len < 0) return fail(PNCE_ERR_INVALID_CONFIG, "chunk_len must be >= 0 (0: one chunk)");
    if (chunk_len > kp4) return fail(PNCE_ERR_INVALID_CONFIG, "chunk_len exceeds padded length");
    if (chunk_len % kBK) return fail(PNCE_ERR_INVALID_CONFIG, "device chunks are whole 64-sample K-blocks");
    if (binary16_accumulator != 0 && binary16_accumulator != 1)
        return fail(PNCE_ERR_INVALID_CONFIG, "accumulator must be 0 (binary32) or 1 (binary16)");
    o = T16Opts{chunk_len ? chunk_len / kBK : p->k_pad / kBK, binary16_accumulator};
    return PNCE_OK;
}

pnce_status_t pnce_process_frames_tensor16(const pnce_plan_t* p, const float* iq, float* taps, const float* truth,
                                           double* stats, int32_t chunk_len, int32_t binary16_accumulator,
                                           int64_t n_frames, void* stream) {
    T16Opts o;
    s_ok_or_return(t16_opts(p, chunk_len, binary16_accumulator, o));
    return process_frames_impl(p, iq, taps, truth, stats, nullptr, n_frames, stream, &o);
}

pnce_status_t pnce_process_bodies_tensor16(const pnce_plan_t* p, const float* bodies, int32_t body_stride,
                                           float* taps, const float* truth, double* stats, int32_t chunk_len,
                                           int32_t binary16_accumulator, int64_t n_frames, void* stream) {
    T16Opts o;
    s_ok_or_return(t16_opts(p, chunk_len, binary16_accumulator, o));
    if (body_stride < p->cfg.m) return fail(PNCE_ERR_DIMENSION, "body_stride must be >= m");
    BodyLayout b{body_stride};
    return process_frames_impl(p, bodies, taps, truth, stats, nullptr, n_frames, stream, &o, &b);
}

}  // extern "C"

static pnce_status_t process_frames_impl(const pnce_plan_t* p, const float* iq, float* taps, const float* truth,
                                         double* stats, float* link_err, int64_t n_frames, void* stream,
                                         const T16Opts* t16, const BodyLayout* bodies, const GatherOpts* gather) {
    if (!p) return fail(PNCE_ERR_INVALID_CONFIG, "null plan");
    if (n_frames < 0) return fail(PNCE_ERR_DIMENSION, "n_frames < 0");
    if (n_frames == 0) return PNCE_OK;
    if (!iq || !taps) return fail(PNCE_ERR_DIMENSION, "null buffer");
    if (reinterpret_cast<uintptr_t>(iq) & 7) return fail(PNCE_ERR_DIMENSION, "iq buffer must be 8-byte aligned");
    s_ok_or_return(check_device(p));
    const Knobs& kn = knobs();
    CorrParams prm;
    // tensor16: scoring moves to the finish kernel (saturated batches are scored as zeros).
    // Scored launches (drain ~2x the main loop) use <= 256-column groups with two TMEM
    // accumulators, so one tile's drain overlaps the next tile's MMAs (knob PNCE_TUNE_SCORED_G)
    const bool scored = !t16 && (truth || stats || link_err);
    // plain launches with few row tiles (a handful of frame-sets: latency-bound): narrower
    // lag-row groups spread over more CTA pairs (same MMAs per output, bit-identical taps)
    const int64_t tiles_fused = (n_frames * p->n_batches * (int64_t)p->cfg.n_r + kBM - 1) / kBM * p->fused.n_groups;
    const bool narrow = !t16 && !scored && kn.narrow == 1 && p->narrow.n_groups > p->fused.n_groups &&
                        tiles_fused * 4 <= p->num_sms / 2;
    // a few more row tiles (5-9 cfg3 frame-sets): 256-column groups, still one wave of CTA
    // pairs (PNCE_TUNE_MID: 0 off, 1 TMA raw ring, 2 LDG converters)
    const int64_t row_tiles = tiles_fused / p->fused.n_groups;
    const bool mid = !t16 && !scored && !narrow && kn.mid >= 1 && p->mid.n_groups > p->fused.n_groups &&
                     row_tiles * p->mid.n_groups <= p->num_sms / 2;
    const Tiling& tiling = t16 ? p->t16
                               : (narrow ? p->narrow : mid ? p->mid
                                         : (scored && kn.scored_g == 256 ? p->packed_ldg : p->fused));
    pnce_status_t s = fill_params(p, tiling, true, taps, t16 ? nullptr : truth, t16 ? nullptr : stats, n_frames, prm);
    if (s != PNCE_OK) return s;
    prm.iq = iq;
    prm.link_err = link_err;
    if (gather) {
        prm.out_nr = gather->n_r_total;
        prm.out_r0 = gather->r0;
        prm.gather_n = gather->n_peers;
        for (int d = 0; d < gather->n_peers; ++d) prm.gather_dst[d] = gather->peers[d];
        prm.n_taps = n_frames * (int64_t)gather->n_r_total * p->cfg.n_t * p->cfg.l;
    }
    if (bodies) {  // compact bodies: sample k of a link's body at row offset k
        prm.samples = bodies->stride;
        prm.c = 0;
    }
    const int samples = prm.samples;
    // the raw f32 rows can be described by a tensor map when the row stride is 16-byte aligned
    const bool map_ok = ((size_t)samples * 8) % 16 == 0 && (reinterpret_cast<uintptr_t>(iq) & 15) == 0;
    if (t16 && !map_ok)
        return fail(PNCE_ERR_INVALID_CONFIG, "tensor16 mode needs 16-byte aligned IQ rows (even P+L-1)");
    bool use_tma = map_ok;
    // (the tensor16 instantiation only exists with the TMA raw ring: the knob never applies to it)
    if (!t16 && kn.fused_mode == kModeFusedLdg) use_tma = false;
    // lone-tile (narrow) launches are latency-bound: the LDG converters (no raw staging ring,
    // all shared memory for A/B stages) shorten the serial K chain, 26 vs 29 us per cfg3
    // frame-set, bit-identical (tools/narrow_mode_trial.sh; PNCE_TUNE_NARROW_LDG=0: TMA ring)
    if (narrow && kn.fused_mode < 0 && kn.narrow_ldg == 1) use_tma = false;
    if (mid && kn.fused_mode < 0 && kn.mid == 2) use_tma = false;
    // plain launches with >= 3 lag-row groups (cfg4': R = 2032, K = 2048) are MMA-bound: the LDG
    // converters (no raw TMA boxes queued ahead of the circulant loads in the TMA engine) beat the
    // TMA raw ring + A-stage reuse, 14.9 vs 15.9 us per cfg4' frame-set, bit-identical
    // (tools/cfg4_probe6.sh; PNCE_TUNE_WIDE_LDG=0: TMA ring).  Scored launches keep the ring
    // (27 vs 37 us: the truth ring needs its shared memory).
    if (!t16 && !scored && kn.fused_mode < 0 && kn.wide_ldg == 1 && tiling.n_groups >= 3 && !narrow && !mid)
        use_tma = false;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamRes* res = stream_res(const_cast<pnce_plan*>(p), st);
    if (scored && stats) s_ok_or_return(scored_prepare(p, res, n_frames, st, prm));
    prm.raw_row_floats = 2 * kRawChunk + ((prm.c & 1) ? 4 : 0);
    if (use_tma) {
        // raw f32 rows as a tensor map, cached per stream (rebuilt when the input changes)
        const uint64_t key[3] = {(uint64_t)samples * 2, (uint64_t)prm.total_links, (uint64_t)prm.raw_row_floats << 1};
        if (res->tm_in_ptr != iq || std::memcmp(res->tm_in_key, key, sizeof(key)) != 0) {
            s = make_tmap_raw(&res->tm_in, iq, key[0], key[1], (uint32_t)prm.raw_row_floats);
            if (s != PNCE_OK) {
                res->tm_in_ptr = nullptr;
                return s;
            }
            res->tm_in_ptr = iq;
            std::memcpy(res->tm_in_key, key, sizeof(key));
        }
        // f32 rows TMA-staged in shared memory (default): A/B ring of up to 3 stages, the
        // rest of shared memory as the raw half-K-block ring (its depth hides HBM latency:
        // ~1.3 us per load vs ~0.4 us of MMA per chunk)
        prm.raw_stage_bytes = (uint32_t)(kLinksPerTile * prm.raw_row_floats * 4);
        int64_t budget = (int64_t)kSmemLimit - 2048;
        // a_reuse (several lag-row groups): convert a row tile once, keep its fp16 A stages in an
        // L2-resident scratch for the other groups (PNCE_TUNE_A_REUSE=0: convert per group)
        // (two groups: tensor16 -- 2.76 vs 2.82 us; with >= 3 groups (cfg4') the re-reads of
        // the raw rows hit L2 (neighbouring clusters take the other groups of the same row tile)
        // and skipping the scratch is faster: scored cfg4' 27.8 -> 25.4 us.  PNCE_TUNE_A_REUSE:
        // 0 never, 1 two groups, 2 any number of groups)
        if (kn.a_reuse >= 1 && !narrow && !mid && tiling.n_groups > 1 && (tiling.n_groups == 2 || kn.a_reuse == 2) &&
            prm.k_blocks <= 64) {
            prm.a_reuse = 1;
            prm.scr_pol = kn.scr_pol;
            prm.scr_slots = kn.scr_slots > 0 ? std::max(1, std::min(2, kn.scr_slots)) : 1;
            prm.bar_bytes = 2048;
            budget -= 1024;
        }
        // scored drain: truth staged through a per-thread LDGSTS ring (epilogue warps x
        // slots x 2 KB) when the truth runs are 16-byte aligned (PNCE_TUNE_TRUTH_SLOTS, 0 = off)
        const int epi_warps = kn.scored_epi == 4 ? 4 : 8;
        if (scored && truth && (p->cfg.l % 2) == 0 && (reinterpret_cast<uintptr_t>(truth) & 15) == 0 &&
            (prm.g_cols & 31) == 0 && kn.truth_slots >= 2 && kn.truth_slots <= 4) {
            prm.truth_slots = kn.truth_slots;
            budget -= (int64_t)epi_warps * prm.truth_slots * 2048;
        }
        // tensor16's 32 KB stages (256-column groups): 4 A/B stages, 2.85 -> 2.76 us per cfg3
        // frame-set (5: same, 6: 2.91 -- the raw ring gets too short; tools/t16_probe.sh)
        int ab = (int)std::min<int64_t>(t16 ? 4 : 3, budget / (int64_t)prm.stage_bytes);
        if (kn.ab_stages > 0) ab = std::min<int>((int)(budget / prm.stage_bytes), kn.ab_stages);
        int raw = (int)std::min<int64_t>(8, (budget - (int64_t)ab * prm.stage_bytes) / prm.raw_stage_bytes);
        if (kn.raw_stages > 0) raw = std::min(raw, kn.raw_stages);
        if (ab < 2 || raw < 2) return fail(PNCE_ERR_INVALID_CONFIG, "shared memory too small for the fused pipeline");
        prm.stages = ab;
        prm.raw_stages = raw;
        // one scratch slot is enough when a K-block's store for row tile r+1 (group 0) comes at
        // least `stages` jobs after the last group's load of it for row tile r: k_blocks >= stages
        if (prm.a_reuse && prm.k_blocks < prm.stages) prm.scr_slots = 2;
        prm.truth_off = (uint32_t)((size_t)prm.stages * prm.stage_bytes + prm.bar_bytes +
                                   (size_t)prm.raw_stages * prm.raw_stage_bytes);
        const size_t smem = 1024 + (size_t)prm.truth_off + (size_t)epi_warps * prm.truth_slots * 2048;
        const int grid = pair_grid(p, prm);
        if (prm.a_reuse) {
            // [slots][clusters][2 CTAs][k_blocks] A stages of 128 rows x 128 B, owned by the
            // (plan, stream) entry: allocated once, not per launch
            const uint64_t rows = (uint64_t)prm.scr_slots * (grid / 2) * 2 * prm.k_blocks * kBM;
            const uint8_t* before = res->scratch;
            s_ok_or_return(ensure_buf(res->scratch, res->scratch_bytes, (size_t)rows * 128, st, "A scratch"));
            if (res->scratch != before || res->tm_scr_rows != rows) {
                s = make_tmap_scr(&res->tm_scr, res->scratch, rows);
                if (s != PNCE_OK) {
                    res->tm_scr_rows = 0;
                    return s;
                }
                res->tm_scr_rows = rows;
            }
            prm.scratch = res->scratch;
            prm.scr_rows = (int64_t)rows;
        }
        if (t16) {
            const int64_t n_fb = n_frames * p->n_batches;
            s_ok_or_return(ensure_buf(res->flags, res->flags_n, (size_t)n_fb, st, "tensor16 flags"));
            CUDA_TRY(cudaMemsetAsync(res->flags, 0, sizeof(uint32_t) * n_fb, st));
            prm.chunk_kb = t16->chunk_kb;
            prm.acc16 = t16->acc16;
            prm.sat_flags = res->flags;
            if (t16->acc16) prm.idesc &= ~(3u << 4);  // c_format = F16: binary16 partials in TMEM
            if (kn.t16_epi == 8)
                k_correlate<kModeFusedTma, false, true, true><<<grid, kThreadsK3, smem, st>>>(
                    res->tm_in, p->t16.tm_circ, prm.a_reuse ? res->tm_scr : p->t16.tm_circ, prm);
            else
                k_correlate<kModeFusedTma, false, false, true><<<grid, kThreadsK3, smem, st>>>(
                    res->tm_in, p->t16.tm_circ, prm.a_reuse ? res->tm_scr : p->t16.tm_circ, prm);
            g_launches++;
            const pnce_cfg_t& c = p->cfg;
            k_t16_finish<<<(unsigned)n_fb, 256, 0, st>>>(taps, truth, stats, res->flags, c.n_r, c.n_t, c.n_batch,
                                                         p->n_batches, c.l);
            CUDA_TRY(cudaGetLastError());
        } else {
            launch_k3<kModeFusedTma>(scored, grid, smem, st, res->tm_in, tiling.tm_circ, prm,
                                     prm.a_reuse ? &res->tm_scr : nullptr);
        }
    } else {
        if (kn.ab_stages > 0) prm.stages = std::min(prm.stages, std::max(2, kn.ab_stages));
        const size_t smem = 1024 + (size_t)prm.stages * prm.stage_bytes + 1024;
        // the LDG variant reads the rows directly (tm_in unused; the circulant map fills the slot)
        launch_k3<kModeFusedLdg>(scored, pair_grid(p, prm), smem, st, tiling.tm_circ, tiling.tm_circ, prm);
    }
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    if (scored && stats) s_ok_or_return(scored_finish(p, res, taps, truth, stats, link_err, n_frames, st));
    diag_dump(st);
    return PNCE_OK;
}
