/*
 * pnce_b200 — C ABI of the B200-native PN-correlation channel estimator.
 *
 * This is the drop-in boundary for the reference's hot path
 *   process_frames -> correlate_rows        (pnce/experiments.py:176-208,
 *                                            pnce/estimator.py:68-86)
 * Plain pointers and sizes only; no torch types.  All device pointers are
 * caller-owned CUDA allocations; `stream` is a cudaStream_t passed as void*.
 * Every entry point is reentrant (no hidden global state beyond a
 * thread-local error string) and returns a pnce_status_t; on failure
 * pnce_last_error() describes the failure on the calling thread.
 *
 * Layouts (row-major, little-endian):
 *   iq     float32 [n_frames][n_batches][n_r][P + L - 1][2]   (I, Q)
 *          = the reference IQ file payload layout (pnce/iqfile.py:9-11),
 *          one frame-set = all n_batches = ceil(n_t / n_batch) received batches.
 *   taps   float32 [n_frames][n_r][n_t][L][2]  (complex64, CirEstimate.taps,
 *          pnce/estimator.py:27-37, already normalised by 1/M).
 *   truth  same layout as taps (ChannelRealization.taps, pnce/channel.py:79-88).
 *   stats  float64 [n_frames][4] accumulated (+=):
 *          {sum |h_est - h|, sum |h_est - h|^2, non-finite tap count, saturations}.
 *          Saturations use the reference's unit (experiments.py:201-205): a (frame-set,
 *          batch) whose estimate went non-finite (e.g. an input beyond the fp16 range) is
 *          scored as all-zero taps and counted as n_r * n_tx.  Saturation accounting needs
 *          `stats`; without it non-finite taps are left as computed.
 *
 * Resources: launch scratch (A-stage reuse, saturation flags, tensor maps) is owned by the
 * plan, one set per calling stream, allocated on the first launch on that stream; no
 * launch allocates afterwards.  Compute calls must run with the plan's device current
 * (PNCE_ERR_DIMENSION otherwise).
 */
#ifndef PNCE_B200_H
#define PNCE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes; each maps to the reference exception class named
 * (pnce/errors.py:4-69) by the Python front end. */
typedef enum pnce_status {
    PNCE_OK = 0,
    PNCE_ERR_INVALID_CONFIG = 1,    /* InvalidConfigError      errors.py:29  */
    PNCE_ERR_INVALID_SPEC = 2,      /* InvalidSpecError        errors.py:25  */
    PNCE_ERR_ZERO_STATE = 3,        /* ZeroStateError          errors.py:17  */
    PNCE_ERR_NOT_MAXIMAL = 4,       /* NotMaximalLengthError   errors.py:21  */
    PNCE_ERR_DIMENSION = 5,         /* DimensionMismatchError  errors.py:45  */
    PNCE_ERR_FRAME_TOO_SHORT = 6,   /* FrameTooShortError      errors.py:49  */
    PNCE_ERR_PLAN_MISMATCH = 7,     /* PlanMismatchError       errors.py:53  */
    PNCE_ERR_ROWS_OUT_OF_RANGE = 8, /* RowsOutOfRangeError     errors.py:41  */
    PNCE_ERR_SATURATION = 9,        /* SaturationDetectedError errors.py:57  */
    PNCE_ERR_CUDA = 10,             /* CUDA runtime/driver failure            */
    PNCE_ERR_UNSUPPORTED_DEVICE = 11/* not an sm_100 device                  */
} pnce_status_t;

/* Operand precision of the tensor-core contraction (fp32 accumulate). */
enum { PNCE_DTYPE_FP16 = 0, PNCE_DTYPE_BF16 = 1 };

/* PilotConfig (pnce/pilots.py:14-47) + receive array size + LfsrSpec
 * (pnce/pn.py:39-71).  tap_mask bit (t-1) set <=> feedback tap t. */
typedef struct pnce_cfg {
    int32_t m;          /* PN length M = 2^degree - 1          */
    int32_t c;          /* cyclic-prefix length C              */
    int32_t n_t;        /* transmit antennas                   */
    int32_t n_r;        /* receive antennas                    */
    int32_t n_batch;    /* transmitters multiplexed per batch  */
    int32_t l;          /* CIR length L                        */
    int32_t degree;     /* LFSR degree k                       */
    uint32_t tap_mask;  /* LFSR feedback taps                  */
    uint32_t state;     /* LFSR start state (nonzero)          */
    int32_t dtype;      /* PNCE_DTYPE_*                        */
} pnce_cfg_t;

typedef struct pnce_plan pnce_plan_t;

/* Library version (major*10000 + minor*100 + patch). */
int32_t pnce_version(void);

/* Thread-local description of the last failure on this thread. */
const char* pnce_last_error(void);

/* Validate a configuration (PilotConfig.__post_init__ pilots.py:30-41,
 * LfsrSpec.__post_init__ pn.py:53-67, build_batch_plan's separation
 * check pilots.py:134-142).  Host only, no device work. */
pnce_status_t pnce_config_check(const pnce_cfg_t* cfg);

/* generate_mseq (pn.py:109-138) on the device: one LFSR period written as
 * chips (+1.0f / -1.0f) to chips_dev[0..m).  Synchronises `stream` to run the
 * period check; returns PNCE_ERR_NOT_MAXIMAL when the period is not 2^k-1. */
pnce_status_t pnce_generate_mseq(int32_t degree, uint32_t tap_mask, uint32_t state,
                                 float* chips_dev, int32_t m, void* stream);

/* Build the correlator state for a configuration (correlator_rows_for_plan,
 * experiments.py:157-173): runs the device LFSR and builds the stacked
 * lag-window circulant rows (batched_lag_rows, estimator.py:114-117) in
 * tensor-core operand layout.  One-time; synchronises `stream`. */
pnce_status_t pnce_plan_create(const pnce_cfg_t* cfg, pnce_plan_t** plan, void* stream);
pnce_status_t pnce_plan_destroy(pnce_plan_t* plan);

/* Operator-level seam: a plan over caller-supplied correlation rows, the `rows` argument of
 * correlate_rows (estimator.py:68-86; build_partial_circulant / batched_lag_rows output).
 * rows_dev: float32 [n_rows][m] on the device (+-1 for PN rows; any values are rounded to
 * the plan dtype), 1 <= n_rows <= m (RowsOutOfRange otherwise); norm_len: the 1/norm_len
 * scale.  From cfg only m, n_r (received columns) and dtype are used.  Correlating y
 * ([n_r] columns of m samples) is pnce_process_bodies with body rows of y's columns:
 * taps[f][col][0][q] = (1/norm_len) sum_k rows[q][k] y[k][col]. */
pnce_status_t pnce_plan_create_rows(const pnce_cfg_t* cfg, const float* rows_dev, int32_t n_rows,
                                    int32_t norm_len, pnce_plan_t** plan, void* stream);

/* Copy the plan's device-generated chips (float32 [m]) into dst_dev. */
pnce_status_t pnce_plan_chips(const pnce_plan_t* plan, float* dst_dev, void* stream);

/* The plan's correlation operand as built on the device (test/inspection seam for the
 * integer work of batched_lag_rows, estimator.py:114-117): 16-bit (plan dtype) rows
 * [n_rows][k_pad], row j*L + l = chips shifted by shift_j + l (A[j*L+l][k] =
 * chip[(k - s_j - l) mod M]), columns >= m and rows >= N_b*L zero.  With dst == NULL
 * only the extents are returned. */
pnce_status_t pnce_plan_operand(const pnce_plan_t* plan, void* dst_dev, int32_t* n_rows, int32_t* k_pad,
                                void* stream);

/* Bytes of the packed 16-bit operand pnce_pack_iq writes for n_frames.
 * Packed layout: K_pad = roundup(m, 64) columns; links q = (f*n_batches + b)*n_r + r are
 * grouped by 8 and each 16-row block holds the block's 8 Re rows then its 8 Im rows
 * (Re of q at row 16*(q/8) + q%8, Im at 16*(q/8) + 8 + q%8); rows of padding links up to
 * a multiple of 8, and columns >= m, are zero.  Rows = 16 * ceil(links / 8). */
size_t pnce_workspace_bytes(const pnce_plan_t* plan, int64_t n_frames);

/* K2 alone: CP removal (remove_cp, estimator.py:40-47) + de-interleave +
 * fp16/bf16 quantisation of received IQ into the contraction operand. */
pnce_status_t pnce_pack_iq(const pnce_plan_t* plan, const float* iq, void* packed,
                           int64_t n_frames, void* stream);

/* K3+K4 alone: tensor-core correlation of packed samples with the PN
 * circulant, fused 1/M normalisation, per-transmitter window demux into taps
 * and (when truth != NULL) per-frame error statistics into stats. */
pnce_status_t pnce_correlate(const pnce_plan_t* plan, const void* packed, float* taps,
                             const float* truth, double* stats, int64_t n_frames,
                             void* stream);

/* Frame-set seam = process_frames (experiments.py:176-208) for n_frames
 * frame-sets in ONE fused kernel: CP strip + quantise (K2) inside the
 * tcgen05 correlation (K3) + demux/normalise/scoring epilogue (K4).  No packed
 * intermediate is written; `workspace` may be NULL (kept for ABI stability). */
pnce_status_t pnce_process_frames(const pnce_plan_t* plan, const float* iq, float* taps,
                                  const float* truth, double* stats, void* workspace,
                                  size_t workspace_bytes, int64_t n_frames, void* stream);

/* Antenna split with the CSI all-gather fused into the epilogue (the paper's multi-GPU
 * scheme: N_r / N_gpu receive antennas per GPU, then Allgather() of the
 * CIRs).  `plan` covers this rank's n_r receivers, which are rows [r0, r0 + n_r) of the
 * n_r_total-row CSI.  Every tap is stored into `csi` (local, complex64
 * [F][n_r_total][n_t][L]) AND into each of the n_peers (<= 7) peer buffers of the same
 * layout (device pointers valid in this context, e.g. CUDA-IPC mappings of the other
 * ranks' `csi`: NVLink stores from the epilogue, no separate collective).  The caller
 * orders the ranks (stream sync + barrier) before reading the gathered CSI.  Plain
 * estimation only (no truth/stats).  Replaces process_frames + allgather over ranks. */
pnce_status_t pnce_process_frames_gather(const pnce_plan_t* plan, const float* iq, float* csi,
                                         float* const* peers, int32_t n_peers, int32_t n_r_total,
                                         int32_t r0, int64_t n_frames, void* stream);

/* process_frames + fused per-link scoring (north star (4)): as pnce_process_frames,
 * and when link_err != NULL (float32 [F][n_r][n_t], zeroed by the caller; needs truth)
 * each entry receives the link's MSE, mean over its L taps of |h_est - h_true|^2,
 * reduced in the epilogue with warp shuffles.  Reference: the mae/MSE scoring of
 * metrics.py:19-25 applied per (r, t) link of CirEstimate.taps (estimator.py:27-37). */
pnce_status_t pnce_process_frames_scored(const pnce_plan_t* plan, const float* iq, float* taps,
                                         const float* truth, double* stats, float* link_err,
                                         int64_t n_frames, void* stream);

/* Host-ingest helpers (remove_cp before PCIe, estimator.py:40-47): pnce_copy_bodies_h2d
 * copies only the CP-stripped bodies of host IQ rows ([F][n_batches][n_r][P+L-1][2] f32,
 * pinned) into compact device rows of body_stride (>= m) samples with one pitched DMA;
 * pnce_process_bodies runs the fused estimator (as pnce_process_frames_scored) on such
 * compact rows. */
pnce_status_t pnce_copy_bodies_h2d(const pnce_plan_t* plan, const float* iq_host, float* bodies_dev,
                                   int32_t body_stride, int64_t n_frames, void* stream);
pnce_status_t pnce_process_bodies(const pnce_plan_t* plan, const float* bodies, int32_t body_stride,
                                  float* taps, const float* truth, double* stats, float* link_err,
                                  int64_t n_frames, void* stream);

/* The reference's tensor16 backend on real tensor cores (halfprec.py:93-125):
 * fp16/bf16 operands, the contraction split into chunk_len-sample chunks (0: one chunk;
 * otherwise a multiple of 64 and <= roundup(m, 4)), each chunk accumulated in TMEM as a
 * binary32 (binary16_accumulator = 0) or binary16 (= 1, the F16 tcgen05 accumulator)
 * partial, then x fp32(1/M) into an fp32 running total.  A (frame-set, batch) whose partial
 * or total goes non-finite is scored as all-zero taps and counted, as process_frames
 * does (experiments.py:201-205).  stats (nullable, zeroed by the caller) [F][4]:
 * sum|e|, sum|e|^2 (when truth != NULL), non-finite taps, saturations (n_r * n_tx per
 * saturated batch, the reference's unit). */
pnce_status_t pnce_process_frames_tensor16(const pnce_plan_t* plan, const float* iq, float* taps,
                                           const float* truth, double* stats, int32_t chunk_len,
                                           int32_t binary16_accumulator, int64_t n_frames,
                                           void* stream);

/* tensor16 mode over compact body rows (pnce_process_bodies layout): the operator seam's
 * correlate_rows with BackendConfig(kind="tensor16") (estimator.py:68-86 -> halfprec.py:127-156). */
pnce_status_t pnce_process_bodies_tensor16(const pnce_plan_t* plan, const float* bodies, int32_t body_stride,
                                           float* taps, const float* truth, double* stats, int32_t chunk_len,
                                           int32_t binary16_accumulator, int64_t n_frames, void* stream);

/* Input synthesis on the device (channel.py:96-214).  Not part of the timed
 * estimation path: it feeds benches and sweeps with statistically equivalent frames
 * (Philox streams instead of numpy's PCG64).
 *
 * pnce_draw_channel: h complex64 [F][n_r][n_t][L] with the draw_channel law
 * (channel.py:96-108): l_nz distinct taps per link, |h| uniform on (0, A_max],
 * A_max^2 = 1 / (n_t sqrt(l_nz)), phase uniform on [0, 2 pi).
 *
 * pnce_simulate_frames: the pilot sweep of simulate_frame (channel.py:186-214) for each
 * frame-set: iq float32 [F][n_batches][n_r][P+L-1][2] = linear convolution of every
 * batch pilot [CP | PN rolled by its shift] with its CIR, plus complex AWGN at snr_db
 * relative to the noise_reference_power (channel.py:175-183); snr_db = +inf: noiseless. */
pnce_status_t pnce_draw_channel(const pnce_plan_t* plan, int32_t l_nz, uint64_t seed, float* h,
                                int64_t n_frames, void* stream);
pnce_status_t pnce_simulate_frames(const pnce_plan_t* plan, const float* h, double snr_db,
                                   uint64_t seed, float* iq, int64_t n_frames, void* stream);

/* Launch-count accounting: number of device kernels this library has
 * launched in the calling process (for bench.py's gpu_launches). */
int64_t pnce_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* PNCE_B200_H */
