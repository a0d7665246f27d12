/*
 * include/mm.h -- C ABI of the MicroMix B200 hot path (libmicromix_b200.so).
 *
 * MicroMix (arXiv 2508.02343) splits the K input channels of a linear layer
 * into three groups P4 | P6 | P8 quantized to MXFP4 (E2M1), MXFP6 (E3M2 or
 * E2M3) and MXFP8 (E4M3 or E5M2) with 32-element blocks and E8M0 shared
 * scales (§3.1 line 91, §4.1, Eq. 1 lines 40-45).  The
 * group sizes come from the quantization thresholds T(4), T(6) (Definition 1,
 * Eq. 5-6, lines 97-106; Eq. 17) and the channel order from the
 * channel-wise absolute means (Eq. 7 and Q3, lines 120-126), both computed
 * offline on calibration data.  Weights are reordered and quantized once
 * offline (Fig. 1 caption line 20, line 151); activations are reordered and
 * quantized online by one fused kernel (§3.2 "Quantization Kernel", line 151,
 * Fig. 6) and multiplied by one block-scaled GEMM that accumulates
 * the three segment contractions in FP32 and writes BFloat16 (§3.2 "GEMM
 * Kernel" line 143, Eq. 2 lines 47-51, abstract line 6).
 *
 * The four calls named by the north star are
 *   mm_calibrate_thresholds, mm_quantize_weight_offline,
 *   mm_reorder_quantize_act, mm_mixed_gemm_bf16.
 *
 * CONVENTIONS (all calls)
 *  - extern "C", never throws; every call returns mm_status; on error nothing
 *    has been enqueued and mm_last_error() (thread-local) has the reason.
 *  - Pointers named d_* are DEVICE pointers, h_* are HOST pointers.  All
 *    buffers are allocated and owned by the caller; the library allocates no
 *    device memory and never synchronizes on the hot calls (mm_reorder_quantize_act,
 *    mm_rmsnorm_reorder_quantize_act, mm_mixed_gemm_bf16 and the N-shard GEMMs), so
 *    they can be captured into CUDA graphs; it keeps no reference after the work
 *    queued on `stream` has completed (buffers are borrowed until then).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Work is
 *    asynchronous on that stream except where stated.
 *  - BF16 matrices are row-major with an element leading dimension ld*
 *    (ld >= number of columns, rows 16-byte aligned: ld % 8 == 0 and the base
 *    pointer 16-byte aligned).
 *  - Requires an sm_100 device (B200); anything else -> MM_ERR_UNSUPPORTED_DEVICE.
 *
 * QUANTIZED OPERAND LAYOUT (mm_mx_tensor, "segment g" = 0:FP4, 1:FP6, 2:FP8)
 *  - Segment g holds n[g] reordered channels stored in Kp[g] = roundup(n[g], 128)
 *    columns; columns >= n[g] hold zero codes and zero scale bytes.
 *  - codes[g]: rows x pitch(g) bytes, pitch = Kp*bits/8 (FP4: Kp/2, FP6: 3Kp/4,
 *    FP8: Kp).  FP4: element 2i in the low nibble of byte i.  FP6: tight LSB-first
 *    bit stream (element i at stream bits [6i, 6i+6), stream bit s = bit s%8 of
 *    byte s/8).  FP8: one byte per element.  Sign bit = top bit of the code.
 *  - sf[g]: E8M0 bytes (value 2^(byte-127)) for roundup(rows,128) x Kp/32 blocks in
 *    128x4 atoms of 512 B: byte (r, kb) lives at
 *       ((r/128)*(Kp/128) + kb/4)*512 + (r%32)*16 + ((r/32)%4)*4 + kb%4.
 *    Rows >= `rows` up to the next multiple of 128 are written as zero.
 *  - codes[g] and sf[g] must be 256-byte aligned and may be NULL iff n[g] == 0.
 */
#ifndef MICROMIX_B200_MM_H
#define MICROMIX_B200_MM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* mm_stream_t; /* == cudaStream_t */

typedef enum {
  MM_OK = 0,
  MM_ERR_INVALID_ARGUMENT = 1, /* NULL pointer, bad enum, non-bijective permutation */
  MM_ERR_SHAPE = 2,            /* K % 32, n[] rules, ld < cols, K > 65536, ...      */
  MM_ERR_ALIGNMENT = 3,        /* see the alignment rules above                    */
  MM_ERR_PLAN_MISMATCH = 4,    /* operands produced by a different plan           */
  MM_ERR_DEGENERATE = 5,       /* calibration data with max|X| == 0  */
  MM_ERR_UNSUPPORTED_DEVICE = 6,
  MM_ERR_CUDA = 7,             /* a CUDA runtime/driver call failed               */
  MM_ERR_NCCL = 8,             /* NCCL missing or an NCCL call failed             */
  MM_ERR_WORKSPACE = 9         /* workspace too small                              */
} mm_status;

typedef enum { MM_E2M1 = 0, MM_E3M2 = 1, MM_E2M3 = 2, MM_E4M3 = 3, MM_E5M2 = 4 } mm_elem_fmt;

/* Offset subtracted from floor(log2 max|X_i|) in Eq. 1:
 * OCP  = exponent of the largest normal (E2M1 2, E3M2 4, E2M3 2, E4M3 8, E5M2 15), default;
 * PAPER_EQ1 = Table 6's exponent bias b taken literally (1, 3, 1, 7, 15).
 * See DESIGN.md reading R1. */
typedef enum { MM_SCALE_OCP = 0, MM_SCALE_PAPER_EQ1 = 1 } mm_scale_rule;

/* A channel plan (§3.1): permutation + segment sizes + formats.
 * Plain value; the callee copies what it needs.  d_perm is borrowed. */
typedef struct {
  int32_t K;            /* in_features, K % 32 == 0, 32 <= K <= 65536            */
  int32_t n[3];         /* n4, n6, n8: multiples of 32 (0 allowed), sum == K      */
  int32_t fmt6;         /* MM_E3M2 (paper default) or MM_E2M3           */
  int32_t fmt8;         /* MM_E4M3 (paper default) or MM_E5M2                     */
  int32_t rule;         /* mm_scale_rule                                          */
  int32_t reserved;
  const int32_t* d_perm;  /* device int32[K]: reordered position j reads channel d_perm[j] */
  uint64_t fingerprint; /* hash(K, n, fmts, rule, perm); set by mm_plan_init / calibrate */
  double tensor_max;    /* calibration diagnostics: max|X| (0 for user plans)     */
  double t4, t6;        /* T(4), T(6) of Eq. 5 (0 for user plans)                 */
  int32_t c[3];         /* raw channel counts before rounding to 32 (calibration) */
  int32_t reserved2;
  const uint32_t* d_layout; /* optional gather-slot layout (mm_plan_set_gather_layout); NULL =
                               natural.  Changes where the RQ keeps values in shared memory only:
                               results are identical with and without it (borrowed). */
} mm_plan;

/* One quantized operand (activation: rows = M; weight: rows = N). */
typedef struct {
  int64_t rows;
  void* codes[3];
  void* sf[3];
  uint64_t fingerprint; /* copied from the plan that produced it */
} mm_mx_tensor;

/* ---- size queries (pure host functions; -1 on invalid arguments) ---------- */
int64_t mm_padded_cols(const mm_plan* plan, int seg);                 /* Kp = roundup(n,128) */
int64_t mm_code_pitch_bytes(const mm_plan* plan, int seg);            /* bytes per code row  */
int64_t mm_codes_bytes(const mm_plan* plan, int64_t rows, int seg);   /* rows * pitch        */
int64_t mm_sf_bytes(const mm_plan* plan, int64_t rows, int seg);      /* roundup(rows,128)*Kp/32 */
int64_t mm_calib_workspace_bytes(int64_t L, int32_t K);

/* Build a plan from a HOST permutation (validated to be a bijection) and copy
 * it into the caller's device buffer d_perm_storage (int32[K]); synchronous. */
mm_status mm_plan_init(mm_plan* plan_out, int32_t K, const int32_t n[3], int32_t fmt6,
                       int32_t fmt8, int32_t rule, const int32_t* h_perm,
                       int32_t* d_perm_storage, mm_stream_t stream);

/* Plan-time gather layout for the reorder-quantize (an implementation choice, not part
 * of the method: DESIGN.md §6.1).  For the plan's permutation, a local search picks,
 * inside every 32-channel line of the RQ's shared-memory rows, a parity-preserving
 * permutation of its eight 4-channel chunks that lowers the bank conflicts of the
 * gather x_r[j] = X[perm[j]].  d_layout_storage: caller device buffer of
 * mm_gather_layout_words(K) u32 words; on success plan->d_layout points to it.  Reads the
 * permutation back and SYNCHRONIZES stream (offline call).  Quantized outputs do not
 * depend on it (the plan fingerprint is unchanged). */
int64_t mm_gather_layout_words(int32_t K);
mm_status mm_plan_set_gather_layout(mm_plan* plan, uint32_t* d_layout_storage, mm_stream_t stream);
/* Host-only forms (diagnostics / tests): the layout for (K, n, permutation) into
 * h_layout_out[K/32], and the gather's bank wavefronts for a layout (NULL = natural);
 * -1 on invalid arguments. */
mm_status mm_gather_layout_host(int32_t K, const int32_t n[3], const int32_t* h_perm, uint32_t* h_layout_out);
int64_t mm_gather_wavefronts(int32_t K, const int32_t n[3], const int32_t* h_perm, const uint32_t* h_layout);

/* Offline calibration (§3.1 Q1-Q3, Eq. 5-7, Eq. 17; §4.1).
 * d_x: BF16 [L, K] calibration activations (ld = ldx).  On the device: exact
 * per-channel max|X| and the per-channel mean of |X| (fp64, double-double
 * accumulation, one final rounding).  On the host: max|X| -> T(4), T(6);
 * channel counts by max (<= T4 -> P4, (T4, T6] -> P6, rest -> P8) rounded to
 * multiples of 32 (n8 up, then n6 up capped, n4 the remainder); permutation =
 * stable ascending argsort of the means.  Writes d_perm_out (int32[K]) and
 * fills *plan_out (plan_out->d_perm = d_perm_out).  Optional h_chmax / h_chmean
 * (host double[K], may be NULL) receive the statistics.  SYNCHRONIZES stream.
 * Errors: MM_ERR_DEGENERATE if max|X| == 0; MM_ERR_WORKSPACE if ws_bytes <
 * mm_calib_workspace_bytes(L, K). */
mm_status mm_calibrate_thresholds(const void* d_x, int64_t L, int32_t K, int64_t ldx,
                                  int32_t fmt6, int32_t fmt8, int32_t rule,
                                  int32_t* d_perm_out, mm_plan* plan_out,
                                  void* d_ws, size_t ws_bytes,
                                  double* h_chmax, double* h_chmean, mm_stream_t stream);

/* Streaming calibration (the paper pools 32 x 2048 calibration tokens per layer,
 * §4.1; pooled statistics, R15).  d_state: caller-owned device
 * buffer of mm_calib_state_bytes(K) bytes, 256-byte aligned, ZEROED before the first
 * batch.  mm_calib_accumulate adds one batch X[L, K] (exact channel max, double-double
 * channel |x| sums, row count) -- asynchronous; d_ws as for mm_calibrate_thresholds.
 * mm_calib_finalize turns the state into a plan exactly as mm_calibrate_thresholds
 * does over the concatenated batches (SYNCHRONIZES stream); h_rows (may be NULL)
 * receives the pooled row count.  MM_ERR_DEGENERATE if no rows or max|X| == 0. */
int64_t mm_calib_state_bytes(int32_t K);
mm_status mm_calib_accumulate(const void* d_x, int64_t L, int32_t K, int64_t ldx, void* d_ws, size_t ws_bytes,
                              void* d_state, mm_stream_t stream);
mm_status mm_calib_finalize(const void* d_state, int32_t K, int32_t fmt6, int32_t fmt8, int32_t rule,
                            int32_t* d_perm_out, mm_plan* plan_out, double* h_chmax, double* h_chmean,
                            int64_t* h_rows, mm_stream_t stream);

/* Plan diagnostics (host only): proportions p4/p6/p8 (§3.1 Q2), average bits per
 * element incl. the 8-bit scale per 32 elements (Table 1 accounting, SPEC.md line
 * 392), stored bytes per row (128-padded segments + scale bytes), and -- when the
 * calibration channel maxima h_chmax[K] and the host permutation h_perm[K] are
 * given -- the Eq. 6 violations: channels placed in P4 (P6) by their mean whose
 * max exceeds T(4) (T(6)). */
typedef struct {
  double p[3];
  double avg_bits;
  int64_t stored_bytes_per_row;
  int32_t eq6_violations[2];
} mm_plan_diag;
mm_status mm_plan_diagnostics(const mm_plan* plan, const double* h_chmax, const int32_t* h_perm,
                              mm_plan_diag* out);

/* Offline weight transform (Fig. 1 caption line 20; line 151): W[N, K] BF16
 * (PyTorch Linear layout, K contiguous, ld = ldw) is reordered with the plan's
 * permutation and block-quantized along K into w_out (rows = N). */
mm_status mm_quantize_weight_offline(const void* d_w, int64_t N, int64_t ldw,
                                     const mm_plan* plan, mm_mx_tensor* w_out,
                                     mm_stream_t stream);

/* Online fused reorder-and-quantize (§3.2, Fig. 6): X[M, K] BF16 ->
 * a_out (rows = M).  Bit-exact with the oracle (codes, scales, padding). */
mm_status mm_reorder_quantize_act(const void* d_x, int64_t M, int64_t ldx,
                                  const mm_plan* plan, mm_mx_tensor* a_out,
                                  mm_stream_t stream);

/* RMSNorm fused into the online reorder-and-quantize (the paper's integration: one
 * RQ after each normalization layer, shared by the following linears, §3.2 / Fig. 7
 * lines 156-163).  Quantizes y = RMSNorm(X) * gamma, where for
 * every row ss = sum_j x_j^2 (exact), r = fp32(1 / sqrt(ss / K + eps)) (IEEE fp64),
 * t_j = bf16_rne(fp32(x_j * r)) and y_j = bf16_rne(fp32(gamma_j * t_j)) (the HF
 * LlamaRMSNorm data flow; reading R27) -- bit-exact with quantizing the
 * separately normalized BF16 rows.  d_gamma: device BF16[K] in the
 * ORIGINAL channel order, 16-byte aligned; eps > 0.  Saves the BF16 write and read of
 * the normalized activation. */
mm_status mm_rmsnorm_reorder_quantize_act(const void* d_x, int64_t M, int64_t ldx, const void* d_gamma, double eps,
                                          const mm_plan* plan, mm_mx_tensor* a_out, mm_stream_t stream);

/* Mixed block-scaled GEMM (§3.2, Eq. 2): Y[M, N] = A W^T over the three
 * K-segments, one FP32 accumulator, BF16 round-to-nearest-even output
 * (row-major, ld = ldy >= N, ldy % 8 == 0).  A and W must come from `plan`
 * (fingerprints equal) -- else MM_ERR_PLAN_MISMATCH.  N % 16 == 0.
 * Small M (<= 128 when the W tiles leave room for >= 2 K splits) runs the swap-AB /
 * split-K kernel: each K split keeps its own FP32 accumulator and the partials are
 * added in split order (deterministic; reading R28) inside the thread-block
 * cluster of the split CTAs (distributed shared memory; no workspace).  The opt-in
 * stream-K schedule's FP32 partials and flags live in the CALLER's workspace d_ws of
 * ws_bytes >= mm_gemm_workspace_bytes(plan, M, N) bytes:
 * 256-byte aligned, ZERO-FILLED once before its first use (the kernels leave every
 * counter at zero), reusable by later calls on the same stream, not shared by calls
 * in flight on different streams.  d_ws may be NULL when the query returns 0.
 * Errors: MM_ERR_WORKSPACE if the workspace is missing, misaligned or too small. */
mm_status mm_mixed_gemm_bf16(const mm_mx_tensor* a, const mm_mx_tensor* w,
                             const mm_plan* plan, void* d_y, int64_t ldy,
                             void* d_ws, size_t ws_bytes, mm_stream_t stream);

/* Workspace bytes mm_mixed_gemm_bf16 needs for an M x N output under the current
 * tile configuration (mm_set_gemm_config); 0 when the chosen kernel needs none;
 * -1 on an invalid plan or negative sizes.  Pure host function. */
int64_t mm_gemm_workspace_bytes(const mm_plan* plan, int64_t M, int64_t N);

/* Test entry: the reorder output x_r[m, j] = X[m, perm[j]] as BF16 [M, K]
 * (ld = ldxr), for bit-exact reorder parity.  Not on the hot path. */
mm_status mm_reorder_act_bf16(const void* d_x, int64_t M, int64_t ldx, const mm_plan* plan,
                              void* d_xr, int64_t ldxr, mm_stream_t stream);

/* GEMM tile configuration override for tuning (0 = automatic).  block_n: 128 or 256
 * = single-CTA 128 x block_n tiles, 512 = CTA-pair (cta_group::2) 256 x 256 tiles,
 * 1 = the small-M swap-AB / split-K kernel (M <= 128; auto for M <= 32);
 * num_stages: smem pipeline depth (kernel-specific set, 0 = default). */
mm_status mm_set_gemm_config(int32_t block_n, int32_t num_stages, int32_t max_ctas);

/* Kernel launches issued by this thread since the last reset (instrumentation). */
int64_t mm_launch_count(void);
void mm_reset_launch_count(void);

const char* mm_last_error(void);
int32_t mm_abi_version(void);

/* ---- multi-GPU N-sharding (BASELINE north star) ----
 * Each rank holds W rows [r*N/G, (r+1)*N/G) quantized with the shared plan and
 * computes Y_r = A W_r^T; the BF16 shards are all-gathered over NVLink with NCCL
 * and laid out as the full row-major Y[M, N] on every rank. */
int32_t mm_nccl_unique_id_bytes(void);                       /* 128 */
mm_status mm_nccl_get_unique_id(void* h_id_out);            /* rank 0 only */
mm_status mm_comm_init(int32_t rank, int32_t world, const void* h_unique_id, void** comm_out);
mm_status mm_comm_destroy(void* comm);
/* d_stage: caller scratch of stage_bytes >= 2*M*N bytes (BF16 [G][M][N/G]),
 * 16-byte aligned.  Y shard is computed into the stage slot of this rank,
 * all-gathered, then permuted into d_y_full [M, N] (ld = ldy, 16-byte aligned).
 * The shard GEMM uses no workspace (tile kernels only).  Errors
 * (MM_ERR_SHAPE / _ALIGNMENT / _WORKSPACE / _NCCL) are detected before anything is
 * enqueued. */
mm_status mm_mixed_gemm_bf16_nshard_allgather(const mm_mx_tensor* a, const mm_mx_tensor* w_shard,
                                              const mm_plan* plan, int64_t n_total,
                                              void* d_y_full, int64_t ldy, void* d_stage,
                                              size_t stage_bytes, void* comm, mm_stream_t stream);

/* ---- fused GEMM + all-gather epilogue over peer memory ----
 * The N-shard of mm_mixed_gemm_bf16_nshard_allgather without a separate
 * collective: every output tile of rank r is TMA-stored straight into EVERY
 * rank's full Y (columns [r*Ns, (r+1)*Ns)) through peer-mapped memory over
 * NVLink/NVSwitch, then a flag barrier tells each rank that all shards have
 * landed.  Results equal the 1-GPU GEMM bit for bit (same tiles, same K order).
 *
 * Peer buffer (one per rank, caller-allocated, 256-B aligned, ZERO-FILLED before
 * the handle exchange, e.g. torch.zeros): [Y: BF16 M x ldy, padded to 256 B]
 * [flags: 64 x u32; word 63 = barrier-timeout record].  mm_peer_buffer_bytes gives its size.
 *
 * Window: this rank's table of all ranks' buffers.  mm_peer_window_open maps the
 * peers' buffers from CUDA IPC handles (mm_ipc_get_handle on each rank, exchanged
 * by the caller, e.g. through torch.distributed); mm_peer_window_from_ptrs takes
 * device pointers valid in this process (already-mapped memory, or several
 * "virtual ranks" on one GPU for testing).  world <= 8.  The window owns the IPC
 * mappings it opened; mm_peer_window_close unmaps them (buffers stay the caller's).
 *
 * mm_mixed_gemm_bf16_nshard_peerstore: a = this rank's (replicated) activation,
 * w_shard = its Ns = n_total / world weight rows, Ns % 16 == 0, ldy >= n_total,
 * ldy % 8 == 0.  barrier = 1 appends the flag barrier on `stream` (the call then
 * completes on every rank only when all ranks have called it: a collective);
 * barrier = 0 leaves it to mm_peer_barrier (same-process virtual ranks, where the
 * barriers of all ranks must run concurrently on different streams).  Y reuse: peers
 * write into this rank's Y as soon as they reach the call, so a rank that still reads
 * its previous Y must separate iterations with mm_peer_barrier (or alternate two
 * windows).  Errors as everywhere: validated before any launch, nothing enqueued on
 * error. */
size_t mm_peer_buffer_bytes(int64_t M, int64_t ldy);
int32_t mm_ipc_handle_bytes(void);                                   /* 72 */
mm_status mm_ipc_get_handle(const void* d_buf, void* h_handle_out);   /* 64 B CUDA IPC handle of the
                                                                          allocation + u64 byte offset */
mm_status mm_peer_window_open(int32_t rank, int32_t world, void* d_local_buf, const void* h_handles,
                              int64_t M, int64_t ldy, void** win_out);
mm_status mm_peer_window_from_ptrs(int32_t rank, int32_t world, void* const* h_dev_bufs, int64_t M,
                                   int64_t ldy, void** win_out);
mm_status mm_peer_window_close(void* win);   /* no queued work may still use the window, on
                                                any rank (e.g. close after a final barrier) */
mm_status mm_mixed_gemm_bf16_nshard_peerstore(const mm_mx_tensor* a, const mm_mx_tensor* w_shard,
                                              const mm_plan* plan, int64_t n_total, void* win,
                                              int32_t barrier, mm_stream_t stream);
mm_status mm_peer_barrier(void* win, mm_stream_t stream);
/* ---- fused all-gather over NVLS / NVLink SHARP (multicast) ----
 * One multicast object spans every rank's buffer ([Y: BF16 M x ldy, padded to 256 B]
 * [flags: 64 x u32], the peer-buffer layout); the CTA-pair GEMM epilogue writes each
 * output element ONCE with multimem.st and the switch replicates it to all ranks
 * (per-GPU egress M*Ns*2 bytes instead of (G-1)*M*Ns*2).  Setup is collective, in two
 * halves separated by a barrier of the caller's process group:
 *   1. mm_mc_window_create on every rank: rank 0 creates the object and writes its
 *      shareable handle (mm_mc_handle_bytes() bytes: a fabric handle, else a POSIX fd
 *      that the peers duplicate with pidfd_getfd) into h_handle; the caller broadcasts
 *      those bytes and the other ranks pass them in; every rank adds its device.
 *   2. (barrier) mm_mc_window_bind on every rank: allocates this rank's buffer with the
 *      driver's virtual-memory API, binds it, maps the multicast and the local views and
 *      zeroes the buffer; (barrier) before the first GEMM.
 * mm_mc_window_local returns this rank's buffer (read Y there).  world <= 8; world 1 is
 * allowed (a one-device multicast object, for testing).  mm_mc_supported() reports
 * whether this device can create multicast objects (attribute + a one-time probe: GPUs
 * not attached to an NVSwitch fabric reject cuMulticastCreate).  Barrier: every rank adds 1 to flag word 0 of all ranks through the
 * multicast view (multimem.red.release.sys) and waits for its own copy to reach
 * world * epoch; with a timeout (mm_mc_window_set_timeout, default off) a barrier that
 * gives up writes 0xFFFF into flag word 63, reported by mm_mc_window_error.
 * mm_mixed_gemm_bf16_nshard_nvls: as mm_mixed_gemm_bf16_nshard_peerstore. */
int32_t mm_mc_supported(void);
int32_t mm_mc_handle_bytes(void);
mm_status mm_mc_window_create(int32_t rank, int32_t world, int64_t M, int64_t ldy, void* h_handle, void** win_out);
mm_status mm_mc_window_bind(void* win);
void* mm_mc_window_local(void* win);
mm_status mm_mc_window_set_timeout(void* win, double seconds);
mm_status mm_mc_window_error(void* win, int32_t* h_timed_out);   /* synchronous; 1 if a barrier gave up */
mm_status mm_mc_window_close(void* win);
mm_status mm_mc_barrier(void* win, mm_stream_t stream);
mm_status mm_mixed_gemm_bf16_nshard_nvls(const mm_mx_tensor* a, const mm_mx_tensor* w_shard, const mm_plan* plan,
                                         int64_t n_total, void* win, int32_t barrier, mm_stream_t stream);

/* Barrier timeout of a window (default 0 = wait forever, like NCCL: a slow rank is
 * not an error).  With a timeout, a barrier whose peer never arrives gives up, and
 * records the missing rank in this rank's buffer instead of trapping (the CUDA
 * context stays usable); mm_peer_window_error (synchronous read, call after the
 * stream completed) returns it in *h_missing_rank, or -1 if every barrier completed. */
mm_status mm_peer_window_set_timeout(void* win, double seconds);
mm_status mm_peer_window_error(void* win, int32_t* h_missing_rank);

#ifdef __cplusplus
}
#endif
#endif /* MICROMIX_B200_MM_H */
