/*
 * qcldpc_b200.h -- C ABI of the B200-native layered BP decoder for QC-MET-LDPC codes.
 *
 * Plain pointers and sizes only; no torch or CUDA types cross this boundary.
 * The reference (/root/reference/pkg/src/qcldpc) is pure Python with no FFI, so
 * each entry point below names the Python interface it replaces; the Python
 * package paper_2004_09084_b200 binds them with ctypes (see INTEGRATION.md for
 * the binding a maintainer of the reference would add).
 *
 * Conventions
 *   - Every function returns QCL_OK (0) or a negative error class; the
 *     thread-local message is available from qcl_last_error().
 *     QCL_EVALUE  -> the reference raises ValueError (same message text)
 *     QCL_ECUDA   -> CUDA runtime failure (Python RuntimeError)
 *     QCL_EUNSUP  -> a shape this build does not handle (RuntimeError)
 *   - Host arrays use the reference layouts (decoder.py:79-83,168-170,275-312):
 *       llr / posterior   (B, n)             n = n_cols * z, row-major
 *       edge messages     (B, total_edges*z) slot-ordered, [edge][k]
 *       syndrome          (B, m) uint8       m = n_rows * z, ORIGINAL check order row*z+k
 *       words             (B, n) uint8
 *   - Plans are immutable after creation and may be shared by host threads;
 *     a qcl_state belongs to one host thread at a time (decoder.py:18-21).
 *   - All device work of a state runs on that state's own CUDA stream.
 */
#ifndef QCLDPC_B200_H
#define QCLDPC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QCL_OK 0
#define QCL_EVALUE (-1)
#define QCL_ECUDA (-2)
#define QCL_EUNSUP (-3)

#define QCL_PREC_FP32 0 /* performance path: FP32 state, exclusive Phi-sums */
#define QCL_PREC_FP64 1 /* parity path: FP64 state, reference formula and fold order */
/* Beyond-parity opt-in: FP32 posteriors, FP16 edge messages (|r| rounded
 * to FP16 before use: 12 instead of 16 bytes per edge and iteration).  Flow engine only
 * (engine 4/6, whole sweeps); decisions are NOT bit-identical to FP32/FP64. */
#define QCL_PREC_FP32_MSG16 2

#define QCL_DTYPE_F64 0
#define QCL_DTYPE_F32 1

typedef struct qcl_plan qcl_plan;
typedef struct qcl_state qcl_state;

/* DecoderConfig (decoder.py:48-63) plus the precision switch. */
typedef struct {
    int32_t max_iterations;    /* >= 1 */
    int32_t early_termination; /* 0/1 */
    double llr_clip;           /* > 0 */
    double phi_epsilon;        /* (0, 1) */
    int32_t precision;         /* QCL_PREC_* */
} qcl_config;

int32_t qcl_abi_version(void);
const char *qcl_last_error(void);
int qcl_device_count(int32_t *count);

/* LayeredDecoder.__init__ (decoder.py:117-189) given build_compact_index output
 * (qc_code.py:249-279): validates the schedule/index match (decoder.py:118-120)
 * and in-layer column disjointness (decoder.py:144-154), then uploads the packed
 * H_compact1 table (per-edge column base + shift, per-slot offset/degree/row,
 * per-layer slot range) to `device`.
 *   edge_shift/edge_col   [n_edges]      EdgeRecord.shift / .base_col
 *   slot_offsets          [n_slots + 1]  CompactIndex.slot_offsets
 *   slot_rows             [n_slots]      CompactIndex.slot_rows
 *   layer_slot_starts     [n_layers + 1] cumulative layer sizes of the schedule
 *   schedule_rows         [n_slots]      concatenated schedule layers (for the match check) */
int qcl_plan_create(int32_t z, int32_t n_cols, int32_t n_slots, int32_t n_layers, int32_t n_edges,
                    const int32_t *edge_shift, const int32_t *edge_col, const int32_t *slot_offsets,
                    const int32_t *slot_rows, const int32_t *layer_slot_starts,
                    const int32_t *schedule_rows, int32_t device, qcl_plan **out);
int qcl_plan_destroy(qcl_plan *plan);
/* n, m, total expanded edges, layers, max row degree */
int qcl_plan_info(const qcl_plan *plan, int64_t *n_vars, int64_t *n_checks, int64_t *n_edges_expanded,
                  int32_t *n_layers, int32_t *max_degree);

/* LayeredDecoder.decode_batch_arrays (decoder.py:275-312): one-shot host-buffer decode.
 * llr0 is (B, n) float64 (QCL_DTYPE_F64) or float32 (QCL_DTYPE_F32); syndrome may be
 * NULL (all-zero target).  Outputs: words (B, n), converged (B), iterations (B).
 * Every host buffer may be pageable (the reference's numpy arrays) or pinned
 * (qcl_host_alloc): pageable ones go through a pinned-chunk pipeline driven by host
 * threads (float64 LLRs converted to float32 there for the FP32 paths); an all-zero
 * syndrome is detected on the host and not copied.  Every entry point of this header runs
 * on its plan's device and restores the calling thread's current device on return. */
int qcl_decode(qcl_plan *plan, const qcl_config *cfg, const void *llr0, int32_t llr_dtype,
               const uint8_t *syndrome, int64_t batch, uint8_t *words, uint8_t *converged,
               int64_t *iterations);

/* ---- device-resident state (DecoderState, decoder.py:75-93) ---------------- */
int qcl_state_create(qcl_plan *plan, int64_t batch, int32_t precision, qcl_state **out);
int qcl_state_destroy(qcl_state *st);
/* Channel LLRs from host (B, n) -> device input buffer (channel.py:54-56 output).  A
 * pageable llr0 is staged before the call returns (the caller may reuse it at once); a
 * pinned one is read asynchronously on the state's stream. */
int qcl_state_set_llr(qcl_state *st, const void *llr0, int32_t llr_dtype);
/* Device BIAWGN generator (replaces channel.py:36-56 on the hot path): frame b of the
 * state is frame (first_frame + b) of the Philox4x32-10 stream keyed by (seed, snr_idx).
 * encode_mode draws a random word per frame and sets the target syndrome to H*word
 * (bench.py:216-228); otherwise the all-zero word / zero syndrome. */
int qcl_state_set_llr_synthetic(qcl_state *st, uint64_t seed, int64_t snr_idx, int64_t first_frame,
                                double snr, int32_t encode_mode);
/* Target syndrome (B, m) original order; NULL = all-zero. */
int qcl_state_set_syndrome(qcl_state *st, const uint8_t *syndrome);
/* new_state (decoder.py:191-202): posterior = clip(llr), messages = 0. */
int qcl_state_reset(qcl_state *st, double llr_clip);
/* Overwrite the device state from reference-layout host arrays (messages may be NULL = 0). */
int qcl_state_upload(qcl_state *st, const double *posterior, const double *messages);
int qcl_state_download(qcl_state *st, double *posterior, double *messages);
/* layer_update (decoder.py:252-257) for layers [first, first + count), in order. */
int qcl_state_layers(qcl_state *st, int32_t first, int32_t count, double llr_clip, double phi_epsilon);
/* hard_decision (decoder.py:264-266) -> (B, n) */
int qcl_state_hard_decision(qcl_state *st, uint8_t *words);
/* syndrome_satisfied (decoder.py:268-273) of the current posterior signs -> (B) */
int qcl_state_syndrome_ok(qcl_state *st, uint8_t *ok);
/* Full decode (decoder.py:275-312) from the state's LLR buffer and syndrome; results stay
 * on the device until qcl_state_results.  elapsed_ms (may be NULL) receives the CUDA-event
 * time of the decode on the state's stream. */
int qcl_state_decode(qcl_state *st, const qcl_config *cfg, float *elapsed_ms);
int qcl_state_results(qcl_state *st, uint8_t *words, uint8_t *converged, int64_t *iterations);
/* The transmitted words of the last synthetic encode-mode fill, (B, n). */
int qcl_state_truths(qcl_state *st, uint8_t *words);
/* Frame pool: n_frames device-generated BIAWGN frames (Philox keyed by (seed, snr_idx,
 * frame), all-zero word, zero syndrome) streamed through the state's lanes with early
 * termination: a lane whose frame converged or hit max_iterations records the outcome at
 * its frame index and takes the next frame.  Per-frame outcomes equal the batch decode's;
 * conv/err are (n_frames) bytes, iters (n_frames) int64; err = frame error (bench.py:236-237).
 * Flow engine only (FP32). */
int qcl_state_decode_pool(qcl_state *st, const qcl_config *cfg, uint64_t seed, int64_t snr_idx, int64_t first_frame,
                          int64_t n_frames, double snr, uint8_t *conv, int64_t *iters, uint8_t *err,
                          float *elapsed_ms);
/* Campaign frame errors (reference bench.py:236-237): mismatch[b] = 1 when the decoded
 * word of frame b (after qcl_state_decode) differs from its transmitted word -- the
 * encode-mode truths of the last synthetic fill, else the all-zero word.  (B) bytes. */
int qcl_state_frame_errors(qcl_state *st, uint8_t *mismatch);
/* Copy the state's device LLR buffer back as float64 (B, n) (tests of the generator). */
int qcl_state_get_llr(qcl_state *st, double *llr);
/* Lanes per group (W) of the state's layout, and whether its decodes run on the flow
 * engine (FP32 or FP16 messages, row degree <= 12, W >= 4, tables fit in shared memory);
 * the frame pool (qcl_state_decode_pool) and FP16 messages need it. */
int qcl_state_info(qcl_state *st, int32_t *lanes, int32_t *flow_engine);
/* Device-time breakdown of the last qcl_state_decode: number of layer-kernel launches and
 * their summed CUDA-event time (ms); used by bench.py's roofline. */
int qcl_state_kernel_stats(qcl_state *st, int64_t *layer_launches, float *layer_ms, int64_t *all_launches);
/* Select the layer-update engine: 4 = flow engine (default: one persistent launch per
 * decode, tiles ordered by completion flags; FP32, row degree <= 12, >= 4 lanes -- other
 * cases and single-layer calls use engine 0), 0 = TMA-pipelined per-layer kernels,
 * 1 = direct register-staged kernels; 2 / 3 / 6 = engine 0 / 1 / 4 with CUDA events
 * around every sweep or flow launch (read by qcl_state_kernel_stats).  FP64 single-codeword
 * and FP32 two-codeword decodes on engine 0 / 4 (lane rows narrower than 16 bytes) run
 * every sweep in one cooperative launch of the direct-kernel arithmetic with grid barriers
 * between layers (QCL_PERSIST=0: one launch per layer, 2: also one FP32 codeword);
 * engine 1 keeps the per-layer launches. */
int qcl_state_set_engine(qcl_state *st, int32_t engine);

/* ---- asynchronous path (streaming / overlapped host<->device copies) ---------------
 * Everything below only enqueues work on the state's stream; qcl_state_wait blocks until
 * all of it has completed (the results requested by qcl_state_results_async have landed;
 * decode_ms: the last decode's device time, 0 if none was queued).  Result buffers should
 * be pinned (qcl_host_alloc) for the copies to overlap device work; pageable LLR inputs
 * are converted and staged through pinned chunks by host threads before the call returns
 * (the caller may reuse them at once), pinned ones are read asynchronously.
 * qcl_state_set_syndrome_hint: the caller states whether the (B, m) target is nonzero
 * (nonzero = 0 or syndrome = NULL: all-zero target, nothing is copied; nonzero < 0: the
 * library checks on the host threads).
 * qcl_state_decode_async: the decode of qcl_state_decode without host synchronisation;
 * with early termination every layer launch after the last convergence returns at once. */
int qcl_state_set_syndrome_hint(qcl_state *st, const uint8_t *syndrome, int32_t nonzero);
int qcl_state_decode_async(qcl_state *st, const qcl_config *cfg);
int qcl_state_results_async(qcl_state *st, uint8_t *words, uint8_t *converged, int64_t *iterations);
int qcl_state_wait(qcl_state *st, float *decode_ms);
int qcl_host_alloc(int64_t bytes, void **out);
int qcl_host_free(void *ptr);

/* phi (decoder.py:96-105) evaluated by the device kernels' own Phi. */
int qcl_phi(const double *x, int64_t n, double phi_epsilon, double llr_clip, int32_t precision,
            int32_t device, double *out);

#ifdef __cplusplus
}
#endif
#endif
