/* isnmf_b200.h — C ABI of the B200-native online / batch Itakura-Saito NMF
 * engine (sm_100a).  This is the drop-in boundary: the C++ API in
 * include/isnmf/ headers (same names and signatures as the reference's
 * proj/include/isnmf) is a thin header-only layer over these entry points,
 * and a cgo / JNI / ctypes binding would bind exactly these symbols
 * (INTEGRATION.md).
 *
 * Conventions
 *  - Plain pointers and sizes; no torch / CUDA types in any signature.
 *  - Host matrices are column-major fp64 (the reference's Eigen::MatrixXd
 *    layout, proj/include/isnmf/matrix.hpp:14-16) unless the name says f32.
 *  - Frames (spectrogram columns) for the hot path are fp32, F contiguous
 *    values per frame with a leading dimension `ldv` (>= F).
 *  - Every call returns ISNMF_OK (0) or an isnmf_status; the message of the
 *    calling thread's last failure is isnmf_last_error().  The codes map 1:1
 *    onto the reference's exception types (proj/include/isnmf/errors.hpp:9-90).
 *  - The engine computes in fp32 on the device (accumulations of the
 *    objective and of the A/B statistics in fp64); results match the
 *    reference's fp64 arithmetic to ~1e-5 relative (tests state 1e-4).
 *  - A context is single-writer: do not call into the same context from two
 *    threads at once (the reference is single-threaded too).
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry fails with ISNMF_E_CUDA.
 */
#ifndef ISNMF_B200_H
#define ISNMF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum isnmf_status {
  ISNMF_OK = 0,
  ISNMF_E_SHAPE_MISMATCH = 1,     /* ShapeMismatch     errors.hpp:61-63 */
  ISNMF_E_EMPTY_DATASET = 2,      /* EmptyDataset      errors.hpp:57-59 */
  ISNMF_E_NEGATIVE_INPUT = 3,     /* NegativeInput     errors.hpp:67-69 */
  ISNMF_E_NON_POSITIVE_INIT = 4,  /* NonPositiveInit   errors.hpp:75-77 */
  ISNMF_E_ZERO_COLUMN = 5,        /* ZeroColumn        errors.hpp:71-73 */
  ISNMF_E_INCONSISTENT_STATS = 6, /* InconsistentStats errors.hpp:79-81 */
  ISNMF_E_NUMERICAL_FAILURE = 7,  /* NumericalFailure  errors.hpp:88-90 */
  ISNMF_E_DIVERGED_OBJECTIVE = 8, /* DivergedObjective errors.hpp:83-85 */
  ISNMF_E_NON_FINITE_ENTRY = 9,   /* NonFiniteEntry    errors.hpp:37-39 */
  ISNMF_E_NEGATIVE_ENTRY = 10,    /* NegativeEntry     errors.hpp:41-43 */
  ISNMF_E_IO = 11,                /* IoError           errors.hpp:25-27 */
  ISNMF_E_UNSUPPORTED_FORMAT = 12, /* UnsupportedFormat errors.hpp:45-47 */
  ISNMF_E_TOO_SHORT = 13,         /* TooShort          errors.hpp:49-51 */
  ISNMF_E_ALL_SILENT = 14,        /* AllSilent         errors.hpp:53-55 */
  ISNMF_E_CUDA = 20,              /* device / driver failure (no reference equivalent) */
  ISNMF_E_INVALID_ARG = 21,       /* bad pointer / size at the C boundary */
  ISNMF_E_UNSUPPORTED = 22        /* shape outside the built kernel family */
} isnmf_status;

/* Restart modes (model.hpp:20-30). */
enum { ISNMF_RESTART_WARM = 0, ISNMF_RESTART_FRESH = 1 };
/* Engine flags: force the generic (W-streaming) solve kernel even when a
 * register-tiled variant would fit (testing / comparison). */
/* solver selection: GENERIC_SOLVE = the shape-generic FP32 kernel; NO_PAIR = never the
 * 2-SM tcgen05 kernel K1C (K1M instead); PAIR = K1C at any mini-batch size it supports */
enum { ISNMF_FLAG_GENERIC_SOLVE = 1, ISNMF_FLAG_NO_PAIR = 2, ISNMF_FLAG_PAIR = 4 };

const char* isnmf_last_error(void);
/* Library / device description: writes a short JSON string. */
int isnmf_device_info(char* buf, int64_t cap);

/* ---------------------------------------------------------------------------
 * Stateless numerical kernels — kernels.hpp:30-159 and model.hpp:73-86.
 * Host fp64 in/out, device fp32 compute.
 * ------------------------------------------------------------------------- */

/* is_divergence (kernels.hpp:30-40): sum_i is_term((y_i-x_i)/(eps+x_i)). */
int isnmf_is_divergence(const double* y, int64_t ny, const double* x, int64_t nx, double epsilon, double* out);

/* objective (kernels.hpp:43-55): (1/N) sum_n d_IS(eps+v_n, eps+W h_n).
 * v F x N, w F x K, h K x N. */
int isnmf_objective(const double* v, const double* w, const double* h, int64_t F, int64_t K, int64_t N,
                    double epsilon, double* out);

/* solve_h (kernels.hpp:62-80), batched: every column n of v (F x N) is solved
 * independently from h0[:, n] (K x N) with `iters` MM iterations at fixed W. */
int isnmf_solve_h(const double* v, const double* w, const double* h0, int64_t F, int64_t K, int64_t N, int iters,
                  double epsilon, double* h_out);

/* sample_stats (kernels.hpp:112-121) summed over the N columns, which is
 * batch_stats (kernels.hpp:125-137): a = ((v+e)/(e+WH)^2 H^T) .* W^2,
 * b = (1/(e+WH)) H^T.  a, b: F x K. */
int isnmf_batch_stats(const double* v, const double* w, const double* h, int64_t F, int64_t K, int64_t N,
                      double epsilon, double* a_out, double* b_out);

/* update_w (kernels.hpp:142-159): W = sqrt(A/B); A=B=0 keeps w_prev;
 * A>0 with B=0 -> ISNMF_E_INCONSISTENT_STATS. */
int isnmf_update_w(const double* a, const double* b, const double* w_prev, int64_t F, int64_t K, double* w_out);

/* rescale_dictionary (model.hpp:73-86), in place; warm_h (K x N) optional. */
int isnmf_rescale_dictionary(double* w, double* a, double* b, int64_t F, int64_t K, double* warm_h, int64_t N);

/* ---------------------------------------------------------------------------
 * Online engine — the state behind OnlineState (online.hpp:224-248) lives on
 * the device; these calls implement make_online_state / online_step /
 * dictionary_commit / online_resume (online.hpp:254-419).
 * ------------------------------------------------------------------------- */
typedef struct isnmf_online isnmf_online;

typedef struct isnmf_online_config {
  int64_t F;             /* frame length (rows of W) */
  int64_t K;             /* atoms, SolverConfig::k */
  int32_t beta;          /* mini-batch size, SolverConfig::beta */
  int32_t inner_iters;   /* effective H iterations per visit (>= 1) */
  double epsilon;        /* SolverConfig::epsilon */
  int32_t restart;       /* ISNMF_RESTART_WARM / ISNMF_RESTART_FRESH */
  int32_t flags;         /* ISNMF_FLAG_* */
  uint64_t seed;         /* SolverConfig::seed (fresh-restart stream) */
  int64_t n_store;       /* warm mode: columns of the activation store (dataset size) */
  int64_t max_chunk;     /* frames per H2D chunk when streaming host frames (0 = 64*beta) */
} isnmf_online_config;

int isnmf_online_create(isnmf_online** out, const isnmf_online_config* cfg);
int isnmf_online_destroy(isnmf_online* ctx);

/* Whole-state set / get (fp64 F x K column-major; NULL skips a field). */
int isnmf_online_set_dictionary(isnmf_online* ctx, const double* w, const double* a, const double* b);
int isnmf_online_get_dictionary(isnmf_online* ctx, double* w, double* a, double* b);
int isnmf_online_set_pending(isnmf_online* ctx, const double* pending_a, const double* pending_b, double pending_div,
                             uint64_t pending_count);
int isnmf_online_get_pending(isnmf_online* ctx, double* pending_a, double* pending_b, double* pending_div,
                             uint64_t* pending_count);
/* t, commits, rho (online.hpp:226-234). */
int isnmf_online_set_counters(isnmf_online* ctx, uint64_t t, uint64_t commits, double rho);
/* t, commits, rho, last_delta, last_minibatch_obj. */
int isnmf_online_get_counters(isnmf_online* ctx, uint64_t* t, uint64_t* commits, double* rho, double* last_delta,
                              double* last_minibatch_obj);
/* Warm activation store (K x n_store).  fill sets every entry to `value`. */
int isnmf_online_set_warm_h(isnmf_online* ctx, const double* warm_h);
int isnmf_online_fill_warm_h(isnmf_online* ctx, double value);
int isnmf_online_get_warm_h(isnmf_online* ctx, double* warm_h);

/* Runs online_step (online.hpp:342-368) over n frames in order, committing
 * every beta samples (dictionary_commit, online.hpp:318-337).
 *   frames   fp32, frame j at frames + j*ldv (host or device memory: the
 *            engine detects which; host frames are streamed in chunks on a
 *            copy stream, double-buffered against compute)
 *   index    dataset index of each frame (warm store column); NULL = identity
 *            order cycling over the store: column (t + j) mod n_store
 *   budget   stop when t reaches it (max_epochs_or_samples)
 *   eta      stop at the first commit whose ||W_t - W_{t-beta}||_F < eta (0 = off)
 * Returns after the device finished (trace / counters readable).  *stopped is
 * set to 1 when the eta rule fired. */
int isnmf_online_run(isnmf_online* ctx, const float* frames, int64_t ldv, int64_t n, const uint64_t* index,
                     uint64_t budget, double eta, int32_t* stopped);

/* Asynchronous variant for pipelines: enqueues the same work, does not wait. */
int isnmf_online_enqueue(isnmf_online* ctx, const float* frames, int64_t ldv, int64_t n, const uint64_t* index,
                         uint64_t budget, double eta);
int isnmf_online_synchronize(isnmf_online* ctx);

/* dictionary_commit (online.hpp:318-337) now, whatever t % beta is: folds the
 * pending statistics into A, B, refreshes and renormalises W. */
int isnmf_online_commit(isnmf_online* ctx);

/* Page-locked host staging memory (so frame uploads overlap compute). */
void* isnmf_host_alloc(int64_t bytes);
void isnmf_host_free(void* p);

/* Trace points recorded at each commit since the last clear: samples seen,
 * mini-batch objective (last_minibatch_obj) and device timestamp (seconds
 * since the context's clock origin). */
int isnmf_online_get_trace(isnmf_online* ctx, uint64_t* samples, double* train_obj, double* seconds, int64_t cap,
                           int64_t* n);
int isnmf_online_clear_trace(isnmf_online* ctx);

/* Last H solved for each frame of the most recent run (K x n, fp64) —
 * test hook for per-mini-batch state-injection parity. */
int isnmf_online_get_last_h(isnmf_online* ctx, double* h, int64_t n);

/* Number of engine kernel launches issued so far (bench accounting). */
int64_t isnmf_online_launch_count(isnmf_online* ctx);
/* Name of the mini-batch solve kernel the context runs ("K1C", "K1M", "K1", "K1L", "K1T",
 * "generic"), NUL-terminated into buf. */
int isnmf_online_solver(isnmf_online* ctx, char* buf, int64_t cap);

/* Profiling: begin() records a CUDA event on the engine's compute stream; with
 * per_kernel != 0 events are also recorded around every K1 (solve) and K2
 * (fold/commit) launch (they add ~2 us per mini-batch).  end() records the
 * closing event, waits for the stream and returns the summed K1 device time,
 * the K1 launch and frame counts, the device time of the whole region on that
 * stream and the summed K2 time (the per-kernel values are 0 without per_kernel). */
int isnmf_online_profile_begin(isnmf_online* ctx, int32_t per_kernel);
int isnmf_online_profile_end(isnmf_online* ctx, double* solve_ms, int64_t* solve_launches, int64_t* solve_frames,
                             double* span_ms, double* tail_ms);

/* ---------------------------------------------------------------------------
 * Batch engine — batch_train (batch.hpp:84-143): per epoch one MM pass over H,
 * fresh statistics, W = sqrt(A/B), l1 rescale (H rows compensated), objective.
 * v: fp32 frames as above (host or device); w0 F x K, h0 K x N fp64.
 * obj_trace receives the objective after each epoch (length >= max_epochs).
 * ------------------------------------------------------------------------- */
int isnmf_batch_train(const float* v, int64_t ldv, int64_t F, int64_t N, int64_t K, const double* w0,
                      const double* h0, uint64_t max_epochs, double epsilon, double eta, double* w_out,
                      double* h_out, double* obj_trace, uint64_t* epochs, double* initial_obj, double* last_delta);

/* Profiling (not part of the reference interface): enable >= 0 switches CUDA-event
 * timing of isnmf_batch_train on (1) or off (0); -1 leaves it.  Returns the device
 * time of the last timed call (its enqueued epochs and final objective pass, without
 * the V / H transfers) and how many engine kernels it launched. */
int isnmf_batch_profile(int32_t enable, double* device_ms, int64_t* launches);

/* ---------------------------------------------------------------------------
 * Held-out fit — evaluate_heldout (harness.hpp:17-37): H from the reference's
 * seed-deterministic uniform stream scaled by max(mean test, eps)/(K mean W),
 * inner_iters MM updates at frozen W (the fused solve kernel, no statistics),
 * then the mean IS divergence per frame.  test: F x N fp32 with leading
 * dimension ldt (host or device); w: F x K fp64.  W is not modified.
 * ------------------------------------------------------------------------- */
int isnmf_evaluate_heldout(const float* test, int64_t ldt, int64_t F, int64_t N, const double* w, int64_t K,
                           double epsilon, int32_t inner_iters, uint64_t seed, double* out);

/* ---------------------------------------------------------------------------
 * Spectrogram front end (audio.hpp:121-187).
 * isnmf_stft_power: sine-windowed one-sided power spectrum of `samples` (fp64,
 * host), frame i = samples [i*hop, i*hop + window); power is window/2+1 bins x
 * frames, column-major fp64, frames = (n_samples - window)/hop + 1.  Windows
 * that are powers of two use an in-shared-memory radix-2 FFT, others a direct
 * DFT; both in fp64 on the device.  Errors: UnsupportedFormat (window odd or
 * < 2, hop outside [1, window]), TooShort (signal shorter than one window).
 * isnmf_discard_silence: indices (ascending) of the frames whose total power is
 * at least max * 10^(threshold_db/10); spec is bins x frames fp64 (host or
 * device).  Errors: AllSilent.
 * ------------------------------------------------------------------------- */
int isnmf_stft_power(const double* samples, int64_t n_samples, int32_t window, int32_t hop, double* power,
                     int64_t frames_cap, int64_t* frames);
int isnmf_discard_silence(const double* spec, int64_t bins, int64_t frames, double threshold_db, int64_t* keep,
                          int64_t* n_keep);

#ifdef __cplusplus
}
#endif
#endif /* ISNMF_B200_H */
