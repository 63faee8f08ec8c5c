/*
 * surrogate.h — C ABI of the B200 (sm_100a) exhaustive FCNN-surrogate sweep.
 *
 * The method (arxiv 2306.14011): a fully connected ReLU network predicts the
 * solver runtime of a SENSEI configuration from its 14 OpenACC scheduling
 * parameters (7 kernels x {gang, vector}, Table "Tuning
 * Parameters" PAPER.md:253-266), after StandardScaler feature scaling
 * (PAPER.md:271-273).  The paper only says the trained model "identifies
 * configurations with the lowest runtime"; this library does
 * that exhaustively: every flat index of the space is mixed-radix decoded,
 * normalised, pushed through the network on tcgen05 tensor cores and reduced
 * to the k fastest predicted configurations.
 *
 * Conventions (all entry points):
 *  - Every call returns surr_status; nothing throws across the ABI.  On error
 *    no output is written and surrogate_last_error() holds the reason.
 *  - Arguments are validated before any launch.
 *  - Input descriptors (surr_space, surr_model and the arrays they point to)
 *    are HOST memory owned by the caller and copied during the call.
 *  - Outputs named *_dev are caller-allocated DEVICE buffers on the handle's
 *    device; *_host outputs are host memory.  Calls taking `stream` (a
 *    cudaStream_t, NULL = legacy default stream) are stream-ordered and
 *    asynchronous unless the name says _host.
 *  - A handle is not thread-safe; distinct handles are independent.  The
 *    handle's device scratch (per-CTA records, the ensemble accumulator) is
 *    shared by its calls, so calls on DIFFERENT streams of one handle must
 *    not overlap in time (calls on one stream are ordered; use one handle
 *    per concurrent stream).
 *  - There is no CPU fallback: without an sm_100 device every call that needs
 *    the GPU returns SURR_E_NO_DEVICE.
 */
#ifndef PAPER_2306_14011_SURROGATE_H
#define PAPER_2306_14011_SURROGATE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct surrogate surrogate_t; /* opaque; owns every device buffer it allocates */

typedef enum {
  SURR_OK = 0,
  SURR_E_INVALID_ARG = 1, /* null pointer, bad shape, k == 0 or k > SURR_K_MAX, begin > end ... */
  SURR_E_RANGE = 2,       /* |S| >= 2^64, or an index split the decoder cannot represent */
  SURR_E_NO_DEVICE = 3,   /* no CUDA device, or the device is not sm_100 */
  SURR_E_CUDA = 4,        /* a CUDA runtime error (text in surrogate_last_error) */
  SURR_E_OOM = 5,         /* device or pinned-host allocation failed */
  SURR_E_NOT_LOADED = 6,  /* no model loaded on this handle */
  SURR_E_UNSUPPORTED = 7  /* shape outside the kernel envelope (widths, layers, params) */
} surr_status;

/* Arithmetic of the hidden layers.  The final H -> 1 layer and the
 * de-standardisation always run in FP32 on CUDA cores. */
typedef enum {
  SURR_PREC_BF16 = 0, /* BF16 operands, FP32 accumulate (tcgen05 kind::f16) */
  SURR_PREC_FP32 = 1, /* "FP32 path" (1e-5): 3xFP16 split hi*hi + lo*hi + hi*lo on kind::f16
                         (hi = fp16(x), lo = fp16(x - hi): 22 significant bits), FP32 accumulate */
  SURR_PREC_TF32 = 2, /* 1xTF32 hidden layers, 3xTF32 first layer */
  SURR_PREC_FP16 = 3, /* IEEE FP16 operands, FP32 accumulate (kind::f16): BF16's tensor rate with
                         11 significant bits instead of 8 (activations must stay below 65504) */
  SURR_PREC_FP32_3XTF32 = 4 /* the FP32 path forced onto the 3xTF32 split */
} surr_precision;

#define SURR_K_MAX 1024u        /* largest top-k */
#define SURR_MAX_PARAMS 30u     /* tuning parameters per config (paper: 14) */
#define SURR_MAX_HIDDEN_LAYERS 4u

/* Search-space descriptor (Table "Tuning Parameters").
 * Flat index I = sum_j d_j * prod_{l>j} r_l with parameter 0 most significant
 * (lexicographic order of value indices).  [begin, end) selects a
 * sub-range; end == 0 means |S|.  */
typedef struct {
  uint32_t num_params;  /* P, 1..SURR_MAX_PARAMS */
  const uint32_t *radix; /* [P] value-list lengths r_j >= 1 */
  const double *values;  /* concatenated value lists, sum_j r_j entries, list j strictly increasing */
  uint64_t begin, end;   /* index sub-range; end == 0 -> |S| */
} surr_space;

/* A trained FCNN, or an ensemble of E members with
 * identical widths whose predictions are averaged in seconds.
 * widths[0] = F = P + num_const_features, widths[1..L-1] = hidden width H
 * (all equal), widths[L] = 1.  W[e*L + l] is row-major fan_in x fan_out,
 * b[e*L + l] has fan_out entries.  The input transform is
 * z = (x - x_shift) / x_scale (StandardScaler: shift = mean, scale = population
 * std; min-max: shift = min, scale = max - min);
 * x_scale == 0 is treated as 1.  The output is t = y_mean + y_scale * yhat
 * (SURVEY G4).  Constant device features are raw
 * values appended after the P tuning parameters; they are folded into the
 * first-layer bias at load time.  Ensembles (E <= 64) run one fused pass per
 * member: members 0..E-2 accumulate t in an fp32 device buffer (chunks of
 * 2^28 configs), the last one averages and emits.  Kernel envelope:
 * H in {32, 64, 128} (256: FP16 / BF16, CTA pairs), 1 <= L-1 <=
 * SURR_MAX_HIDDEN_LAYERS, P + 1 <= 16; a net whose weight image in the
 * precision's operand format does not fit shared memory is refused here
 * (SURR_E_UNSUPPORTED).  FP16 operands add a per-space range check (any
 * activation that can reach 65504 -> SURR_E_RANGE at the first sweep). */
typedef struct {
  uint32_t num_layers;           /* L affine layers */
  const uint32_t *widths;        /* [L + 1] */
  const double *const *W;        /* [E * L] */
  const double *const *b;        /* [E * L] */
  const double *x_shift;         /* [F] */
  const double *x_scale;         /* [F] */
  double y_mean, y_scale;        /* (0, 1) = identity */
  uint32_t num_const_features;   /* F - P */
  const double *const_features;  /* [F - P] raw values, or NULL when 0 */
  uint32_t ensemble;             /* E >= 1 */
  surr_precision precision;
} surr_model;

/* One result record as written by the sweep kernels: the k best of a
 * sub-range, sorted ascending by (t, idx); NaN ranks after +inf; unused
 * slots hold the sentinel (idx = UINT64_MAX, key = 0xFFFFFFFF). key is the
 * order-preserving uint32 image of the float time. */
typedef struct {
  uint64_t idx;
  uint32_t key;
  uint32_t pad;
} surr_record;

/* Create a handle on CUDA device `cuda_device` (must be sm_100). */
surr_status surrogate_create(int cuda_device, surrogate_t **out);
void surrogate_destroy(surrogate_t *h);
const char *surrogate_last_error(const surrogate_t *h);

/* Validate the model against the kernel envelope, fold constant features, b_1,
 * y_mean / y_scale into the layer parameters, convert to the precision's
 * operand format, pack the UMMA shared-memory image (K-major, no swizzle) and
 * upload it (complete on return) into the other of two device slots: sweeps
 * queued earlier keep reading the weights their launch captured, and no
 * device-wide synchronisation happens.  Non-finite weights, biases or scaler
 * entries -> SURR_E_INVALID_ARG.  PAPER.md:54, :63, :273. */
surr_status surrogate_load_weights(surrogate_t *h, const surr_model *model);

/* Predict an explicit batch: x_dev holds n rows of P raw parameter values
 * (row-major float32, device); t_dev receives n predicted times in seconds.
 * Row-wise pure.  n == 0 is a no-op. */
surr_status surrogate_predict(surrogate_t *h, const float *x_dev, uint64_t n, float *t_dev, void *stream);

/* Exhaustive sweep of [begin, end): the k smallest (t, I), sorted.
 * idx_dev[k], t_dev[k]; *count_host = min(k, end - begin).
 * k in 1..SURR_K_MAX.  The space's value lookup table is cached on the
 * handle and re-uploaded only when the descriptor changes, stream-ordered on
 * `stream` into the other of two device slots (sweeps queued earlier, on any
 * stream, keep reading the table their launch captured; the slot being
 * rewritten is first waited for by its own events, never the whole device).
 * A descriptor that fails validation leaves no cached space behind. */
surr_status surrogate_sweep(surrogate_t *h, const surr_space *space, uint32_t k, uint64_t *idx_dev, float *t_dev,
                            uint32_t *count_host, void *stream);

/* The same sweep end to end with HOST outputs: rebuilds and uploads the value
 * table, runs the sweep and copies the k results back; synchronous. */
surr_status surrogate_sweep_host(surrogate_t *h, const surr_space *space, uint32_t k, uint64_t *idx_host,
                                 float *t_host, uint32_t *count_host, void *stream);

/* Parity hook: the fused sweep kernel in dense-output mode writes t(I) for
 * every I in [begin, end) to t_dev[I - begin]. */
surr_status surrogate_eval_range(surrogate_t *h, const surr_space *space, float *t_dev, void *stream);

/* Parity hook of the decoder and the normalisation prologue (SURVEY §8(a)
 * a2, a3; PAPER.md:241 mixed-radix space, :273 StandardScaler): the fused
 * sweep kernel itself, in the launch configuration surrogate_sweep uses for
 * [begin, end), writes for every stride-th I (I - begin = q stride) the
 * layer-1 operand row it built from its in-register digits and the value
 * table: ops_dev[q * 16 + w], w =
 * 0..7 the eight packed 16-bit hi column pairs (slot 2w in the low half, slot
 * 2w+1 in the high half: z_j for parameter j, 1.0 in slot P, zeros after),
 * w = 8..15 the lo pairs of the 3xFP16 FP32 path (0 for FP16 / BF16).  The
 * row is exactly the UMMA operand, so comparing it with the oracle's decoded
 * tuple mapped through the documented rounding checks
 * decoded tuples bit-exactly; stride > 1 samples a whole-space launch.
 * ops_dev: device, caller-owned, ceil((end - begin) / stride) * 64 bytes.
 * SURR_E_INVALID_ARG for stride 0; SURR_E_UNSUPPORTED for the TF32 kernels
 * (not covered). */
surr_status surrogate_sweep_operands(surrogate_t *h, const surr_space *space, uint64_t stride, uint32_t *ops_dev,
                                     void *stream);

/* Merge `lists` sorted record lists of k_in entries each (device, contiguous)
 * into the k best, sorted (used after the NCCL
 * allgather).  k <= k_in * lists is not required: short results are padded
 * with sentinels. */
surr_status surrogate_merge_topk(surrogate_t *h, const surr_record *recs_dev, uint32_t lists, uint32_t k_in,
                                 uint32_t k, uint64_t *idx_dev, float *t_dev, surr_record *recs_out_dev,
                                 void *stream);

/* Records of the last surrogate_sweep before the final merge is converted:
 * copies the k merged records (device) — used by the multi-GPU path to feed
 * the allgather without a float->key round trip. */
surr_status surrogate_sweep_records(surrogate_t *h, const surr_space *space, uint32_t k, surr_record *recs_dev,
                                    void *stream);

/* Decoder hook: digits of n consecutive indices starting at `first`, computed
 * by the kernels' device decoder (super-digit magic division), written as
 * uint8 digits_dev[n * P] (parameter 0 first).  SURR_E_UNSUPPORTED when a
 * radix exceeds 256 (a digit would not fit its byte). */
surr_status surrogate_decode_range(surrogate_t *h, const surr_space *space, uint64_t first, uint64_t n,
                                   uint8_t *digits_dev, void *stream);

/* Exact |S| = prod r_j; SURR_E_RANGE if it does not fit u64. */
surr_status surrogate_space_size(const surr_space *space, uint64_t *out);

/* Timing of the fused sweep kernel alone (CUDA events recorded on the launch
 * stream around every K1 launch while enabled).  get synchronises the events
 * and returns the summed milliseconds and launch count since the last reset. */
surr_status surrogate_kernel_timing(surrogate_t *h, int enable);
surr_status surrogate_kernel_timing_get(surrogate_t *h, double *total_ms, uint32_t *launches);

/* Debug hook: record a clock64 timeline of CTA 0's pipeline events into
 * trace_dev[n] (device, caller-owned) on subsequent sweeps; NULL disables.
 * Layout: (round * 4 + slot) * 16 + event (see sweep_kernel3.cuh). */
surr_status surrogate_debug_trace(surrogate_t *h, unsigned long long *trace_dev, uint32_t n);

/* Drop the cached value table: the next sweep call rebuilds it from the
 * descriptor and uploads it again (used to time end-to-end sweeps). */
surr_status surrogate_reset_cache(surrogate_t *h);

/* Bytes of the value lookup table of the cached space (the per-sweep H2D of
 * surrogate_sweep_host). */
uint32_t surrogate_table_bytes(const surrogate_t *h);

/* Tensor-core arithmetic the loaded model runs on: *mma_kind = 0 for
 * tcgen05 kind::f16 (BF16 / FP16 operands), 1 for kind::tf32; *passes = UMMA
 * passes per hidden-layer K step (1, or 3 for the split FP32 path: 3xFP16 or
 * 3xTF32); *issued_flops = 2 x the MACs the sweep kernel issues to the tensor
 * cores per config and ensemble member (K padding 14 -> 16, bias K blocks and
 * split passes included; the FP32 final layer runs on CUDA cores).  The bench
 * derives the roofline peak of the dtype and the issued rate from it.
 * SURR_E_NOT_LOADED without a model. */
surr_status surrogate_arith(const surrogate_t *h, uint32_t *mma_kind, uint32_t *passes, double *issued_flops);

/* Number of kernel launches the last call issued on the GPU (for the bench's
 * gpu_launches count). */
uint32_t surrogate_last_launches(const surrogate_t *h);

/* Self-test of one tcgen05 GEMM (test infrastructure for the UMMA encodings):
 * D[128 x N] = A[128 x K] * B[K x N] with A staged in TMEM, B in shared memory
 * (K-major, no swizzle), FP32 accumulate.  precision BF16 or TF32 (one pass).
 * a_host / b_host / d_host are host float arrays (row-major). */
surr_status surrogate_selftest_umma(int cuda_device, int precision, uint32_t n, uint32_t k, const float *a_host,
                                    const float *b_host, float *d_host);

/* ---------------------------------------------------------------- training
 * GPU-side training of one F-H-H-1 FCNN, the step before
 * the sweep: the paper's scikit-learn MLPRegressor recipe (Table
 * "Hyperparameter" PAPER.md:212-235) in FP32 — minibatches in the given
 * epoch orders (the last batch of an epoch short), loss 1/2 mean squared error
 * + alpha/(2B) sum ||W||^2 (biases excluded), backpropagation with the ReLU
 * subgradient 0 at 0, Adam with lr_t = lr0 sqrt(1 - beta2^t) / (1 - beta1^t),
 * epoch loss = sample-weighted mean of the batch losses, stop after more than
 * n_iter_no_change epochs without improving the best epoch loss by tol, or
 * after max_epochs.  One launch of an H/16-CTA thread-block cluster runs the
 * whole fit. */
typedef struct {
  double alpha, beta1, beta2, lr0, eps, tol; /* paper: 1e-4, 0.95, 0.90, 0.0009, 1e-9, 1e-6 */
  uint32_t batch_size;                       /* 1..200 (paper: 200) */
  uint32_t max_epochs;                       /* >= 1 (paper: 200) */
  uint32_t n_iter_no_change;                 /* scikit-learn default 10 */
} surr_train_hyper;

/* widths = {F, H, H, 1} with F in 1..20 and H in {32, 64, 128}; E >= 1
 * ensemble members trained at once on the same data, each with
 * its own initial values and epoch orders (one cluster per member).
 * W[3 e + l], b[3 e + l] (l = 0..2): HOST float64, row-major fan_in x fan_out;
 * read as member e's initial parameters and overwritten with the trained ones.
 * X: HOST n x F row-major, y: HOST n — already standardised (the scalers are
 * the caller's).  perms: HOST E x max_epochs x n row indices
 * (member e, epoch p visits rows perms[(e max_epochs + p) n + i] in order i;
 * each row a permutation of 0..n-1), or NULL for the identity order.
 * Outputs (host): loss_history[E x max_epochs] (epochs beyond a member's
 * epochs_run left untouched), epochs_run[E], stop_reason[E] (0 = max_epochs,
 * 1 = tol).  Synchronous.  Errors: SURR_E_INVALID_ARG (null, n == 0, E == 0,
 * bad hyper, an index >= n in perms), SURR_E_UNSUPPORTED (widths outside the
 * envelope), SURR_E_RANGE when a member's epoch loss is non-finite (the fit
 * diverged: the error names the member and epoch, W / b are left untouched).
 * Members are independent clusters: more than fit at once run in
 * further waves. */
surr_status surrogate_train(surrogate_t *h, const uint32_t *widths, uint32_t E, double *const *W, double *const *b,
                            const double *X, const double *y, uint64_t n, const uint32_t *perms,
                            const surr_train_hyper *hyper, double *loss_history, uint32_t *epochs_run,
                            uint32_t *stop_reason);

#ifdef __cplusplus
}
#endif
#endif
