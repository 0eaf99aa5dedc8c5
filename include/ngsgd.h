/*
 * ngsgd.h -- C ABI of libngsgd.so: the data-parallel hot path of arXiv 1410.7455
 * (Povey, Zhang & Khudanpur, "Parallel training of DNNs with natural gradient and
 * parameter averaging") on NVIDIA B200 (sm_100a).
 *
 * Citations: "P:n" = line n of the paper's PAPER.md, with the section / equation label.
 *
 * Conventions (all entry points)
 *  - Every call returns ng_status and never throws across the ABI.  On failure,
 *    ng_last_error() returns a thread-local, human-readable message.
 *  - Plain pointers only.  "device" pointers are CUDA global-memory addresses on the
 *    device that was current when the handle was created; "host" pointers are ordinary
 *    CPU memory.  No pointer is retained after the call returns unless stated.
 *  - Matrices are row-major, one frame (minibatch element) per row, with an
 *    explicit leading dimension `ld` (elements between consecutive rows, ld >= cols).
 *  - Work is enqueued on the CUDA stream given at create time and is asynchronous unless
 *    stated; the caller keeps argument buffers alive until that stream has consumed them.
 *  - Argument/shape errors are detected on the host before anything is enqueued.
 *    Device-detected conditions (non-finite data, label out of range, a failed Cholesky
 *    in the re-orthogonalisation) raise a sticky device flag that is reported by the next
 *    synchronising call (ngsgd_get_state, nnet_get_params, nnet_average, or
 *    nnet_forward_backward with objective_out != NULL).
 *  - One stream owns a handle; handles are not thread-safe (the paper's try-lock of
 *    B.3.4, is a CPU-Hogwild device and has no counterpart here).
 */
#ifndef NGSGD_H_
#define NGSGD_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ common ---- */

typedef enum {
  NG_OK = 0,
  NG_EINVAL = 1,      /* bad argument (NULL handle, negative size, bad enum)          */
  NG_ESHAPE = 2,      /* inconsistent dimensions / leading dimension / n > max rows    */
  NG_ENONFINITE = 3,  /* NaN/Inf seen in device data (sticky flag)                     */
  NG_ELABEL = 4,      /* label outside [0, num_classes) (sticky flag)                  */
  NG_ECUDA = 5,       /* CUDA runtime error                                            */
  NG_ENCCL = 6,       /* NCCL error / communicator not initialised                     */
  NG_ENOTPD = 7,      /* Cholesky of O_t failed in B.3.1 repair: corrupted NG state    */
  NG_ESTATE = 8,      /* operation not valid in the handle's current state             */
  NG_ENOMEM = 9       /* device allocation failed                                      */
} ng_status;

/* Thread-local message describing the last failure on this thread ("" if none). */
const char* ng_last_error(void);
/* Library version / build string (static storage). */
const char* ng_version(void);

/* ------------------------------------ online NG-SGD preconditioner (Appendix B) ---- */

/* Configuration of one preconditioner ("one Kronecker side of one weight matrix",
 * P:913-919).  Defaults per B.4/B.5 are filled in by
 * ngsgd_config_default(). */
typedef struct {
  int32_t rank;                /* R, rank of the non-identity part; 20 input /
                                  80 output side.  Clipped to dim-1.  <= 112. */
  float alpha;                 /* identity smoothing, 4               */
  float s_samples;             /* S; forgetting factor eta = 1-exp(-N/S), 2000*/
  int32_t update_period;       /* J = 4                             */
  int32_t always_update_first; /* 10: always update on the first 10 minibatches  */
  float epsilon;               /* floor of rho and d, 1e-10      */
  int32_t precision;           /* ng_precision (below).  NG_FP32 and NG_TF32: the projections
                                  H = X W^T, J = H^T X and X_hat = X - H W on tcgen05 tensor
                                  cores in 3xTF32 (FP32-grade: X_hat is a difference of nearly
                                  equal terms when the subspace holds most of X's energy);
                                  needs ld % 4 == 0 and R % 4 == 0, otherwise that call uses
                                  CUDA cores.  NG_FP32_SIMT: CUDA cores in FP32 throughout.
                                  K, L, A_t B_t are FP32 CUDA-core, the R x R math FP64.     */
} ngsgd_config;

void ngsgd_config_default(ngsgd_config* cfg, int32_t rank);

typedef struct ngsgd_ctx* ngsgd_t;

/* Create one online NG-SGD state for vectors of logical dimension `dim` (D; on the input
 * side of a weight matrix D includes the appended 1 of the bias, e.g. 301).
 * `max_rows` bounds the minibatch size N of later calls (workspaces are sized here so
 * the hot path never allocates).  `cuda_stream` is a cudaStream_t (NULL = legacy default
 * stream).  The state is uninitialised until the first minibatch with tr(X^T X) > 0
 * (B.3.2; reading R7); earlier minibatches pass through unchanged
 * but are counted in t (the update schedule is per minibatch).  Owns all its
 * device memory. */
ng_status ngsgd_create(int32_t dim, int32_t max_rows, const ngsgd_config* cfg,
                       void* cuda_stream, ngsgd_t* out);
ng_status ngsgd_destroy(ngsgd_t h);

/* Precondition one minibatch X (B.5 summary), in place.
 *   x          device float, n rows x dim columns, leading dimension ld (ld >= dim).
 *              On return holds X_hat = X - X W_t^T W_t (eqn:hatxt:compute),
 *              NOT multiplied by gamma: "we actually output gamma_t and let the user do the
 *              scaling later on".  Columns dim..ld-1 are not touched.
 *   gamma_out  device float[1] or NULL: gamma_t = sqrt(tr(X X^T)/tr(X_hat X_hat^T))
 *              (eqn:gammat), 1 if the denominator is 0.
 *   p_out      device float[n] or NULL: p_i = ||x_hat_i||^2 (eqn:pi), the
 *              UNSCALED row products; gamma^2 p_i = ||x_bar_i||^2.
 *   update     -1: internal policy "t < always_update_first or J divides t";
 *              0 / 1: force the non-update / update branch.
 * The first call with non-zero X initialises the state from that X (t = 0) and, unlike
 * every other call, synchronises the stream once (to test tr(X^T X) > 0).
 * Errors: NG_ESHAPE if n < 1, n > max_rows or ld < dim. */
ng_status ngsgd_precondition(ngsgd_t h, int32_t n, float* x, int64_t ld,
                             float* gamma_out, float* p_out, int32_t update);

/* Enqueue on the handle's stream a wait for the state's internal side-stream work (the
 * R x R refresh and W_{t+1} = A_t B_t of the last update step run on a side stream and
 * are otherwise joined lazily by the next call on this state).  Asynchronous. */
ng_status ngsgd_join(ngsgd_t h);

/* Host snapshot of a state (B.5: the stored variables are rho_t, D_t, W_t). */
typedef struct {
  int32_t dim, rank, t, initialized;
  double rho;        /* rho_t                                                      */
  double* d;         /* host double[rank]  caller-allocated: diag(D_t), descending */
  float* w;          /* host float[rank*dim] caller-allocated: W_t row-major        */
  int32_t last_updated, last_floored, last_reorth_checked, last_reorthogonalized;
  int32_t last_jacobi_sweeps;   /* sweeps the R x R eigensolver used in the last update */
} ngsgd_state_host;

/* Copy the state to the host (synchronises the handle's stream).  d / w may be NULL to
 * query only the scalar fields.  Also reports sticky device errors (NG_ENONFINITE,
 * NG_ENOTPD). */
ng_status ngsgd_get_state(ngsgd_t h, ngsgd_state_host* out);
/* Overwrite the state from the host (e.g. to inject an oracle state for parity tests).
 * rank must equal the handle's effective rank; initialized != 0 marks it initialised. */
ng_status ngsgd_set_state(ngsgd_t h, const ngsgd_state_host* in);

/* ---------------------------------- simple NG-SGD preconditioner (Appendix A) ---- */

/* The simple natural-gradient method (A.2), computed by its efficient form A.3
 * (P:843-887): per minibatch X (n x dim) the Fisher estimate of every row is formed from
 * the OTHER rows (held-out, reading R1), regularised by beta = alpha max(tr X^T X, 1e-20)
 * / (n dim); Q = X (beta I + X^T X/(n-1))^{-1} if n > dim, else
 * (beta I + X X^T/(n-1))^{-1} X (strict n > dim, reading R11);
 * x_hat_i = (1 + a_i / (n-1-a_i)) q_i with a_i = x_i^T q_i;
 * gamma = sqrt(tr X^T X / tr X_hat^T X_hat).  Stateless apart from its
 * workspace (FP64 Gram / Cholesky factor of min(n, dim)^2 and dim x max_rows solves).
 * Arithmetic: FP64 on the device (Gram, Cholesky, substitutions); I/O FP32. */
typedef struct ngsimple_ctx* ngsimple_t;
/* max_rows >= 2 (a held-out estimate needs another row); alpha > 0 (4). */
ng_status ngsimple_create(int32_t dim, int32_t max_rows, float alpha, void* cuda_stream, ngsimple_t* out);
ng_status ngsimple_destroy(ngsimple_t h);
/* x: device, n x dim, leading dimension ld >= dim, 2 <= n <= max_rows.  In place:
 * x <- X_hat (NOT scaled by gamma, as ngsgd_precondition); gamma_out: device float[1] or
 * NULL; row_sq_out: device float[n] (||x_hat_i||^2) or NULL.  Asynchronous. */
ng_status ngsimple_precondition(ngsimple_t h, int32_t n, float* x, int64_t ld, float* gamma_out,
                                float* row_sq_out);
/* Synchronise the handle's stream and report sticky device errors (non-positive pivot:
 * NG_ENOTPD; non-finite data: NG_ENONFINITE). */
ng_status ngsimple_read_flags(ngsimple_t h);

/* ---------------------------------------- p-norm / softmax DNN training step ---- */

/* NG_FP32: FP32-grade (paper-faithful; parity 1e-4): every GEMM on tcgen05 tensor
 *          cores in 3xTF32 (hi/lo split of both operands in shared memory, three MMAs
 *          accumulated in FP32 TMEM).
 * NG_TF32: the DNN GEMMs (forward, backward-data, weight update) on tcgen05 tensor cores
 *          reading the FP32 buffers as TF32, FP32 accumulation (parity bar 2e-2 of the
 *          north star for reduced-precision tensor-core inputs); NG projections 3xTF32.
 * NG_FP32_SIMT: every GEMM on FP32 CUDA cores (the round-1 reference path).
 * NG_BF16: reserved. */
typedef enum { NG_FP32 = 0, NG_BF16 = 1, NG_TF32 = 2, NG_FP32_SIMT = 3 } ng_precision;

/* Network: input_dim -> num_hidden x [affine hidden_dim -> p-norm /pnorm_group
 * (-> renormalisation)] -> affine num_classes -> softmax (p = 2,
 * DESIGN.md R19).  renorm != 0 adds the renormalisation layer that follows each p-norm
 * layer in the paper's networks (R32): y = s a, s = sqrt(D/||a||^2)
 * per row (unit root-mean-square; s = 0 for an all-zero row). */
typedef struct {
  int32_t input_dim, num_hidden, hidden_dim, pnorm_group, num_classes;
  int32_t max_minibatch;        /* N bound; 512 on GPU              */
  int32_t precond;              /* 0: plain SGD, 1: online NG-SGD (Appendix B),
                                   2: simple NG-SGD (Appendix A; ng_in.alpha is its alpha) */
  ngsgd_config ng_in, ng_out;   /* R_in = 20, R_out = 80                    */
  int32_t precision;            /* ng_precision of the DNN GEMMs                          */
  uint64_t seed;                /* weight-init seed (C.6)                    */
  int32_t renorm;               /* 1: renormalisation layer after each p-norm (R32)       */
} nnet_config;

typedef struct nnet_ctx* nnet_t;

/* Create a network with C.6 initialisation: N(0, 1/fan-in) with the bias
 * column counted in the fan-in (R20), softmax layer zero.  Parameters live in
 * one contiguous FP32 device arena (for nnet_average).  NG_ESHAPE if hidden_dim or
 * num_classes exceeds 50000 (one activation row is staged in shared memory). */
ng_status nnet_create(const nnet_config* cfg, void* cuda_stream, nnet_t* out);
ng_status nnet_destroy(nnet_t h);

/* Forward + backward for one minibatch with the current weights: fills, for
 * every weight matrix, X_i (derivative of sum_i log p(y_i|x_i) w.r.t. its output) and Y_i
 * (its input with the appended 1), kept inside the handle for nnet_update.
 *   frames       device float, n x input_dim, leading dimension ld.
 *   labels       device int32[n] in [0, num_classes).
 *   objective_out host double* or NULL. If non-NULL the call synchronises and returns
 *                sum_i log p(y_i | x_i) (a sum, not a mean). */
ng_status nnet_forward_backward(nnet_t h, const float* frames, int64_t ld,
                                const int32_t* labels, int32_t n, double* objective_out);

/* Input descriptor of nnet_forward_backward_ex (the step before the hot path, C.2,
 * P:1459-1485):
 *   frames  device; format 0: float32 [rows][ld]; format 1: uint8 codes [rows][ld] of the
 *           1-byte lossy compression (R36), decoded in the input
 *           kernel as float(lo[c] + step[c] * q) with lo, step device double[input_dim]
 *           (see ng_compress_frames).
 *   rows    device int32[n] or NULL: minibatch row r is frame row rows[r] (a block of the
 *           N x M randomisation, resident in device memory); NULL = rows 0..n-1.
 *   labels  device int32, indexed like the frame rows. */
typedef struct {
  const void* frames;
  int32_t format;
  int64_t ld;
  const double* lo;
  const double* step;
  const int32_t* rows;
  const int32_t* labels;
} nnet_input;
ng_status nnet_forward_backward_ex(nnet_t h, const nnet_input* in, int32_t n, double* objective_out);

/* ------------------------------------------ generalised model combination (C.4) ---- */
/* The parameter arena (all W_l, FP32, layout of nnet_create) as a flat vector: its length,
 * and a copy to (direction 0) or from (direction 1) a caller-owned device buffer -- the
 * snapshots of the last P outer iterations' models.  Stream-ordered. */
ng_status nnet_arena_size(nnet_t h, int64_t* count);
ng_status nnet_copy_arena(nnet_t h, float* dev, int32_t direction);
/* W_l = sum_p weights[l P + p] W_l^(p): models is a HOST array of P <= 32
 * device arena pointers (snapshots), weights host float[L x P].  Stream-ordered. */
ng_status nnet_set_combination(nnet_t h, const float* const* models, int32_t P, const float* weights);
/* After nnet_forward_backward: grad[l P + p] = <X_l^T Y_l, W_l^(p)>_F, the derivative of the
 * minibatch objective w.r.t. the combination weight w[l][p] (chain rule through
 * W_l = sum_p w[l][p] W_l^(p)); host double[L x P].  Synchronises.  The L-BFGS search over
 * the weights is host logic (driver.combine_models). */
ng_status nnet_combination_grad(nnet_t h, const float* const* models, int32_t P, double* grad);

/* 1-byte compression of n frames (R36): per column lo = min, step = (max - min)/255 (FP64),
 * q = clamp(round_half_even((x - lo)/step), 0, 255).  All pointers device; x is n x dim
 * (ld ldx), q n x dim (ld ldq), lo/step double[dim].  Stream-ordered on `stream`. */
ng_status ng_compress_frames(int32_t n, int32_t dim, const float* x, int64_t ldx, uint8_t* q, int64_t ldq,
                             double* lo, double* step, void* stream);

/* The objective of the last nnet_forward_backward, without synchronising: enqueues the
 * fixed-order sum over the minibatch's rows (same value as objective_out above) and an
 * asynchronous device-to-host copy into `host_out` (host double*, should be pinned) on the
 * handle's stream.  The value is valid once the stream reaches this point (e.g. after a
 * cudaEventSynchronize on an event recorded after the call); lets a caller overlap the next
 * step's input copy and launches with the readback of this step's result. */
ng_status nnet_objective_async(nnet_t h, double* host_out);

typedef struct {
  float alpha_t[16];      /* max-change scale per weight matrix (C.3)        */
  float gamma_in[16];     /* gamma of the input side (eqn:gammat)                        */
  float gamma_out[16];    /* gamma of the output side                                    */
  int32_t updated_in[16], updated_out[16];  /* Fisher factor refreshed this step         */
} nnet_update_stats;

/* Precondition both sides of every weight matrix (2I calls), compute the
 * max-change scale alpha_t from the preconditioned row norms, and apply
 * W_i += alpha_t * lr * gamma_x * gamma_y * X_hat_i^T Y_hat_i (eqn:add:w).
 *   lr   per-job learning rate = n_jobs x effective rate.
 *   max_change_per_sample  0.075.
 *   stats_or_null  host; if non-NULL the call synchronises and fills it. */
ng_status nnet_update(nnet_t h, float lr, float max_change_per_sample,
                      nnet_update_stats* stats_or_null);

/* Make the network's stream wait for all internal side-stream work (NG refreshes).
 * Asynchronous; use before timing the stream or handing buffers to other streams. */
ng_status nnet_join(nnet_t h);

/* Number of weight matrices I and the shape (rows = D_out, cols = D_in + 1) of each. */
ng_status nnet_num_layers(nnet_t h, int32_t* out);
ng_status nnet_layer_shape(nnet_t h, int32_t layer, int32_t* rows, int32_t* cols);

/* Copy weight matrix `layer` (rows x cols, row-major, bias last column) to / from the
 * host.  count must equal rows*cols.  get_params synchronises. */
ng_status nnet_get_params(nnet_t h, int32_t layer, float* host, int64_t count);
ng_status nnet_set_params(nnet_t h, int32_t layer, const float* host, int64_t count);
/* Borrowed handle of the input-side (side = 0) or output-side (side = 1) preconditioner
 * of weight matrix `layer`; valid while the network lives; NULL-equivalent error if
 * precond == 0. */
ng_status nnet_get_ngsgd(nnet_t h, int32_t layer, int32_t side, ngsgd_t* out);

/* ----------------------------------------------- parameter averaging (3.1) ---- */

/* Size in bytes of the NCCL unique id expected by nnet_comm_init (128). */
int32_t nnet_comm_id_bytes(void);
/* Create an NCCL unique id into host buffer `id_out` (nnet_comm_id_bytes() bytes), to
 * be broadcast by the caller (e.g. torch.distributed) to all ranks. */
ng_status nnet_comm_get_unique_id(void* id_out);
/* Join the communicator of `nranks` jobs as `rank` (one process per GPU), 1 <= nranks <= 64
 * (any count, e.g. the paper's 6 jobs).  The arena is split into nranks shards of
 * ceil(count / nranks) floats rounded up to 64; the last shard(s) are ragged.  Allocates two
 * device staging buffers of nranks x shard floats. */
ng_status nnet_comm_init(nnet_t h, const void* nccl_unique_id, int32_t rank, int32_t nranks);
/* In-place average of all parameters over the ranks (3.1): W <- (sum_r W^r)/n
 * with the sum taken in a fixed pairwise-tree order over rank index (R18), so
 * every rank ends with bit-identical parameters equal to the host tree sum.  NG states
 * are per-job and untouched.  mode 0: deterministic
 * (all-to-all of shards, fixed-order sum kernel, all-gather); mode 1: ncclAllReduce(sum)
 * then scale (speed reference; order not fixed).  Synchronises the stream. */
ng_status nnet_average(nnet_t h, int32_t mode);

/* Best-of-n in place of the average on an outer iteration that follows a random
 * initialisation: every rank passes the objective of its job on the data it
 * trained on (host double, e.g. the mean log-likelihood per frame of its last outer
 * iteration); the objectives are all-gathered, the best one wins (ties: the lowest rank)
 * and its parameters are broadcast to every rank (NCCL, in place).  NG states untouched.
 * winner_out (host, may be NULL) receives the winning rank.  Synchronises. */
ng_status nnet_select_best(nnet_t h, double objective, int32_t* winner_out);

/* The n networks `nets` (same shapes, same device, n <= 64) all receive the average of
 * their parameters, summed in the fixed pairwise tree order of nnet_average (bit-exact
 * with it): the single-device form of the every-K average, for running several jobs on one
 * GPU (experiments).  Stream-ordered on nets[0]'s stream after
 * synchronising the others. */
ng_status nnet_average_local(nnet_t* nets, int32_t n);


/* The fixed-order sum kernel of nnet_average on its own, for bit-exact tests on one GPU:
 * out[i] = (sum over r of in[r * count + i]) * (1.0f / nr), summed in the pairwise tree order
 * of DESIGN.md R18 (oracle/training.py tree_sum).  in: device float[nr * count]; out: device
 * float[count]; 1 <= nr <= 64; asynchronous on `stream`. */
ng_status ng_debug_tree_avg(int32_t nr, int64_t count, const float* in, float* out, void* cuda_stream);

/* ------------------------------------------------ instrumentation (bench.py) ---- */

/* Kernel groups for live per-group timing.  Each group's algorithmic FLOPs and bytes
 * are counted per launch from the shapes. */
typedef enum {
  NG_PROF_FWD_GEMM = 0,   /* Z_l = Y_l W_l^T (+ p-norm)                               */
  NG_PROF_BWD_GEMM = 1,   /* g = X_l W_l (+ p-norm backward)                           */
  NG_PROF_UPD_GEMM = 2,   /* W_l += s X_hat^T Y_hat                                    */
  NG_PROF_NG_PROJ = 3,    /* H = X W^T                                                 */
  NG_PROF_NG_APPLY = 4,   /* X_hat = X - H W, p_i, traces, gamma                       */
  NG_PROF_NG_REFRESH = 5, /* J, K, L, one-CTA refresh, W_{t+1} = A_t B_t, B.3.1         */
  NG_PROF_NG_INIT = 6,    /* B.3.2 initialisation (once per state)                     */
  NG_PROF_ELEMWISE = 7,   /* input, p-norm, softmax/objective, max-change              */
  NG_PROF_AVERAGE = 8,    /* parameter averaging                                       */
  NG_PROF_NG_EIG = 9,     /* the one-CTA R x R refresh (Z_t, Jacobi eigensolver, A_t)   */
  NG_PROF_NUM = 10
} ng_prof_group;

typedef struct {
  int64_t launches[16];   /* launches recorded per group since enable                 */
  double ms[16];          /* summed CUDA-event durations (ms) per group                */
  double flops[16];       /* summed algorithmic FLOPs per group                        */
  double bytes[16];       /* summed algorithmic HBM bytes per group                    */
} ng_profile_stats;

/* Enable CUDA-event timing around every launch of the groups in `group_mask` (bit g =
 * group g); 0 disables.  Resets the accumulators.  Events are recorded on the stream
 * each kernel is launched on. */
ng_status ng_profile_enable(uint32_t group_mask);
/* Synchronise the recorded events and return the accumulated statistics. */
ng_status ng_profile_read(ng_profile_stats* out);
/* Number of kernels this library has launched since it was loaded. */
int64_t ng_kernel_launches(void);

/* ------------------------------------------------------------ diagnostics ---- */

/* One tensor-core GEMM C = A B exactly as the DNN's TF32 path runs it (tcgen05.mma
 * kind::tf32 fed by TMA, FP32 accumulation in TMEM); exposed for unit tests.
 *   A is M x K: a_kmajor != 0 -> A[m][k] = A[m*lda + k], else A[m][k] = A[k*lda + m].
 *   B is K x N: b_kmajor != 0 -> B[k][n] = B[n*ldb + k], else B[k][n] = B[k*ldb + n].
 *   C (device, M x N, ldc) is overwritten.  bn in {64, 128}; splits >= 1 (split-K with a
 *   fixed-order reduction).  All pointers device, 16-byte aligned, lda/ldb % 4 == 0. */
ng_status ng_debug_gemm_tf32(int32_t M, int32_t N, int32_t K, const float* A, int64_t lda, int32_t a_kmajor,
                             const float* B, int64_t ldb, int32_t b_kmajor, float* C, int64_t ldc,
                             int32_t bn, int32_t splits, void* cuda_stream);
/* The same with split3 != 0 selecting 3xTF32 (each operand split in shared memory into a
 * TF32 hi part and the exact remainder, A_lo B_hi + A_hi B_lo + A_hi B_hi accumulated in
 * TMEM): the FP32-grade tensor-core GEMM of the NG_FP32 mode and of the NG projections. */
ng_status ng_debug_gemm_tc(int32_t M, int32_t N, int32_t K, const float* A, int64_t lda, int32_t a_kmajor,
                           const float* B, int64_t ldb, int32_t b_kmajor, float* C, int64_t ldc,
                           int32_t bn, int32_t splits, int32_t split3, void* cuda_stream);

/* The refresh's default eigensolver (Householder + relatively robust representation +
 * twisted-factorisation eigenvectors, FP64, one CTA; eqn:zt:eig) on its own,
 * for unit tests: z device double[n*n] (row major, symmetric), lam device double[n], vt device
 * double[n*n]; lam / vt come out UNORDERED
 * (vt row i = unit eigenvector of lam[i]); ok device int[4]: ok[0] = 1 when the solve passed
 * its orthogonality check (0 = the refresh would fall back to Jacobi; lam / vt undefined),
 * ok[1] = cycles spent (clock64, whole solve), ok[2..5] = cycles of the phases
 * (tridiagonalisation, eigenvalues + vectors of T, orthogonality check, V = X Q^T); ok: int[8].  n in [1, 80]; asynchronous on `stream`. */
ng_status ng_debug_eig_tri(const double* z, int32_t n, double* lam, double* vt, int32_t* ok, void* stream);

/* Diagnostics of the refresh's Jacobi fallback (eig_tri failed its checks): z_host double[80*80]
 * gets the last such Z_t (row major, n x n with n = info_host[0]); info_host int[5] = {n, number
 * of fallbacks so far, reason of the last one: 1 no positive definite root representation,
 * 2 an eigenvalue did not converge, 3 orthogonality check; the largest relative-cluster
 * position and 1000 x RQI-loop iterations + twisted solves of any eigenvalue since the last
 * call (both reset)}.  Synchronises the device. */
ng_status ng_debug_tri_fail(double* z_host, int32_t* info_host);

/* Device-clock (globaltimer, ns) start / end of the last refresh CTAs: out host
 * uint64[256*9] ring of {R | D << 16, start, end, eigensolve start, eigensolve end, then the
 * eigensolver's phases in SM cycles: tridiagonalisation, split..multisection, RQI + vectors,
 * clusters + check + back-transformation} (slot = refresh index mod 256; the eigensolver
 * stamps are 0 outside the default solver), count = refreshes so far.  Synchronises the
 * device.  For tools/refresh_timeline.py. */
ng_status ng_debug_refresh_times(uint64_t* out, int32_t* count);

#ifdef __cplusplus
}
#endif
#endif /* NGSGD_H_ */
