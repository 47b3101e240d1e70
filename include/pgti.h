/*
 * pgti.h -- C ABI of libpgti, the B200-native index-batched DCRNN training step
 * of PGT-I (arXiv 2507.11683).  "P:n" = PAPER.md line n, "S:n" = SPEC.md line n,
 * "cN" / "ON" = reading / oracle row N of DESIGN.md (= SURVEY.md 8(c)).
 *
 * Conventions (every entry point):
 *  - Returns pgti_status; PGTI_OK == 0.  No C++ exception crosses the ABI.  On
 *    error, pgti_last_error() returns a thread-local message naming the
 *    offending argument / row / offset.
 *  - Argument and shape checks are synchronous and happen before any launch; a
 *    failed check launches nothing.  Conditions only the device can see (a
 *    window start outside the rank's rows, a non-finite loss) set a sticky
 *    device flag that pgti_check_device_error() reports.
 *  - Memory: every device buffer is allocated and owned by the CALLER (torch
 *    tensors in the Python binding) and must stay alive until the stream work
 *    using it completes.  The library keeps no device allocation beyond (a) a
 *    series handle's error flag and (b) NCCL's internal buffers; pgti_make_index
 *    takes transient sort scratch from the stream-ordered allocator.
 *  - Streams: `stream` is a cudaStream_t passed as void*; all device work is
 *    enqueued on it, in order; nothing synchronises the host except
 *    pgti_check_device_error and pgti_load_series from pageable memory.
 *  - Layouts are row-major, dimensions listed outermost first.  "ld" is the
 *    series row pitch in floats: ld >= N*F and ld % 4 == 0, so every time row
 *    starts 16-byte aligned (pads are +0.0).
 */
#ifndef PGTI_H
#define PGTI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PGTI_OK = 0,
  PGTI_ERR_INVALID_ARG = 1,     /* null pointer, negative size, bad enum */
  PGTI_ERR_TOO_FEW_ENTRIES = 2, /* rows < T_in + T_out */
  PGTI_ERR_ZERO_VARIANCE = 3,   /* sigma <= 0 or not finite */
  PGTI_ERR_NONFINITE = 4,       /* non-finite input / loss */
  PGTI_ERR_OUT_OF_RANGE = 5,    /* window start outside the held rows */
  PGTI_ERR_SHAPE = 6,           /* inconsistent dimensions */
  PGTI_ERR_TOO_FEW_WINDOWS = 7, /* fewer windows than one batch */
  PGTI_ERR_ALIGNMENT = 8,       /* ld % 4 != 0 or a device pointer not 16-byte aligned */
  PGTI_ERR_WORKSPACE = 9,       /* workspace too small; message reports the bytes needed */
  PGTI_ERR_CUDA = 10,           /* CUDA runtime error (message has cudaGetErrorString) */
  PGTI_ERR_NCCL = 11,           /* NCCL error */
  PGTI_ERR_UNSUPPORTED = 12     /* valid request this build does not implement */
} pgti_status;

/* Thread-local text of the last error on this thread ("" if none). */
const char *pgti_last_error(void);
/* Library version string. */
const char *pgti_version(void);
/* Synchronises `stream`, then reads and clears the sticky device error flags set by
 * kernels: PGTI_ERR_OUT_OF_RANGE (gather saw a start outside the series rows),
 * PGTI_ERR_NONFINITE (the step produced a non-finite loss). */
pgti_status pgti_check_device_error(void *stream);

/* ------------------------------------------------------------------ graph (host) */
/* Transition matrices of the diffusion convolution (reading c1/c4/c5; Li et al.
 * Eq. 2 [ext]): A[i][j] = w of the directed edge src->dst;
 * P_f = D_O^-1 A, P_b = D_I^-1 A^T, zero degree -> zero row.  Computed on the
 * host in double, stored as float, on two CSR patterns:
 *   pattern(A)  : row i lists j with A[i][j] != 0   -> values P_f and P_b^T
 *   pattern(A^T): row i lists j with A[j][i] != 0   -> values P_b and P_f^T
 * (P_f^T and P_b^T drive the backward adjoint diffusion.)  Column indices within
 * a row are ascending.  Inputs: nnz edges (no duplicates; self loops allowed).
 * Outputs (caller-allocated HOST arrays): *_rowptr [N+1], *_col / *_val [nnz].
 * Errors: INVALID_ARG (null, nnz < 0, node id out of [0,N), negative or
 * non-finite weight, duplicate edge). */
pgti_status pgti_graph_build(int32_t N, int64_t nnz, const int32_t *src, const int32_t *dst,
                             const float *w, int32_t *a_rowptr, int32_t *a_col, float *Pf_val,
                             float *PbT_val, int32_t *at_rowptr, int32_t *at_col, float *Pb_val,
                             float *PfT_val);

/* Shared-memory staging plan of the diffusion SpMM (the north star's "shared-
 * memory staging of the dense operand") on ONE CSR pattern (host arrays): rows
 * are cut into windows of rows_per_window consecutive nodes (1..64); window w
 * stages the ascending union of its rows' columns, written to
 * win_nodes[win_ptr[w] .. win_ptr[w+1]) (win_ptr has ceil(N/rows_per_window)+1
 * entries; win_nodes needs at most rowptr[N] entries), and lcol[e] (rowptr[N]
 * entries) is the position of col[e] in its window's union.  *max_union = the
 * largest union.  Index bookkeeping only (no values).  Errors: INVALID_ARG (null,
 * rows_per_window outside [1,64], column outside [0,N), a union > 65535). */
pgti_status pgti_graph_windows(int32_t N, const int32_t *rowptr, const int32_t *col,
                               int32_t rows_per_window, int32_t *win_ptr, int32_t *win_nodes,
                               uint16_t *lcol, int32_t *max_union);

/* ----------------------------------------------------------------- the series */
typedef struct pgti_series pgti_series; /* opaque; BORROWS dev_buf */

/* GPU-index-batching's single consolidated H2D copy (A5): rows
 * [row0, row0+nrows) of the raw float32 series v[E][N][F] (host_rows holds
 * exactly those rows, [nrows][N][F]; pinned memory gives an async copy) are
 * copied into dev_buf[nrows][ld] (caller-allocated, >= nrows*ld floats, 16-byte
 * aligned) and the pad columns [N*F, ld) are set to +0.0.  Under halo sharding
 * (BASELINE.json north_star) row0/nrows are the rank's window range plus a halo
 * of T_in+T_out-1 rows.  Errors: INVALID_ARG, ALIGNMENT, CUDA. */
pgti_status pgti_load_series(pgti_series **out, const float *host_rows, int64_t row0,
                             int64_t nrows, int64_t N, int64_t F, float *dev_buf, int64_t ld,
                             void *stream);

/* Window-weighted statistics of Alg. 1 lines 199-202 (reading c9)
 * without stacking: global row t is covered by
 *   w(t) = max(0, min(t, S_tr-1) - max(0, t-T_in+1) + 1)
 * training windows' x slices.  Over the held global rows
 * [row_lo, row_hi) it accumulates, in float64,
 *   dev_sums[0] += sum_t w(t) * N*F,
 *   dev_sums[1] += sum_t w(t) * sum_{n,f} (v - shift),
 *   dev_sums[2] += sum_t w(t) * sum_{n,f} (v - shift)^2
 * into the caller's device double[3] (zero it first).  Ranks sum disjoint row
 * ranges, all-reduce the three sums, then mu = shift + s1/s0 and
 * sigma^2 = s2/s0 - (s1/s0)^2 (population variance); run once with shift 0 and
 * again with shift = mu for a cancellation-free variance.  Must run before
 * pgti_series_normalize.  Errors: INVALID_ARG, OUT_OF_RANGE (rows not held). */
pgti_status pgti_series_stats(const pgti_series *s, int64_t S_tr, int T_in, int64_t row_lo,
                              int64_t row_hi, double shift, double *dev_sums, void *stream);

/* Alg. 1 lines 201-202 (reading c9) finished from the three sums of
 * pgti_series_stats (HOST double[3], already summed over ranks) taken about
 * `shift`:  *mean = shift + s1/s0,  *var = max(0, s2/s0 - (s1/s0)^2)  (population
 * variance, ddof 0).  Pure host arithmetic, no device work.
 * Errors: INVALID_ARG (null), TOO_FEW_ENTRIES (s0 <= 0: no training window covers
 * the rows), NONFINITE (a sum or the shift not finite). */
pgti_status pgti_stats_finalize(const double sums[3], double shift, double *mean, double *var);

typedef struct pgti_comm pgti_comm;
/* The whole of Alg. 1's statistics for a (possibly halo-sharded)
 * series: pass 1 = pgti_series_stats over this rank's rows [row_lo, row_hi) about
 * shift 0, in-place NCCL SUM of the three sums over the ranks when comm is
 * non-null (every rank of comm must call with its own disjoint rows), then
 * pgti_stats_finalize; pass 2 the same about shift = the pass-1 mean (cancellation-
 * free variance).  Results on the HOST: *mu, *sigma = sqrt(var) -- identical on
 * every rank.  dev_sums: caller-owned device double[3] scratch.  Synchronises
 * `stream` twice.  Errors: as pgti_series_stats and pgti_stats_finalize, NCCL,
 * CUDA, ZERO_VARIANCE (sigma == 0). */
pgti_status pgti_series_moments(const pgti_series *s, int64_t S_tr, int T_in, int64_t row_lo,
                                int64_t row_hi, pgti_comm *comm, double *dev_sums, double *mu,
                                double *sigma, void *stream);

/* Mean of per-batch losses over every rank (the per-epoch validation MAE of
 * distributed-index-batching and its AllReduce): the n device
 * floats dev_losses are summed in float64 in a fixed order into dev_scratch[0]
 * (dev_scratch[1] = n; caller-owned device double[2]), the pair is NCCL-summed
 * over the ranks when comm is non-null, and *mean (HOST) = sum / count (NaN when
 * no rank had a batch).  Every batch must have the same element count (equal-
 * weight mean).  Synchronises `stream`.  Errors: INVALID_ARG, NCCL, CUDA. */
pgti_status pgti_mean_losses(pgti_comm *comm, const float *dev_losses, int64_t n,
                             double *dev_scratch, double *mean, void *stream);

/* In-place z-score (Alg. 1 lines 203-204 applied once to the single copy, the
 * in-place standardisation of P:249): v <- fl32(fl32(v - fl32(mu)) / fl32(sigma)),
 * IEEE round-to-nearest float32 sub and div (reading O4); pads stay +0.0.
 * Errors: ZERO_VARIANCE (sigma <= 0 or not finite), NONFINITE (mu). */
pgti_status pgti_series_normalize(pgti_series *s, double mu, double sigma, void *stream);

pgti_status pgti_series_info(const pgti_series *s, int64_t *row0, int64_t *nrows, int64_t *N,
                             int64_t *F, int64_t *ld);
pgti_status pgti_series_destroy(pgti_series *s);

/* -------------------------------------------------------------- index batching */
/* Per-epoch index plan ("array of graph IDs", "shuffled at the start
 * of each epoch"; reading c16/c17, oracle O6).  For the global window
 * starts [win_lo, win_hi) of this rank, writes dev_idx[i] (int32, caller
 * allocated, >= win_hi-win_lo entries) = win_lo + pi(i) where pi is the stable
 * argsort of the Philox4x32-10 keys
 *   key_i = (w0 << 32) | w1,  (w0,w1,..) = Philox4x32-10(ctr = (i, epoch_lo,
 *           epoch_hi, rank), key = (seed_lo, seed_hi))
 * (shuffle = 1), or the identity (shuffle = 0).  shuffle = 2 is the generalized
 * variant's local batch shuffle: batch membership
 * is frozen to consecutive windows and only the batch ORDER is permuted --
 * dev_idx[jB + u] = win_lo + rho(j) B + u with rho the stable argsort of the
 * same Philox keys over batch indices j < floor(n/B) (entries past n_used are
 * left untouched).  The replicated placement's global shuffle (SURVEY
 * f1) is this call with [win_lo, win_hi) = all training windows and rank = 0 on
 * every rank, each rank then visiting its slice of the one plan.  *n_used (host) =
 * floor((win_hi-win_lo)/B)*B: batch j is dev_idx[jB, (j+1)B).  Every window must
 * lie inside the series' rows: win_lo >= row0, win_hi-1+T_in+T_out <= row0+nrows.
 * Errors: INVALID_ARG, OUT_OF_RANGE, TOO_FEW_WINDOWS (fewer than B), CUDA. */
pgti_status pgti_make_index(const pgti_series *s, int64_t win_lo, int64_t win_hi, int T_in,
                            int T_out, int B, uint64_t seed, uint64_t epoch, int rank,
                            int shuffle, int32_t *dev_idx, int64_t *n_used, void *stream);

/* Index-batching's runtime snapshot construction (x = data[s:s+T_in],
 * y = data[s+T_in : s+T_in+T_out]) on the device: for b < B, the contiguous slab
 * of T_in+T_out rows starting at global row dev_idx[b] is copied bit-exactly into
 * x[b] ([B][T_in][ld]) and y[b] ([B][T_out][ld]) -- pads included.  x, y 16-byte
 * aligned, caller-allocated.  A start outside the held rows writes nothing for
 * that sample and sets the OUT_OF_RANGE device flag.  Errors: INVALID_ARG,
 * ALIGNMENT, CUDA. */
pgti_status pgti_gather_batch(const pgti_series *s, const int32_t *dev_idx, int B, int T_in,
                              int T_out, float *x, float *y, void *stream);

/* --------------------------------------------------------------- DCRNN model */
/* Stepwise stacked DCGRU (PGT-DCRNN; Li et al. Eq. 2-3 [ext]; readings
 * c1-c7):  for t < T_in, layer l < L, with Z = [in, H] (in = x_t for l = 0,
 * H^{l-1}_t otherwise) and T(Z) = [Z, P_f Z..P_f^K Z, P_b Z..P_b^K Z]:
 *   r|u = sigma(T(Z) W_ru + b_ru),  c = tanh(T([in, r*H]) W_c + b_c),
 *   H <- u*H + (1-u)*c;   yhat_{t-(T_in-T_out)} = H^{L-1}_t W_out + b_out for the
 * last T_out steps; loss = mean |yhat - y[..., :F_out]|.
 * Parameter layout (flat float32): per layer W_ru[M][C_in][2H], b_ru[2H],
 * W_c[M][C_in][H], b_c[H]; then W_out[H][F_out], b_out[F_out]; M = 2K+1,
 * C_in = F+H (layer 0) or 2H; block 0 = identity, 1..K = P_f^k, K+1..2K = P_b^k;
 * C_in lists input channels first; gate columns r = [0,H), u = [H,2H). */
typedef struct {
  int32_t N, F, F_out, L, H, K, T_in, T_out, B;
  int32_t precision;                 /* 0 = fp32 SIMT (1e-5 parity path); 1 = bf16 tcgen05 */
  int64_t ld, nnz;
  const int32_t *a_rowptr, *a_col;   /* pattern(A)   device CSR: [N+1], [nnz] */
  const float *Pf_val, *PbT_val;     /*   values of P_f and P_b^T on it         */
  const int32_t *at_rowptr, *at_col; /* pattern(A^T) device CSR                  */
  const float *Pb_val, *PfT_val;     /*   values of P_b and P_f^T on it         */
  /* Optional shared-memory staging plan of the SpMM (pgti_graph_windows on each
   * pattern, same rows_per_window; device arrays).  win_rows = 0 or any null
   * pointer -> the SpMM reads neighbour rows straight from global memory.  The
   * plan changes where operands are read from, never the arithmetic or its order:
   * results are bit-identical either way. */
  int32_t win_rows;                  /* rows per window, 1..64 (0 = no plan)      */
  int32_t win_max;                   /* max window union size over both patterns */
  const int32_t *a_win_ptr, *a_win_nodes;   /* pattern(A) plan                   */
  const uint16_t *a_lcol;
  const int32_t *at_win_ptr, *at_win_nodes; /* pattern(A^T) plan                 */
  const uint16_t *at_lcol;
  /* Model family.  0 = the stepwise stacked PGT-DCRNN above.  1 = Li et al.'s
   * DCRNN encoder-decoder (reading c24): the L-layer
   * stack above run as the encoder over x_0..x_{T_in-1} (no readout), then a
   * second L-layer stack (the decoder, own parameters, layer-0 C_in = F_out + H)
   * for T_out steps starting from the encoder's final states; its layer-0 input
   * is the GO symbol (zeros) at step 0, then for step s >= 1 the previous
   * prediction, or the previous target y[..., :F_out] when bit s-1 of the
   * teacher_forcing mask is set (all bits: teacher forcing; the caller's
   * per-step coin flips: Li et al.'s scheduled sampling); yhat_s = H^L_s W_out +
   * b_out on every decoder step.
   * Parameters: encoder layers, decoder layers, W_out, b_out.  T_out may exceed
   * T_in.  act_dump covers the T_in + T_out steps.  Both precisions. */
  int32_t model;
  int32_t teacher_forcing;  /* bit mask over decoder steps 1..T_out-1 (model 1) */
  /* Diffusion blocks (reading c25; Li et al.'s DCRNN code [ext]): 0 = plain powers
   * P^k Z; 1 = the Chebyshev recurrence T_1 = P Z, T_k = 2 P T_{k-1} - T_{k-2}
   * per direction (T_0 = Z); the adjoint is the same polynomial in P^T. */
  int32_t cheb;
} pgti_dcrnn_desc;

/* sizeof(pgti_dcrnn_desc) as this build lays it out: bindings check their mirror of the
 * struct against it before the first call (fields are only ever appended). */
size_t pgti_dcrnn_desc_size(void);

/* Number of float parameters of the layout above (0 if desc invalid). */
size_t pgti_dcrnn_num_params(const pgti_dcrnn_desc *d);
/* Bytes of device workspace pgti_dcrnn_step needs (0 if desc invalid). */
size_t pgti_dcrnn_workspace_bytes(const pgti_dcrnn_desc *d);

/* One forward + backward (BPTT) pass over one batch ("each worker
 * computes the gradients of the loss with respect to the model parameters").
 * x [B][T_in][ld], y [B][T_out][ld] (as written by pgti_gather_batch),
 * params/grads [num_params] float32 (grads OVERWRITTEN with d loss / d theta of
 * this rank's mean loss -- unscaled by 1/R), *loss_dev (device float) = loss.
 * act_dump (nullable, test-only): if non-null it receives, after the step,
 * for t < T_in, l < L: H, r, u, c each [N][B][H] (layout [T_in][L][4][N][B][H]),
 * then yhat [T_out][N][B][F_out].  Errors: INVALID_ARG, SHAPE, ALIGNMENT,
 * WORKSPACE, UNSUPPORTED (precision), CUDA. */
pgti_status pgti_dcrnn_step(const pgti_dcrnn_desc *d, const float *params, float *grads,
                            const float *x, const float *y, float *loss_dev, void *workspace,
                            size_t ws_bytes, float *act_dump, void *stream);

/* Zero-copy index-batched step ("views, not copies"):
 * the same forward + BPTT as pgti_dcrnn_step, but the first layer's inputs and
 * the loss targets are read straight from the resident series by window start
 * -- sample b's x_t is series row dev_idx[b] + t and its y_t row dev_idx[b] +
 * T_in + t -- so no x / y batch buffers and no gather launch.  dev_idx: B device
 * int32 window starts (global rows; windows must be held by `series`, else the
 * sample reads zeros and the OUT_OF_RANGE device flag is raised).  series N, F,
 * ld must equal the desc's.  Results are bit-identical to pgti_gather_batch +
 * pgti_dcrnn_step.  Errors: as pgti_dcrnn_step, plus SHAPE (series vs desc). */
pgti_status pgti_dcrnn_step_indexed(const pgti_dcrnn_desc *d, const float *params, float *grads,
                                    const pgti_series *series, const int32_t *dev_idx,
                                    float *loss_dev, void *workspace, size_t ws_bytes,
                                    float *act_dump, void *stream);

/* Forward pass and loss only (the validation MAE of distributed-index-batching,
 * P:424): the same forward as pgti_dcrnn_step -- same kernels, same
 * workspace (workspace_bytes), same *loss_dev -- with no backward and no
 * gradients.  Errors: INVALID_ARG, SHAPE, ALIGNMENT, WORKSPACE, UNSUPPORTED, CUDA. */
pgti_status pgti_dcrnn_loss(const pgti_dcrnn_desc *d, const float *params, const float *x,
                            const float *y, float *loss_dev, void *workspace, size_t ws_bytes,
                            void *stream);

/* Diffusion features alone (test / profiling hook for the SpMM kernel):
 * X [N][W] -> out [M][N][W] = T(X) (block order as above). */
pgti_status pgti_diffuse(const pgti_dcrnn_desc *d, const float *X, int64_t W, float *out,
                         void *stream);
/* Its adjoint: dT [M][N][W] -> dZ [N][W] = sum_m (P^k)^T dT_m (Horner form). */
pgti_status pgti_diffuse_adjoint(const pgti_dcrnn_desc *d, const float *dT, int64_t W,
                                 float *dZ, void *stream);

/* ----------------------------------------------------- distributed + optimiser */
/* NCCL unique id (rank 0), to be broadcast to the other ranks (torch PG). */
pgti_status pgti_comm_unique_id(uint8_t id[128]);
/* ncclCommInitRank on CUDA device `device`.  Errors: INVALID_ARG, NCCL, CUDA. */
pgti_status pgti_comm_init(pgti_comm **out, const uint8_t id[128], int rank, int world,
                           int device);
/* Distributed-index-batching's gradient exchange ("averaged across all
 * workers through an all-reduce operation"): in-place SUM of grads[n] over the
 * ranks (NCCL, NVLink); the 1/R of the mean is applied by pgti_adam_step's
 * grad_scale.  Errors: INVALID_ARG, NCCL. */
pgti_status pgti_allreduce_grads(pgti_comm *c, float *grads, size_t n, void *stream);
/* Same collective on a float64 buffer (the stats sums of pgti_series_stats). */
pgti_status pgti_allreduce_f64(pgti_comm *c, double *buf, size_t n, void *stream);
pgti_status pgti_comm_destroy(pgti_comm *c);

/* torch-default Adam (reading c21), fp32, in place:
 *   g = grad_scale*grads; m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
 *   params -= lr * (m / (1-b1^t)) / (sqrt(v / (1-b2^t)) + eps)
 * with t = step (1-based) if step > 0; if step <= 0, t = *dev_step + 1 is read
 * from device memory and *dev_step is incremented afterwards on the stream (so
 * a captured CUDA graph replays correctly).  Errors: INVALID_ARG, CUDA. */
pgti_status pgti_adam_step(float *params, const float *grads, float *m, float *v, size_t n,
                           int64_t step, int64_t *dev_step, float lr, float beta1, float beta2,
                           float eps, float grad_scale, void *stream);

/* ----------------------------------------------------------------- instrumentation */
/* Per-kernel-class timing for the roofline report (bench.py).  While enabled, every EAGER
 * launch (not while a stream is being captured into a CUDA graph) is bracketed by two CUDA
 * events on its own stream and attributed to one class (gather, spmm, gemm_fwd, ...) with its
 * ALGORITHMIC bytes and flops.  pgti_profile_read synchronises on the
 * recorded events, writes per-class totals (ms, bytes, flops, launches; arrays of >=
 * pgti_profile_num_classes() entries) and clears the record.  Errors: INVALID_ARG, CUDA. */
pgti_status pgti_profile_enable(int on);
int pgti_profile_num_classes(void);
const char *pgti_profile_class_name(int c);
pgti_status pgti_profile_read(double *ms, double *bytes, double *flops, int64_t *launches, int n);
/* Number of kernel launches libpgti has issued (captured launches included) since load. */
uint64_t pgti_launch_count(void);
/* Per-launch timeline of the recorded (not yet read) eager launches, in launch order:
 * class, start / end in ms relative to the first record's start, and the stream handle
 * (as an integer).  *count = the number recorded; at most cap entries are written (cap 0:
 * count only).  Call before pgti_profile_read, which clears the records.  Errors:
 * INVALID_ARG, CUDA. */
pgti_status pgti_profile_timeline(int *cls, double *start_ms, double *end_ms, int64_t *stream,
                                  int cap, int *count);

#ifdef __cplusplus
}
#endif
#endif /* PGTI_H */
