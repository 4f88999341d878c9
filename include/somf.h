/*
 * somf.h -- C ABI of the B200-native SOMF hot path.
 *
 * SOMF = subsampled online matrix factorisation (Mensch, Mairal, Thirion,
 * Varoquaux, arXiv 1701.05363).  Citations "P:n" are lines of that paper's
 * source; "R<n>" are the readings listed in DESIGN.md §2.
 *
 * Problem (Eq. 1-4): X ~ D A with X p x n, D p x k in the set
 *   C = { D : ||d_j|| = (1-mu)||d_j||_1 + mu/2 ||d_j||_2^2 <= 1 (, D >= 0) }
 * and codes penalised by lambda * Omega(a), Omega(a) = (1-nu)||a||_1 + nu/2 ||a||_2^2
 * (, a >= 0).  One call of somf_partial_fit is one iteration t of Alg. 3
 * with estimator (a) (Eq. a) followed by the partial
 * dictionary update of Alg. 4 on the rows selected by M_t.
 *
 * Conventions shared by every entry point
 *  - Precision: float32 storage of D, Bbar, X and codes; Cbar, the slack
 *    norms n_j, G and beta are accumulated / kept in float64.
 *  - Layout: every p x m matrix crossing the ABI is ROW-MAJOR with a leading
 *    dimension `ld` (elements): element (row i, column s) is at ptr[i*ld + s].
 *    A handle owns rows [row_lo, row_hi) of the p features (one GPU: [0, p)),
 *    and row-major arguments hold only those rows (local row i - row_lo).
 *    Codes (k x m) are row-major with leading dimension m.
 *  - Pointers: "device" = cudaMalloc'd memory of the handle's device or
 *    pinned host memory mapped into the device address space (torch
 *    pin_memory tensors qualify; the kernels then read over PCIe/C2C).
 *    "host" = ordinary host memory.  The caller keeps ownership of every
 *    pointer it passes; inputs are only read, and only until the call's work
 *    on the stream has completed.
 *  - Ordering: all work is enqueued on config.stream (a cudaStream_t owned by
 *    the caller, e.g. torch's current stream).  Calls return after enqueueing
 *    unless they document that they synchronise (those writing host memory).
 *  - Errors: every call returns a somf_status; nothing throws across the ABI.
 *    somf_last_error(h) returns the handle's last message (thread-unsafe,
 *    valid until the next call on the handle).  A CUDA error from a kernel is
 *    reported by the next synchronising call as SOMF_E_CUDA.
 */
#ifndef SOMF_H_
#define SOMF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SOMF_ABI_VERSION 3

typedef struct somf_ctx* somf_handle;

typedef enum {
  SOMF_OK = 0,
  SOMF_E_ARG = 1,         /* invalid configuration value or argument           */
  SOMF_E_DIM = 2,         /* inconsistent size / leading dimension             */
  SOMF_E_NONFINITE = 3,   /* non-finite input detected (debug mode only)       */
  SOMF_E_STATE = 4,       /* call out of order (e.g. partial_fit before init)  */
  SOMF_E_CUDA = 5,        /* CUDA runtime / kernel error                       */
  SOMF_E_NCCL = 6,        /* collective error (sharded handles)                */
  SOMF_E_OOM = 7,         /* device allocation failed                          */
  SOMF_E_UNSUPPORTED = 8  /* valid request this build does not implement       */
} somf_status;

/* Which rows of Bbar an iteration updates (reading R5, Eq. somf_partial
 * and Alg. 3's last line P:612). */
typedef enum {
  SOMF_B_MASKED = 0,      /* P_t Bbar only: BASELINE north star (hot path)      */
  SOMF_B_UNBIASED = 1,    /* unbiased masked update (reading R6):
                           Bbar <- (1-w) Bbar on every row, kept lazily as
                           one scale sigma_t, plus (w r / eta) X_M A^T on the
                           masked rows; same bytes as MASKED, tracks FULL.
                           somf_get_state returns the true (scaled) Bbar, Cbar */
  SOMF_B_FULL = 2         /* P_t Bbar and P_t^perp Bbar: Alg. 3 as printed      */
} somf_bmode;

typedef struct somf_config {
  int64_t p;              /* rows (features)                          */
  int32_t k;              /* atoms, 1 <= k <= 256                                */
  int32_t eta;            /* mini-batch size, P:396-400, 1 <= eta <= 4096        */
  double lambda;          /* code penalty strength lambda >= 0, Eq. 1            */
  double nu;              /* Omega mix in [0,1]: 1 = ridge, 0 = lasso, Eq. 2     */
  int32_t pos_code;       /* 1: codes >= 0                            */
  double mu;              /* atom norm mix in [0,1]: 0 = l1 ball, 1 = l2 ball    */
  int32_t pos_dict;       /* 1: D >= 0                                */
  double r;               /* reduction factor r >= 1, Eq. mt           */
  double u;               /* weights w_t = t^-u, u in (0,1], P:797-799           */
  int32_t b_mode;         /* somf_bmode                                          */
  int32_t perm_cyclic;    /* 1: atoms in index order instead of Alg. 4's
                             random permutation (R13)                            */
  double cd_tol;          /* coordinate-descent stop: max|delta| <= cd_tol *
                             max(1, ||alpha||_inf) (R14; paper silent)           */
  int32_t cd_max_sweeps;  /* coordinate-descent sweep cap                        */
  uint64_t seed;          /* Philox key of every random draw (R1)                */
  int64_t row_lo;         /* first row owned by this handle (sharding)           */
  int64_t row_hi;         /* one past the last owned row; 0 means p              */
  int32_t device;         /* CUDA device ordinal                                 */
  void* stream;           /* cudaStream_t (NULL = legacy default stream)         */
  int32_t debug;          /* 1: synchronise and check after every call          */
  int32_t bcd_kernel;     /* Alg. 4 kernel: 0 = auto (simultaneous-threshold
                             when k <= 128 and the masked rows fit on chip, else
                             kernel 4, else on-chip per-atom, else global), 1 = global-memory
                             per-atom kernel, 2 = on-chip per-atom kernel,
                             3 = simultaneous-threshold kernel (k <= 128, rows
                             on chip), 4 = simultaneous-threshold kernel for
                             k <= 256 with streamed Cbar chunks and streamed
                             row tiles (auto picks it when 3 does not fit)
                             (SOMF_E_UNSUPPORTED at create if it cannot fit)   */
  /* Kernel selection of the other phases (0 = auto everywhere).  Every value
   * computes the same step (parity tests force each one); a forced variant
   * whose shape limits the call violates returns SOMF_E_UNSUPPORTED from the
   * call that needs it.                                                     */
  int32_t contract_kernel;/* (a1) beta, G (Eq. a): 0 auto, 1 tcgen05 3xTF32
                             (k <= 128, eta + k <= 512, eta % 4 == 0),
                             2 FFMA whole-slice (fused split-K), 3 FFMA tiled
                             (register tiles + reduce kernel), 4 generic FFMA */
  int32_t bbar_kernel;    /* (a3) P_t Bbar (Eq. somf_partial): 0 auto,
                             1 tcgen05 bf16x3, 2 FFMA whole-slice, 3 FFMA
                             tiled, 4 generic; mode FULL with a value other
                             than 0 / 1 runs the complement rows on a side
                             stream beside Alg. 4 (k_bbar_comp)             */
  int32_t codes_kernel;   /* (a2) codes (Eq. somf_alpha): 0 auto, 1 ridge
                             Cholesky (nu = 1, no positivity, k <= 160),
                             2 coordinate descent with exact support jumps
                             (k >= 32), 3 plain cyclic coordinate descent     */
  double bcd_lam_tol;     /* simultaneous-threshold Alg. 4: relative
                             tolerance on each projection multiplier between
                             two rounds (0 = default 1e-5)     */
  int32_t bcd_copies;     /* simultaneous-threshold Alg. 4: copies of each
                             per-atom grid accumulator (1..16, 0 = 2); a
                             performance knob only: the sums are fixed-point
                             integers, so results are bit-identical for any
                             value and any CTA arrival order                 */
  /* Code-step estimator (Table I): 0 = (a) masked G and beta
   * (Eq. a, the hot path), 1 = (b) per-sample averaged G^(i) and beta^(i)
   * (Eq. b; n_samples x k x k float64 of device memory), 2 = (c) exact Gram
   * D^T D maintained through Alg. 4's partial updates + averaged beta^(i)
   * (Eq. c; n_samples x k float64).  (b) / (c) need somf_partial_fit_ids. */
  int32_t estimator;
  int64_t n_samples;      /* n: sample ids of the stream lie in [0, n)        */
  double v;               /* gamma_c = c^-v of the per-sample averages,
                             v in (0, 1] (0.751 in P:1361)        */
  int32_t bcd_tile_rows;  /* bcd_kernel 4 (k <= 256 / streamed rows): masked
                             rows per on-chip tile (0 = as many as fit); a
                             CTA with more rows streams its tiles from an
                             L2 / HBM scratch every round.  Performance /
                             test knob only: the result does not depend on it */
  int32_t bcd_group;      /* bcd_kernel 3: threads per masked row of the
                             recurrence (0 auto, 1 one thread per row, 2 two
                             threads per row, 4 the v5 groups of 4 (8) threads
                             x 2 rows).  Performance knob; SOMF_E_UNSUPPORTED
                             when the requested group does not fit        */
} somf_config;

/* Fills *cfg with defaults: u = 0.917, r = 1, nu = 1, mu = 0,
 * lambda = 0.1, b_mode = SOMF_B_MASKED, cd_tol = 1e-7, cd_max_sweeps = 4000, v = 0.751,
 * seed = 0, row range [0, p), device 0, stream NULL, debug 0.  p, k, eta are
 * left 0 and must be set. */
void somf_config_default(somf_config* cfg);

int32_t somf_abi_version(void);
/* sizeof(somf_config) of this build, for bindings to check their layout. */
int64_t somf_config_size(void);
const char* somf_status_string(somf_status s);
const char* somf_last_error(somf_handle h);

/* Validates *cfg and allocates the handle's device state on cfg->device:
 * D and Bbar (rows x k, float32, k padded to a multiple of 4), Cbar (k x k
 * float64), slack norms n (k, float64), t = 0 and scratch.
 * SOMF_E_ARG: p < 1, k < 1 or k > 256, eta < 1 or eta > 4096, lambda < 0,
 * nu or mu outside [0,1], r < 1, u outside (0,1], unknown b_mode, empty or
 * out-of-range row range.  SOMF_E_OOM / SOMF_E_CUDA as named. */
somf_status somf_create(const somf_config* cfg, somf_handle* out);
somf_status somf_destroy(somf_handle h);

/* D_0 := D0 (device, rows x k row-major, ld >= k), each atom projected onto C
 * (reading R15: the paper leaves D_0 to the user), n_j = 1 - ||d_j||
 * (P:850-851), Bbar = 0, Cbar = 0, t = 0 (R4: w_1 = 1 overwrites them).
 * Sharded handles: the projection is of the local rows only (single-GPU
 * builds require row range [0, p)). */
somf_status somf_set_components(somf_handle h, const float* D0, int64_t ld);

/* One SOMF iteration (Alg. 3 + Alg. 4) on the mini-batch X (device,
 * rows x eta row-major, ld >= eta): t <- t+1, w_t = t^-u, draw M_t (Eq. mt),
 * beta = D^T M_t X, G = D^T M_t D (Eq. a), codes (Eq. somf_alpha: ridge closed
 * form by Cholesky when nu = 1 and no positivity and k <= 160, coordinate
 * descent otherwise), Cbar and Bbar (Eq. somf_partial; b_mode), then Alg. 4 on
 * the selected rows.  Only the selected rows of X are read (b_mode MASKED or
 * UNBIASED):
 * X may be mapped pinned host memory, in which case the q selected rows are
 * first gathered into device memory (phase SOMF_PH_STAGE), each crossing the
 * host link once.  SOMF_E_STATE before somf_set_components / somf_set_state. */
somf_status somf_partial_fit(somf_handle h, const float* X, int64_t ld);

/* somf_partial_fit for estimators (b) / (c): ids (host or device, int64[eta])
 * are the sample ids in [0, n_samples) of the batch's columns -- distinct
 * within one batch (reading R25; a repeat or an out-of-range id makes the next
 * synchronising call fail with SOMF_E_ARG).  Per column s, sample i = ids[s]:
 * c^(i) += 1, gamma = c^(i)^-v, beta^(i) <- (1 - gamma) beta^(i) + gamma beta_s
 * ((b): also G^(i)); codes from (G^(i), beta^(i)) ((b)) or
 * (D^T D, beta^(i)) ((c)); (c) then updates D^T D by the rows Alg. 4 moved
 * (P:754-756).  somf_set_components / somf_set_state reset every sample's
 * statistics (and recompute D^T D).  Estimator (a) handles accept it too
 * (ids ignored). */
somf_status somf_partial_fit_ids(somf_handle h, const float* X, int64_t ld, const int64_t* ids);

/* Draws the mask M_{t+1} of the NEXT iteration now, writes its size to
 * *q_out and, when idx_out is not NULL, its ascending local row indices
 * (host int32 array of capacity row_hi - row_lo).  Synchronises.  The next
 * partial_fit / partial_fit_masked reuses this draw (it is the same draw:
 * counter-based, R1). */
somf_status somf_next_mask(somf_handle h, int64_t* q_out, int32_t* idx_out);

/* Like somf_partial_fit, but X_M (device, q x eta row-major, ld >= eta) holds
 * only the q selected rows of the batch, in ascending row order, where q and
 * the rows are those returned by the preceding somf_next_mask.  Requires
 * b_mode MASKED or UNBIASED (FULL reads every row: SOMF_E_STATE).  SOMF_E_STATE without a preceding somf_next_mask. */
somf_status somf_partial_fit_masked(somf_handle h, const float* X_M, int64_t ld);

/* Codes alpha_t of the last iteration's batch, k x eta row-major float32,
 * copied into A_out (host or device, detected).  Synchronises when host. */
somf_status somf_get_codes(somf_handle h, float* A_out);

/* Codes of X (device, rows x m) on the current D with the exact G* = D^T D,
 * beta* = D^T X (Eq. regression), written to A_out (device,
 * k x m row-major).  Uses cd_tol / 100 for coordinate descent. */
somf_status somf_transform(somf_handle h, const float* X, int64_t ld, int64_t m,
                           float* A_out);

/* Held-out objective fbar(D) = mean_s min_a 1/2||x_s - D a||^2 + lambda Omega(a)
 * (Eq. 3) over the m columns of X (device, rows x m),
 * residuals formed directly and summed in float64, written to *obj_out
 * (host).  Synchronises. */
somf_status somf_objective(somf_handle h, const float* X, int64_t ld, int64_t m,
                           double* obj_out);

/* Current D (rows x k) into D_out (device, row-major, ld >= k). */
somf_status somf_components(somf_handle h, float* D_out, int64_t ld);

/* Whole iterate (host buffers, any may be NULL): D and Bbar rows x k
 * row-major (ld = k), Cbar k x k, n k, t.  Synchronises.  For checkpoints and
 * for parity tests that start from a mid-trajectory state. */
somf_status somf_get_state(somf_handle h, float* D, float* Bbar, double* Cbar,
                           double* n, int64_t* t);
somf_status somf_set_state(somf_handle h, const float* D, const float* Bbar,
                           const double* Cbar, const double* n, int64_t t);

/* Diagnostics of the last iteration (host out-params, any may be NULL):
 * q = |S_t|, bcd_reductions = grid-wide reductions spent in Alg. 4, w = w_t. */
somf_status somf_last_step_info(somf_handle h, int64_t* q, int64_t* bcd_reductions,
                                double* w);

/* Alg. 4 kernel this handle launches: 1 = global-memory (per-atom grid
 * reductions, rows re-read from L2/HBM), 2 = on-chip per-atom (masked rows
 * resident in registers + shared memory), 3 = on-chip simultaneous-threshold
 * rounds (all k thresholds per grid reduction).  0 on a null handle. */
int32_t somf_bcd_variant(somf_handle h);

/* Kernel variants the last somf_partial_fit ran (host int32 out[7]):
 * out[0] contraction (1 tcgen05, 2 FFMA whole-slice, 3 FFMA tiled, 4 generic),
 * out[1] codes (1 ridge Cholesky, 2 CD with support jumps, 3 plain CD),
 * out[2] P_t Bbar (1 tcgen05, 2 FFMA whole-slice, 3 FFMA tiled, 4 generic),
 * out[3] Alg. 4 (as somf_bcd_variant; 4 = row-sharded rounds),
 * out[4] 1 when mode FULL ran the complement rows on the side stream,
 * out[5], out[6] the simultaneous-threshold kernel's group shape: T threads
 * own M masked rows (1 x 1 and 2 x 1: packed-FFMA2 recurrence; 4 x 2 and
 * 8 x 2: shuffle recurrence), 0 for the other Alg. 4 kernels,
 * out[7] 1 when the Alg. 4 kernel was a programmatic dependent launch of the
 * kernel before it (its prologue overlapping that kernel's tail).
 * 0 before the first step (out holds 8 entries).  Does not synchronise. */
somf_status somf_last_kernels(somf_handle h, int32_t* out);

/* SM-cycle breakdown of the simultaneous-threshold BCD kernel (CTA 0), summed
 * over the launches made while somf_profile_enable(h, 1) was on, then reset:
 * [0] setup + residual, [1] recurrence, [2] statistics + partial reductions,
 * [3] grid barrier, [4] threshold update, [5] finish, [6] write-back,
 * [7] launches, [8 + r] atoms not yet converged after round r (r < 64);
 * [72..75] ridge code kernel (CTA 0): load, factorisation, substitutions,
 * Cbar partial; [76..78] the setup of [0] split: parameters, row gathers,
 * permutation (the residual GEMM is [0] minus these); [84..91] lasso / nonneg
 * CD (cd_as): columns, sweeps, face solves, summed face size, sweep cycles,
 * jump cycles, largest face, accepted jumps; [92] k_bcd_big rounds whose first
 * unconverged atom moved back; k_bcd_big per round r < 64: [8 + r] also holds
 * the first unconverged position << 16, [96 + r] / [160 + r] its lambda and
 * next lambda (double bits); at its round cap [72..79] that atom's state;
 * [224..231] tcgen05 contraction (CTA 0): row indices + load issue, wait for
 * the rows, wait for a buffer's previous MMAs, transpose / split, epilogue,
 * grid barrier, fixed-order reduction, launches, and [241] the MMA warp's
 * issue time ([240] reserved); [232..239] tcgen05
 * B-bar kernel (CTA 0): X rows staged, wait for the code solver, codes
 * staged, MMA issue, Cbar update, MMA + old rows wait, epilogue, launches.
 * cycles must hold SOMF_PROF_SLOTS entries.  Synchronises.  Zeros for the
 * kernels not launched. */
#define SOMF_PROF_SLOTS 248
somf_status somf_bcd_phase_cycles(somf_handle h, int64_t* cycles);

/* ---- per-phase timing of somf_partial_fit (CUDA events on config.stream) ---- */
enum {
  SOMF_PH_STAGE = 0,     /* gather of the selected rows of a host-resident batch   */
  SOMF_PH_MASK = 1,      /* t, w_t, M_t, atom permutation              (a0)        */
  SOMF_PH_CONTRACT = 2,  /* beta, G                                     (a1) Eq. a  */
  SOMF_PH_CODES = 3,     /* code solve                                  (a2)        */
  SOMF_PH_CBAR = 4,      /* Cbar                                        (a3)        */
  SOMF_PH_BBAR = 5,      /* Bbar rows                                   (a3)        */
  SOMF_PH_BCD = 6,       /* Alg. 4                                      (a4)        */
  SOMF_NPHASE = 7
};
/* on != 0: record an event pair around every phase of every following
 * iteration (a few hundred ns per phase); on == 0: stop recording. */
somf_status somf_profile_enable(somf_handle h, int32_t on);
/* Synchronises, then writes the milliseconds (ms[SOMF_NPHASE]) and kernel
 * launches (launches[SOMF_NPHASE]) accumulated per phase since the last read
 * and the number of iterations covered (*steps), and resets the counters.
 * Any pointer may be NULL.  Launch counts are kept even when timing is off. */
somf_status somf_profile_read(somf_handle h, double* ms, int64_t* launches, int64_t* steps);

/* ---- row sharding -------------------------------------------
 * A handle that owns rows [row_lo, row_hi) of a p-row problem computes only
 * the contributions of its rows to every grid-wide quantity of the step.  The
 * reducer combines them over the ranks IN PLACE, elementwise, on `stream`
 * (the handle's stream; work may be enqueued, the call may return before it
 * completes), and returns 0 on success.  dtype: SOMF_DT_F64 (double) or
 * SOMF_DT_I32 (non-negative int32: float bit patterns of values >= 0, whose
 * integer order is their float order); op: SOMF_OP_SUM / MIN / MAX.
 * Exchange points of one somf_partial_fit (every rank calls in the same order):
 *   [beta | G]  k*eta + k*k doubles, SUM            (Eq. a)
 *   radius sums ||P d_j||  2k doubles, SUM
 *   per BCD round: 3k doubles SUM, k MIN, k MAX     (R17 threshold sums)
 * and of somf_transform / somf_objective: [beta | G] of X, SUM; the residual
 * column sums, m doubles, SUM.  The code solve, Cbar and the threshold
 * updates then run identically on every rank.  fn == NULL restores the
 * single-GPU path.  With a reducer, Alg. 4 runs as one kernel per round; the
 * host reads the convergence flag once per 8 rounds (rounds after convergence
 * are no-ops whose sums are zero, so every rank still makes the same calls):
 * one or two host synchronisations per step at the configs' round counts. */
typedef int32_t (*somf_reduce_fn)(void* user, void* buf, int64_t count, int32_t dtype, int32_t op,
                                  void* stream);
enum { SOMF_DT_F64 = 0, SOMF_DT_I32 = 1 };
enum { SOMF_OP_SUM = 0, SOMF_OP_MIN = 1, SOMF_OP_MAX = 2 };
somf_status somf_set_reducer(somf_handle h, somf_reduce_fn fn, void* user);

/* ---- stateless kernels (same arithmetic as the handle's; parity tests) ---- */

/* Ascending global row indices i in [row_lo, row_hi) selected by M_t
 * (Eq. mt, R1-R2) into idx (device int32, capacity row_hi-row_lo);
 * *q_out (host) gets their number.  Synchronises. */
somf_status somf_mask_rows(uint64_t seed, int64_t t, int64_t row_lo, int64_t row_hi,
                           double r, int32_t* idx, int64_t* q_out, void* stream);

/* Alg. 4's atom order "permutation([1,k])" (R13) into perm (device int32[k]). */
somf_status somf_atom_permutation(uint64_t seed, int64_t t, int32_t k, int32_t cyclic,
                                  int32_t* perm, void* stream);

/* Column ids of stream positions s0 .. s0+count-1 (R16) into ids
 * (device int64[count]). */
somf_status somf_column_ids(uint64_t seed, int64_t n, int64_t s0, int64_t count,
                            int64_t* ids, void* stream);

/* Projects each of the m columns of U (device, len x m row-major, ld) onto
 * {d : (1-mu)||d||_1 + mu/2||d||^2 <= radius[j]} (, d >= 0), radius device
 * float64[m], writing Out (device, same layout; may alias U).  The
 * enet_projection of Alg. 4 (R17). */
somf_status somf_project_columns(const float* U, int64_t len, int32_t m, int64_t ld,
                                 const double* radius, double mu, int32_t positive,
                                 float* Out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SOMF_H_ */
