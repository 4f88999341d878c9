// somf_capi.cu -- engine and C ABI of the SOMF hot path (include/somf.h).
//
// One SOMF iteration (Alg. 3 + Alg. 4 of arXiv 1701.05363) is the launch
// sequence below, all on the caller's stream, with no host synchronisation
// (dynamic sizes such as q = |S_t| stay on the device).  Steady state at
// cfgC: four launches, the mask / t / coefficients / atom order of step t
// having been drawn by step t-1's BCD kernel (or, first step, by
// k_step_mask_count + k_mask_scatter: Eq. mt):
//   k_contract_tc     [beta | G] = r D_M^T [X_M | D_M]        (Eq. a)
//   k_ridge_codes | k_cd_as | k_cd   codes                    (Eq. somf_alpha)
//   k_bbar_tc         P_t Bbar (+ P_t^perp Bbar, mode F) and Cbar, as a
//                     programmatic dependent of the code solver
//   k_bcd_newton | k_bcd_big | k_bcd_onchip | k_bcd_seq      Alg. 4 on S_t
//                     (cooperative; draws M_{t+1} ahead)
// (FFMA fallbacks of each step, the row-sharded rounds and the estimator (b)
// / (c) kernels are selected by shape and configuration below.)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/somf.h"
#include "common.cuh"
#include "mask.cuh"
#include "gemm.cuh"
#include "contract.cuh"
#include "codes.cuh"
#include "bbar.cuh"
#include "solve.cuh"
#include "bcd.cuh"
#include "bcd_onchip.cuh"
#include "bcd_newton.cuh"
#include "bcd_big.cuh"
#include "bcd_shard.cuh"
#include "bbar_tc.cuh"
#include "contract_tc.cuh"
#include "cd_as.cuh"
#include "estimators.cuh"

using namespace somf;

#define SOMF_EXPORT extern "C" __attribute__((visibility("default")))

// ---------------------------------------------------------------------------
// small kernels
// ---------------------------------------------------------------------------
__global__ void k_step_begin(int64_t* t, double* w, double u) {
  const int64_t tt = *t + 1;
  *t = tt;
  *w = pow((double)tt, -u);
}

__global__ void k_set_scalar_i64(int64_t* p, int64_t v) { *p = v; }

// X_M[m][:] = X[idx[m]][:] for m < q: one warp per row, the rows of a host
// batch read once over the host link (many independent 4-byte requests in
// flight per warp; rows are contiguous so requests coalesce per row).
__global__ void __launch_bounds__(256)
k_gather_rows(const int32_t* __restrict__ idx, const int64_t* __restrict__ q_dev, const float* __restrict__ X,
              int64_t ldx, int eta, float* __restrict__ Xm) {
  const int64_t q = *q_dev;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec = (eta & 3) == 0 && (ldx & 3) == 0 && ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Xm)) & 15) == 0;
  if (vec) {
    // 16-byte requests (fewer, larger reads over the host link), all of a row in flight
    const int e4 = eta >> 2;
    for (int64_t m = warp; m < q; m += nwarps) {
      const float4* src = reinterpret_cast<const float4*>(X + (int64_t)idx[m] * ldx);
      float4* dst = reinterpret_cast<float4*>(Xm + m * eta);
      float4 v[4];
      for (int s0 = 0; s0 < e4; s0 += 128) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (s0 + 32 * u + lane < e4) v[u] = src[s0 + 32 * u + lane];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (s0 + 32 * u + lane < e4) dst[s0 + 32 * u + lane] = v[u];
      }
    }
    return;
  }
  for (int64_t m = warp; m < q; m += nwarps) {
    const float* src = X + (int64_t)idx[m] * ldx;
    float* dst = Xm + m * eta;
    for (int s = lane; s < eta; s += 32) dst[s] = src[s];
  }
}

__global__ void k_objective_final(const double* __restrict__ colsq, const double* __restrict__ A64,
                                  int k, int m, double lam, double nu, double* __restrict__ out) {
  __shared__ double scratch[32];
  double s[1] = {0.0};
  for (int c = threadIdx.x; c < m; c += blockDim.x) {
    double pen = 0.0;
    for (int a = 0; a < k; ++a) {
      const double v = A64[(int64_t)a * m + c];
      pen += (1.0 - nu) * fabs(v) + 0.5 * nu * v * v;
    }
    s[0] += 0.5 * colsq[c] + lam * pen;
  }
  block_sum<1>(s, scratch);
  if (threadIdx.x == 0) *out = s[0] / m;
}

// ---------------------------------------------------------------------------
// handle
// ---------------------------------------------------------------------------
struct somf_ctx {
  somf_config cfg{};
  int64_t rows = 0;          // local rows
  int kp = 0;                // k padded to a multiple of 4
  int dev = 0, nsm = 148;
  cudaStream_t st = nullptr;
  cudaStream_t st2 = nullptr;        // side stream: mode F complement rows beside the BCD
  cudaEvent_t ev_codes = nullptr, ev_comp = nullptr;
  bool comp_pending = false;
  std::string err;
  bool initialized = false;
  bool mask_ready = false;   // idx/q hold the draw of iteration t+1
  bool begin_ready = false;  // t_dev / w_dev / perm hold iteration t+1 (drawn ahead)
  bool ahead_ready = false;  // the *_next buffers hold iteration t+1 (BCD draw-ahead)
  int32_t* idx_next = nullptr;
  int* cnt_next = nullptr;
  unsigned* ct_bar = nullptr;   // fused contract reduction barrier [arrivals, exits]
  int ct_launches = 2;          // kernels the last launch_contract issued
  int kern[8] = {};             // kernel variants of the last step: contract, codes, bbar, bcd, bbar complement, BCD T, M, BCD PDL
  int64_t* q_next = nullptr;
  int64_t* t_next = nullptr;
  double* w_next = nullptr;
  int nt_mbits_off = 0;
  int64_t t_host = 0;
  double sig = 1.0;          // mode U: sigma_{t_host}, the lazy scale of the stored Bbar / Cbar (R6)
  // iterate
  float* D = nullptr;
  float* Bbar = nullptr;
  double* C64 = nullptr;
  float* C32 = nullptr;
  double* nslack = nullptr;
  // per-step scratch
  int64_t* t_dev = nullptr;
  double* w_dev = nullptr;
  int64_t* q_dev = nullptr;
  int64_t* nred_dev = nullptr;
  int* err_dev = nullptr;
  int* sweeps_dev = nullptr;
  int32_t* idx = nullptr;
  int32_t* tile_counts = nullptr;
  int ntiles = 0;
  int32_t* perm = nullptr;
  float* partial = nullptr;
  size_t partial_cap = 0;    // floats
  double* G64 = nullptr;
  double* beta64 = nullptr;
  double* A64 = nullptr;
  float* A32 = nullptr;
  float* AT32 = nullptr;     // codes transposed, eta x kp (bbar v3)
  double* cpart = nullptr;   // per-CTA partial A A^T of the ridge code kernel
  int cpart_n = 0;           // partials written by the last partial_fit code solve (0: none)
  bool at_valid = false;     // AT32 holds the last solve's codes (transposed)
  double* red = nullptr;
  unsigned* bar = nullptr;
  int bcd_grid = 0;
  int rows_cap = 0;          // rows per BCD CTA upper bound
  // on-chip BCD (bcd_onchip.cuh): chosen when the masked rows fit on chip
  int64_t q_cap = 0;         // masked-row capacity (mean + 10 sigma of |S_t|)
  const void* oc_fn = nullptr;
  int oc_cap_rows = 0, oc_cs = 0, oc_rpw = 0, oc_kc = 0;
  size_t oc_smem = 0;
  double* theta_ws = nullptr;
  const void* nt_fn = nullptr;   // simultaneous-threshold BCD (bcd_newton.cuh)
  double nt_lam_tol = kNtLamTol;
  int nt_rd_h = 1, nt_cap_rows = 0, nt_kpt = 0, nt_threads = 0, nt_ct_in_w = 0, nt_part_in_cpi = 0, nt_T = 0, nt_M = 0;
  size_t nt_smem = 0;
  double* lam_ws = nullptr;
  unsigned long long* nt_acc = nullptr;
  int nt_ncopy = 2;
  bool nt_pdl = true;            // launch k_bcd_newton as a programmatic dependent (until refused)
  // per-kernel dynamic shared memory already granted and occupancy already
  // queried (the per-step launch paths ask once, not every partial_fit)
  std::unordered_map<const void*, int> smem_set;
  std::unordered_map<uint64_t, int> occ_cache;
  // simultaneous-threshold BCD for k <= 256 / streamed rows (bcd_big.cuh)
  const void* nb_fn = nullptr;
  int nb_kpt = 0, nb_T = 0, nb_ch = 0, nb_blk = 0, nb_tr = 0, nb_threads = 0, nb_rd_h = 1;
  size_t nb_smem = 0;
  float *nb_cpi = nullptr, *nb_ctg = nullptr, *nb_invc = nullptr, *nb_scr = nullptr;
  long long* bcd_prof = nullptr;   // SM cycles per BCD phase (somf_bcd_phase_cycles)
  // row sharding (somf_set_reducer): the caller's allreduce over the ranks
  somf_reduce_fn reducer = nullptr;
  void* reducer_user = nullptr;
  ShState sh{};
  bool sh_alloc = false;
  int* sh_conv_host = nullptr;     // pinned
  unsigned long long* oc_acc = nullptr;
  unsigned* oc_accmin = nullptr;
  unsigned long long* oc_rho = nullptr;
  unsigned* oc_bar = nullptr;
  // evaluation scratch (objective / transform)
  int64_t eval_cap = 0;
  double *Ge = nullptr, *betae = nullptr, *Ae64 = nullptr, *colsq = nullptr, *objd = nullptr;
  float* Ae32 = nullptr;
  int64_t* qfull_dev = nullptr;
  // estimators (b) / (c) (estimators.cuh): per-sample statistics
  int64_t* ids_dev = nullptr;       // eta sample ids of the current batch
  int* est_cnt = nullptr;           // n visit counts c^(i)
  int* est_stamp = nullptr;         // n: iteration of the last visit (repeat check)
  double* est_bcache = nullptr;     // n x k averaged beta^(i)
  double* est_gcache = nullptr;     // n x k x k averaged G^(i)  ((b) only)
  double* est_beta = nullptr;       // k x eta: the batch's averaged beta
  double* est_G = nullptr;          // eta x k x k: the batch's averaged G ((b) only)
  double* Gex = nullptr;            // k x k exact Gram D^T D ((c) only)
  double* gnew = nullptr;           // k x 4 + k x k: contraction of the updated rows ((c) only)
  uint64_t T = 0;            // mask threshold floor(2^32 / r)
  float* Xstage = nullptr;   // device copy of the selected rows of a host batch
  // profiling
  bool prof_on = false;
  struct Ev { int ph; cudaEvent_t a, b; };
  std::vector<Ev> evs;
  std::vector<cudaEvent_t> pool;
  int64_t launches[SOMF_NPHASE] = {};
  int64_t steps_prof = 0;
};

static cudaEvent_t take_event(somf_ctx* h) {
  if (!h->pool.empty()) {
    cudaEvent_t e = h->pool.back();
    h->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) { cudaGetLastError(); return nullptr; }
  return e;
}

static void set_err(somf_ctx* h, const char* fmt, ...) {
  if (!h) return;
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  h->err = buf;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      set_err(h, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return e_ == cudaErrorMemoryAllocation ? SOMF_E_OOM : SOMF_E_CUDA;                \
    }                                                                                   \
  } while (0)

#define CKL()  CK(cudaGetLastError())

// Device-side flags: err_dev (numerical) and bar[2] (grid-barrier watchdog).
// A flag is reported once, then cleared (the call that reports it fails; the
// handle's state after a failed step is whatever the kernels left, so callers
// restore a checkpoint with somf_set_state).
static somf_status check_flags(somf_ctx* h) {
  int e = 0;
  unsigned b = 0;
  CK(cudaStreamSynchronize(h->st));
  CK(cudaMemcpy(&e, h->err_dev, sizeof(int), cudaMemcpyDeviceToHost));
  unsigned b2 = 0;
  CK(cudaMemcpy(&b, h->bar + 2, sizeof(unsigned), cudaMemcpyDeviceToHost));
  if (h->oc_bar) CK(cudaMemcpy(&b2, h->oc_bar + 2, sizeof(unsigned), cudaMemcpyDeviceToHost));
  if (!(b || b2 || e)) return SOMF_OK;
  CK(cudaMemset(h->err_dev, 0, sizeof(int)));
  CK(cudaMemset(h->bar + 2, 0, sizeof(unsigned)));
  if (h->oc_bar) CK(cudaMemset(h->oc_bar + 2, 0, sizeof(unsigned)));
  if (b || b2) { set_err(h, "grid barrier watchdog fired in the BCD kernel (results invalid)"); return SOMF_E_CUDA; }
  if (e == 2) { set_err(h, "more masked rows than the on-chip BCD capacity (q > mean + 10 sigma)"); return SOMF_E_CUDA; }
  if (e == 3 || e == 4) { set_err(h, "projection threshold search hit its round cap"); return SOMF_E_CUDA; }
  if (e == 7) { set_err(h, "a sample id is outside [0, n_samples)"); return SOMF_E_ARG; }
  if (e == 8) { set_err(h, "a sample id repeats within one mini-batch (reading R25)"); return SOMF_E_ARG; }
  if (e == 6) { set_err(h, "a BCD threshold sum left the fixed-point range [0, 2^48)"); return SOMF_E_NONFINITE; }
  if (e == 5) { set_err(h, "grid barrier watchdog fired in the contraction kernel (results invalid)"); return SOMF_E_CUDA; }
  set_err(h, "device numerical error flag %d (non-SPD system in the code solve)", e);
  return SOMF_E_NONFINITE;
}

static somf_status post_call(somf_ctx* h) {
  CKL();
  if (h->cfg.debug) {
    CK(cudaStreamSynchronize(h->st));
    return check_flags(h);
  }
  return SOMF_OK;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size
static cudaError_t smem_attr(somf_ctx* h, const void* fn, size_t smem) {
  auto it = h->smem_set.find(fn);
  if (it != h->smem_set.end() && it->second >= (int)smem) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) h->smem_set[fn] = (int)smem;
  return e;
}

// resident CTAs per SM of (fn, threads, smem), queried once (0 on error)
static int occupancy(somf_ctx* h, const void* fn, int threads, size_t smem) {
  const uint64_t key = (uint64_t)(uintptr_t)fn * 1000003ull ^ ((uint64_t)threads << 40) ^ (uint64_t)smem;
  auto it = h->occ_cache.find(key);
  if (it != h->occ_cache.end()) return it->second;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    occ = 0;
  }
  h->occ_cache[key] = occ;
  return occ;
}

// Device-readable address for a pointer that is device memory or mapped pinned host memory.
static somf_status resolve_in(somf_ctx* h, const void* p, const void** out, bool* is_host = nullptr) {
  if (is_host) *is_host = false;
  cudaPointerAttributes at{};
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) { cudaGetLastError(); set_err(h, "pointer query failed"); return SOMF_E_ARG; }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) { *out = p; return SOMF_OK; }
  if (at.type == cudaMemoryTypeHost) {
    void* d = nullptr;
    if (cudaHostGetDevicePointer(&d, const_cast<void*>(p), 0) != cudaSuccess || !d) {
      cudaGetLastError();
      set_err(h, "pinned host pointer is not mapped into the device address space");
      return SOMF_E_ARG;
    }
    *out = d;
    if (is_host) *is_host = true;
    return SOMF_OK;
  }
  set_err(h, "input must be device memory or pinned (page-locked) host memory");
  return SOMF_E_ARG;
}

template <typename T>
static cudaError_t dalloc(T** p, size_t n) {
  return cudaMalloc((void**)p, std::max<size_t>(n, 1) * sizeof(T));
}

static int split_count(const somf_ctx* h, int tiles, int64_t q_est) {
  int ns = std::max(1, (2 * h->nsm) / std::max(1, tiles));
  ns = (int)std::min<int64_t>(ns, std::max<int64_t>(1, q_est / TK));
  return std::max(1, ns);
}

static somf_status ensure_partial(somf_ctx* h, size_t floats) {
  if (floats <= h->partial_cap) return SOMF_OK;
  if (h->partial) CK(cudaFree(h->partial));
  h->partial = nullptr;
  CK(dalloc(&h->partial, floats));
  h->partial_cap = floats;
  return SOMF_OK;
}

// v2 Bbar variants (bbar.cuh): KC atoms per lane, RT rows per warp and pass
typedef void (*BbFn)(const int32_t*, const int64_t*, const float*, int64_t, int, const float*, int, float*, int,
                     const double*);
struct BbVariant { int kc, rt; BbFn fn[3]; };   // [0] gather+compact X, [1] gather, [2] all rows
#define BBV(KC, RT) {KC, RT, {k_bbar_v2<KC, RT, true, true>, k_bbar_v2<KC, RT, true, false>, \
                              k_bbar_v2<KC, RT, false, false>}}
static const BbVariant kBbVariants[] = {
    BBV(1, 2), BBV(1, 4), BBV(1, 8), BBV(1, 16), BBV(2, 2), BBV(2, 4), BBV(2, 8), BBV(2, 16),
    BBV(3, 2), BBV(3, 4), BBV(3, 8), BBV(3, 16), BBV(4, 2), BBV(4, 4), BBV(4, 8), BBV(4, 16),
    BBV(8, 2), BBV(8, 4), BBV(8, 8)};
#undef BBV

typedef void (*Bb3Fn)(const int32_t*, const int64_t*, const float*, int64_t, int, const float*, int, int, float*,
                      const double*, int, CbarFold);
struct Bb3Variant { int kc, rt; Bb3Fn fn[2]; };   // [0] compact X, [1] gathered X
#define BB3(KC, RT) {KC, RT, {k_bbar_v3<KC, RT, true>, k_bbar_v3<KC, RT, false>}}
static const Bb3Variant kBb3Variants[] = {BB3(1, 4), BB3(1, 8), BB3(1, 16), BB3(2, 4), BB3(2, 8), BB3(2, 16),
                                          BB3(3, 4), BB3(3, 8), BB3(3, 16), BB3(4, 4), BB3(4, 8), BB3(4, 16)};
#undef BB3

// shared memory of the tensor-core Bbar kernel (0: it does not apply)
static size_t bbar_tc_smem(const somf_ctx* h, const float* X, int64_t ldx) {
  const int k = h->cfg.k, eta = h->cfg.eta;
  const int sel = h->cfg.bbar_kernel;
  if ((eta % 4) || (ldx % 4) || (((uintptr_t)X) & 15) || !(sel == 0 || sel == 1) || k > 256) return 0;
  const int np = (k + 15) & ~15, ep = (eta + 15) & ~15;
  const size_t smem = (size_t)2 * (kBtM + np) * ep * 2 + (size_t)kBtM * h->kp * sizeof(float);
  return smem <= 220 * 1024 ? smem : 0;
}

// Bbar rows (masked list, or all rows when !gather) -- bbar.cuh.  false when
// the layout does not allow the 16-byte path (caller uses k_bbar_update).
// *folded (optional) is set when the Cbar update rode along (v3 kernel, cpart ready)
// all_rows: the tensor-core kernel over every row (mode F: the same update for
// the rows in and outside M_t); returns false, launching nothing, if it does
// not apply
static bool launch_bbar_v2(somf_ctx* h, bool gather, bool xcompact, const int64_t* q_dev, int64_t q_est,
                           const float* X, int64_t ldx, bool* folded = nullptr, bool all_rows = false) {
  if (folded) *folded = false;
  const int k = h->cfg.k, eta = h->cfg.eta;
  const int sel = h->cfg.bbar_kernel;      // 0 auto, 1 tc, 2 slice, 3 tiled (4 generic: the caller)
  if ((eta % 4) || (ldx % 4) || (((uintptr_t)X) & 15)) return false;
  const size_t tc_smem = bbar_tc_smem(h, X, ldx);
  if ((gather || all_rows) && tc_smem > 0) {
    // tensor cores (bbar_tc.cuh): bf16x3 tcgen05 GEMM per 128 masked rows
    BtArgs a{};
    a.np = (k + 15) & ~15;
    a.ep = (eta + 15) & ~15;
    const size_t smem = tc_smem;
    if (smem_attr(h, (const void*)k_bbar_tc, smem) == cudaSuccess) {
      a.idx = all_rows ? nullptr : h->idx;
      a.xcompact = all_rows ? 0 : xcompact;
      a.q_dev = q_dev;
      a.X = X;
      a.ldx = ldx;
      a.eta = eta;
      a.k = k;
      a.kp = h->kp;
      a.A = h->A32;
      a.Bbar = h->Bbar;
      a.w_dev = h->w_dev;
      if (folded) {
        // Cbar from the fp64 codes, every CTA a slice of the k x k entries
        a.cf = CbarFold{nullptr, 0, k * k, h->C64, h->C32, h->A64, k, eta};
        *folded = true;
      }
      // programmatic dependent launch: the CTAs stage their first X tile while
      // the code solver still runs (k_bbar_tc waits before reading the codes)
      a.pdl = 1;
      a.prof = h->prof_on ? h->bcd_prof + 232 : nullptr;   // slots 232..239 (B-bar phases)
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(h->nsm);
      cfg.blockDim = dim3(kBtThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = h->st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (cudaLaunchKernelEx(&cfg, k_bbar_tc, a) != cudaSuccess) {
        cudaGetLastError();
        if (folded) *folded = false;
        return false;
      }
      h->kern[2] = 1;
      return true;
    }
    cudaGetLastError();
  }
  if (all_rows) return false;
  int kc = (k + 31) / 32;
  if (kc > 4) kc = 8;
  const int64_t per = ceil_div(std::max<int64_t>(q_est, 1), h->nsm);
  if (gather && kc <= 4 && (sel == 0 || sel == 2) && h->at_valid) {
    // v3: whole slice in shared memory (rows of one segment per warp: RT <= 16)
    const int rt = per <= 32 ? 4 : per <= 64 ? 8 : 16;
    const int64_t seg = 8 * rt;
    const size_t smem = ((size_t)eta * 32 * kc + (size_t)seg * eta) * sizeof(float);
    const Bb3Variant* v3 = nullptr;
    for (const Bb3Variant& bv : kBb3Variants)
      if (bv.kc == kc && bv.rt == rt) v3 = &bv;
    if (v3 && smem <= 200 * 1024) {
      Bb3Fn fn = v3->fn[xcompact ? 0 : 1];
      if (smem_attr(h, (const void*)fn, smem) == cudaSuccess) {
        CbarFold cf{};
        if (folded && h->cpart_n > 0) {
          cf = CbarFold{h->cpart, h->cpart_n, k * k, h->C64, h->C32, nullptr, k, eta};
          *folded = true;
        }
        fn<<<h->nsm, kBbThreads, smem, h->st>>>(h->idx, q_dev, X, ldx, eta, h->AT32, h->kp, k, h->Bbar, h->w_dev,
                                                (int)seg, cf);
        h->kern[2] = 2;
        return true;
      }
      cudaGetLastError();
    }
  }
  if (sel != 0 && sel != 3) return false;
  const BbVariant* v = nullptr;
  for (const BbVariant& bv : kBbVariants) {
    if (bv.kc != kc) continue;
    v = &bv;                                   // largest RT for this kc if none covers per
    if (8 * bv.rt >= per) break;
  }
  const int rt = v->rt;
  const size_t smem = ((size_t)2 * kBbWarps * rt * kBbSC + (size_t)2 * kBbSC * 32 * kc) * sizeof(float);
  BbFn fn = v->fn[gather ? (xcompact ? 0 : 1) : 2];
  if (smem_attr(h, (const void*)fn, smem) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  fn<<<h->nsm, kBbThreads, smem, h->st>>>(gather ? h->idx : nullptr, q_dev, X, ldx, eta, h->A32, k, h->Bbar,
                                          h->kp, h->w_dev);
  h->kern[2] = 3;
  return true;
}

// v2 contraction variants (contract.cuh): MT = atoms / 8 per thread, NT = columns / 32 per thread
typedef void (*CtFn)(const int32_t*, const int64_t*, const float*, int, int, const float*, int64_t, int, float*);
struct CtVariant { int mt, nt; CtFn fn[3]; };   // fn[0] gather+compact X, [1] gather, [2] contiguous
#define CTV(MT, NT) {MT, NT, {k_contract_v2<MT, NT, true, true>, k_contract_v2<MT, NT, true, false>, \
                              k_contract_v2<MT, NT, false, false>}}
static const CtVariant kCtVariants[] = {
    CTV(2, 2), CTV(2, 4), CTV(2, 6), CTV(2, 9), CTV(4, 2), CTV(4, 4), CTV(4, 6), CTV(4, 9),
    CTV(9, 2), CTV(9, 4), CTV(9, 6), CTV(9, 9), CTV(16, 2), CTV(16, 4), CTV(16, 6)};
#undef CTV

// v3 (whole-slice staging) variants: single output tile per CTA
typedef void (*Ct3Fn)(const int32_t*, const int64_t*, const float*, int, int, const float*, int64_t, int, float*,
                      int, CtFuse);
struct Ct3Variant { int mt, nt; Ct3Fn fn[2]; };   // [0] compact X, [1] gathered X
#define CT3(MT, NT) {MT, NT, {k_contract_v3<MT, NT, true>, k_contract_v3<MT, NT, false>}}
static const Ct3Variant kCt3Variants[] = {CT3(2, 2), CT3(2, 4), CT3(2, 6), CT3(2, 9), CT3(4, 2), CT3(4, 4),
                                          CT3(4, 6), CT3(4, 9), CT3(9, 2), CT3(9, 4), CT3(9, 6), CT3(9, 9)};
#undef CT3

// [beta | G] over rows given by idx (or all rows), scaled by r.
// sel: 0 auto, 1 tcgen05, 2 FFMA whole-slice, 3 FFMA tiled, 4 generic (somf_config.contract_kernel)
static somf_status launch_contract(somf_ctx* h, bool gather, bool xcompact, const int64_t* q_dev,
                                   int64_t q_est, const float* X, int64_t ldx, int m, double r,
                                   double* beta, double* G, int sel = 0) {
  const int k = h->cfg.k;
  const int nc = m + k;
  h->ct_launches = 2;
  if (gather && (sel == 0 || sel == 1) && k <= kTcM) {
    // tensor cores (contract_tc.cuh): bf16x3 tcgen05 GEMMs + fused split-K reduction
    CtTcArgs a{};
    a.ep = (m + 15) & ~15;
    a.kn = (k + 15) & ~15;
    const size_t smem = (size_t)kTcBuf * 2 * (kTcM + a.ep) * kTcK * 4 + (size_t)kTcChunk * (a.ep + h->kp) * 4;
    if (a.ep + a.kn <= 512 && smem <= 226 * 1024 && m % 4 == 0 &&
        smem_attr(h, (const void*)k_contract_tc, smem) == cudaSuccess) {
      if (occupancy(h, (const void*)k_contract_tc, kCtThreads, smem) >= 1) {
        somf_status s = ensure_partial(h, (size_t)h->nsm * k * (a.ep + a.kn));
        if (s) return s;
        a.idx = h->idx;
        a.q_dev = q_dev;
        a.D = h->D;
        a.kp = h->kp;
        a.k = k;
        a.X = X;
        a.ldx = ldx;
        a.eta = m;
        a.xcompact = xcompact;
        a.partial = h->partial;
        a.fz = CtFuse{h->ct_bar, r, beta, G, h->err_dev};
        a.prof = h->prof_on ? h->bcd_prof + 224 : nullptr;  // slots 224..231 (contraction phases)
        void* args[] = {&a};
        CK(cudaLaunchCooperativeKernel((const void*)k_contract_tc, dim3(h->nsm), dim3(kCtThreads), args, smem,
                                       h->st));
        h->ct_launches = 1;
        h->kern[0] = 1;
        return SOMF_OK;
      }
    }
    cudaGetLastError();
  }
  const bool fast = (m % 4 == 0) && (ldx % 4 == 0) && (((uintptr_t)X & 15) == 0);
  if (sel == 1) {
    set_err(h, "contract_kernel = tcgen05 does not apply (k <= 128, eta + k <= 512, eta %% 4 == 0 required)");
    return SOMF_E_UNSUPPORTED;
  }
  if (fast && gather && (sel == 0 || sel == 2)) {
    const Ct3Variant* v3 = nullptr;
    for (const Ct3Variant& cv : kCt3Variants)
      if (8 * cv.mt >= k && 32 * cv.nt >= nc && (!v3 || cv.mt * cv.nt < v3->mt * v3->nt)) v3 = &cv;
    const int LDY = m + h->kp;
    const int64_t per = ceil_div(std::max<int64_t>(q_est, 1), h->nsm) + 8;
    const int64_t fit = (200 * 1024) / ((int64_t)LDY * 4 + 4);
    const int seg = (int)std::min<int64_t>(per, fit);
    if (v3 && seg >= 32) {
      somf_status s = ensure_partial(h, (size_t)h->nsm * k * nc);
      if (s) return s;
      const size_t smem = (size_t)seg * LDY * sizeof(float) + (size_t)seg * sizeof(int);
      Ct3Fn fn = v3->fn[xcompact ? 0 : 1];
      CK(smem_attr(h, (const void*)fn, smem));
      h->kern[0] = 2;
      const int occ = occupancy(h, (const void*)fn, kCtThreads, smem);
      if (occ >= 1) {
        // split-K reduction fused behind one grid barrier (cooperative launch)
        CtFuse fz{h->ct_bar, r, beta, G, h->err_dev};
        const int32_t* idxp = h->idx;
        float* Dp = h->D;
        int kp = h->kp, kk = k, mm = m, sg = seg;
        float* part = h->partial;
        int64_t ld = ldx;
        void* args[] = {(void*)&idxp, (void*)&q_dev, (void*)&Dp, (void*)&kp, (void*)&kk, (void*)&X, (void*)&ld,
                        (void*)&mm, (void*)&part, (void*)&sg, (void*)&fz};
        CK(cudaLaunchCooperativeKernel((const void*)fn, dim3(h->nsm), dim3(kCtThreads), args, smem, h->st));
        h->ct_launches = 1;
        return SOMF_OK;
      }
      cudaGetLastError();
      fn<<<h->nsm, kCtThreads, smem, h->st>>>(h->idx, q_dev, h->D, h->kp, k, X, ldx, m, h->partial, seg, CtFuse{});
      CKL();
      const int64_t tot = (int64_t)k * nc;
      k_contract_reduce2<<<(unsigned)ceil_div(tot, 32), 256, 0, h->st>>>(h->partial, h->nsm, k, m, r, beta, G);
      CKL();
      return SOMF_OK;
    }
  }
  if (sel == 2) {
    set_err(h, "contract_kernel = slice does not apply (eta %% 4 == 0, aligned rows, >= 32 rows per SM slice)");
    return SOMF_E_UNSUPPORTED;
  }
  if (fast && (sel == 0 || sel == 3)) {
    h->kern[0] = 3;
    // the fewest tiles (each gathered row is staged once per tile), then the
    // least padding; register tile MT x NT <= 96 accumulators
    const CtVariant* v = nullptr;
    long best_tiles = 0, best_pad = 0;
    for (const CtVariant& cv : kCtVariants) {
      const long ta_ = ceil_div(k, 8 * cv.mt), tc_ = ceil_div(nc, 32 * cv.nt);
      const long pad = ta_ * 8 * cv.mt * tc_ * 32 * cv.nt;
      const long tiles = ta_ * tc_;
      if (!v || tiles < best_tiles || (tiles == best_tiles && pad < best_pad)) {
        v = &cv;
        best_tiles = tiles;
        best_pad = pad;
      }
    }
    const int mt = v->mt, nt = v->nt;
    const int ta = (int)ceil_div(k, 8 * mt), tc = (int)ceil_div(nc, 32 * nt);
    // one CTA per SM in total (the row slices balance exactly)
    int ns = std::max(1, (int)(h->nsm / (ta * tc)));
    ns = (int)std::min<int64_t>(ns, std::max<int64_t>(1, q_est / (2 * kCtTK)));
    somf_status s = ensure_partial(h, (size_t)ns * k * nc);
    if (s) return s;
    const size_t smem = (size_t)kCtStages * kCtTK * (8 * mt + 32 * nt) * sizeof(float);
    CtFn fn = v->fn[gather ? (xcompact ? 0 : 1) : 2];
    CK(smem_attr(h, (const void*)fn, smem));
    fn<<<dim3(ta, tc, ns), kCtThreads, smem, h->st>>>(h->idx, q_dev, h->D, h->kp, k, X, ldx, m, h->partial);
    CKL();
    const int64_t tot = (int64_t)k * nc;
    k_contract_reduce2<<<(unsigned)ceil_div(tot, 32), 256, 0, h->st>>>(h->partial, ns, k, m, r, beta, G);
    CKL();
    return SOMF_OK;
  }
  if (sel == 3) {
    set_err(h, "contract_kernel = tiled does not apply (eta %% 4 == 0 and aligned rows required)");
    return SOMF_E_UNSUPPORTED;
  }
  h->kern[0] = 4;
  const int ta = (int)ceil_div(k, TM), tc = (int)ceil_div(nc, TN);
  const int ns = split_count(h, ta * tc, q_est);
  somf_status s = ensure_partial(h, (size_t)ns * k * nc);
  if (s) return s;
  dim3 grid(ta, tc, ns);
  if (gather) {
    if (xcompact)
      k_contract<true, true><<<grid, kGemmThreads, 0, h->st>>>(h->idx, q_dev, h->D, h->kp, k, X, ldx, m, h->partial);
    else
      k_contract<true, false><<<grid, kGemmThreads, 0, h->st>>>(h->idx, q_dev, h->D, h->kp, k, X, ldx, m, h->partial);
  } else {
    k_contract<false, false><<<grid, kGemmThreads, 0, h->st>>>(nullptr, q_dev, h->D, h->kp, k, X, ldx, m, h->partial);
  }
  CKL();
  const int64_t tot = (int64_t)k * nc;
  k_contract_reduce<<<(unsigned)ceil_div(tot, 256), 256, 0, h->st>>>(h->partial, ns, k, m, r, beta, G);
  CKL();
  return SOMF_OK;
}

// sel: 0 auto, 1 ridge Cholesky, 2 CD with support jumps, 3 plain CD (somf_config.codes_kernel)
// gstride > 0: column s uses the Gram G + s gstride (estimator (b)), one column per CTA
static somf_status launch_codes(somf_ctx* h, const double* G, const double* beta, int m, double tol,
                                double* A64, float* A32, bool want_cpart = false, int64_t gstride = 0) {
  const somf_config& c = h->cfg;
  const int k = c.k;
  const int sel = c.codes_kernel;
  h->at_valid = want_cpart;
  const int nw = kSolveThreads / 32;
  const int grid = (int)std::max<int64_t>(1, ceil_div(m, nw));
  h->cpart_n = 0;
  const bool ridge_ok = c.nu == 1.0 && !c.pos_code && k <= kRcMaxK;
  if (sel == 1 && !ridge_ok) {
    set_err(h, "codes_kernel = ridge requires nu = 1, no positivity and k <= %d", kRcMaxK);
    return SOMF_E_UNSUPPORTED;
  }
  if (ridge_ok && (sel == 0 || sel == 1)) {
    // ridge closed form (v3): every CTA factorises and solves cpc right-hand sides
    const int k4 = (k + kRcB - 1) & ~(kRcB - 1);
    const size_t smem = rc_smem_doubles(k4) * sizeof(double);
    // right-hand sides per CTA: as few as fill the SMs once (the substitution
    // chain is per warp; each CTA factorises, in parallel)
    const int cpc = gstride > 0 ? 1 : (int)std::min<int64_t>(8, std::max<int64_t>(1, ceil_div(m, h->nsm)));
    const int g = (want_cpart || gstride > 0) ? (int)ceil_div(m, cpc)
                                              : (int)std::min<int64_t>(ceil_div(m, cpc), 4 * h->nsm);
    if (want_cpart) {
      if (!h->cpart) CK(dalloc(&h->cpart, (size_t)c.eta * k * k));      // up to one partial per column
      h->cpart_n = g;
    }
    double* cp = want_cpart ? h->cpart : nullptr;
    const void* fn = nullptr;
    switch ((k4 + 31) / 32) {
      case 1: fn = (const void*)k_ridge_codes<1>; break;
      case 2: fn = (const void*)k_ridge_codes<2>; break;
      case 3: fn = (const void*)k_ridge_codes<3>; break;
      case 4: fn = (const void*)k_ridge_codes<4>; break;
      default: fn = (const void*)k_ridge_codes<5>; break;
    }
    CK(smem_attr(h, fn, smem));
    double lam = c.lambda;
    long long* rprof = h->prof_on ? h->bcd_prof + 72 : nullptr;    // slots 72..75 (ridge phases)
    float* at = want_cpart ? h->AT32 : nullptr;
    int ldt = h->kp;
    int cpc_a = cpc;
    void* args[] = {(void*)&G, (void*)&beta, (void*)&k, (void*)&m, (void*)&lam, (void*)&A64, (void*)&A32,
                    (void*)&at, (void*)&ldt, (void*)&cp, (void*)&h->err_dev, (void*)&rprof, (void*)&gstride,
                    (void*)&cpc_a};
    CK(cudaLaunchKernel(fn, dim3(g), dim3(kRcThreads), args, smem, h->st));
    h->kern[1] = 1;
    return SOMF_OK;
  }
  const double l1 = c.lambda * (1.0 - c.nu), l2 = c.lambda * c.nu;
  // the packed Gram in fp64 when it fits next to the face scratch, else fp32
  // (k = 256: 132 KB); face capacity nmax = min(k, 128) (a column whose support
  // outgrows it runs plain CD), as many warps (columns) per CTA as fit, <= 4
  const size_t np = (size_t)k * (k + 1) / 2;
  const int kpl = (int)ceil_div(k, 32);
  // Policy: enough warps per CTA that the columns fill the SMs in one wave
  // (<= 4), with the largest face that still leaves them room, but a face of
  // at least min(k, 96) (the supports at cfgB / cfgE reach ~40 / ~90); fp64
  // Gram first.
  const size_t budget = 220 * 1024;
  const int nw_want = (int)std::min<int64_t>(4, std::max<int64_t>(1, ceil_div(m, h->nsm)));
  const int nm_floor = std::min(k, 96);
  bool g64 = true;
  int nmax = 0, nw_as = 0;
  for (int gi = 0; gi < 2; ++gi) {
    const bool g = gi == 0;
    const size_t gb = np * (g ? sizeof(double) : sizeof(float));
    if (gb >= budget) continue;
    for (int nw = nw_want; nw >= 1; --nw) {
      int best = 0;
      for (int nm = std::min(k, 128); nm >= nm_floor; nm -= 8)
        if ((size_t)nw * cd_as_warp_bytes(nm, k) + gb <= budget) { best = nm; break; }
      if (best && nw > nw_as) { nmax = best; nw_as = nw; g64 = g; }
      if (best) break;
    }
    if (nw_as == nw_want) break;
  }
  if (gstride > 0) nw_as = std::min(nw_as, 1);      // a Gram per column: one column per CTA
  const size_t smem_as = nw_as > 0 ? (size_t)nw_as * cd_as_warp_bytes(nmax, k) +
                                         np * (g64 ? sizeof(double) : sizeof(float))
                                   : 0;
  const bool as_ok = k >= 8 && nw_as > 0;
  if (sel == 2 && !as_ok) {
    set_err(h, "codes_kernel = cd_jump does not fit k = %d", k);
    return SOMF_E_UNSUPPORTED;
  }
  if (as_ok && (sel == 0 || sel == 2)) {
    // CD with exact support jumps and line search (cd_as.cuh)
    const int tas = 32 * nw_as;
    const int gas = (int)ceil_div(m, nw_as);
#define LAUNCH_AS(N, GT)                                                                               \
  {                                                                                                    \
    CK(smem_attr(h, (const void*)k_cd_as<N, GT>, smem_as));                                          \
    k_cd_as<N, GT><<<gas, tas, smem_as, h->st>>>(G, beta, k, m, l1, l2, c.pos_code, tol,              \
                                                 c.cd_max_sweeps, nmax, A64, A32, h->sweeps_dev,      \
                                                 want_cpart ? h->AT32 : nullptr, h->kp, gstride,      \
                                                 h->prof_on ? h->bcd_prof : nullptr);                 \
  }
#define CASE_AS(N) \
  case N: if (g64) LAUNCH_AS(N, double) else LAUNCH_AS(N, float) break;
    switch (kpl) {
      CASE_AS(1) CASE_AS(2) CASE_AS(3) CASE_AS(4)
      CASE_AS(5) CASE_AS(6) CASE_AS(7) CASE_AS(8)
      default: set_err(h, "k too large for the CD kernel"); return SOMF_E_ARG;
    }
#undef CASE_AS
#undef LAUNCH_AS
    CKL();
    h->kern[1] = 2;
    return SOMF_OK;
  }
  const bool g64cd = np * sizeof(double) <= 200 * 1024;
  const size_t smem_cd = np * (g64cd ? sizeof(double) : sizeof(float));
#define LAUNCH_CD(N, GT)                                                                      \
  {                                                                                           \
    CK(smem_attr(h, (const void*)k_cd<N, GT>, smem_cd));                                   \
    k_cd<N, GT><<<gstride > 0 ? m : grid, gstride > 0 ? 32 : kSolveThreads, smem_cd, h->st>>>( \
        G, beta, k, m, l1, l2, c.pos_code, tol, c.cd_max_sweeps, A64, A32, h->sweeps_dev,     \
        want_cpart ? h->AT32 : nullptr, h->kp, gstride);                                     \
  }
#define CASE_CD(N) \
  case N: if (g64cd) LAUNCH_CD(N, double) else LAUNCH_CD(N, float) break;
  switch (kpl) {
    CASE_CD(1) CASE_CD(2) CASE_CD(3) CASE_CD(4)
    CASE_CD(5) CASE_CD(6) CASE_CD(7) CASE_CD(8)
    default: set_err(h, "k too large for the CD kernel"); return SOMF_E_ARG;
  }
#undef CASE_CD
#undef LAUNCH_CD
  CKL();
  h->kern[1] = 3;
  return SOMF_OK;
}

static somf_status launch_mask(somf_ctx* h, const int64_t* t_dev_ptr, int64_t idx_offset,
                               int64_t row_lo, int64_t row_hi, uint64_t T, int32_t* idx,
                               int32_t* tile_counts, int64_t* q_out, cudaStream_t st) {
  const int64_t nblk = ((row_hi - 1) >> 2) - (row_lo >> 2) + 1;
  const int ntiles = (int)ceil_div(nblk, kMaskThreads);
  k_mask_count<<<ntiles, kMaskThreads, 0, st>>>(h->cfg.seed, t_dev_ptr, row_lo, row_hi, T, tile_counts);
  CKL();
  k_mask_scatter<<<ntiles, kMaskThreads, 0, st>>>(h->cfg.seed, t_dev_ptr, row_lo, row_hi, T, tile_counts,
                                                  idx_offset, idx, q_out);
  CKL();
  return SOMF_OK;
}

// ---------------------------------------------------------------------------
// on-chip BCD variants: KC = columns per lane (ceil(kp/32), 5..7 -> 8),
// RPW = masked rows per warp; R lives in RPW*KC registers per thread.
// ---------------------------------------------------------------------------
// on-chip BCD variants (bcd_onchip_inst.cu): KC = columns per lane
// (ceil(kp/32), 5..7 -> 8), RPW = masked rows per warp; R lives in RPW*KC
// registers per thread.
struct OcVariant { int kc, rpw; };
static const OcVariant kOcVariants[] = {
    {1, 2}, {1, 4}, {1, 8}, {1, 12}, {1, 16}, {1, 24}, {1, 32},
    {2, 2}, {2, 4}, {2, 8}, {2, 12}, {2, 16}, {2, 24}, {2, 32},
    {3, 2}, {3, 4}, {3, 8}, {3, 12}, {3, 16}, {3, 24},
    {4, 2}, {4, 4}, {4, 8}, {4, 12}, {4, 16},
    {8, 2}, {8, 4}, {8, 8}};
const void* somf_oc_kernel(int kc, int rpw);

// simultaneous-threshold BCD variants (bcd_newton_inst.cu, one object per KPT)
#define NT_DECL(K) const void* somf_nt_kernel_##K(int T, int M, int gen);
NT_DECL(16) NT_DECL(32) NT_DECL(48) NT_DECL(64) NT_DECL(72) NT_DECL(80) NT_DECL(96) NT_DECL(128)
#undef NT_DECL
struct NtVariant { int kpt; const void* (*get)(int, int, int); };
static const NtVariant kNtVariants[] = {{16, somf_nt_kernel_16}, {32, somf_nt_kernel_32}, {48, somf_nt_kernel_48},
                                        {64, somf_nt_kernel_64}, {72, somf_nt_kernel_72}, {80, somf_nt_kernel_80},
                                        {96, somf_nt_kernel_96}, {128, somf_nt_kernel_128}};

static void choose_newton(somf_ctx* h) {
  const int k = h->cfg.k;
  const int cap = (int)ceil_div(h->q_cap, h->nsm);
  const int gen = h->cfg.mu > 0.0 || h->cfg.pos_dict;
  const int max_thr = NtCfg<1, 1>::kThreads;
  for (const NtVariant& v : kNtVariants) {
    if (v.kpt < k) continue;
    // (T threads, M rows) per group in order of preference: v6 one thread
    // per row (no shuffles) when the rows fill >= 3 warps, v6 two threads per
    // row, v5 4 x 2 (8 x 2 at KPT = 128)
    const int cands[3][2] = {{1, 1}, {2, 1}, {v.kpt > 96 ? 8 : 4, 2}};
    for (const auto& tm : cands) {
      const int Tv = tm[0], M = tm[1];
      const int want = h->cfg.bcd_group;
      if (want && !(want == Tv || (want == 4 && M == 2))) continue;
      if (Tv == 1 && (v.kpt > 96 || (cap < 96 && !want))) continue;
      const int64_t groups = ceil_div(cap, M);
      if (Tv * groups > max_thr) continue;
      // >= k threads: the per-atom statistics and threshold updates run one
      // thread per atom; v6 launches the full 384 (the warps past the rows skip
      // the recurrence but share the setup and the per-atom statistics)
      const int nthr = M == 1 ? max_thr
                              : (int)std::max<int64_t>(ceil_div(std::max(64, k), 32) * 32,
                                                       ceil_div((int64_t)Tv * groups, 32) * 32);
      if (nthr > max_thr) continue;
      const void* fn = v.get(Tv, M, gen);
      if (!fn) continue;
      const int LD = v.kpt + 1;
      const int KT = v.kpt / Tv, KTS = (KT + 3) & ~3;
      const size_t blk = ((size_t)(cap + 1) * LD + 3) & ~(size_t)3;
      const size_t ct = (size_t)Tv * ((((size_t)v.kpt * KTS + 31) & ~(size_t)31) + 8);   // T x CTS (bcd_newton.cuh)
      const int ct_in_w = ct <= blk;
      const size_t H = std::max(1, nthr / k);
      // stats partials (words); after the barrier the same area holds the
      // cooperative record read's partials (12 rd_h k words)
      const size_t part = std::max<size_t>(5 * H * v.kpt, (size_t)12 * k);
      const int part_in_cpi = part <= (size_t)k * v.kpt;
      const size_t avail = part_in_cpi ? (size_t)k * v.kpt : part;
      const int rd_h = (int)std::max<size_t>(1, std::min<size_t>({avail / (12 * (size_t)k), (size_t)h->nt_ncopy,
                                                                    (size_t)nthr / k}));
      const size_t base = ((size_t)4 * blk + (size_t)k * v.kpt + (ct_in_w ? 0 : ct) + (part_in_cpi ? 0 : part)) *
                              sizeof(float) + (size_t)cap * sizeof(int) + 16;
      // mask-bit scratch of the draw-ahead: one byte per Philox block of my slice
      const int64_t nb = ((h->cfg.row_hi - 1) >> 2) - (h->cfg.row_lo >> 2) + 1;
      const size_t mb_off = (base + 15) & ~(size_t)15;
      const size_t smem = mb_off + (size_t)ceil_div(nb, h->nsm) + 16;
      if (smem > 220 * 1024) continue;
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      int occ = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, nthr, smem) != cudaSuccess || occ < 1) {
        cudaGetLastError();
        continue;
      }
      h->nt_fn = fn;
      h->nt_cap_rows = cap;
      h->nt_kpt = v.kpt;
      h->nt_T = Tv;
      h->nt_M = M;
      h->nt_smem = smem;
      h->nt_threads = nthr;
      h->nt_ct_in_w = ct_in_w;
      h->nt_mbits_off = (int)mb_off;
      if (h->cfg.bcd_lam_tol > 0.0) h->nt_lam_tol = h->cfg.bcd_lam_tol;
      h->nt_part_in_cpi = part_in_cpi;
      h->nt_rd_h = rd_h;
      return;
    }
    return;     // the smallest KPT >= k did not fit: no simultaneous-threshold kernel
  }
}

#define NB_DECL(K) const void* somf_nb_kernel_##K(int gen, int* T, int* ch, int* blk);
NB_DECL(72) NB_DECL(128) NB_DECL(192) NB_DECL(256)
#undef NB_DECL
struct NbVariant { int kpt; const void* (*get)(int, int*, int*, int*); };
static const NbVariant kNbVariants[] = {{72, somf_nb_kernel_72}, {128, somf_nb_kernel_128},
                                        {192, somf_nb_kernel_192}, {256, somf_nb_kernel_256}};

// The simultaneous-threshold kernel for k <= 256 and for masked rows that do
// not fit on chip (bcd_big.cuh): the smallest KPT >= k; tile rows TR as many
// as the shared memory and the 384 threads hold (several tiles per CTA:
// streamed from the scratch).  Shared-memory layout: bcd_big.cuh.
static bool choose_big(somf_ctx* h) {
  const int k = h->cfg.k;
  const int cap = (int)ceil_div(h->q_cap, h->nsm);
  const int gen = h->cfg.mu > 0.0 || h->cfg.pos_dict;
  const int64_t nb = ((h->cfg.row_hi - 1) >> 2) - (h->cfg.row_lo >> 2) + 1;
  const size_t mb = (size_t)ceil_div(nb, h->nsm) + 16;
  for (const NbVariant& v : kNbVariants) {
    if (v.kpt < k) continue;
    int T = 0, ch = 0, blk = 0;
    const void* fn = v.get(gen, &T, &ch, &blk);
    cudaFuncAttributes fa{};
    if (!fn || cudaFuncGetAttributes(&fa, fn) != cudaSuccess) { cudaGetLastError(); return false; }
    const int kpt = v.kpt, LD = kpt + 4;          // 16-byte rows (bcd_big.cuh)
    const size_t cstr = (size_t)nb_cstr(kpt, T);
    const size_t cbf = blk ? (size_t)2 * kNbCB * kpt
                           : ch >= kpt ? (size_t)kpt * T * cstr : (size_t)2 * ch * T * cstr;
    const size_t limit = 227 * 1024 - fa.sharedSizeBytes - 512;
    int TR = std::min(cap, blk ? kNbThreads : 2 * (kNbThreads / T));
    if (h->cfg.bcd_tile_rows > 0) TR = std::max(2, std::min(TR, (int)h->cfg.bcd_tile_rows));
    size_t smem = 0;
    int nthr = 0;
    for (; TR >= 2; --TR) {
      nthr = blk ? kNbThreads
                 : (int)std::max<int64_t>(ceil_div((int64_t)T * ceil_div(TR, 2), 32) * 32, ceil_div(k, 32) * 32);
      const size_t H = std::max(1, nthr / k);
      const size_t partw = std::max<size_t>(5 * H * kpt, (size_t)12 * k);
      const size_t blkf = ((size_t)(TR + 1) * LD + 3) & ~(size_t)3;
      const size_t dlf = blk ? (size_t)(TR + 1) * kNbCB : 0;
      smem = (3 * blkf + cbf + dlf + ((partw + 3) & ~(size_t)3) + (size_t)((TR + 3) & ~3)) * sizeof(float) + mb;
      if (smem <= limit && nthr <= kNbThreads) break;
    }
    if (TR < 2) return false;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, nthr, smem) != cudaSuccess || occ < 1) {
      cudaGetLastError();
      return false;
    }
    if (dalloc(&h->nb_cpi, (size_t)kpt * kpt) != cudaSuccess || dalloc(&h->nb_invc, (size_t)kpt) != cudaSuccess ||
        (!blk && dalloc(&h->nb_ctg, (size_t)kpt * T * cstr) != cudaSuccess))
      return false;
    if ((blk || cap > TR) && dalloc(&h->nb_scr, (size_t)h->q_cap * 2 * kpt) != cudaSuccess) return false;
    const int H = std::max(1, nthr / k);
    const size_t partw = std::max<size_t>(5 * (size_t)H * kpt, (size_t)12 * k);
    h->nb_rd_h = (int)std::max<size_t>(1, std::min<size_t>({partw / (12 * (size_t)k), (size_t)h->nt_ncopy,
                                                              (size_t)nthr / k}));
    h->nb_fn = fn;
    h->nb_kpt = kpt;
    h->nb_T = T;
    h->nb_ch = ch;
    h->nb_blk = blk;
    h->nb_tr = TR;
    h->nb_threads = nthr;
    h->nb_smem = smem;
    return true;
  }
  return false;
}

// Picks the on-chip variant for this handle (h->oc_fn stays null when the
// masked rows cannot stay on chip; the global-memory kernel k_bcd_seq is used).
static void choose_onchip(somf_ctx* h) {
  const int k = h->cfg.k, kp = h->kp;
  int kc = (kp + 31) / 32;
  if (kc > 4) kc = 8;
  const int need = (int)ceil_div(h->q_cap, h->nsm);
  const int cs = k <= 160;
  for (const OcVariant& ov : kOcVariants) {
    if (ov.kc != kc || ov.rpw * kOcWarps < need) continue;
    const struct { int kc, rpw; const void* fn; } v{ov.kc, ov.rpw, somf_oc_kernel(ov.kc, ov.rpw)};
    if (!v.fn) return;
    const int cap = need;
    size_t smem = (size_t)cap * kp * sizeof(float) + (cs ? (size_t)((k * k + 3) & ~3) * sizeof(float) : 0) +
                  (size_t)((cap + 1) & ~1) * sizeof(float) + (size_t)k * (2 * sizeof(double) + sizeof(int));
    if (smem > 220 * 1024) return;
    if (cudaFuncSetAttribute(v.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, v.fn, kOcThreads, smem) != cudaSuccess || occ < 1) {
      cudaGetLastError();
      return;
    }
    h->oc_fn = v.fn;
    h->oc_cap_rows = cap;
    h->oc_cs = cs;
    h->oc_smem = smem;
    h->oc_rpw = v.rpw;
    h->oc_kc = v.kc;
    return;
  }
}

static somf_status reduce(somf_ctx* h, void* buf, int64_t n, int32_t dt, int32_t op) {
  if (!h->reducer || n <= 0) return SOMF_OK;
  const int32_t rc = h->reducer(h->reducer_user, buf, n, dt, op, (void*)h->st);
  if (rc != 0) {
    set_err(h, "reducer failed with %d", rc);
    return SOMF_E_NCCL;
  }
  return SOMF_OK;
}

static somf_status shard_alloc(somf_ctx* h) {
  if (h->sh_alloc) return SOMF_OK;
  const int k = h->cfg.k;
  const int64_t qc = std::max<int64_t>(h->q_cap, 1);
  ShState& S = h->sh;
  CK(dalloc(&S.jmap, (size_t)k));
  CK(dalloc(&S.pinv, (size_t)k));
  CK(dalloc(&S.invc, (size_t)k));
  CK(dalloc(&S.vlo, (size_t)k));
  CK(dalloc(&S.thf, (size_t)k));
  CK(dalloc(&S.scf, (size_t)k));
  CK(dalloc(&S.lam, (size_t)k));
  CK(dalloc(&S.rho, (size_t)k));
  CK(dalloc(&S.mode, (size_t)k));
  CK(dalloc(&S.Cpi, (size_t)k * k));
  CK(dalloc(&S.Dold, (size_t)qc * k));
  CK(dalloc(&S.Dn, (size_t)qc * k));
  CK(dalloc(&S.Rini, (size_t)qc * k));
  CK(dalloc(&S.acc, (size_t)3 * k));
  CK(dalloc(&S.last, (size_t)3 * k));
  CK(dalloc(&S.mn, (size_t)k));
  CK(dalloc(&S.mx, (size_t)k));
  CK(dalloc(&S.rho_acc, (size_t)2 * k));
  CK(dalloc(&S.conv, 2));
  CK(cudaMallocHost((void**)&h->sh_conv_host, 2 * sizeof(int)));
  h->sh_alloc = true;
  return SOMF_OK;
}

// Projection of the local rows of D onto C with thresholds over all ranks
// (somf_set_components on a row shard).
static somf_status project_sharded(somf_ctx* h) {
  if (somf_status s = shard_alloc(h)) return s;
  const somf_config& c = h->cfg;
  const int k = c.k;
  const double a = 1.0 - c.mu, b = c.mu;
  ShState& S = h->sh;
  k_proj_init<<<1, 256, 0, h->st>>>(S, k);
  CKL();
  bool conv = false;
  for (int it = 0; it < 200 && !conv; ++it) {
    k_proj_stats<<<k, 256, 0, h->st>>>(S, h->D, h->rows, h->kp, a, c.pos_dict);
    CKL();
    if (somf_status s = reduce(h, S.acc, 3 * k, SOMF_DT_F64, SOMF_OP_SUM)) return s;
    if (somf_status s = reduce(h, S.mn, k, SOMF_DT_I32, SOMF_OP_MIN)) return s;
    if (somf_status s = reduce(h, S.mx, k, SOMF_DT_I32, SOMF_OP_MAX)) return s;
    k_shard_update<<<1, 256, 0, h->st>>>(S, k, a, b, it, 0);
    CKL();
    CK(cudaMemcpyAsync(h->sh_conv_host, S.conv, sizeof(int), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    conv = *h->sh_conv_host != 0;
  }
  if (!conv) {
    set_err(h, "sharded projection of D0 did not converge");
    return SOMF_E_CUDA;
  }
  k_proj_apply<<<(unsigned)std::max<int64_t>(1, ceil_div(h->rows * k, 256)), 256, 0, h->st>>>(
      S, h->D, h->rows, h->kp, k, a, b, c.pos_dict, h->nslack);
  CKL();
  return SOMF_OK;
}

// Alg. 4 on a row shard (bcd_shard.cuh): one kernel per round, the caller's
// reducer between them, a host read of the convergence flag per round.
static somf_status bcd_sharded(somf_ctx* h) {
  const somf_config& c = h->cfg;
  const int k = c.k;
  const double a = 1.0 - c.mu, b = c.mu;
  const int64_t qc = std::max<int64_t>(h->q_cap, 1);
  ShState& S = h->sh;
  if (somf_status s = shard_alloc(h)) return s;
  k_shard_init<<<1, 256, 0, h->st>>>(S, h->perm, h->C64, h->C32, h->lam_ws, h->nslack, k, a, b, c.pos_dict);
  CKL();
  const int rb = 128;
  k_shard_setup<<<(unsigned)ceil_div(qc, rb), rb, 0, h->st>>>(S, h->idx, h->q_dev, h->D, h->Bbar, k, h->kp);
  CKL();
  if (somf_status s = reduce(h, S.rho_acc, 2 * k, SOMF_DT_F64, SOMF_OP_SUM)) return s;
  k_shard_rho<<<1, 256, 0, h->st>>>(S, k, a, b);
  CKL();
  const int rr = k <= 96 ? 128 : 64;
  const size_t smem = (size_t)2 * rr * (k + 1) * sizeof(float);
  CK(smem_attr(h, (const void*)k_shard_round, smem));
  int64_t launched = 0;
  const int max_rounds = 8 * k + 40;
  h->sh_conv_host[0] = h->sh_conv_host[1] = 0;
  for (int r = 0; r < max_rounds; ++r) {
    k_shard_round<<<(unsigned)ceil_div(qc, rr), rr, smem, h->st>>>(S, h->q_dev, k, a);
    CKL();
    if (somf_status s = reduce(h, S.acc, 3 * k, SOMF_DT_F64, SOMF_OP_SUM)) return s;
    if (somf_status s = reduce(h, S.mn, k, SOMF_DT_I32, SOMF_OP_MIN)) return s;
    if (somf_status s = reduce(h, S.mx, k, SOMF_DT_I32, SOMF_OP_MAX)) return s;
    k_shard_update<<<1, 256, 0, h->st>>>(S, k, a, b, r, 1);
    CKL();
    ++launched;
    if ((r + 1) % kShBatch == 0 || r + 1 == max_rounds) {
      // one host synchronisation per kShBatch rounds
      CK(cudaMemcpyAsync(h->sh_conv_host, S.conv, 2 * sizeof(int), cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
      if (h->sh_conv_host[0]) break;
    }
  }
  const bool capped = !h->sh_conv_host[0];
  const int64_t rounds = h->sh_conv_host[1];
  k_shard_finish<<<(unsigned)ceil_div(qc, rb), rb, 0, h->st>>>(S, h->idx, h->q_dev, h->D, k, h->kp, a, b,
                                                               h->nslack, h->lam_ws);
  CKL();
  k_set_scalar_i64<<<1, 1, 0, h->st>>>(h->nred_dev, rounds + 1);
  CKL();
  h->launches[SOMF_PH_BCD] += 4 + 2 * launched;
  if (capped) {
    set_err(h, "projection threshold rounds hit their cap (%d)", max_rounds);
    return SOMF_E_CUDA;
  }
  return SOMF_OK;
}

__global__ void k_init_nt_rec(unsigned long long* rec, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) nt_rec_reset(rec + (size_t)i * kNtRec);
}
static cudaError_t init_nt_rec(unsigned long long* rec, int n) {
  k_init_nt_rec<<<(n + 255) / 256, 256>>>(rec, n);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
SOMF_EXPORT void somf_config_default(somf_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->lambda = 0.1;
  c->nu = 1.0;
  c->mu = 0.0;
  c->r = 1.0;
  c->u = 0.917;
  c->v = 0.751;
  c->b_mode = SOMF_B_MASKED;
  c->cd_tol = 1e-7;
  c->cd_max_sweeps = 4000;
}

SOMF_EXPORT int32_t somf_abi_version(void) { return SOMF_ABI_VERSION; }
SOMF_EXPORT int64_t somf_config_size(void) { return (int64_t)sizeof(somf_config); }

SOMF_EXPORT const char* somf_status_string(somf_status s) {
  switch (s) {
    case SOMF_OK: return "ok";
    case SOMF_E_ARG: return "invalid argument";
    case SOMF_E_DIM: return "dimension mismatch";
    case SOMF_E_NONFINITE: return "non-finite value";
    case SOMF_E_STATE: return "invalid state";
    case SOMF_E_CUDA: return "CUDA error";
    case SOMF_E_NCCL: return "NCCL error";
    case SOMF_E_OOM: return "out of device memory";
    case SOMF_E_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

SOMF_EXPORT const char* somf_last_error(somf_handle h) { return h ? h->err.c_str() : "null handle"; }

SOMF_EXPORT somf_status somf_create(const somf_config* cfg, somf_handle* out) {
  if (!cfg || !out) return SOMF_E_ARG;
  *out = nullptr;
  somf_config c = *cfg;
  if (c.row_hi == 0) c.row_hi = c.p;
  const bool bad =
      c.p < 1 || c.k < 1 || c.k > 256 || c.eta < 1 || c.eta > 4096 || !(c.lambda >= 0.0) ||
      !(c.nu >= 0.0 && c.nu <= 1.0) || !(c.mu >= 0.0 && c.mu <= 1.0) || !(c.r >= 1.0) ||
      !(c.u > 0.0 && c.u <= 1.0) || c.row_lo < 0 || c.row_hi > c.p || c.row_lo >= c.row_hi ||
      !(c.cd_tol > 0.0) || c.cd_max_sweeps < 1 || c.row_hi - c.row_lo > (int64_t)INT32_MAX;
  if (bad) return SOMF_E_ARG;
  if (c.bcd_kernel < 0 || c.bcd_kernel > 4) return SOMF_E_ARG;
  if (c.codes_kernel < 0 || c.codes_kernel > 3 || c.contract_kernel < 0 || c.contract_kernel > 4 ||
      c.bbar_kernel < 0 || c.bbar_kernel > 4)
    return SOMF_E_ARG;
  if (c.b_mode != SOMF_B_MASKED && c.b_mode != SOMF_B_FULL && c.b_mode != SOMF_B_UNBIASED) return SOMF_E_ARG;
  if (c.estimator < 0 || c.estimator > 2) return SOMF_E_ARG;
  if (c.bcd_tile_rows < 0) return SOMF_E_ARG;
  if (c.bcd_group != 0 && c.bcd_group != 1 && c.bcd_group != 2 && c.bcd_group != 4) return SOMF_E_ARG;
  if (c.estimator != 0 && (c.n_samples < 1 || !(c.v > 0.0 && c.v <= 1.0))) return SOMF_E_ARG;
  somf_ctx* h = new somf_ctx();
  h->cfg = c;
  h->rows = c.row_hi - c.row_lo;
  h->kp = (c.k + 3) & ~3;
  h->st = (cudaStream_t)c.stream;
  h->dev = c.device;
  h->T = (uint64_t)std::floor(4294967296.0 / c.r);   // R2
  auto fail = [&](somf_status s) { *out = h; return s; };
  if (cudaSetDevice(c.device) != cudaSuccess) { set_err(h, "cudaSetDevice failed"); return fail(SOMF_E_CUDA); }
  if (cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_codes, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_comp, cudaEventDisableTiming) != cudaSuccess) {
    set_err(h, "stream / event creation failed");
    return fail(SOMF_E_CUDA);
  }
  cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, c.device);
  const int k = c.k;
  const int64_t rows = h->rows;
#define A(call) do { if ((call) != cudaSuccess) { set_err(h, "allocation failed: %s", #call); return fail(SOMF_E_OOM); } } while (0)
  A(dalloc(&h->D, (size_t)rows * h->kp));
  A(dalloc(&h->Bbar, (size_t)rows * h->kp));
  A(dalloc(&h->C64, (size_t)k * k));
  A(dalloc(&h->C32, (size_t)k * k + 4));   // +4: 16-byte staging reads in the BCD
  A(dalloc(&h->nslack, (size_t)k));
  A(dalloc(&h->t_dev, 1));
  A(dalloc(&h->w_dev, kCoefN));
  A(dalloc(&h->q_dev, 1));
  A(dalloc(&h->nred_dev, 1));
  A(dalloc(&h->err_dev, 1));
  A(dalloc(&h->sweeps_dev, 1));
  A(dalloc(&h->idx, (size_t)rows));
  A(dalloc(&h->idx_next, (size_t)rows));
  A(dalloc(&h->q_next, 1));
  A(dalloc(&h->t_next, 1));
  A(dalloc(&h->w_next, kCoefN));
  h->ntiles = (int)ceil_div(((c.row_hi - 1) >> 2) - (c.row_lo >> 2) + 1, kMaskThreads);
  A(dalloc(&h->tile_counts, (size_t)h->ntiles));
  A(dalloc(&h->perm, (size_t)k));
  A(dalloc(&h->cnt_next, (size_t)h->nsm));
  A(cudaMemset(h->cnt_next, 0, (size_t)h->nsm * sizeof(int)));
  A(dalloc(&h->ct_bar, 2));
  A(cudaMemset(h->ct_bar, 0, 2 * sizeof(unsigned)));
  // [beta | G] contiguous: one allreduce when row-sharded
  A(dalloc(&h->beta64, (size_t)k * c.eta + (size_t)k * k));
  h->G64 = h->beta64 + (size_t)k * c.eta;
  A(dalloc(&h->A64, (size_t)k * c.eta));
  A(dalloc(&h->A32, (size_t)k * c.eta));
  A(dalloc(&h->AT32, (size_t)c.eta * ((k + 3) & ~3)));
  A(dalloc(&h->bar, 4));
  A(dalloc(&h->qfull_dev, 1));
  // BCD grid: co-resident CTAs (cooperative launch), at most 2 per SM
  int occ = 0;
  h->rows_cap = (int)ceil_div(rows, h->nsm) + 1;
  size_t smem = ((size_t)((k + 3) & ~3) + h->rows_cap) * sizeof(float);
  if (smem > 200 * 1024) { set_err(h, "too many rows per SM for the v1 BCD kernel"); return fail(SOMF_E_UNSUPPORTED); }
  cudaFuncSetAttribute(k_bcd_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bcd_seq, kBcdThreads, smem);
  occ = std::max(1, std::min(occ, 2));
  h->bcd_grid = occ * h->nsm;
  h->rows_cap = (int)ceil_div(rows, h->bcd_grid) + 1;
  A(dalloc(&h->red, (size_t)2 * h->bcd_grid * kRedStride));
  {
    // |S_t| ~ Binomial(rows, 1/r): capacity mean + 10 sigma (+32)
    const double mean = (double)rows / c.r, sd = std::sqrt(mean * (1.0 - 1.0 / c.r));
    h->q_cap = c.r == 1.0 ? rows : std::min<int64_t>(rows, (int64_t)std::ceil(mean + 10.0 * sd) + 32);
  }
  A(dalloc(&h->theta_ws, (size_t)k));
  A(dalloc(&h->oc_acc, (size_t)kRing * kNC * 5));
  A(dalloc(&h->oc_accmin, (size_t)kRing * kNC));
  A(dalloc(&h->oc_rho, (size_t)4 * k));
  A(dalloc(&h->oc_bar, 4));
  A(dalloc(&h->lam_ws, (size_t)k));
  A(dalloc(&h->bcd_prof, SOMF_PROF_SLOTS));
  h->nt_ncopy = c.bcd_copies > 0 ? std::min(c.bcd_copies, kNtMaxCopies) : 2;
  A(dalloc(&h->nt_acc, (size_t)(kNtRing + 1) * h->nt_ncopy * k * kNtRec));
  if (c.estimator != 0) {
    const size_t n = (size_t)c.n_samples;
    A(dalloc(&h->ids_dev, (size_t)c.eta));
    A(dalloc(&h->est_cnt, n));
    A(dalloc(&h->est_stamp, n));
    A(dalloc(&h->est_bcache, n * k));
    A(dalloc(&h->est_beta, (size_t)k * c.eta));
    if (c.estimator == 1) {
      A(dalloc(&h->est_gcache, n * k * k));
      A(dalloc(&h->est_G, (size_t)c.eta * k * k));
    } else {
      A(dalloc(&h->Gex, (size_t)k * k));
      A(dalloc(&h->gnew, (size_t)k * 4 + (size_t)k * k));
    }
  }
  if (c.bcd_kernel == 0 || c.bcd_kernel == 3) choose_newton(h);
  if ((c.bcd_kernel == 0 && !h->nt_fn) || c.bcd_kernel == 4) choose_big(h);
  if (c.bcd_kernel == 0 ? (!h->nt_fn && !h->nb_fn) : c.bcd_kernel == 2) choose_onchip(h);
  if ((c.bcd_kernel == 2 && !h->oc_fn) || (c.bcd_kernel == 3 && !h->nt_fn) || (c.bcd_kernel == 4 && !h->nb_fn)) {
    set_err(h, "requested BCD kernel does not fit: %lld masked rows x k = %d", (long long)h->q_cap, k);
    return fail(SOMF_E_UNSUPPORTED);
  }
#undef A
  if (cudaMemset(h->bar, 0, 4 * sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(h->oc_bar, 0, 4 * sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(h->oc_acc, 0, (size_t)kRing * kNC * 5 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemset(h->oc_accmin, 0xff, (size_t)kRing * kNC * sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(h->oc_rho, 0, (size_t)4 * k * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemset(h->theta_ws, 0, (size_t)k * sizeof(double)) != cudaSuccess ||
      cudaMemset(h->lam_ws, 0, (size_t)k * sizeof(double)) != cudaSuccess ||
      cudaMemset(h->AT32, 0, (size_t)c.eta * ((k + 3) & ~3) * sizeof(float)) != cudaSuccess ||
      cudaMemset(h->bcd_prof, 0, SOMF_PROF_SLOTS * sizeof(long long)) != cudaSuccess ||
      init_nt_rec(h->nt_acc, (kNtRing + 1) * h->nt_ncopy * k) != cudaSuccess ||
      cudaMemset(h->D, 0, (size_t)rows * h->kp * sizeof(float)) != cudaSuccess ||
      cudaMemset(h->Bbar, 0, (size_t)rows * h->kp * sizeof(float)) != cudaSuccess ||
      cudaMemset(h->C64, 0, (size_t)k * k * sizeof(double)) != cudaSuccess ||
      cudaMemset(h->C32, 0, (size_t)k * k * sizeof(float)) != cudaSuccess ||
      cudaMemset(h->t_dev, 0, sizeof(int64_t)) != cudaSuccess ||
      cudaMemset(h->err_dev, 0, sizeof(int)) != cudaSuccess ||
      cudaMemset(h->sweeps_dev, 0, sizeof(int)) != cudaSuccess ||
      cudaMemset(h->nred_dev, 0, sizeof(int64_t)) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    set_err(h, "initialisation failed");
    return fail(SOMF_E_CUDA);
  }
  *out = h;
  return SOMF_OK;
}

SOMF_EXPORT somf_status somf_destroy(somf_handle h) {
  if (!h) return SOMF_E_ARG;
  void* ptrs[] = {h->D, h->Bbar, h->C64, h->C32, h->nslack, h->t_dev, h->w_dev, h->q_dev,
                  h->nred_dev, h->err_dev, h->sweeps_dev, h->idx, h->tile_counts, h->perm,
                  h->partial, h->beta64, h->A64, h->A32, h->red, h->bar,
                  h->betae, h->Ae64, h->Ae32, h->colsq, h->objd, h->qfull_dev, h->Xstage,
                  h->theta_ws, h->oc_acc, h->oc_accmin, h->oc_rho, h->oc_bar,
                  h->lam_ws, h->nt_acc, h->bcd_prof, h->idx_next, h->cnt_next, h->q_next, h->t_next, h->w_next, h->ct_bar, h->cpart, h->AT32,
                  h->ids_dev, h->est_cnt, h->est_stamp, h->est_bcache, h->est_gcache, h->est_beta, h->est_G,
                  h->Gex, h->gnew, h->nb_cpi, h->nb_ctg, h->nb_invc, h->nb_scr};
  if (h->st2) cudaStreamDestroy(h->st2);
  if (h->ev_codes) cudaEventDestroy(h->ev_codes);
  if (h->ev_comp) cudaEventDestroy(h->ev_comp);
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (h->sh_alloc) {
    void* sp[] = {h->sh.jmap, h->sh.pinv, h->sh.invc, h->sh.vlo, h->sh.thf, h->sh.scf, h->sh.lam, h->sh.rho,
                  h->sh.mode, h->sh.Cpi, h->sh.Dold, h->sh.Dn, h->sh.Rini, h->sh.acc, h->sh.last, h->sh.mn,
                  h->sh.mx, h->sh.rho_acc, h->sh.conv};
    for (void* p : sp)
      if (p) cudaFree(p);
    cudaFreeHost(h->sh_conv_host);
  }
  for (auto& e : h->evs) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
  for (auto e : h->pool) cudaEventDestroy(e);
  delete h;
  return SOMF_OK;
}

// Estimators (b) / (c): forget every sample's statistics; (c): G = D^T D of
// the current D (one contraction over all rows).
static somf_status reset_estimator(somf_ctx* h) {
  const somf_config& c = h->cfg;
  if (c.estimator == 0) return SOMF_OK;
  const int k = c.k;
  const size_t n = (size_t)c.n_samples;
  CK(cudaMemsetAsync(h->est_cnt, 0, n * sizeof(int), h->st));
  CK(cudaMemsetAsync(h->est_stamp, 0xff, n * sizeof(int), h->st));
  CK(cudaMemsetAsync(h->est_bcache, 0, n * k * sizeof(double), h->st));
  if (c.estimator == 1) CK(cudaMemsetAsync(h->est_gcache, 0, n * k * k * sizeof(double), h->st));
  if (c.estimator == 2) {
    k_set_scalar_i64<<<1, 1, 0, h->st>>>(h->qfull_dev, h->rows);
    CKL();
    if (somf_status s = launch_contract(h, false, false, h->qfull_dev, h->rows, h->D, h->kp, 4, 1.0, h->gnew,
                                        h->Gex))
      return s;
    if (somf_status s = reduce(h, h->Gex, (int64_t)k * k, SOMF_DT_F64, SOMF_OP_SUM)) return s;
  }
  return SOMF_OK;
}

SOMF_EXPORT somf_status somf_set_components(somf_handle h, const float* D0, int64_t ld) {
  if (!h || !D0) return SOMF_E_ARG;
  const int k = h->cfg.k;
  if (ld < k) { set_err(h, "ld < k"); return SOMF_E_DIM; }
  const void* src = nullptr;
  if (somf_status s = resolve_in(h, D0, &src)) return s;
  CK(cudaMemsetAsync(h->D, 0, (size_t)h->rows * h->kp * sizeof(float), h->st));
  CK(cudaMemcpy2DAsync(h->D, h->kp * sizeof(float), src, ld * sizeof(float), k * sizeof(float),
                       h->rows, cudaMemcpyDefault, h->st));
  if (h->reducer) {
    if (somf_status s = project_sharded(h)) return s;
  } else {
    k_project_columns<<<k, kBcdThreads, 0, h->st>>>(h->D, h->rows, h->kp, nullptr, 1.0, 1.0 - h->cfg.mu,
                                                    h->cfg.mu, h->cfg.pos_dict, h->D, h->nslack);
    CKL();
  }
  CK(cudaMemsetAsync(h->Bbar, 0, (size_t)h->rows * h->kp * sizeof(float), h->st));
  CK(cudaMemsetAsync(h->C64, 0, (size_t)k * k * sizeof(double), h->st));
  CK(cudaMemsetAsync(h->C32, 0, (size_t)k * k * sizeof(float), h->st));
  CK(cudaMemsetAsync(h->t_dev, 0, sizeof(int64_t), h->st));
  CK(cudaMemsetAsync(h->theta_ws, 0, (size_t)k * sizeof(double), h->st));
  CK(cudaMemsetAsync(h->lam_ws, 0, (size_t)k * sizeof(double), h->st));
  h->t_host = 0;
  h->sig = 1.0;
  h->mask_ready = h->begin_ready = h->ahead_ready = false;
  h->initialized = true;
  if (somf_status s = reset_estimator(h)) return s;
  return post_call(h);
}

// Phase timing (somf_profile_*): an event pair around each phase.
struct PhaseScope {
  somf_ctx* h;
  int ph;
  cudaEvent_t a = nullptr, b = nullptr;
  PhaseScope(somf_ctx* h_, int ph_) : h(h_), ph(ph_) {
    if (h->prof_on) {
      a = take_event(h);
      b = take_event(h);
      if (a) cudaEventRecord(a, h->st);
    }
  }
  ~PhaseScope() {
    if (a && b) {
      cudaEventRecord(b, h->st);
      h->evs.push_back({ph, a, b});
    }
  }
};

// Alg. 4's atom order pi_t on the host (R13): Fisher-Yates from the top with
// j = floor(word_w (i+1) / 2^32), word w of Philox((w>>2, t, 2, 0)) -- the
// arithmetic of atom_perm_cta (mask.cuh), bit for bit.
static void host_atom_perm(uint64_t seed, uint64_t t, int k, int cyclic, int32_t* pi) {
  for (int i = 0; i < k; ++i) pi[i] = i;
  if (cyclic) return;
  for (int w = 0; w < k - 1; ++w) {
    const U4 x = philox4x32_10(U4{(uint32_t)(w >> 2), (uint32_t)t, kStreamPerm, 0u}, seed);
    const uint32_t word = u4_word(x, w & 3);
    const int i = k - 1 - w;
    const int j = (int)(((uint64_t)word * (uint64_t)(i + 1)) >> 32);
    std::swap(pi[i], pi[j]);
  }
}

// the draw-ahead buffers of the BCD kernel become the current ones
// Aggregation coefficients of iteration t (common.cuh StepCoef), from
// sigma_{t-1} = h->sig (mode U; a stored scale below kURenorm is folded back
// into Bbar / Cbar by u_renorm before iteration t aggregates, so t's
// coefficients start from sigma = 1 then).  *sig_t = sigma_t.
constexpr double kURenorm = 1e-20;
static StepCoef step_coef(const somf_ctx* h, int64_t t, double* sig_t = nullptr) {
  const somf_config& c = h->cfg;
  const double w = std::pow((double)t, -c.u);
  StepCoef cf{};
  cf.v[kCoefW] = w;
  double sg = 1.0;
  if (c.b_mode != SOMF_B_UNBIASED) {
    cf.v[kCoefKeep] = 1.0 - w;                                               // Eq. somf_partial
    cf.v[kCoefGainB] = w;
    cf.v[kCoefGainC] = w;
  } else {
    // R6: Bbar = sigma Btilde, Cbar = sigma Ctilde, sigma_t = sigma_{t-1} (1 - w_t);
    // Btilde[S] += (w r / (eta sigma_t)) X_S A^T, Ctilde += (w / (eta sigma_t)) A A^T
    const double base = h->sig < kURenorm ? 1.0 : h->sig;
    sg = base * (1.0 - w);
    if (!(sg > 0.0)) {
      // w_t = 1 (t = 1): Bbar <- 0 on every row (u_begin zeroes the stored
      // rows), Cbar <- A A^T / eta, sigma restarts at 1
      sg = 1.0;
      cf.v[kCoefKeep] = 0.0;
      cf.v[kCoefGainB] = w * c.r;
      cf.v[kCoefGainC] = w;
    } else {
      cf.v[kCoefKeep] = 1.0;
      cf.v[kCoefGainB] = w * c.r / sg;
      cf.v[kCoefGainC] = w / sg;
    }
  }
  if (sig_t) *sig_t = sg;
  return cf;
}

__global__ void k_set_coef(double* dst, StepCoef cf) { store_coef(dst, cf); }

__global__ void k_scale_state(float* __restrict__ Bbar, int64_t n, double* __restrict__ C64,
                              float* __restrict__ C32, int kk, double s) {
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = i0; i < n; i += st) Bbar[i] = (float)(s * (double)Bbar[i]);
  for (int64_t i = i0; i < kk; i += st) {
    const double c = s * C64[i];
    C64[i] = c;
    C32[i] = (float)c;
  }
}

// Mode U: fold the stored scale back (Bbar <- sigma Btilde, Cbar <- sigma Ctilde,
// sigma <- 1) and rewrite the coefficients already drawn for iteration t+1.
static somf_status u_renorm(somf_ctx* h) {
  if (h->cfg.b_mode != SOMF_B_UNBIASED || h->sig == 1.0) return SOMF_OK;
  const int64_t n = h->rows * h->kp;
  const int kk = h->cfg.k * h->cfg.k;
  k_scale_state<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 8 * h->nsm), 256, 0, h->st>>>(
      h->Bbar, n, h->C64, h->C32, kk, h->sig);
  CKL();
  h->sig = 1.0;
  if (h->ahead_ready || h->begin_ready) {
    k_set_coef<<<1, 1, 0, h->st>>>(h->ahead_ready ? h->w_next : h->w_dev, step_coef(h, h->t_host + 1));
    CKL();
  }
  return SOMF_OK;
}

static void swap_ahead(somf_ctx* h) {
  std::swap(h->idx, h->idx_next);
  std::swap(h->q_dev, h->q_next);
  std::swap(h->t_dev, h->t_next);
  std::swap(h->w_dev, h->w_next);
  h->ahead_ready = false;
}

static somf_status partial_fit_impl(somf_handle h, const float* X, int64_t ld, bool compact,
                                    const int64_t* ids = nullptr) {
  const somf_config& c = h->cfg;
  const int k = c.k, eta = c.eta;
  if (!h->initialized) { set_err(h, "partial_fit before set_components / set_state"); return SOMF_E_STATE; }
  if (c.estimator != 0 && !ids) {
    set_err(h, "estimators (b) / (c) need the batch's sample ids: somf_partial_fit_ids");
    return SOMF_E_STATE;
  }
  if (ids) {
    // the batch's sample ids into device memory (host or device pointer)
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, ids) != cudaSuccess) cudaGetLastError();
    const bool dev = at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
    CK(cudaMemcpyAsync(h->ids_dev, ids, (size_t)eta * sizeof(int64_t),
                       dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->st));
  }
  if (ld < eta) { set_err(h, "ld < eta"); return SOMF_E_DIM; }
  bool host = false;
  const void* xs = nullptr;
  if (somf_status s = resolve_in(h, X, &xs, &host)) return s;
  const float* Xd = (const float*)xs;
  const int64_t q_est = (int64_t)std::ceil(h->rows / c.r) + 64;
  {
    PhaseScope ps(h, SOMF_PH_MASK);
    // t <- t+1, w_t, atom order and (unless drawn ahead by somf_next_mask) the
    // tile counts of M_t in one launch; the scatter of the index list in a second
    h->t_host += 1;
    if (h->ahead_ready) {
      // drawn ahead by the previous iteration's BCD kernel: swap the buffers in
      swap_ahead(h);
      h->begin_ready = h->mask_ready = true;
    }
    double sig_t = 1.0;
    if (c.b_mode == SOMF_B_UNBIASED && h->sig < kURenorm) {
      // (t's coefficients, drawn ahead or not, were computed from sigma = 1)
      const bool br = h->begin_ready;
      h->begin_ready = false;
      if (somf_status s = u_renorm(h)) return s;
      h->begin_ready = br;
    }
    const StepCoef cf = step_coef(h, h->t_host, &sig_t);
    if (c.b_mode == SOMF_B_UNBIASED && cf.v[kCoefKeep] == 0.0)                 // w_t = 1: Bbar <- 0 (R6)
      CK(cudaMemsetAsync(h->Bbar, 0, (size_t)h->rows * h->kp * sizeof(float), h->st));
    h->sig = sig_t;
    const int nt = h->mask_ready ? 0 : h->ntiles;
    if (!h->begin_ready) {
      k_step_mask_count<<<nt + 1, kMaskThreads, 0, h->st>>>(c.seed, h->t_host, cf, c.row_lo, c.row_hi, h->T, nt,
                                                            h->tile_counts, h->t_dev, h->w_dev, k, c.perm_cyclic,
                                                            h->perm);
      CKL();
      h->launches[SOMF_PH_MASK] += 1;
    }
    h->begin_ready = false;
    if (!h->mask_ready) {                                                    // M_t (Eq. mt)
      k_mask_scatter<<<h->ntiles, kMaskThreads, 0, h->st>>>(c.seed, h->t_dev, c.row_lo, c.row_hi, h->T,
                                                            h->tile_counts, c.row_lo, h->idx, h->q_dev);
      CKL();
      h->launches[SOMF_PH_MASK] += 1;
    }
    h->mask_ready = false;
  }
  if (host && !compact && c.b_mode != SOMF_B_FULL) {
    // the selected rows of a host-resident batch cross the link once
    PhaseScope ps(h, SOMF_PH_STAGE);
    if (!h->Xstage) CK(dalloc(&h->Xstage, (size_t)h->rows * eta));
    const int grid = std::max(1, std::min<int>((int)ceil_div(q_est, 8), 8 * h->nsm));
    k_gather_rows<<<grid, 256, 0, h->st>>>(h->idx, h->q_dev, Xd, ld, eta, h->Xstage);
    CKL();
    h->launches[SOMF_PH_STAGE] += 1;
    Xd = h->Xstage;
    ld = eta;
    compact = true;
  }
  {
    PhaseScope ps(h, SOMF_PH_CONTRACT);                                      // Eq. (a)
    if (somf_status s = launch_contract(h, true, compact, h->q_dev, q_est, Xd, ld, eta, c.r, h->beta64, h->G64,
                                        c.contract_kernel))
      return s;
    if (somf_status s = reduce(h, h->beta64, (int64_t)k * eta + (int64_t)k * k, SOMF_DT_F64, SOMF_OP_SUM))
      return s;
    h->launches[SOMF_PH_CONTRACT] += h->ct_launches;
  }
  // mode F: the all-rows B-bar kernel reads its row count before
  // griddepcontrol.wait, so it is written before the code solver (its primary)
  if (c.b_mode == SOMF_B_FULL) {
    k_set_scalar_i64<<<1, 1, 0, h->st>>>(h->qfull_dev, h->rows);
    CKL();
    h->launches[SOMF_PH_MASK] += 1;
  }
  h->kern[2] = 4;
  h->kern[4] = 0;
  const double* Gcodes = h->G64;
  const double* bcodes = h->beta64;
  int64_t gstride = 0;
  if (c.estimator != 0) {
    // estimators (b) / (c): per-sample averages of this step's masked estimates
    PhaseScope ps(h, SOMF_PH_CODES);
    k_est_average<<<eta, kEstThreads, 0, h->st>>>(h->ids_dev, c.n_samples, h->beta64, h->G64, k, eta, c.v,
                                                  h->t_dev, h->est_cnt, h->est_stamp, h->est_bcache,
                                                  h->est_gcache, h->est_beta, h->est_G, h->err_dev);
    CKL();
    h->launches[SOMF_PH_CODES] += 1;
    bcodes = h->est_beta;
    if (c.estimator == 1) {
      Gcodes = h->est_G;                                                     // Eq. (b): a Gram per column
      gstride = (int64_t)k * k;
    } else {
      Gcodes = h->Gex;                                                       // Eq. (c): D_{t-1}^T D_{t-1}
    }
  }
  {
    PhaseScope ps(h, SOMF_PH_CODES);                                         // Eq. somf_alpha
    // the tensor-core Bbar kernel folds Cbar from the fp64 codes itself: no
    // per-CTA partials (nor the transposed fp32 codes) from the solver then
    const bool cpart = bbar_tc_smem(h, Xd, ld) == 0;
    if (somf_status s = launch_codes(h, Gcodes, bcodes, eta, c.cd_tol, h->A64, h->A32, cpart, gstride)) return s;
    h->launches[SOMF_PH_CODES] += 1;
  }
  bool cbar_folded = false;
  {
    PhaseScope ps(h, SOMF_PH_BBAR);
    const int grid_a = (int)ceil_div(k, TN);
    if (c.b_mode == SOMF_B_FULL) {
      // mode F (P:602 + P:612): every row gets the same update.  On the tensor
      // cores in one launch over all rows when the bf16x3 kernel applies ...
      const bool all_tc = c.bbar_kernel == 0 || c.bbar_kernel == 1;
      if (all_tc && launch_bbar_v2(h, false, false, h->qfull_dev, h->rows, Xd, ld, &cbar_folded, true)) {
        h->launches[SOMF_PH_BBAR] += 1;
      } else {
        // ... else the rows in M_t first (the BCD reads them) and the rows
        // outside M_t on the side stream beside the BCD (k_bbar_comp)
        if (launch_bbar_v2(h, true, compact, h->q_dev, q_est, Xd, ld, &cbar_folded)) {
          h->launches[SOMF_PH_BBAR] += 1;
        } else {
          const int grid_r = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(q_est, TM), 8 * h->nsm));
          k_bbar_update<true, false><<<dim3(grid_r, grid_a), kGemmThreads, 0, h->st>>>(
              h->idx, h->q_dev, Xd, ld, eta, h->A32, k, h->Bbar, h->kp, h->w_dev);
          h->launches[SOMF_PH_BBAR] += 1;
          h->kern[2] = 4;
        }
        h->kern[4] = 1;
        CK(cudaEventRecord(h->ev_codes, h->st));
        CK(cudaStreamWaitEvent(h->st2, h->ev_codes, 0));
        const int grid_c = (int)std::min<int64_t>(ceil_div(h->rows, TM), 2 * h->nsm);
        k_bbar_comp<<<dim3(grid_c, grid_a), kGemmThreads, 0, h->st2>>>(Xd, ld, eta, h->A32, k, h->Bbar, h->kp,
                                                                       h->w_dev, h->rows, c.row_lo, c.seed,
                                                                       h->t_dev, h->T);
        CK(cudaEventRecord(h->ev_comp, h->st2));
        h->comp_pending = true;
        h->launches[SOMF_PH_BBAR] += 1;
      }
    } else if (launch_bbar_v2(h, true, compact, h->q_dev, q_est, Xd, ld, &cbar_folded)) {
      // (Cbar rides along when cbar_folded: Eq. somf_partial)
      h->launches[SOMF_PH_BBAR] += 1;
    } else {
      const int grid_r = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(q_est, TM), 8 * h->nsm));
      if (compact)
        k_bbar_update<true, true><<<dim3(grid_r, grid_a), kGemmThreads, 0, h->st>>>(
            h->idx, h->q_dev, Xd, ld, eta, h->A32, k, h->Bbar, h->kp, h->w_dev);
      else
        k_bbar_update<true, false><<<dim3(grid_r, grid_a), kGemmThreads, 0, h->st>>>(
            h->idx, h->q_dev, Xd, ld, eta, h->A32, k, h->Bbar, h->kp, h->w_dev);
      h->launches[SOMF_PH_BBAR] += 1;
      h->kern[2] = 4;
    }
    CKL();
    if (c.bbar_kernel != 0 && h->kern[2] != c.bbar_kernel) {
      set_err(h, "bbar_kernel %d does not apply to this shape / input (ran variant %d)", c.bbar_kernel, h->kern[2]);
      return SOMF_E_UNSUPPORTED;
    }
  }
  if (!cbar_folded) {
    PhaseScope ps(h, SOMF_PH_CBAR);                                          // Eq. somf_partial
    if (h->cpart_n > 0)
      k_cbar_finalize<<<(unsigned)ceil_div((int64_t)k * k, 256), 256, 0, h->st>>>(h->cpart, h->cpart_n, k, eta,
                                                                                h->w_dev, h->C64, h->C32);
    else
      k_cbar_update<<<dim3((unsigned)ceil_div(k, kCbT), (unsigned)ceil_div(k, kCbT)), 256, 0, h->st>>>(
          h->A64, k, eta, h->w_dev, h->C64, h->C32);
    CKL();
    h->launches[SOMF_PH_CBAR] += 1;
  }
  {
    PhaseScope ps(h, SOMF_PH_BCD);                                           // Alg. 4
    h->kern[3] = h->reducer ? 4 : h->nt_fn ? 3 : h->nb_fn ? 5 : h->oc_fn ? 2 : 1;
    h->kern[7] = 0;
    h->kern[5] = h->kern[3] == 3 ? h->nt_T : 0;
    h->kern[6] = h->kern[3] == 3 ? h->nt_M : 0;
    if (h->reducer) {
      if (somf_status s = bcd_sharded(h)) return s;
    } else if (h->nt_fn || h->nb_fn) {
      NtArgs na{};
      na.idx = h->idx;
      na.q_dev = h->q_dev;
      na.D = h->D;
      na.Bbar = h->Bbar;
      na.C64 = h->C64;
      na.C32 = h->C32;
      na.nslack = h->nslack;
      na.lam_ws = h->lam_ws;
      na.perm = h->perm;
      // pi_t drawn on the host (same Philox words and swaps as atom_perm_cta, R13)
      if (h->nt_fn) host_atom_perm(c.seed, (uint64_t)h->t_host, k, c.perm_cyclic, na.perm_v);   // (k <= 128)
      na.perm_by_value = h->nt_fn ? 1 : 0;
      na.k = k;
      na.kp = h->kp;
      na.a = 1.0 - c.mu;
      na.b = c.mu;
      na.pos = c.pos_dict;
      na.cap_rows = h->nt_cap_rows;
      na.ct_in_w = h->nt_ct_in_w;
      na.max_rounds = 8 * k + 40;          // (R22: the locked prefix advances every few rounds)
      na.lam_tol = h->nt_lam_tol;
      // draw-ahead of t+1 (mask, atom order, t, w) inside the rounds
      na.idx_next = h->idx_next;
      na.q_next = h->q_next;
      na.cnt_next = h->cnt_next;
      na.t_next = h->t_next;
      na.w_next = h->w_next;
      na.seed = c.seed;
      na.Tthr = h->T;
      na.tn = h->t_host + 1;
      na.row_lo = c.row_lo;
      na.row_hi = c.row_hi;
      na.cf_next = step_coef(h, h->t_host + 1);
      na.cyclic = c.perm_cyclic;
      na.mbits_off = h->nt_mbits_off;
      na.rec = h->nt_acc;
      na.ncopy = h->nt_ncopy;
      na.part_in_cpi = h->nt_part_in_cpi;
      na.rd_h = h->nt_rd_h;
      na.bar = h->oc_bar;
      na.nred_out = h->nred_dev;
      na.err = h->err_dev;
      na.prof = h->prof_on ? h->bcd_prof : nullptr;
      if (h->nt_fn) {
        void* kargs[] = {&na};
        // programmatic dependent launch of the cooperative grid: its prologue
        // (index list, D rows, warm starts, M_{t+1}) overlaps the B-bar
        // kernel's tail; the driver may refuse the combination (then a plain
        // cooperative launch, once and for all)
        bool launched = false;
        if (h->nt_pdl) {
          na.pdl = 1;
          cudaLaunchConfig_t lc = {};
          lc.gridDim = dim3(h->nsm);
          lc.blockDim = dim3(h->nt_threads);
          lc.dynamicSmemBytes = h->nt_smem;
          lc.stream = h->st;
          cudaLaunchAttribute at[2];
          at[0].id = cudaLaunchAttributeCooperative;
          at[0].val.cooperative = 1;
          at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[1].val.programmaticStreamSerializationAllowed = 1;
          lc.attrs = at;
          lc.numAttrs = 2;
          launched = cudaLaunchKernelExC(&lc, h->nt_fn, kargs) == cudaSuccess;
          if (!launched) {
            cudaGetLastError();
            h->nt_pdl = false;
          }
        }
        if (!launched) {
          na.pdl = 0;
          CK(cudaLaunchCooperativeKernel(h->nt_fn, dim3(h->nsm), dim3(h->nt_threads), kargs, h->nt_smem, h->st));
        }
        h->kern[7] = launched ? 1 : 0;
      } else {
        // pi, Cbar in pi order and prescaled per thread parity, then the rounds
        NbPerm pv{};
        host_atom_perm(c.seed, (uint64_t)h->t_host, k, c.perm_cyclic, pv.v);
        k_nb_prep<<<h->nb_kpt, 256, 0, h->st>>>(pv, k, h->nb_kpt, h->nb_T, h->nb_blk, h->C32, h->C64, h->perm,
                                                  h->nb_cpi, h->nb_ctg, h->nb_invc);
        CKL();
        h->launches[SOMF_PH_BCD] += 1;
        na.perm = h->perm;
        na.perm_by_value = 0;
        na.rd_h = h->nb_rd_h;
        na.cap_rows = h->nb_tr;
        NbArgs nba{};
        nba.Cpi = h->nb_cpi;
        nba.Ctg = h->nb_ctg;
        nba.invc = h->nb_invc;
        nba.scr = h->nb_scr;
        nba.tile_rows = h->nb_tr;
        nba.ch = h->nb_ch;
        void* kargs[] = {&na, &nba};
        CK(cudaLaunchCooperativeKernel(h->nb_fn, dim3(h->nsm), dim3(h->nb_threads), kargs, h->nb_smem, h->st));
      }
      h->ahead_ready = true;
    } else if (h->oc_fn) {
      OcArgs oa{};
      oa.idx = h->idx;
      oa.q_dev = h->q_dev;
      oa.D = h->D;
      oa.Bbar = h->Bbar;
      oa.C64 = h->C64;
      oa.C32 = h->C32;
      oa.nslack = h->nslack;
      oa.theta_ws = h->theta_ws;
      oa.perm = h->perm;
      oa.k = k;
      oa.kp = h->kp;
      oa.a = 1.0 - c.mu;
      oa.b = c.mu;
      oa.pos = c.pos_dict;
      oa.cs_smem = h->oc_cs;
      oa.cap_rows = h->oc_cap_rows;
      oa.acc = h->oc_acc;
      oa.accmin = h->oc_accmin;
      oa.rho_acc = h->oc_rho;
      oa.bar = h->oc_bar;
      oa.nred_out = h->nred_dev;
      oa.err = h->err_dev;
      void* kargs[] = {&oa};
      CK(cudaLaunchCooperativeKernel(h->oc_fn, dim3(h->nsm), dim3(kOcThreads), kargs, h->oc_smem, h->st));
    } else {
    BcdArgs args{};
    args.idx = h->idx;
    args.q_dev = h->q_dev;
    args.D = h->D;
    args.Bbar = h->Bbar;
    args.C64 = h->C64;
    args.C32 = h->C32;
    args.nslack = h->nslack;
    args.perm = h->perm;
    args.k = k;
    args.kp = h->kp;
    args.a = 1.0 - c.mu;
    args.b = c.mu;
    args.pos = c.pos_dict;
    args.red = h->red;
    args.bar = h->bar;
    args.nred_out = h->nred_dev;
    const size_t smem = ((size_t)((k + 3) & ~3) + h->rows_cap) * sizeof(float);
    void* kargs[] = {&args};
    CK(cudaLaunchCooperativeKernel((const void*)k_bcd_seq, dim3(h->bcd_grid), dim3(kBcdThreads), kargs,
                                   smem, h->st));
    }
    h->launches[SOMF_PH_BCD] += 1;
  }
  if (c.estimator == 2) {
    // Eq. (c): the exact Gram follows Alg. 4's partial update of the rows S_t
    PhaseScope ps(h, SOMF_PH_CONTRACT);
    if (somf_status s = launch_contract(h, true, false, h->q_dev, q_est, h->D, h->kp, 4, 1.0, h->gnew,
                                        h->gnew + (size_t)k * 4))
      return s;
    if (somf_status s = reduce(h, h->gnew + (size_t)k * 4, (int64_t)k * k, SOMF_DT_F64, SOMF_OP_SUM)) return s;
    k_gex_update<<<(unsigned)ceil_div((int64_t)k * k, 256), 256, 0, h->st>>>(h->Gex, h->G64,
                                                                            h->gnew + (size_t)k * 4, k * k,
                                                                            1.0 / c.r);
    CKL();
    h->launches[SOMF_PH_CONTRACT] += h->ct_launches + 1;
  }
  if (h->comp_pending) {
    // the caller's stream sees the complete Bbar when the call's work is done
    CK(cudaStreamWaitEvent(h->st, h->ev_comp, 0));
    h->comp_pending = false;
  }
  h->steps_prof += 1;
  return post_call(h);
}

SOMF_EXPORT somf_status somf_partial_fit(somf_handle h, const float* X, int64_t ld) {
  if (!h || !X) return SOMF_E_ARG;
  return partial_fit_impl(h, X, ld, false);
}

SOMF_EXPORT somf_status somf_partial_fit_ids(somf_handle h, const float* X, int64_t ld, const int64_t* ids) {
  if (!h || !X || !ids) return SOMF_E_ARG;
  return partial_fit_impl(h, X, ld, false, ids);
}

SOMF_EXPORT somf_status somf_next_mask(somf_handle h, int64_t* q_out, int32_t* idx_out) {
  if (!h) return SOMF_E_ARG;
  const somf_config& c = h->cfg;
  if (h->ahead_ready) {
    swap_ahead(h);                                  // M_{t+1}, pi_{t+1}, t+1, w_{t+1} already drawn
    h->begin_ready = h->mask_ready = true;
  }
  if (!h->mask_ready) {
    // draw M_{t+1}: the mask kernels read t from a device scalar
    k_set_scalar_i64<<<1, 1, 0, h->st>>>(h->qfull_dev, h->t_host + 1);
    CKL();
    if (somf_status s = launch_mask(h, h->qfull_dev, c.row_lo, c.row_lo, c.row_hi, h->T, h->idx,
                                    h->tile_counts, h->q_dev, h->st))
      return s;
    h->mask_ready = true;
  }
  int64_t q = 0;
  CK(cudaMemcpyAsync(&q, h->q_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (q_out) *q_out = q;
  if (idx_out && q > 0) {
    CK(cudaMemcpyAsync(idx_out, h->idx, (size_t)q * sizeof(int32_t), cudaMemcpyDefault, h->st));
    CK(cudaStreamSynchronize(h->st));
  }
  return SOMF_OK;
}

SOMF_EXPORT somf_status somf_partial_fit_masked(somf_handle h, const float* X_M, int64_t ld) {
  if (!h || !X_M) return SOMF_E_ARG;
  if (!h->mask_ready) { set_err(h, "partial_fit_masked without a preceding somf_next_mask"); return SOMF_E_STATE; }
  if (h->cfg.b_mode == SOMF_B_FULL) { set_err(h, "partial_fit_masked: b_mode FULL reads every row"); return SOMF_E_STATE; }
  return partial_fit_impl(h, X_M, ld, true);
}

SOMF_EXPORT somf_status somf_get_codes(somf_handle h, float* A_out) {
  if (!h || !A_out) return SOMF_E_ARG;
  CK(cudaMemcpyAsync(A_out, h->A32, (size_t)h->cfg.k * h->cfg.eta * sizeof(float), cudaMemcpyDefault, h->st));
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, A_out) != cudaSuccess) cudaGetLastError();
  if (at.type != cudaMemoryTypeDevice) CK(cudaStreamSynchronize(h->st));
  return post_call(h);
}

static somf_status ensure_eval(somf_ctx* h, int64_t m) {
  if (m <= h->eval_cap) return SOMF_OK;
  void* ps[] = {h->betae, h->Ae64, h->Ae32, h->colsq, h->objd};
  for (void* p : ps)
    if (p) CK(cudaFree(p));
  const int k = h->cfg.k;
  CK(dalloc(&h->betae, (size_t)k * m + (size_t)k * k));
  h->Ge = h->betae + (size_t)k * m;
  CK(dalloc(&h->Ae64, (size_t)k * m));
  CK(dalloc(&h->Ae32, (size_t)k * m));
  CK(dalloc(&h->colsq, (size_t)m));
  CK(dalloc(&h->objd, 1));
  h->eval_cap = m;
  return SOMF_OK;
}

static somf_status eval_codes(somf_ctx* h, const float* X, int64_t ld, int64_t m) {
  if (!h->initialized) { set_err(h, "no dictionary yet"); return SOMF_E_STATE; }
  if (m < 1 || m > (1 << 20)) { set_err(h, "m out of range"); return SOMF_E_ARG; }
  if (ld < m) { set_err(h, "ld < m"); return SOMF_E_DIM; }
  if (somf_status s = ensure_eval(h, m)) return s;
  k_set_scalar_i64<<<1, 1, 0, h->st>>>(h->qfull_dev, h->rows);
  CKL();
  if (somf_status s = launch_contract(h, false, false, h->qfull_dev, h->rows, X, ld, (int)m, 1.0, h->betae, h->Ge))
    return s;
  if (somf_status s = reduce(h, h->betae, (int64_t)h->cfg.k * m + (int64_t)h->cfg.k * h->cfg.k, SOMF_DT_F64,
                             SOMF_OP_SUM))
    return s;
  return launch_codes(h, h->Ge, h->betae, (int)m, h->cfg.cd_tol * 1e-2, h->Ae64, h->Ae32);
}

SOMF_EXPORT somf_status somf_transform(somf_handle h, const float* X, int64_t ld, int64_t m, float* A_out) {
  if (!h || !X || !A_out) return SOMF_E_ARG;
  const void* xs = nullptr;
  if (somf_status s = resolve_in(h, X, &xs)) return s;
  if (somf_status s = eval_codes(h, (const float*)xs, ld, m)) return s;
  CK(cudaMemcpyAsync(A_out, h->Ae32, (size_t)h->cfg.k * m * sizeof(float), cudaMemcpyDefault, h->st));
  return post_call(h);
}

SOMF_EXPORT somf_status somf_objective(somf_handle h, const float* X, int64_t ld, int64_t m, double* obj_out) {
  if (!h || !X || !obj_out) return SOMF_E_ARG;
  const void* xs = nullptr;
  if (somf_status s = resolve_in(h, X, &xs)) return s;
  if (somf_status s = eval_codes(h, (const float*)xs, ld, m)) return s;
  const int k = h->cfg.k;
  CK(cudaMemsetAsync(h->colsq, 0, (size_t)m * sizeof(double), h->st));
  const int grid_r = (int)std::min<int64_t>(ceil_div(h->rows, TM), 4 * h->nsm);
  k_residual<<<dim3(grid_r, (unsigned)ceil_div(m, TN)), kGemmThreads, 0, h->st>>>(
      h->D, h->kp, k, h->rows, (const float*)xs, ld, (int)m, h->Ae32, h->colsq);
  CKL();
  if (somf_status s = reduce(h, h->colsq, m, SOMF_DT_F64, SOMF_OP_SUM)) return s;
  k_objective_final<<<1, 256, 0, h->st>>>(h->colsq, h->Ae64, k, (int)m, h->cfg.lambda, h->cfg.nu, h->objd);
  CKL();
  CK(cudaMemcpyAsync(obj_out, h->objd, sizeof(double), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return post_call(h);
}

SOMF_EXPORT somf_status somf_components(somf_handle h, float* D_out, int64_t ld) {
  if (!h || !D_out) return SOMF_E_ARG;
  if (ld < h->cfg.k) { set_err(h, "ld < k"); return SOMF_E_DIM; }
  CK(cudaMemcpy2DAsync(D_out, ld * sizeof(float), h->D, h->kp * sizeof(float), h->cfg.k * sizeof(float),
                       h->rows, cudaMemcpyDefault, h->st));
  return post_call(h);
}

SOMF_EXPORT somf_status somf_get_state(somf_handle h, float* D, float* Bbar, double* Cbar, double* n,
                                       int64_t* t) {
  if (!h) return SOMF_E_ARG;
  const int k = h->cfg.k;
  if (somf_status s = u_renorm(h)) return s;      // mode U: the true Bbar / Cbar (R6)
  if (D)
    CK(cudaMemcpy2DAsync(D, k * sizeof(float), h->D, h->kp * sizeof(float), k * sizeof(float), h->rows,
                         cudaMemcpyDefault, h->st));
  if (Bbar)
    CK(cudaMemcpy2DAsync(Bbar, k * sizeof(float), h->Bbar, h->kp * sizeof(float), k * sizeof(float), h->rows,
                         cudaMemcpyDefault, h->st));
  if (Cbar) CK(cudaMemcpyAsync(Cbar, h->C64, (size_t)k * k * sizeof(double), cudaMemcpyDefault, h->st));
  if (n) CK(cudaMemcpyAsync(n, h->nslack, (size_t)k * sizeof(double), cudaMemcpyDefault, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (t) *t = h->t_host;
  if (somf_status st = check_flags(h)) return st;
  return post_call(h);
}

__global__ void k_c64_to_c32(const double* a, float* b, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (float)a[i];
}

SOMF_EXPORT somf_status somf_set_state(somf_handle h, const float* D, const float* Bbar, const double* Cbar,
                                       const double* n, int64_t t) {
  if (!h || !D || !Bbar || !Cbar || !n || t < 0) return SOMF_E_ARG;
  const int k = h->cfg.k;
  CK(cudaMemsetAsync(h->D, 0, (size_t)h->rows * h->kp * sizeof(float), h->st));
  CK(cudaMemsetAsync(h->Bbar, 0, (size_t)h->rows * h->kp * sizeof(float), h->st));
  CK(cudaMemcpy2DAsync(h->D, h->kp * sizeof(float), D, k * sizeof(float), k * sizeof(float), h->rows,
                       cudaMemcpyDefault, h->st));
  CK(cudaMemcpy2DAsync(h->Bbar, h->kp * sizeof(float), Bbar, k * sizeof(float), k * sizeof(float), h->rows,
                       cudaMemcpyDefault, h->st));
  CK(cudaMemcpyAsync(h->C64, Cbar, (size_t)k * k * sizeof(double), cudaMemcpyDefault, h->st));
  CK(cudaMemcpyAsync(h->nslack, n, (size_t)k * sizeof(double), cudaMemcpyDefault, h->st));
  k_c64_to_c32<<<(unsigned)ceil_div((int64_t)k * k, 256), 256, 0, h->st>>>(h->C64, h->C32, k * k);
  CKL();
  k_set_scalar_i64<<<1, 1, 0, h->st>>>(h->t_dev, t);
  CKL();
  CK(cudaMemsetAsync(h->theta_ws, 0, (size_t)k * sizeof(double), h->st));
  CK(cudaMemsetAsync(h->lam_ws, 0, (size_t)k * sizeof(double), h->st));
  CK(cudaStreamSynchronize(h->st));
  h->t_host = t;
  h->sig = 1.0;
  h->mask_ready = h->begin_ready = h->ahead_ready = false;
  h->initialized = true;
  if (somf_status s = reset_estimator(h)) return s;
  return post_call(h);
}

SOMF_EXPORT somf_status somf_last_step_info(somf_handle h, int64_t* q, int64_t* nred, double* w) {
  if (!h) return SOMF_E_ARG;
  if (q) CK(cudaMemcpyAsync(q, h->q_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, h->st));
  if (nred) CK(cudaMemcpyAsync(nred, h->nred_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, h->st));
  if (w) CK(cudaMemcpyAsync(w, h->w_dev, sizeof(double), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return check_flags(h);
}

SOMF_EXPORT somf_status somf_set_reducer(somf_handle h, somf_reduce_fn fn, void* user) {
  if (!h) return SOMF_E_ARG;
  h->reducer = fn;
  h->reducer_user = user;
  // the next step redraws t+1 (mask and the device copy of pi) itself: the
  // draw-ahead buffers of the single-GPU kernel are not used by the sharded path
  h->mask_ready = h->begin_ready = h->ahead_ready = false;
  return SOMF_OK;
}

SOMF_EXPORT somf_status somf_bcd_phase_cycles(somf_handle h, int64_t* cycles) {
  if (!h || !cycles) return SOMF_E_ARG;
  CK(cudaStreamSynchronize(h->st));
  long long v[SOMF_PROF_SLOTS];
  CK(cudaMemcpy(v, h->bcd_prof, sizeof(v), cudaMemcpyDeviceToHost));
  CK(cudaMemset(h->bcd_prof, 0, sizeof(v)));
  for (int i = 0; i < SOMF_PROF_SLOTS; ++i) cycles[i] = v[i];
  return SOMF_OK;
}

SOMF_EXPORT int32_t somf_bcd_variant(somf_handle h) { return h ? (h->nt_fn ? 3 : h->nb_fn ? 5 : h->oc_fn ? 2 : 1) : 0; }

SOMF_EXPORT somf_status somf_last_kernels(somf_handle h, int32_t* out) {
  if (!h || !out) return SOMF_E_ARG;
  for (int i = 0; i < 8; ++i) out[i] = h->kern[i];
  return SOMF_OK;
}

SOMF_EXPORT somf_status somf_profile_enable(somf_handle h, int32_t on) {
  if (!h) return SOMF_E_ARG;
  h->prof_on = on != 0;
  return SOMF_OK;
}

SOMF_EXPORT somf_status somf_profile_read(somf_handle h, double* ms, int64_t* launches, int64_t* steps) {
  if (!h) return SOMF_E_ARG;
  CK(cudaStreamSynchronize(h->st));
  double acc[SOMF_NPHASE] = {};
  for (auto& e : h->evs) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, e.a, e.b));
    acc[e.ph] += t;
    h->pool.push_back(e.a);
    h->pool.push_back(e.b);
  }
  h->evs.clear();
  for (int i = 0; i < SOMF_NPHASE; ++i) {
    if (ms) ms[i] = acc[i];
    if (launches) launches[i] = h->launches[i];
    h->launches[i] = 0;
  }
  if (steps) *steps = h->steps_prof;
  h->steps_prof = 0;
  return SOMF_OK;
}

// ---- stateless -------------------------------------------------------------
SOMF_EXPORT somf_status somf_mask_rows(uint64_t seed, int64_t t, int64_t row_lo, int64_t row_hi, double r,
                                       int32_t* idx, int64_t* q_out, void* stream) {
  if (!idx || !q_out || row_lo < 0 || row_hi <= row_lo || !(r >= 1.0)) return SOMF_E_ARG;
  somf_ctx tmp;
  somf_ctx* h = &tmp;
  h->cfg.seed = seed;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t* td = nullptr;
  int64_t* qd = nullptr;
  int32_t* tiles = nullptr;
  const int ntiles = (int)ceil_div(((row_hi - 1) >> 2) - (row_lo >> 2) + 1, kMaskThreads);
  CK(dalloc(&td, 1));
  CK(dalloc(&qd, 1));
  CK(dalloc(&tiles, (size_t)ntiles));
  k_set_scalar_i64<<<1, 1, 0, st>>>(td, t);
  const uint64_t T = (uint64_t)std::floor(4294967296.0 / r);
  somf_status s = launch_mask(h, td, 0, row_lo, row_hi, T, idx, tiles, qd, st);
  if (s == SOMF_OK) {
    CK(cudaMemcpyAsync(q_out, qd, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  cudaFree(td);
  cudaFree(qd);
  cudaFree(tiles);
  return s;
}

SOMF_EXPORT somf_status somf_atom_permutation(uint64_t seed, int64_t t, int32_t k, int32_t cyclic, int32_t* perm,
                                              void* stream) {
  if (!perm || k < 1 || k > 4096) return SOMF_E_ARG;
  somf_ctx tmp;
  somf_ctx* h = &tmp;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t* td = nullptr;
  CK(dalloc(&td, 1));
  k_set_scalar_i64<<<1, 1, 0, st>>>(td, t);
  k_atom_perm<<<1, 32, (size_t)2 * k * sizeof(uint32_t), st>>>(seed, td, k, cyclic, perm);
  CKL();
  CK(cudaStreamSynchronize(st));
  cudaFree(td);
  return SOMF_OK;
}

SOMF_EXPORT somf_status somf_column_ids(uint64_t seed, int64_t n, int64_t s0, int64_t count, int64_t* ids,
                                        void* stream) {
  if (!ids || n < 1 || s0 < 0 || count < 0) return SOMF_E_ARG;
  if (count == 0) return SOMF_OK;
  somf_ctx tmp;
  somf_ctx* h = &tmp;
  int b = 2;
  while ((1ll << b) < n) ++b;
  b += b & 1;
  k_column_ids<<<(unsigned)ceil_div(count, 256), 256, 0, (cudaStream_t)stream>>>(seed, n, s0, count, b / 2, ids);
  CKL();
  return SOMF_OK;
}

SOMF_EXPORT somf_status somf_project_columns(const float* U, int64_t len, int32_t m, int64_t ld,
                                             const double* radius, double mu, int32_t positive, float* Out,
                                             void* stream) {
  if (!U || !Out || !radius || len < 1 || m < 1 || ld < m || !(mu >= 0.0 && mu <= 1.0)) return SOMF_E_ARG;
  somf_ctx tmp;
  somf_ctx* h = &tmp;
  k_project_columns<<<m, kBcdThreads, 0, (cudaStream_t)stream>>>(U, len, ld, radius, 0.0, 1.0 - mu, mu,
                                                                 positive, Out, nullptr);
  CKL();
  return SOMF_OK;
}
