// contract.cuh -- (a1) masked code step, Eq. (a), v2:
//   [beta | G] = r * D_M^T [X_M | D_M]        (k x (eta + k), split-K over q rows)
//
// CTA tile = TM atoms x TN columns (TM = 8 MT, TN = 32 NT), 256 threads in an
// 8 x 32 grid, each thread an MT x NT register tile.  The q masked rows are
// split into nsplit contiguous slices (grid.z); each slice streams its rows in
// chunks of TK = 32 through a two-stage cp.async pipeline (16-byte chunks,
// rows gathered through the index list, out-of-range chunks zero-filled), so
// the next chunk's gathers are in flight while the current one is multiplied.
// Fast path requirements (checked by the host): eta % 4 == 0, ldx % 4 == 0,
// X 16-byte aligned.  Otherwise the v1 kernel k_contract is used.
#pragma once
#include "common.cuh"

namespace somf {

constexpr int kCtThreads = 256;
constexpr int kCtTK = 32;

__device__ __forceinline__ void ct_cp_async16(void* smem_dst, const void* gmem_src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int n = valid ? 16 : 0;     // src-size 0: zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem_src), "r"(n) : "memory");
}
__device__ __forceinline__ void ct_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void ct_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void ct_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// partial[split][a][c], a < k, c < eta + k
constexpr int kCtStages = 3;
constexpr int kCtSeg = 512;      // row indices staged in shared memory per segment

template <int MT, int NT, bool kGather, bool kXCompact>
__global__ void __launch_bounds__(kCtThreads)
k_contract_v2(const int32_t* __restrict__ idx, const int64_t* __restrict__ q_dev, const float* __restrict__ D,
              int kp, int k, const float* __restrict__ X, int64_t ldx, int eta, float* __restrict__ partial) {
  constexpr int TM = 8 * MT, TN = 32 * NT, TK = kCtTK;
  extern __shared__ __align__(16) float ct_smem[];
  float* As = ct_smem;                              // [S][TK][TM]
  float* Bs = ct_smem + kCtStages * TK * TM;        // [S][TK][TN]
  __shared__ int gidx[kCtSeg];
  const int nc = eta + k;
  const int a0 = blockIdx.x * TM, c0 = blockIdx.y * TN;
  const int64_t q = *q_dev;
  const int nsplit = gridDim.z, s = blockIdx.z;
  const int64_t m_lo = q * s / nsplit, m_hi = q * (s + 1) / nsplit;
  const int tid = threadIdx.x, ta = tid >> 5, tc = tid & 31;

  // rows [sb, sb + seg) of the current segment; gidx holds their global rows
  auto load_chunk = [&](int64_t sb, int seg, int ch, int stage) {
    float* A = As + stage * TK * TM;
    float* B = Bs + stage * TK * TN;
    constexpr int ca = TM / 4, cb = TN / 4;
    for (int e = tid; e < TK * ca; e += kCtThreads) {
      const int rr = e / ca, c = e % ca;
      const int lr = ch * TK + rr;
      const int col = a0 + 4 * c;
      const bool ok = lr < seg && col < kp;
      const int64_t g = ok ? (int64_t)gidx[lr] : 0;
      ct_cp_async16(A + rr * TM + 4 * c, D + g * kp + (ok ? col : 0), ok);
    }
    for (int e = tid; e < TK * cb; e += kCtThreads) {
      const int rr = e / cb, c = e % cb;
      const int lr = ch * TK + rr;
      const int col = c0 + 4 * c;
      const bool inrow = lr < seg;
      const int64_t g = inrow ? (int64_t)gidx[lr] : 0;
      const float* src = D;
      bool ok = false;
      if (inrow && col < eta) {
        src = X + (kXCompact ? sb + lr : g) * ldx + col;
        ok = true;
      } else if (inrow && col < nc) {
        src = D + g * kp + (col - eta);
        ok = true;
      }
      ct_cp_async16(B + rr * TN + 4 * c, src, ok);
    }
  };

  float acc[MT][NT];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j] = 0.f;

  for (int64_t sb = m_lo; sb < m_hi; sb += kCtSeg) {
    const int seg = (int)(m_hi - sb < (int64_t)kCtSeg ? m_hi - sb : (int64_t)kCtSeg);
    __syncthreads();                       // previous segment's readers of gidx are done
    for (int r = tid; r < seg; r += kCtThreads) gidx[r] = kGather ? idx[sb + r] : (int)(sb + r);
    __syncthreads();
    const int nch = (seg + TK - 1) / TK;
#pragma unroll
    for (int st = 0; st < kCtStages - 1; ++st) {
      if (st < nch) load_chunk(sb, seg, st, st);
      ct_commit();
    }
    for (int ch = 0; ch < nch; ++ch) {
      const int stage = ch % kCtStages;
      if (ch + kCtStages - 1 < nch) load_chunk(sb, seg, ch + kCtStages - 1, (ch + kCtStages - 1) % kCtStages);
      ct_commit();
      asm volatile("cp.async.wait_group %0;" ::"n"(kCtStages - 1) : "memory");
      __syncthreads();
      const float* A = As + stage * TK * TM + ta * MT;
      const float* B = Bs + stage * TK * TN + tc;
#pragma unroll 4
      for (int kk = 0; kk < TK; ++kk) {
        float av[MT], bv[NT];
#pragma unroll
        for (int i = 0; i < MT; ++i) av[i] = A[kk * TM + i];
#pragma unroll
        for (int j = 0; j < NT; ++j) bv[j] = B[kk * TN + 32 * j];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
    ct_wait0();
  }
  float* out = partial + (int64_t)s * k * nc;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int a = a0 + ta * MT + i;
    if (a >= k) continue;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int c = c0 + tc + 32 * j;
      if (c < nc) out[(int64_t)a * nc + c] = acc[i][j];
    }
  }
}

// Fixed-order fp64 reduction of the split-K partials, scaled by r:
// beta (k x eta) and G (k x k), row-major.  32 outputs per CTA (lane =
// output, coalesced); warp w sums splits w, w + 8, ...; then warp 0 adds the 8
// warp sums in order.
__global__ void __launch_bounds__(256)
k_contract_reduce2(const float* __restrict__ partial, int nsplit, int k, int eta, double r,
                   double* __restrict__ beta, double* __restrict__ G) {
  __shared__ double ws[8][32];
  const int nc = eta + k;
  const int64_t tot = (int64_t)k * nc;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (e < tot) {
#pragma unroll 8
    for (int i = w; i < nsplit; i += 8) s += (double)__ldcs(partial + (int64_t)i * tot + e);
  }
  ws[w][lane] = s;
  __syncthreads();
  if (w == 0 && e < tot) {
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += ws[i][lane];
    t *= r;
    const int a = (int)(e / nc), c = (int)(e % nc);
    if (c < eta) beta[(int64_t)a * eta + c] = t;
    else G[(int64_t)a * k + (c - eta)] = t;
  }
}

}  // namespace somf

namespace somf {

// ---------------------------------------------------------------------------
// v3: one CTA per SM owns a slice of ~q/#SMs masked rows and stages the WHOLE
// slice ([X row | D row] per row, 16-byte cp.async, every row's loads in
// flight at once -- the gather is latency-bound otherwise, see
// tests/tools/gather_bench.cu) in two commit groups, then computes the full
// k x (eta + k) output tile (8 x 32 threads, MT x NT registers each) while the
// second half lands.  Used when the tile covers k and eta + k and the slice
// fits in shared memory; rows beyond one slice are processed in segments.
// ---------------------------------------------------------------------------
// Optional fused split-K reduction (cooperative launch, bar != null): after
// the partial tiles are written, one grid barrier, then CTA b reduces the
// outputs [tot b / G, tot (b+1) / G) over the G partials in the fixed order
// of k_contract_reduce2 (lane = output, warp w sums splits w, w + 8, ...,
// then the 8 warp sums in order) and writes r x [beta | G] in fp64.
struct CtFuse {
  unsigned* bar;            // [0] arrivals, [1] exits (zero between launches); null = no fusion
  double r;
  double* beta;             // k x eta
  double* G;                // k x k
  int* err;                 // watchdog: set to 5 when the barrier times out (protocol bug)
};

// Fused fixed-order split-K reduction (CtFuse): grid barrier, then CTA b
// reduces the outputs [tot b / G, tot (b+1) / G) over the G partial tiles.
// Partial tile layout: k rows of ncp columns; column c < eta is beta[:, c],
// column ep + j (j < k) is G[:, j], other columns are padding.  Order: warp w
// sums the splits w, w + 8, ... ascending (fp64), then the 8 warp sums in
// order -- the same bits for any timing.
__device__ __forceinline__ void ct_store_out(const CtFuse& fz, int64_t e, double t, int k, int eta, int ncp,
                                             int ep) {
  const int a = (int)(e / ncp), c = (int)(e % ncp);
  t *= fz.r;
  if (c < eta) fz.beta[(int64_t)a * eta + c] = t;
  else if (c >= ep && c - ep < k) fz.G[(int64_t)a * k + (c - ep)] = t;
}

// scratch: >= 16 KB of shared memory the caller no longer needs
__device__ __forceinline__ void ct_fused_reduce(const float* __restrict__ partial, int k, int eta, int ncp, int ep,
                                                const CtFuse& fz, double* scratch,
                                                long long* barrier_cycles = nullptr) {
  const int tid = threadIdx.x, ta = tid >> 5, tc = tid & 31;
  const int G = gridDim.x;
  const long long tb0 = barrier_cycles ? clock64() : 0;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(fz.bar), "r"(1u) : "memory");
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_gpu(fz.bar) < (unsigned)G) {
      if (globaltimer_ns() - t0 > 2000000000ull) {          // protocol bug: do not hang the GPU
        if (fz.err) atomicExch(fz.err, 5);
        break;
      }
    }
  }
  __syncthreads();
  if (barrier_cycles) *barrier_cycles += clock64() - tb0;      // the calling thread's wait (diagnostics)
  const int64_t tot = (int64_t)k * ncp;
  if ((ncp & 3) == 0) {
    // lane = 2 x 4 consecutive outputs (16-byte loads; outputs e and e + 32),
    // up to 20 loads of a thread in flight: a CTA's ~tot / (4 G) outputs (34 at
    // cfgC) take ONE pass of two L2 round trips (a 32-output pass needed two
    // passes of three)
    static_assert(kCtThreads == 256, "8 warps; 64 outputs x 4 in the combine");
    double (*ws4)[64][4] = reinterpret_cast<double (*)[64][4]>(scratch);     // [8][64][4]
    const int64_t t4 = tot / 4;
    const int64_t e0 = t4 * blockIdx.x / G, e1 = t4 * (blockIdx.x + 1) / G;
    for (int64_t g0 = e0; g0 < e1; g0 += 64) {
      const int64_t ea = g0 + tc, eb = ea + 32;
      double s[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
      const float4* p4 = reinterpret_cast<const float4*>(partial);
      // (predicated loads, no branch on the lane: a divergent second output
      // would serialise the two groups of lanes)
      const bool ha = ea < e1, hb = eb < e1;
      const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
      // batches of 10 splits, fully unrolled with predicated loads (a partial
      // unroll of the runtime-length loop leaves a one-load-at-a-time remainder:
      // 9 serial L2 round trips at G = 148)
      for (int i0 = ta; i0 < G; i0 += 80) {
        float4 v[10], u[10];
#pragma unroll
        for (int x = 0; x < 10; ++x) {
          const int i = i0 + 8 * x;
          v[x] = (ha && i < G) ? __ldcg(p4 + (int64_t)i * t4 + ea) : z4;
          u[x] = (hb && i < G) ? __ldcg(p4 + (int64_t)i * t4 + eb) : z4;
        }
#pragma unroll
        for (int x = 0; x < 10; ++x) {
          s[0][0] += (double)v[x].x;
          s[0][1] += (double)v[x].y;
          s[0][2] += (double)v[x].z;
          s[0][3] += (double)v[x].w;
          s[1][0] += (double)u[x].x;
          s[1][1] += (double)u[x].y;
          s[1][2] += (double)u[x].z;
          s[1][3] += (double)u[x].w;
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        ws4[ta][tc][j] = s[0][j];
        ws4[ta][tc + 32][j] = s[1][j];
      }
      __syncthreads();
      {
        const int l = tid >> 2, j = tid & 3;         // 256 threads = 64 outputs x 4
        const int64_t ee = g0 + l;
        if (ee < e1) {
          double t = 0.0;
#pragma unroll
          for (int w = 0; w < 8; ++w) t += ws4[w][l][j];
          ct_store_out(fz, 4 * ee + j, t, k, eta, ncp, ep);
        }
      }
      __syncthreads();
    }
  } else {
    constexpr int kOpl = 8;                      // outputs per lane (>= ceil(tot / G / 32))
    double (*ws)[32 * kOpl] = reinterpret_cast<double (*)[32 * kOpl]>(scratch);   // [8][32 kOpl]
    const int64_t e0 = tot * blockIdx.x / G, e1 = tot * (blockIdx.x + 1) / G;
    for (int64_t g0 = e0; g0 < e1; g0 += 32 * kOpl) {
      double sacc[kOpl];
#pragma unroll
      for (int o = 0; o < kOpl; ++o) sacc[o] = 0.0;
#pragma unroll 5
      for (int i = ta; i < G; i += 8) {
        float v[kOpl];
#pragma unroll
        for (int o = 0; o < kOpl; ++o) {
          const int64_t e = g0 + 32 * o + tc;
          v[o] = e < e1 ? __ldcg(partial + (int64_t)i * tot + e) : 0.f;
        }
#pragma unroll
        for (int o = 0; o < kOpl; ++o) sacc[o] += (double)v[o];
      }
#pragma unroll
      for (int o = 0; o < kOpl; ++o) ws[ta][32 * o + tc] = sacc[o];
      __syncthreads();
      for (int x = tid; x < 32 * kOpl; x += kCtThreads) {
        const int64_t e = g0 + x;
        if (e < e1) {
          double t = 0.0;
#pragma unroll
          for (int i = 0; i < 8; ++i) t += ws[i][x];
          ct_store_out(fz, e, t, k, eta, ncp, ep);
        }
      }
      __syncthreads();
    }
  }
  // last CTA out resets the barrier for the next launch
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(fz.bar + 1, 1u) == (unsigned)G - 1) {
      fz.bar[0] = 0u;
      fz.bar[1] = 0u;
      __threadfence();
    }
  }
}

template <int MT, int NT, bool kXCompact>
__global__ void __launch_bounds__(kCtThreads)
k_contract_v3(const int32_t* __restrict__ idx, const int64_t* __restrict__ q_dev, const float* __restrict__ D,
              int kp, int k, const float* __restrict__ X, int64_t ldx, int eta, float* __restrict__ partial,
              int seg_rows, CtFuse fz) {
  extern __shared__ __align__(16) float c3_smem[];
  const int LDY = eta + kp;                 // [X row | D row], 16-byte multiple
  float* Ys = c3_smem;                      // seg_rows x LDY
  int* gidx = reinterpret_cast<int*>(Ys + (size_t)seg_rows * LDY);
  const int nc = eta + k;
  const int64_t q = *q_dev;
  const int G = gridDim.x;
  const int64_t m_lo = q * blockIdx.x / G, m_hi = q * (blockIdx.x + 1) / G;
  const int tid = threadIdx.x, ta = tid >> 5, tc = tid & 31;
  float acc[MT][NT];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j] = 0.f;
  const int cx = eta / 4, cd = kp / 4, cr = cx + cd;
  for (int64_t sb = m_lo; sb < m_hi; sb += seg_rows) {
    const int n = (int)(m_hi - sb < (int64_t)seg_rows ? m_hi - sb : (int64_t)seg_rows);
    __syncthreads();
    for (int r = tid; r < n; r += kCtThreads) gidx[r] = idx[sb + r];
    __syncthreads();
    const int half = (n + 1) / 2;
    for (int part = 0; part < 2; ++part) {
      const int rb = part ? half : 0, re = part ? n : half;
      for (int e = tid; e < (re - rb) * cr; e += kCtThreads) {
        const int r = rb + e / cr, c = e % cr;
        const int64_t g = gidx[r];
        const float* src = c < cx ? X + (kXCompact ? sb + r : g) * ldx + 4 * c : D + g * kp + 4 * (c - cx);
        ct_cp_async16(Ys + (size_t)r * LDY + 4 * c, src, true);
      }
      ct_commit();
    }
    for (int part = 0; part < 2; ++part) {
      if (part == 0) ct_wait1();
      else ct_wait0();
      __syncthreads();
      const int rb = part ? half : 0, re = part ? n : half;
#pragma unroll 2
      for (int r = rb; r < re; ++r) {
        const float* y = Ys + (size_t)r * LDY;
        float av[MT], bv[NT];
#pragma unroll
        for (int i = 0; i < MT; ++i) av[i] = y[eta + ta * MT + i];
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int c = tc + 32 * j;
          bv[j] = c < nc ? y[c] : 0.f;
        }
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
    }
  }
  float* out = partial + (int64_t)blockIdx.x * k * nc;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int a = ta * MT + i;
    if (a >= k) continue;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int c = tc + 32 * j;
      if (c < nc) out[(int64_t)a * nc + c] = acc[i][j];
    }
  }
  if (fz.bar == nullptr) return;
  ct_fused_reduce(partial, k, eta, eta + k, eta, fz, reinterpret_cast<double*>(c3_smem));
}

}  // namespace somf
