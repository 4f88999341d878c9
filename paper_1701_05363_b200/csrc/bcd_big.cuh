// bcd_big.cuh -- (a4) Alg. 4 with all k projection thresholds
// solved SIMULTANEOUSLY (the rounds of bcd_newton.cuh) for the shapes the
// on-chip kernel does not cover:
//   * k up to 256 (cfgB hyperspectral, cfgE): the prescaled Cbar rows in pi
//     order (256 KB at k = 256) no longer fit shared memory next to the rows,
//     so they stream from L2 in chunks of CH positions (cp.async, double
//     buffered, one CTA barrier per chunk);
//   * masked rows that do not fit on chip (cfgC r <= 4, cfgE on one GPU):
//     every CTA walks its rows in tiles of TR rows; the tile's d_old and its
//     prescaled initial residual (pi order) are written once to an L2/HBM
//     scratch at setup and re-read every round (they do not change over the
//     rounds), the per-atom statistics are accumulated over the tiles in a
//     fixed order, and the final D is written by one more pass with the
//     converged thresholds.
// Round structure, convergence test and the deterministic fixed-point grid
// sums are the ones of k_bcd_newton (shared helpers in bcd_newton.cuh).
#pragma once
#include "bcd_newton.cuh"

namespace somf {

constexpr int kNbMaxK = 256;
constexpr int kNbThreads = 384;

// prescaled Cbar rows per thread parity: row PP of Ctg holds, for each parity
// t < T, the KTS values c_{PP, iT+t} / c_{iT+t, iT+t} (i < KT, zero padded) at
// stride CSTR floats (CSTR = 4 mod 8: the 16-byte loads of 8 consecutive
// parities hit disjoint banks)
__host__ __device__ constexpr int nb_kts(int kpt, int t) { return ((kpt / t) + 3) & ~3; }
__host__ __device__ constexpr int nb_cstr(int kpt, int t) { return (nb_kts(kpt, t) % 8 == 0) ? nb_kts(kpt, t) + 4 : nb_kts(kpt, t); }

struct NbArgs {
  const float* Cpi;         // KPT x KPT, pi order: Cbar (NbRec mode) or Cbar prescaled by
                            // 1 / c_ll per column l (blocked mode)
  const float* Ctg;         // KPT x T x CSTR: prescaled Cbar rows per parity (NbRec mode)
  const float* invc;        // KPT: 1 / c_pp in pi order (0 for dead atoms)
  float* scr;               // per masked row 2 x KPT floats (d_old | R0), pi order: streamed
                            // tiles (NbRec mode) / every tile (blocked mode)
  int tile_rows;            // TR: rows per tile (rows of a CTA beyond TR => several tiles)
  int ch;                   // positions per Cbar chunk (== KPT: resident)
};

// pi in the device array, Cbar permuted and prescaled, 1/c_pp; one CTA per
// position row.  Dead atoms (R10) get 1/c = 0 (their residual is zero, so d
// stays d_old).  blocked: Cpi[p][l] = c_{pi p, pi l} / c_{pi l, pi l} and no
// Ctg; else Cpi unscaled and Ctg = the parity layout of the prescaled rows.
struct NbPerm { int32_t v[kNbMaxK]; };
static __global__ void k_nb_prep(NbPerm pi, int k, int kpt, int T, int blocked, const float* __restrict__ C32,
                                 const double* __restrict__ C64, int32_t* __restrict__ perm, float* __restrict__ Cpi,
                                 float* __restrict__ Ctg, float* __restrict__ invc) {
  const int p = blockIdx.x;                    // position (row of Cpi / Ctg)
  __shared__ double dmax_s;
  __shared__ float inv_s[kNbMaxK];
  if (threadIdx.x < 32) {
    double dm = 1.0;
    for (int j = threadIdx.x; j < k; j += 32) dm = fmax(dm, C64[(int64_t)j * k + j]);
    dm = warp_max(dm);
    if (threadIdx.x == 0) dmax_s = dm;
  }
  __syncthreads();
  for (int l = threadIdx.x; l < kpt; l += blockDim.x) {
    float iv = 0.f;
    if (l < k) {
      const double c = C64[(int64_t)pi.v[l] * k + pi.v[l]];
      iv = c > 1e-12 * dmax_s ? (float)(1.0 / c) : 0.f;
    }
    inv_s[l] = iv;
  }
  __syncthreads();
  if (p == 0)
    for (int l = threadIdx.x; l < kpt; l += blockDim.x) {
      if (l < k) perm[l] = pi.v[l];
      invc[l] = inv_s[l];
    }
  const int jp = p < k ? pi.v[p] : 0;
  for (int l = threadIdx.x; l < kpt; l += blockDim.x) {
    const float c = (p < k && l < k) ? C32[(int64_t)jp * k + pi.v[l]] : 0.f;
    Cpi[(int64_t)p * kpt + l] = blocked ? c * inv_s[l] : c;
  }
  if (blocked) return;
  const int kt = kpt / T, kts = nb_kts(kpt, T), cstr = nb_cstr(kpt, T);
  for (int e = threadIdx.x; e < T * cstr; e += blockDim.x) {
    const int t = e / cstr, i = e % cstr;
    const int l = i * T + t;
    float v = 0.f;
    if (p < k && i < kt && i < kts && l < k) v = C32[(int64_t)jp * k + pi.v[l]] * inv_s[l];
    Ctg[(int64_t)p * T * cstr + e] = v;
  }
}

__device__ __forceinline__ void nb_cp16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}

// The recurrence of one tile (v5 layout: a group of T lanes owns M rows; R and
// d_old in registers), with the prescaled Cbar rows either resident (CH =
// KPT) or streamed in double-buffered chunks of CH positions (one CTA barrier
// per chunk: every thread of the CTA runs this, rows past the tile on the
// spare zero row).
template <int KPT, int T, int M, bool kGen, int CH, int PP, int END>
struct NbRec {
  static constexpr int KT = KPT / T;
  static constexpr int KTS = nb_kts(KPT, T);
  static constexpr int CSTR = nb_cstr(KPT, T);
  static constexpr int CHB = CH * T * CSTR;           // floats per chunk buffer
  static __device__ __forceinline__ void run(float (&R)[M][KT], const float (&Do)[M][KT], int t, float* __restrict__ v0,
                                             int vstride, float* __restrict__ cbuf, const float* __restrict__ Ctg,
                                             const NtPar<kGen>* __restrict__ par) {
    if constexpr (CH < KPT && PP % CH == 0) {
      // chunk PP / CH is (being) loaded into buffer (PP / CH) & 1: wait for it;
      // then every thread is past chunk PP / CH - 1, whose buffer takes the next
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
      if (PP + CH < KPT) {
        float* dst = cbuf + (((PP / CH) + 1) & 1) * CHB;
        const float* src = Ctg + (size_t)(PP + CH) * T * CSTR;
        constexpr int n4 = CHB / 4;
        for (int e = threadIdx.x; e < n4; e += blockDim.x) nb_cp16(dst + 4 * e, src + 4 * e);
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
    }
    constexpr int own = PP % T, ii = PP / T;
    {
      const NtPar<kGen> pr = par[PP];
      float delta[M];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const float u = R[m][ii] + Do[m][ii];        // P:861 (valid in the owner)
        const float v = pr.v_of(u);
        const float d = pr.d_of(u);
        if (t == own) v0[m * vstride + PP] = v;
        delta[m] = __shfl_sync(0xffffffffu, d - Do[m][ii], own, T);
      }
      const float* crow = cbuf + ((PP / CH) & 1) * CHB + (PP % CH) * T * CSTR + t * CSTR;
#pragma unroll
      for (int j4 = ii / 4; j4 < KTS / 4; ++j4) {
        const float4 c = *reinterpret_cast<const float4*>(crow + 4 * j4);
        const float cc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = 4 * j4 + e;
          if (i < KT) {
#pragma unroll
            for (int m = 0; m < M; ++m) {
              if (i > ii) {
                R[m][i] = fmaf(-delta[m], cc[e], R[m][i]);
              } else if (i == ii) {
                const float up = fmaf(-delta[m], cc[e], R[m][i]);
                R[m][i] = t > own ? up : R[m][i];
              }
            }
          }
        }
      }
    }
    NbRec<KPT, T, M, kGen, CH, PP + 1, END>::run(R, Do, t, v0, vstride, cbuf, Ctg, par);
  }
};
// (positions in runs of <= 128 template instantiations: nvcc's recursion limit)
template <int KPT, int T, int M, bool kGen, int CH, int END>
struct NbRec<KPT, T, M, kGen, CH, END, END> {
  static __device__ __forceinline__ void run(float (&)[M][KPT / T], const float (&)[M][KPT / T], int, float*, int,
                                             float*, const float*, const NtPar<kGen>*) {}
};

// ---------------------------------------------------------------------------
// Blocked recurrence (k > 128: the unrolled per-position code of NbRec would
// not fit the instruction cache).  Positions in chunks of 16:
//   (a) one thread per masked row runs the chunk's 16 positions in order (its
//       16 residuals and d_old in registers, the chunk's 16 x 16 block of the
//       prescaled Cbar broadcast from shared memory), writes v and
//       delta = d - d_old of the 16 positions;
//   (b) the rows' later residuals take the chunk's rank-16 update
//       R[:, l] -= delta[:, chunk] Cpre[chunk, l] (l past the chunk), register
//       tiles of 2 rows x 4 positions over all threads.
// Same arithmetic as the sequential recurrence, grouped.
// ---------------------------------------------------------------------------
constexpr int kNbCB = 16;        // positions per chunk

// R[r][l] -= sum_j S[r][j] C[j][l]  for r < nr, l in [l0, l1) (multiples of 4),
// j < 16; S rows at stride lds (16-byte aligned), C the 16 chunk rows (stride
// KPT).  tid / nthr: this thread's share of the (row pair, 4 positions) items.
template <int KPT>
__device__ __forceinline__ void nb_rank16(float* __restrict__ R, int ldr, const float* __restrict__ S, int lds,
                                          const float* __restrict__ C, int nr, int l0, int l1, int tid, int nthr) {
  const int nq = (l1 - l0) >> 2, npair = (nr + 1) >> 1;
  for (int it = tid; it < npair * nq; it += nthr) {
    const int r0 = 2 * (it / nq), lq = l0 + 4 * (it % nq);
    const bool two = r0 + 1 < nr;
    float4 a0 = *reinterpret_cast<const float4*>(R + (size_t)r0 * ldr + lq);
    float4 a1 = two ? *reinterpret_cast<const float4*>(R + (size_t)(r0 + 1) * ldr + lq) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j4 = 0; j4 < 4; ++j4) {
      const float4 s0 = *reinterpret_cast<const float4*>(S + (size_t)r0 * lds + 4 * j4);
      const float4 s1 = two ? *reinterpret_cast<const float4*>(S + (size_t)(r0 + 1) * lds + 4 * j4)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
      const float sv0[4] = {s0.x, s0.y, s0.z, s0.w}, sv1[4] = {s1.x, s1.y, s1.z, s1.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float4 c = *reinterpret_cast<const float4*>(C + (size_t)(4 * j4 + e) * KPT + lq);
        a0.x = fmaf(-sv0[e], c.x, a0.x);
        a0.y = fmaf(-sv0[e], c.y, a0.y);
        a0.z = fmaf(-sv0[e], c.z, a0.z);
        a0.w = fmaf(-sv0[e], c.w, a0.w);
        a1.x = fmaf(-sv1[e], c.x, a1.x);
        a1.y = fmaf(-sv1[e], c.y, a1.y);
        a1.z = fmaf(-sv1[e], c.z, a1.z);
        a1.w = fmaf(-sv1[e], c.w, a1.w);
      }
    }
    *reinterpret_cast<float4*>(R + (size_t)r0 * ldr + lq) = a0;
    if (two) *reinterpret_cast<float4*>(R + (size_t)(r0 + 1) * ldr + lq) = a1;
  }
}

// chunk c of the prescaled Cbar (16 rows x KPT) into buffer c & 1 (cp.async)
template <int KPT>
__device__ __forceinline__ void nb_load_chunk(float* cbuf, const float* __restrict__ Cpre, int c, int tid, int nthr) {
  float* dst = cbuf + (c & 1) * kNbCB * KPT;
  const float* src = Cpre + (size_t)c * kNbCB * KPT;
  for (int e = tid; e < kNbCB * KPT / 4; e += nthr) nb_cp16(dst + 4 * e, src + 4 * e);
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// one recurrence pass of the blocked mode over the tile's rows (R: the
// tile's R0, overwritten; Dold; V receives v; Dl: nr x 16 deltas)
template <int KPT, bool kGen>
__device__ __forceinline__ void nb_blk_pass(float* R, const float* Dold, float* V, float* Dl, float* cbuf,
                                            const float* __restrict__ Cpre, const NtPar<kGen>* par, int nr,
                                            int tid, int nthr) {
  constexpr int LDB = KPT + 4, NC = KPT / kNbCB;
  nb_load_chunk<KPT>(cbuf, Cpre, 0, tid, nthr);
#pragma unroll 1
  for (int c = 0; c < NC; ++c) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();                                   // chunk c landed; chunk c - 1 consumed
    if (c + 1 < NC) nb_load_chunk<KPT>(cbuf, Cpre, c + 1, tid, nthr);
    const float* Cb = cbuf + (c & 1) * kNbCB * KPT;
    const int p0 = c * kNbCB;
    if (tid < nr) {
      float rr[kNbCB], dd[kNbCB], vv[kNbCB], dl[kNbCB];
      const float* Rr = R + (size_t)tid * LDB + p0;
      const float* Dr = Dold + (size_t)tid * LDB + p0;
#pragma unroll
      for (int i4 = 0; i4 < kNbCB / 4; ++i4) {
        const float4 x = *reinterpret_cast<const float4*>(Rr + 4 * i4);
        const float4 y = *reinterpret_cast<const float4*>(Dr + 4 * i4);
        rr[4 * i4] = x.x; rr[4 * i4 + 1] = x.y; rr[4 * i4 + 2] = x.z; rr[4 * i4 + 3] = x.w;
        dd[4 * i4] = y.x; dd[4 * i4 + 1] = y.y; dd[4 * i4 + 2] = y.z; dd[4 * i4 + 3] = y.w;
      }
#pragma unroll
      for (int j = 0; j < kNbCB; ++j) {
        const NtPar<kGen> pr = par[p0 + j];
        const float u = rr[j] + dd[j];
        vv[j] = pr.v_of(u);
        const float delta = pr.d_of(u) - dd[j];
        dl[j] = delta;
        const float* crow = Cb + (size_t)j * KPT + p0;
#pragma unroll
        for (int i4 = (j + 1) / 4; i4 < kNbCB / 4; ++i4) {
          const float4 cc = *reinterpret_cast<const float4*>(crow + 4 * i4);
          const float cv[4] = {cc.x, cc.y, cc.z, cc.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (4 * i4 + e > j) rr[4 * i4 + e] = fmaf(-delta, cv[e], rr[4 * i4 + e]);
        }
      }
      float* Vr = V + (size_t)tid * LDB + p0;
      float* Dlr = Dl + (size_t)tid * kNbCB;
#pragma unroll
      for (int i4 = 0; i4 < kNbCB / 4; ++i4) {
        *reinterpret_cast<float4*>(Vr + 4 * i4) = make_float4(vv[4 * i4], vv[4 * i4 + 1], vv[4 * i4 + 2], vv[4 * i4 + 3]);
        *reinterpret_cast<float4*>(Dlr + 4 * i4) = make_float4(dl[4 * i4], dl[4 * i4 + 1], dl[4 * i4 + 2], dl[4 * i4 + 3]);
      }
    }
    __syncthreads();
    if (c + 1 < NC) nb_rank16<KPT>(R, LDB, Dl, kNbCB, Cb, nr, p0 + kNbCB, KPT, tid, nthr);
  }
  __syncthreads();
}

// shared-memory layout (floats unless noted), host mirror in somf_capi.cu
//   NbRec mode:   Dold, Rini, V   3 x (TR + 1) x (KPT + 4); cbuf 2 x CHB or KPT x T x CSTR
//   blocked mode: Dold, R, V      3 x (TR + 1) x (KPT + 4); cbuf 2 x 16 x KPT; Dl (TR + 1) x 16
//   part          max(5 H KPT, 12 k) words (stats partials / record read)
//   rows_s        TR ints; mbits: one byte per Philox block of my slice
template <int KPT, int T>
__host__ __device__ constexpr size_t nb_cbuf_floats(int ch, bool blk) {
  return blk ? (size_t)2 * kNbCB * KPT
             : ch >= KPT ? (size_t)KPT * T * nb_cstr(KPT, T) : (size_t)2 * ch * T * nb_cstr(KPT, T);
}

// One recurrence pass over tile tl: loads it from the scratch when streamed,
// leaves v in V; returns the tile's row count.
// Streamed tiles of the unrolled mode (!kBlk) are double buffered through
// the registers: a tile's d_old / R0 rows are cp.async'd into Dold / Rini
// while the PREVIOUS tile's recurrence runs (its rows already sit in
// registers), so the scratch read overlaps the arithmetic.  nb_prefetch
// issues tile tl's copy; the pass waits for it, loads its registers and
// issues tile (tl + 1) % ntile's.  (Blocked mode updates R in shared memory
// during the pass: its loads stay synchronous.)
template <int KPT>
__device__ __forceinline__ void nb_prefetch(const float* __restrict__ scr, int tl, int TR, int nr_all, int64_t lo,
                                            float* Dold, float* Rini, int tid, int nthr) {
  constexpr int LD = KPT + 4;
  constexpr int q4 = KPT / 4;
  const int r0 = tl * TR, nr = min(TR, nr_all - r0);
  const float* sc = scr + (size_t)(lo + r0) * 2 * KPT;
  for (int e = tid; e < nr * 2 * q4; e += nthr) {
    const int row = e / (2 * q4), c = e % (2 * q4);
    float* dst = c < q4 ? Dold + (size_t)row * LD + 4 * c : Rini + (size_t)row * LD + 4 * (c - q4);
    nb_cp16(dst, sc + (size_t)row * 2 * KPT + 4 * c);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int KPT, int T, int M, bool kGen, int CH, bool kBlk>
__device__ __forceinline__ int nb_tile_pass(const float* __restrict__ scr, const float* __restrict__ Cpi,
                                            const float* __restrict__ Ctg, int tl, int TR, int nr_all, int64_t lo,
                                            bool streamed, float* Dold, float* Rini, float* V, float* cbuf, float* Dl,
                                            const NtPar<kGen>* par, int g, int tq, int ngroups, int tid, int nthr,
                                            long long* ld_cyc = nullptr) {
  constexpr int LD = KPT + 4;
  const long long t_ld = ld_cyc ? clock64() : 0;
  constexpr int KT = KPT / T;
  constexpr int CSTR = nb_cstr(KPT, T);
  const int r0 = tl * TR, nr = min(TR, nr_all - r0);
  if (streamed && kBlk) {
    __syncthreads();                               // V / Dold / Rini of the previous tile consumed
    nb_prefetch<KPT>(scr, tl, TR, nr_all, lo, Dold, Rini, tid, nthr);   // every row in flight at once
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (streamed) {
    asm volatile("cp.async.wait_all;" ::: "memory");   // this tile's prefetch
  }
  if constexpr (kBlk) {
    __syncthreads();
    if (ld_cyc) *ld_cyc += clock64() - t_ld;
    nb_blk_pass<KPT, kGen>(Rini, Dold, V, Dl, cbuf, Cpi, par, nr, tid, nthr);
    return nr;
  } else {
    if (CH < KPT) {
      // chunk 0 of the prescaled Cbar into buffer 0
      constexpr int n4 = CH * T * CSTR / 4;
      for (int e = tid; e < n4; e += nthr) nb_cp16(cbuf + 4 * e, Ctg + 4 * e);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    __syncthreads();
    if (ld_cyc) *ld_cyc += clock64() - t_ld;
    int rowx[M];
#pragma unroll
    for (int m = 0; m < M; ++m) rowx[m] = (g < ngroups && g * M + m < nr) ? g * M + m : TR;
    const int vstride = rowx[M - 1] - rowx[0];
    float Do[M][KT], R[M][KT];
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
      for (int i = 0; i < KT; ++i) {
        Do[m][i] = Dold[(size_t)rowx[m] * LD + i * T + tq];
        R[m][i] = Rini[(size_t)rowx[m] * LD + i * T + tq];
      }
    if (streamed) {
      // every thread holds its rows: the next tile's rows may overwrite Dold / Rini
      __syncthreads();
      const int ntile = (nr_all + TR - 1) / TR;
      nb_prefetch<KPT>(scr, tl + 1 < ntile ? tl + 1 : 0, TR, nr_all, lo, Dold, Rini, tid, nthr);
    }
    // threads past the groups: same code on the spare row (their v goes to the spare row)
    constexpr int H1 = KPT > 128 ? 128 : KPT;
    NbRec<KPT, T, M, kGen, CH, 0, H1>::run(R, Do, tq, V + (size_t)rowx[0] * LD, vstride * LD, cbuf, Ctg, par);
    if constexpr (KPT > 128)
      NbRec<KPT, T, M, kGen, CH, H1, KPT>::run(R, Do, tq, V + (size_t)rowx[0] * LD, vstride * LD, cbuf, Ctg, par);
    __syncthreads();
    return nr;
  }
}

template <int KPT, int T, int M, bool kGen, int CH, bool kBlk>
__global__ void __launch_bounds__(kNbThreads, 1)
k_bcd_big(NtArgs P, NbArgs A) {
  constexpr int LD = KPT + 4;                       // 16-byte rows (cp.async of streamed tiles)
  constexpr int KT = KPT / T;
  constexpr int CSTR = nb_cstr(KPT, T);
  static_assert(KPT % T == 0 && M == 2, "groups of T lanes x 2 rows");
  static_assert(!kBlk || KPT % kNbCB == 0, "blocked mode: KPT a multiple of 16");
  extern __shared__ __align__(16) float nb_smem[];
  __shared__ __align__(16) NtPar<kGen> par_s[2][KPT];
  __shared__ double lam_s[KPT], rho_s[KPT];
  __shared__ double acc1_s[KPT], acc2_s[KPT];       // per-atom sums over my tiles (fixed order)
  __shared__ unsigned acn_s[KPT], amn_s[KPT], amx_s[KPT];
  __shared__ float vlo_s[KPT];
  __shared__ int mode_s[KPT], jmap_s[KPT], pinv_s[KPT];
  __shared__ int mcnt_s;
  __shared__ int lockF_s, firstU_s, prevF_s;   // locked prefix (R22), first unconverged position
  // phase clock of CTA 0 (slots as k_bcd_newton's 0..7; 8 = streamed tile loads, part of 1;
  // 9..12 = setup: staging, pi-order permutes, R0, radii + scratch write, part of 0)
  __shared__ long long nbp_s[13];
  long long t_mark = clock64();
  long long* const ldp = (P.prof && blockIdx.x == 0 && threadIdx.x == 0) ? &nbp_s[8] : nullptr;
#define NB_MARK(slot)                                                              \
  do {                                                                             \
    if (P.prof && blockIdx.x == 0 && threadIdx.x == 0) {                           \
      const long long now_ = clock64();                                            \
      nbp_s[slot] += now_ - t_mark;                                                \
      t_mark = now_;                                                               \
    }                                                                              \
  } while (0)
  if (P.prof && blockIdx.x == 0 && threadIdx.x < 13) nbp_s[threadIdx.x] = 0;
  const int k = P.k, kp = P.kp;
  const int nthr = blockDim.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = gridDim.x;
  const int64_t q = *P.q_dev;
  const int64_t lo = q * blockIdx.x / G, hi = q * (blockIdx.x + 1) / G;
  const int nr_all = (int)(hi - lo);
  const int TR = A.tile_rows;
  const int ntile = nr_all > 0 ? (nr_all + TR - 1) / TR : 0;
  const bool streamed = kBlk || ntile > 1;          // tiles re-read from the scratch every round
  // host sizing errors (uniform over the CTAs: every CTA returns before any barrier)
  if ((!kBlk && T * ((TR + M - 1) / M) > nthr) || (kBlk && TR > nthr) || nthr < k ||
      ((kBlk || (q + G - 1) / G > TR) && A.scr == nullptr)) {
    if (tid == 0) atomicExch(P.err, 2);
    return;
  }
  const size_t blk = ((size_t)(TR + 1) * LD + 3) & ~(size_t)3;
  float* Dold = nb_smem;
  float* Rini = Dold + blk;
  float* V = Rini + blk;
  float* cbuf = V + blk;
  const size_t cbf = nb_cbuf_floats<KPT, T>(CH, kBlk);
  float* Dl = cbuf + cbf;                                       // blocked mode: (TR + 1) x 16
  const size_t dlf = kBlk ? (size_t)(TR + 1) * kNbCB : 0;
  const int H = max(1, nthr / max(k, 1));
  const size_t partw = (size_t)5 * H * KPT > (size_t)12 * k ? (size_t)5 * H * KPT : (size_t)12 * k;
  unsigned* pcn = reinterpret_cast<unsigned*>(Dl + dlf);
  float* ps1 = reinterpret_cast<float*>(pcn + H * KPT);
  float* ps2 = ps1 + H * KPT;
  unsigned* pmn = reinterpret_cast<unsigned*>(ps2 + H * KPT);
  unsigned* pmx = pmn + H * KPT;
  int* rows_s = reinterpret_cast<int*>(Dl + dlf + ((partw + 3) & ~(size_t)3));
  uint8_t* mbits_s = reinterpret_cast<uint8_t*>(rows_s + ((TR + 3) & ~3));
  const double a = P.a, b = P.b;
  if (tid == 0) mcnt_s = 0;

  // ---- setup: parameters, warm-start thresholds, M_{t+1} of my Philox slice --------
  for (int p = tid; p < KPT; p += nthr) {
    if (p < k) {
      const int j = P.perm[p];
      jmap_s[p] = j;
      pinv_s[j] = p;
      const bool dead = !(A.invc[p] > 0.f);                          // R10
      const double lw = dead ? 0.0 : P.lam_ws[j];
      lam_s[p] = lw;
      rho_s[p] = P.nslack[j];
      const int mode = dead ? kModeDead : (lw > 0.0 ? kModeShrink : kModeCopy);
      mode_s[p] = mode;
      vlo_s[p] = P.pos ? 0.f : -INFINITY;
      par_s[0][p] = par_s[1][p] = nt_make_par<kGen>(mode, a, b, lw, vlo_s[p]);
    } else {
      jmap_s[p] = 0;
      mode_s[p] = kModeDead;
      lam_s[p] = 0.0;
      rho_s[p] = 0.0;
      vlo_s[p] = -INFINITY;
      par_s[0][p] = par_s[1][p] = nt_make_par<kGen>(kModeDead, a, b, 0.0, -INFINITY);
    }
    acc1_s[p] = acc2_s[p] = 0.0;
  }
  // resident prescaled Cbar (NbRec mode): staged once
  if (!kBlk && CH >= KPT) {
    const int n4 = (int)(cbf / 4);
    for (int e = tid; e < n4; e += nthr) nb_cp16(cbuf + 4 * e, A.Ctg + 4 * e);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  int64_t mb0 = 0;
  int nmb = 0;
  if (P.idx_next) {
    const int64_t b0 = P.row_lo >> 2, nb = ((P.row_hi - 1) >> 2) - b0 + 1;
    mb0 = b0 + nb * blockIdx.x / G;
    nmb = (int)(b0 + nb * (blockIdx.x + 1) / G - mb0);
    int c = 0;
    for (int i = tid; i < nmb; i += nthr) {
      const uint32_t bits = mask_bits(P.seed, (uint64_t)P.tn, mb0 + i, P.row_lo, P.row_hi, P.Tthr);
      mbits_s[i] = (uint8_t)bits;
      c += __popc(bits);
    }
    c = (int)__reduce_add_sync(0xffffffffu, (unsigned)c);
    if (lane == 0 && c) atomicAdd(&mcnt_s, c);
  }
  __syncthreads();

  // ---- setup per tile: d_old and the prescaled residual in pi order ----------------
  // R0 = (P Bbar - P D Cbar) / c_pp, radii sums ||P d_j|| (R9)
  for (int e = tid; e < LD; e += nthr) {
    Dold[(size_t)TR * LD + e] = 0.f;
    Rini[(size_t)TR * LD + e] = 0.f;
  }
  for (int tl = 0; tl < ntile; ++tl) {
    const int r0 = tl * TR, nr = min(TR, nr_all - r0);
    for (int r = tid; r < nr; r += nthr) rows_s[r] = P.idx[lo + r0 + r];
    __syncthreads();
    // natural-order rows: D into V, Bbar into Rini (stride kp)
    {
      const int c4 = kp / 4;
      for (int e = tid; e < nr * c4; e += nthr) {
        const int row = e / c4, c = e % c4;
        const int64_t goff = (int64_t)rows_s[row] * kp + 4 * c;
        nb_cp16(V + (size_t)row * kp + 4 * c, P.D + goff);
        nb_cp16(Rini + (size_t)row * kp + 4 * c, P.Bbar + goff);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
    }
    NB_MARK(9);
    // d_old in pi order
    for (int e = tid; e < nr * KPT; e += nthr) {
      const int row = e / KPT, p = e % KPT;
      Dold[(size_t)row * LD + p] = p < k ? V[(size_t)row * kp + jmap_s[p]] : 0.f;
    }
    __syncthreads();
    // Bbar in pi order into V (row stride LD); blocked mode: prescaled by 1 / c_pp
    for (int e = tid; e < nr * KPT; e += nthr) {
      const int row = e / KPT, p = e % KPT;
      const float bb = p < k ? Rini[(size_t)row * kp + jmap_s[p]] : 0.f;
      V[(size_t)row * LD + p] = kBlk ? bb * A.invc[p] : bb;
    }
    __syncthreads();
    NB_MARK(10);
    if constexpr (kBlk) {
      // R0 = Bbar / c - Dold Cpre: rank-16 updates over every chunk of positions
      for (int e = tid; e < nr * LD; e += nthr) Rini[e] = V[e];
      int c = 0;
      nb_load_chunk<KPT>(cbuf, A.Cpi, 0, tid, nthr);
#pragma unroll 1
      for (; c < KPT / kNbCB; ++c) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        if (c + 1 < KPT / kNbCB) nb_load_chunk<KPT>(cbuf, A.Cpi, c + 1, tid, nthr);
        nb_rank16<KPT>(Rini, LD, Dold + c * kNbCB, LD, cbuf + (c & 1) * kNbCB * KPT, nr, 0, KPT, tid, nthr);
      }
      __syncthreads();
    } else {
      // R0[l] = Bbar[l] / c_ll - sum_p Dold[p] C[p][l] / c_ll from the resident
      // prescaled Cbar (cbuf, parity layout: (p, l = i T + t) at
      // p T CSTR + t CSTR + i; staged at the start, landed with the first
      // tile's rows).  Item = RT rows x 4 positions (one parity t, i0..i0+3),
      // 4 p per step: 4 + RT 16-byte shared loads per 16 RT FMAs.  (The
      // global-memory Cpi version was bound by L2 loads: L1 is ~30 KB next to
      // this kernel's shared memory; 187 us of setup per step at cfgC r=1.)
      constexpr int RT = 16, NIB = nb_kts(KPT, T) / 4;
      const int nrb = (nr + RT - 1) / RT;
      for (int it = tid; it < nrb * T * NIB; it += nthr) {
        const int ib = it % NIB, t = (it / NIB) % T, rb = (it / (NIB * T)) * RT;
        float acc[RT][4];
#pragma unroll
        for (int i = 0; i < RT; ++i)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[i][c] = 0.f;
        const float* cb = cbuf + (size_t)t * CSTR + 4 * ib;
        for (int p = 0; p < k; p += 4) {               // Dold and Cbar are zero past k (KPT % 4 == 0)
          float cv[4][4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 c4 = *reinterpret_cast<const float4*>(cb + (size_t)(p + j) * T * CSTR);
            cv[j][0] = c4.x; cv[j][1] = c4.y; cv[j][2] = c4.z; cv[j][3] = c4.w;
          }
#pragma unroll
          for (int i = 0; i < RT; ++i) {
            const float4 d = *reinterpret_cast<const float4*>(Dold + (size_t)min(rb + i, TR) * LD + p);
            const float dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int c = 0; c < 4; ++c) acc[i][c] = fmaf(dv[j], cv[j][c], acc[i][c]);
          }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int l = (4 * ib + c) * T + t;
          if (4 * ib + c >= KPT / T || l >= k) continue;
          const float iv = A.invc[l];
#pragma unroll
          for (int i = 0; i < RT; ++i) {
            const int row = rb + i;
            if (row < nr) Rini[(size_t)row * LD + l] = V[(size_t)row * LD + l] * iv - acc[i][c];
          }
        }
      }
      __syncthreads();
    }
    for (int e = tid; e < nr * LD; e += nthr) {                 // padding positions of R0
      const int p = e % LD;
      if (p >= k) Rini[e] = 0.f;
    }
    NB_MARK(11);
    // radii sums of this tile (fp64, fixed order: tile by tile)
    {
      const int nwarp = nthr >> 5;
      for (int p = wid; p < k; p += nwarp) {
        double d1 = 0.0, d2 = 0.0;
        for (int row = lane; row < nr; row += 32) {
          const double d = Dold[(size_t)row * LD + p];
          d1 += fabs(d);
          d2 += d * d;
        }
        d1 = warp_sum(d1);
        d2 = warp_sum(d2);
        if (lane == 0) {
          acc1_s[p] += d1;
          acc2_s[p] += d2;
        }
      }
    }
    __syncthreads();
    if (streamed) {
      // the tile's d_old | R0 rows to the scratch (2 KPT floats per row)
      float* sc = A.scr + (size_t)(lo + r0) * 2 * KPT;
      for (int e = tid; e < nr * KPT; e += nthr) {
        const int row = e / KPT, p = e % KPT;
        sc[(size_t)row * 2 * KPT + p] = Dold[(size_t)row * LD + p];
        sc[(size_t)row * 2 * KPT + KPT + p] = Rini[(size_t)row * LD + p];
      }
      __syncthreads();
    }
    NB_MARK(12);
  }
  if (nr_all > 0 && tid < k) {
    unsigned long long* rr = P.rec + (((size_t)kNtRing * P.ncopy + blockIdx.x % P.ncopy) * k + tid) * kNtRec;
    const bool ok = fx_red(rr + 1, acc1_s[tid]) & fx_red(rr + 3, acc2_s[tid]);
    if (!ok) atomicExch(P.err, 6);
  }
  if (!kBlk && CH >= KPT) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (P.idx_next && tid == 0) P.cnt_next[blockIdx.x] = mcnt_s;   // before round 0's barrier

  // my rows within a tile (NbRec mode): M consecutive rows of group g; rows >= nr use the spare row
  const int g = tid / T, tq = tid % T;
  const int ngroups = (TR + M - 1) / M;

  unsigned nbar = 0;
  int round = 0, cur = 0;
  bool done = q == 0;
  if (tid == 0) {
    lockF_s = 0;
    prevF_s = 0;
  }
  if (done && P.idx_next) {
    ++nbar;
    nt_barrier(P.bar, nbar * G);
  }
#pragma unroll 1
  __syncthreads();
  if (!kBlk && streamed && ntile > 0) nb_prefetch<KPT>(A.scr, 0, TR, nr_all, lo, Dold, Rini, tid, nthr);
  NB_MARK(0);
  while (!done) {
    const int ring = round % kNtRing;
    for (int p = tid; p < k; p += nthr) {
      acn_s[p] = 0u;
      amn_s[p] = 0xffffffffu;
      amx_s[p] = 0u;
      acc1_s[p] = acc2_s[p] = 0.0;
    }
    for (int tl = 0; tl < ntile; ++tl) {
      const int nr = nb_tile_pass<KPT, T, M, kGen, CH, kBlk>(A.scr, A.Cpi, A.Ctg, tl, TR, nr_all, lo, streamed, Dold, Rini, V, cbuf,
                                                            Dl, par_s[cur], g, tq, ngroups, tid, nthr, ldp);
      NB_MARK(1);
      // per-atom statistics of the tile, added to the CTA sums in tile order
      if (tid < H * k) {
        const int p = tid % k, h = tid / k;
        const double th = a * lam_s[p];
        const float thf = th > 0.0 ? __double2float_rd(th) : 0.f;
        unsigned cnt = 0, mn = 0xffffffffu, mx = 0u;
        float s1 = 0.f, s2 = 0.f;
        for (int r = h; r < nr; r += H) {
          const float av = fabsf(V[(size_t)r * LD + p]);
          const bool above = av > thf;
          cnt += above;
          s1 += above ? av : 0.f;
          s2 = fmaf(above ? av : 0.f, av, s2);
          mn = above ? min(mn, __float_as_uint(av)) : mn;
          mx = above ? mx : max(mx, __float_as_uint(av));
        }
        pcn[h * KPT + p] = cnt;
        ps1[h * KPT + p] = s1;
        ps2[h * KPT + p] = s2;
        pmn[h * KPT + p] = mn;
        pmx[h * KPT + p] = mx;
      }
      __syncthreads();
      if (tid < k) {
        const int p = tid;
        unsigned cnt = acn_s[p], mn = amn_s[p], mx = amx_s[p];
        double S1 = 0.0, S2 = 0.0;
        for (int h = 0; h < H; ++h) {
          cnt += pcn[h * KPT + p];
          S1 += (double)ps1[h * KPT + p];
          S2 += (double)ps2[h * KPT + p];
          mn = min(mn, pmn[h * KPT + p]);
          mx = max(mx, pmx[h * KPT + p]);
        }
        acn_s[p] = cnt;
        amn_s[p] = mn;
        amx_s[p] = mx;
        acc1_s[p] += S1;
        acc2_s[p] += S2;
      }
      __syncthreads();
      NB_MARK(2);
    }
    if (nr_all > 0 && tid < k) {
      const int p = tid;
      unsigned long long* rc = P.rec + (((size_t)ring * P.ncopy + blockIdx.x % P.ncopy) * k + p) * kNtRec;
      unsigned* mm = reinterpret_cast<unsigned*>(rc + 5);
      if (acn_s[p] > 0) {
        nt_red_u64(rc, (unsigned long long)acn_s[p]);
        const bool ok = fx_red(rc + 1, acc1_s[p]) & fx_red(rc + 3, acc2_s[p]);
        if (!ok) atomicExch(P.err, 6);
        atomicMin(mm, amn_s[p]);
      }
      if (amx_s[p]) atomicMax(mm + 1, amx_s[p]);
    }
    ++nbar;
    nt_barrier(P.bar, nbar * G);
    NB_MARK(3);
    {
      const int rz = (round + 2) % kNtRing;          // (see k_bcd_newton)
      for (int e = blockIdx.x + G * tid; e < P.ncopy * k; e += G * nthr)
        nt_rec_reset(P.rec + ((size_t)rz * P.ncopy * k + e) * kNtRec);
    }
    // ---- the same Michelot step for every atom in every CTA ----
    int conv = 1, nmode = 0;
    double nlam = 0.0, cnt = 0.0, S1 = 0.0, S2 = 0.0, mn_d = 0.0, mx_d = 0.0;
    const int p = tid;
    const bool act = tid < k;
    unsigned long long* rdp = reinterpret_cast<unsigned long long*>(pcn);
    if (round == 0) {
      nt_read_coop(P.rec + (size_t)kNtRing * P.ncopy * k * kNtRec, P.ncopy, k, P.rd_h, rdp);
      __syncthreads();
      if (act) {
        const NtSums rs = nt_combine(rdp, P.rd_h, k, p);
        rho_s[p] = fmax(0.0, rho_s[p] + a * rs.S1 + 0.5 * b * rs.S2);     // P:860, R9
      }
      __syncthreads();
    }
    nt_read_coop(P.rec + (size_t)ring * P.ncopy * k * kNtRec, P.ncopy, k, P.rd_h, rdp);
    __syncthreads();
    if (act) {
      const NtSums sm = nt_combine(rdp, P.rd_h, k, p);
      cnt = sm.cnt;
      S1 = sm.S1;
      S2 = sm.S2;
      const double mnv = cnt > 0.0 ? (double)__uint_as_float(sm.mn) : INFINITY;
      const double mxv = (double)__uint_as_float(sm.mx);
      mn_d = mnv;
      mx_d = mxv;
      conv = nt_atom_update(a, b, rho_s[p], cnt, S1, S2, mnv, mxv, mode_s[p], lam_s[p], &nmode, &nlam, P.lam_tol,
                            round >= kNtRelaxRound);
      if (p < lockF_s) conv = 1;                  // locked prefix: parameters final (R22)
    }
    // first unconverged position; after kNtRelaxRound every position before it
    // is locked for the rest of the step (R22): in exact arithmetic the prefix
    // never regresses (the recurrence is triangular and converged atoms keep
    // their parameters), so the lock only guarantees termination
    if (tid == 0) firstU_s = k;
    __syncthreads();
    if (act && !conv) atomicMin(&firstU_s, p);
    const bool all_conv = __syncthreads_and(conv);
    if (tid == 0) {
      if (P.prof && blockIdx.x == 0 && firstU_s < prevF_s)
        atomicAdd(reinterpret_cast<unsigned long long*>(P.prof + 92), 1ull);   // prefix regressions
      prevF_s = firstU_s;
      if (round >= kNtRelaxRound) lockF_s = max(lockF_s, firstU_s);
    }
    const bool capped = round + 1 >= P.max_rounds && !all_conv;
    if (P.prof && blockIdx.x == 0) {
      // diagnostics: unconverged atoms per round (slots 8..71); at the round
      // cap, the first unconverged position's state (slots 72..79, raw bits)
      const int nun = __syncthreads_count(act && !conv);
      if (tid == 0 && round < 64) atomicAdd(reinterpret_cast<unsigned long long*>(P.prof + 8 + round),
                                            (unsigned long long)nun + ((unsigned long long)firstU_s << 16));
      if (act && round < 64 && p == firstU_s) {
        P.prof[96 + round] = __double_as_longlong(lam_s[p]);
        P.prof[160 + round] = __double_as_longlong(nlam);
      }
      if (capped) {
        if (tid == 0) mcnt_s = k;
        __syncthreads();
        if (act && !conv) atomicMin(&mcnt_s, p);
        __syncthreads();
        if (act && p == mcnt_s) {
          const double dv[8] = {(double)p + 1000.0 * nmode + 100000.0 * mode_s[p], lam_s[p], nlam, cnt,
                                mn_d, mx_d, rho_s[p], S1};
          for (int i = 0; i < 8; ++i) P.prof[72 + i] = __double_as_longlong(dv[i]);
        }
        __syncthreads();
      }
    }
    if (act) {
      if (all_conv || capped) {
        if (mode_s[p] != kModeDead && blockIdx.x == 0) {
          const int j = jmap_s[p];
          P.nslack[j] = rho_s[p] - nt_norm_d(a, b, mode_s[p], lam_s[p], cnt, S1, S2);
          P.lam_ws[j] = lam_s[p];
        }
        par_s[cur ^ 1][p] = par_s[cur][p];
      } else if (conv) {
        // converged atoms keep their parameters while others move: the v of
        // the atoms after them then only change when an unconverged atom
        // before them does (no tolerance-level jitter propagating down the
        // chain; at cfgE it kept later atoms from ever settling)
        par_s[cur ^ 1][p] = par_s[cur][p];
      } else {
        lam_s[p] = nlam;
        mode_s[p] = nmode;
        par_s[cur ^ 1][p] = nt_make_par<kGen>(nmode, a, b, nlam, vlo_s[p]);
      }
    }
    ++round;
    if (all_conv) {
      done = true;
    } else if (capped) {
      if (tid == 0 && blockIdx.x == 0) atomicExch(P.err, 4);
      done = true;
    }
    if (!done) cur ^= 1;
    __syncthreads();
    NB_MARK(4);
  }
  // ---- final D: v of the final round through its parameters (several tiles: one
  // more pass per tile with the final parameters) ----
  if (q > 0) {
    const NtPar<kGen>* pr = par_s[cur];
    for (int tl = 0; tl < ntile; ++tl) {
      int nr = min(TR, nr_all - tl * TR);
      if (ntile > 1) nr = nb_tile_pass<KPT, T, M, kGen, CH, kBlk>(A.scr, A.Cpi, A.Ctg, tl, TR, nr_all, lo, streamed, Dold, Rini, V,
                                                                cbuf, Dl, pr, g, tq, ngroups, tid, nthr);
      if (ntile > 1) {
        for (int r = tid; r < nr; r += nthr) rows_s[r] = P.idx[lo + tl * TR + r];
        __syncthreads();
      }
      for (int r = wid; r < nr; r += (nthr >> 5)) {
        float* dst = P.D + (int64_t)rows_s[r] * kp;
        const float* src = V + (size_t)r * LD;
        for (int j = lane; j < k; j += 32) {
          const int pp = pinv_s[j];
          dst[j] = pr[pp].d_of(src[pp]);
        }
      }
      __syncthreads();
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");      // (the last pass prefetched tile 0 again)
  NB_MARK(5);
  // ---- draw-ahead of t+1: scatter of my slice of M_{t+1}, t+1, w_{t+1} ----
  if (P.idx_next) {
    if (wid == 0) {
      int64_t off = 0;
      for (int i = lane; i < (int)blockIdx.x; i += 32) off += __ldcg(P.cnt_next + i);
      off = warp_sum(off);
      const int i0 = nmb * lane / 32, i1 = nmb * (lane + 1) / 32;
      int c = 0;
      for (int i = i0; i < i1; ++i) c += __popc((unsigned)mbits_s[i]);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int64_t pos = off + incl - c;
      for (int i = i0; i < i1; ++i) {
        const unsigned bits = mbits_s[i];
        for (int l = 0; l < 4; ++l)
          if (bits & (1u << l)) P.idx_next[pos++] = (int32_t)((mb0 + i) * 4 + l - P.row_lo);
      }
      if (blockIdx.x == G - 1 && lane == 31) *P.q_next = pos;
    }
    if (blockIdx.x == 0 && tid == 0) {
      *P.t_next = P.tn;
      store_coef(P.w_next, P.cf_next);
    }
  }
  // ---- exit: last CTA resets counters and accumulators ----
  __syncthreads();
  NB_MARK(6);
  if (P.prof && blockIdx.x == 0 && threadIdx.x == 0) {
    nbp_s[7] = 1;
    for (int i = 0; i < 8; ++i) P.prof[i] += nbp_s[i];
    P.prof[82] += nbp_s[8];
    P.prof[83] += nbp_s[9];
    P.prof[93] += nbp_s[10];
    P.prof[94] += nbp_s[11];
    P.prof[95] += nbp_s[12];
  }
#undef NB_MARK
  if (tid == 0) {
    __threadfence();
    const unsigned old = atomicAdd(P.bar + 1, 1u);
    mcnt_s = old == (unsigned)G - 1;
  }
  __syncthreads();
  if (mcnt_s) {
    __threadfence();
    for (int e = tid; e < (kNtRing + 1) * P.ncopy * k; e += nthr) nt_rec_reset(P.rec + (size_t)e * kNtRec);
    if (tid == 0) {
      if (P.nred_out) *P.nred_out = nbar;
      P.bar[0] = 0u;
      P.bar[1] = 0u;
    }
    __threadfence();
  }
}

}  // namespace somf
