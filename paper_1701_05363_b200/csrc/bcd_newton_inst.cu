// bcd_newton_inst.cu -- instantiates the simultaneous-threshold BCD kernel
// k_bcd_newton<NT_KPT, T, M, gen> (bcd_newton.cuh) for groups of T = 4 (8 at
// KPT = 128) threads owning M = 2 masked rows.  Compiled once per NT_KPT (-DNT_KPT=...) so the variants build in
// parallel; the C ABI (somf_capi.cu) picks one through somf_nt_kernel_<KPT>.
#include "bcd_newton.cuh"

#ifndef NT_KPT
#error "compile with -DNT_KPT=<positions per row>"
#endif
#define NT_CAT2(a, b) a##b
#define NT_CAT(a, b) NT_CAT2(a, b)

// T threads x M rows per group; gen = generic parameters (mu > 0 or D >= 0).
// v6 (M = 1, packed FFMA2): T = 1 (one thread per row) for KPT <= 96, T = 2
// (two threads per row, also KPT = 128); v5 (M = 2): 4 x 2, and 8 x 2 at
// KPT = 128 (the residual of 4 x 2 would not fit the registers).
const void* NT_CAT(somf_nt_kernel_, NT_KPT)(int T, int M, int gen) {
#if NT_KPT > 96
  if (T == 8 && M == 2) return gen ? (const void*)somf::k_bcd_newton<NT_KPT, 8, 2, true>
                                   : (const void*)somf::k_bcd_newton<NT_KPT, 8, 2, false>;
  if (T == 2 && M == 1) return gen ? (const void*)somf::k_bcd_newton<NT_KPT, 2, 1, true>
                                   : (const void*)somf::k_bcd_newton<NT_KPT, 2, 1, false>;
#else
  if (T == 4 && M == 2) return gen ? (const void*)somf::k_bcd_newton<NT_KPT, 4, 2, true>
                                   : (const void*)somf::k_bcd_newton<NT_KPT, 4, 2, false>;
  if (T == 1 && M == 1) return gen ? (const void*)somf::k_bcd_newton<NT_KPT, 1, 1, true>
                                   : (const void*)somf::k_bcd_newton<NT_KPT, 1, 1, false>;
  if (T == 2 && M == 1) return gen ? (const void*)somf::k_bcd_newton<NT_KPT, 2, 1, true>
                                   : (const void*)somf::k_bcd_newton<NT_KPT, 2, 1, false>;
#endif
  return nullptr;
}
