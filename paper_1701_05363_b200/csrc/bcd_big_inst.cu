// bcd_big_inst.cu -- instantiates k_bcd_big<NB_KPT, T, 2, gen, CH> (bcd_big.cuh):
// groups of T = 4 (KPT <= 72), 8 (KPT <= 128) or 16 lanes owning 2 masked rows;
// the prescaled Cbar rows resident (CH = KPT) up to KPT = 128, else streamed
// from L2 in chunks of CH = 16 positions.  Compiled once per NB_KPT so the
// variants build in parallel; somf_capi.cu picks one through somf_nb_kernel_<KPT>.
#include "bcd_big.cuh"

#ifndef NB_KPT
#error "compile with -DNB_KPT=<positions per row>"
#endif
#define NB_CAT2(a, b) a##b
#define NB_CAT(a, b) NB_CAT2(a, b)

namespace {
constexpr int kT = NB_KPT <= 72 ? 4 : NB_KPT <= 128 ? 8 : 16;
constexpr int kCH = NB_KPT <= 128 ? NB_KPT : 16;
}

// (gen: mu > 0 or D >= 0) -> kernel; *T, *ch: its group width and Cbar chunk
const void* NB_CAT(somf_nb_kernel_, NB_KPT)(int gen, int* T, int* ch) {
  *T = kT;
  *ch = kCH;
  return gen ? (const void*)somf::k_bcd_big<NB_KPT, kT, 2, true, kCH>
             : (const void*)somf::k_bcd_big<NB_KPT, kT, 2, false, kCH>;
}
