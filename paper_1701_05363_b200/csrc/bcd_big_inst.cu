// bcd_big_inst.cu -- instantiates k_bcd_big (bcd_big.cuh) for one NB_KPT:
//   KPT <= 128: unrolled per-position recurrence, groups of T = 4 (KPT <= 72)
//               or 8 lanes owning 2 masked rows, prescaled Cbar resident;
//   KPT >  128: blocked recurrence (chunks of 16 positions, one thread per
//               row + rank-16 updates), Cbar streamed from L2 in 16-row chunks.
// Compiled once per NB_KPT so the variants build in parallel; somf_capi.cu
// picks one through somf_nb_kernel_<KPT>.
#include "bcd_big.cuh"

#ifndef NB_KPT
#error "compile with -DNB_KPT=<positions per row>"
#endif
#define NB_CAT2(a, b) a##b
#define NB_CAT(a, b) NB_CAT2(a, b)

namespace {
constexpr bool kBlk = NB_KPT > 128;
constexpr int kT = kBlk ? 1 : NB_KPT <= 72 ? 4 : 8;
constexpr int kCH = kBlk ? somf::kNbCB : NB_KPT;
}

// (gen: mu > 0 or D >= 0) -> kernel; *T, *ch, *blk: its group width, Cbar chunk, mode
const void* NB_CAT(somf_nb_kernel_, NB_KPT)(int gen, int* T, int* ch, int* blk) {
  *T = kT;
  *ch = kCH;
  *blk = kBlk;
  return gen ? (const void*)somf::k_bcd_big<NB_KPT, kT, 2, true, kCH, kBlk>
             : (const void*)somf::k_bcd_big<NB_KPT, kT, 2, false, kCH, kBlk>;
}
