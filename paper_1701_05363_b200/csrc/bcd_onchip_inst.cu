// bcd_onchip_inst.cu -- instantiates the on-chip per-atom BCD kernel
// k_bcd_onchip<KC, RPW> (bcd_onchip.cuh) in its own translation unit so the
// library builds in parallel; somf_capi.cu asks for a variant by (KC, RPW).
#include "bcd_onchip.cuh"

#define OCV(KC, RPW) \
  if (kc == KC && rpw == RPW) return (const void*)somf::k_bcd_onchip<KC, RPW>;

const void* somf_oc_kernel(int kc, int rpw) {
  OCV(1, 2) OCV(1, 4) OCV(1, 8) OCV(1, 12) OCV(1, 16) OCV(1, 24) OCV(1, 32)
  OCV(2, 2) OCV(2, 4) OCV(2, 8) OCV(2, 12) OCV(2, 16) OCV(2, 24) OCV(2, 32)
  OCV(3, 2) OCV(3, 4) OCV(3, 8) OCV(3, 12) OCV(3, 16) OCV(3, 24)
  OCV(4, 2) OCV(4, 4) OCV(4, 8) OCV(4, 12) OCV(4, 16)
  OCV(8, 2) OCV(8, 4) OCV(8, 8)
  return nullptr;
}
