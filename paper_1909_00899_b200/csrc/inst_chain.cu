// Strip-pipeline (long pair) kernel instances.
#include "sw_chain32.cuh"
using namespace swb;

#ifndef SWB_CHAIN_SPLIT
#define SWB_CHAIN_SPLIT 1  // 32-bit strips: carry-split column schedule (sw_chain32.cuh)
#endif

void swb_fill_chain(const void* (&tab)[2][6], const void* (&ptab)[2], const void* (&so)[6]) {
  tab[0][0] = (const void*)&sw_chain_kernel<W16, 1, VAR_SCAN>;
  tab[0][1] = (const void*)&sw_chain_kernel<W16, 2, VAR_SCAN>;
  tab[0][2] = (const void*)&sw_chain_kernel<W16, 4, VAR_SCAN>;
  tab[0][3] = (const void*)&sw_chain_kernel<W16, 8, VAR_SCAN>;
  tab[0][4] = (const void*)&sw_chain_kernel<W16, 16, VAR_SCAN>;
  tab[0][5] = (const void*)&sw_chain_kernel<W16, 32, VAR_SCAN>;
  tab[1][0] = SWB_CHAIN_SPLIT ? (const void*)&sw_chain32_kernel<1> : (const void*)&sw_chain_kernel<W32, 1, VAR_SCAN>;
  tab[1][1] = SWB_CHAIN_SPLIT ? (const void*)&sw_chain32_kernel<2> : (const void*)&sw_chain_kernel<W32, 2, VAR_SCAN>;
  tab[1][2] = SWB_CHAIN_SPLIT ? (const void*)&sw_chain32_kernel<4> : (const void*)&sw_chain_kernel<W32, 4, VAR_SCAN>;
  tab[1][3] = SWB_CHAIN_SPLIT ? (const void*)&sw_chain32_kernel<8> : (const void*)&sw_chain_kernel<W32, 8, VAR_SCAN>;
  tab[1][4] = SWB_CHAIN_SPLIT ? (const void*)&sw_chain32_kernel<16> : (const void*)&sw_chain_kernel<W32, 16, VAR_SCAN>;
  tab[1][5] = SWB_CHAIN_SPLIT ? (const void*)&sw_chain32_kernel<32> : (const void*)&sw_chain_kernel<W32, 32, VAR_SCAN>;
  // score-only 32-bit strips (no end-coordinate tracking)
  so[0] = (const void*)&sw_chain32_kernel<1, false>;
  so[1] = (const void*)&sw_chain32_kernel<2, false>;
  so[2] = (const void*)&sw_chain32_kernel<4, false>;
  so[3] = (const void*)&sw_chain32_kernel<8, false>;
  so[4] = (const void*)&sw_chain32_kernel<16, false>;
  so[5] = (const void*)&sw_chain32_kernel<32, false>;
  ptab[0] = (const void*)&sw_chain_profile_kernel<W16>;
  ptab[1] = (const void*)&sw_chain_profile_kernel<W32>;
}
