// Strip-pipeline (long pair) kernel instances.
#include "sw_chain.cuh"
using namespace swb;

void swb_fill_chain(const void* (&tab)[2][6], const void* (&ptab)[2]) {
  tab[0][0] = (const void*)&sw_chain_kernel<W16, 1, VAR_SCAN>;
  tab[0][1] = (const void*)&sw_chain_kernel<W16, 2, VAR_SCAN>;
  tab[0][2] = (const void*)&sw_chain_kernel<W16, 4, VAR_SCAN>;
  tab[0][3] = (const void*)&sw_chain_kernel<W16, 8, VAR_SCAN>;
  tab[0][4] = (const void*)&sw_chain_kernel<W16, 16, VAR_SCAN>;
  tab[0][5] = (const void*)&sw_chain_kernel<W16, 32, VAR_SCAN>;
  tab[1][0] = (const void*)&sw_chain_kernel<W32, 1, VAR_SCAN>;
  tab[1][1] = (const void*)&sw_chain_kernel<W32, 2, VAR_SCAN>;
  tab[1][2] = (const void*)&sw_chain_kernel<W32, 4, VAR_SCAN>;
  tab[1][3] = (const void*)&sw_chain_kernel<W32, 8, VAR_SCAN>;
  tab[1][4] = (const void*)&sw_chain_kernel<W32, 16, VAR_SCAN>;
  tab[1][5] = (const void*)&sw_chain_kernel<W32, 32, VAR_SCAN>;
  ptab[0] = (const void*)&sw_chain_profile_kernel<W16>;
  ptab[1] = (const void*)&sw_chain_profile_kernel<W32>;
}
