// Strip-pipeline (long pair) kernel instances with the gap-extend penalty fixed at 1.
#include "sw_chain32.cuh"
using namespace swb;

void swb_fill_chain_g1(const void* (&tab)[6], const void* (&so)[6]) {
  tab[0] = (const void*)&sw_chain32_kernel<1, true, 1>;
  tab[1] = (const void*)&sw_chain32_kernel<2, true, 1>;
  tab[2] = (const void*)&sw_chain32_kernel<4, true, 1>;
  tab[3] = (const void*)&sw_chain32_kernel<8, true, 1>;
  tab[4] = (const void*)&sw_chain32_kernel<16, true, 1>;
  tab[5] = (const void*)&sw_chain32_kernel<32, true, 1>;
  so[0] = (const void*)&sw_chain32_kernel<1, false, 1>;
  so[1] = (const void*)&sw_chain32_kernel<2, false, 1>;
  so[2] = (const void*)&sw_chain32_kernel<4, false, 1>;
  so[3] = (const void*)&sw_chain32_kernel<8, false, 1>;
  so[4] = (const void*)&sw_chain32_kernel<16, false, 1>;
  so[5] = (const void*)&sw_chain32_kernel<32, false, 1>;
}
