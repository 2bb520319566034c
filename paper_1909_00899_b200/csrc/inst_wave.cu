// Strip-pipeline wavefront (long pair) kernel instances: rows per lane L = 1, 2, 4, 8.
#include "sw_wave.cuh"
using namespace swb;

void swb_fill_wave(const void* (&tab)[4]) {
  tab[0] = (const void*)&sw_wave_kernel<1>;
  tab[1] = (const void*)&sw_wave_kernel<2>;
  tab[2] = (const void*)&sw_wave_kernel<4>;
  tab[3] = (const void*)&sw_wave_kernel<8>;
}
