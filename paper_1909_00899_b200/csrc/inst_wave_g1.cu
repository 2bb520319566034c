// Wavefront strip instances with the gap-extend penalty fixed at 1.
#include "sw_wave.cuh"
using namespace swb;

template <int L, int KC>
static void put(const void* (&tab)[4][4], int li, int ki) {
  tab[li][ki] = (const void*)&sw_wave_kernel<L, KC, 1>;
}

void swb_fill_wave_g1(const void* (&tab)[4][4]) {
  put<1, 1>(tab, 0, 0); put<1, 2>(tab, 0, 1); put<1, 4>(tab, 0, 2); put<1, 8>(tab, 0, 3);
  put<2, 1>(tab, 1, 0); put<2, 2>(tab, 1, 1); put<2, 4>(tab, 1, 2); put<2, 8>(tab, 1, 3);
  put<4, 1>(tab, 2, 0); put<4, 2>(tab, 2, 1); put<4, 4>(tab, 2, 2); put<4, 8>(tab, 2, 3);
  put<8, 1>(tab, 3, 0); put<8, 2>(tab, 3, 1); put<8, 4>(tab, 3, 2); put<8, 8>(tab, 3, 3);
}
