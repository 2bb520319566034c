// Block / cluster scan kernel instances (32-bit): segment length L = 1..16, three variants.
#include "sw_block.cuh"
using namespace swb;

void swb_fill_block32(const void* (&tab)[3][16]) {
  tab[0][0] = (const void*)&sw_block_kernel<W32, 1, VAR_SCAN>;
  tab[0][1] = (const void*)&sw_block_kernel<W32, 2, VAR_SCAN>;
  tab[0][2] = (const void*)&sw_block_kernel<W32, 3, VAR_SCAN>;
  tab[0][3] = (const void*)&sw_block_kernel<W32, 4, VAR_SCAN>;
  tab[0][4] = (const void*)&sw_block_kernel<W32, 5, VAR_SCAN>;
  tab[0][5] = (const void*)&sw_block_kernel<W32, 6, VAR_SCAN>;
  tab[0][6] = (const void*)&sw_block_kernel<W32, 7, VAR_SCAN>;
  tab[0][7] = (const void*)&sw_block_kernel<W32, 8, VAR_SCAN>;
  tab[0][8] = (const void*)&sw_block_kernel<W32, 9, VAR_SCAN>;
  tab[0][9] = (const void*)&sw_block_kernel<W32, 10, VAR_SCAN>;
  tab[0][10] = (const void*)&sw_block_kernel<W32, 11, VAR_SCAN>;
  tab[0][11] = (const void*)&sw_block_kernel<W32, 12, VAR_SCAN>;
  tab[0][12] = (const void*)&sw_block_kernel<W32, 13, VAR_SCAN>;
  tab[0][13] = (const void*)&sw_block_kernel<W32, 14, VAR_SCAN>;
  tab[0][14] = (const void*)&sw_block_kernel<W32, 15, VAR_SCAN>;
  tab[0][15] = (const void*)&sw_block_kernel<W32, 16, VAR_SCAN>;
  tab[1][0] = (const void*)&sw_block_kernel<W32, 1, VAR_LAZYF>;
  tab[1][1] = (const void*)&sw_block_kernel<W32, 2, VAR_LAZYF>;
  tab[1][2] = (const void*)&sw_block_kernel<W32, 3, VAR_LAZYF>;
  tab[1][3] = (const void*)&sw_block_kernel<W32, 4, VAR_LAZYF>;
  tab[1][4] = (const void*)&sw_block_kernel<W32, 5, VAR_LAZYF>;
  tab[1][5] = (const void*)&sw_block_kernel<W32, 6, VAR_LAZYF>;
  tab[1][6] = (const void*)&sw_block_kernel<W32, 7, VAR_LAZYF>;
  tab[1][7] = (const void*)&sw_block_kernel<W32, 8, VAR_LAZYF>;
  tab[1][8] = (const void*)&sw_block_kernel<W32, 9, VAR_LAZYF>;
  tab[1][9] = (const void*)&sw_block_kernel<W32, 10, VAR_LAZYF>;
  tab[1][10] = (const void*)&sw_block_kernel<W32, 11, VAR_LAZYF>;
  tab[1][11] = (const void*)&sw_block_kernel<W32, 12, VAR_LAZYF>;
  tab[1][12] = (const void*)&sw_block_kernel<W32, 13, VAR_LAZYF>;
  tab[1][13] = (const void*)&sw_block_kernel<W32, 14, VAR_LAZYF>;
  tab[1][14] = (const void*)&sw_block_kernel<W32, 15, VAR_LAZYF>;
  tab[1][15] = (const void*)&sw_block_kernel<W32, 16, VAR_LAZYF>;
  tab[2][0] = (const void*)&sw_block_kernel<W32, 1, VAR_LAZYF_MIRROR>;
  tab[2][1] = (const void*)&sw_block_kernel<W32, 2, VAR_LAZYF_MIRROR>;
  tab[2][2] = (const void*)&sw_block_kernel<W32, 3, VAR_LAZYF_MIRROR>;
  tab[2][3] = (const void*)&sw_block_kernel<W32, 4, VAR_LAZYF_MIRROR>;
  tab[2][4] = (const void*)&sw_block_kernel<W32, 5, VAR_LAZYF_MIRROR>;
  tab[2][5] = (const void*)&sw_block_kernel<W32, 6, VAR_LAZYF_MIRROR>;
  tab[2][6] = (const void*)&sw_block_kernel<W32, 7, VAR_LAZYF_MIRROR>;
  tab[2][7] = (const void*)&sw_block_kernel<W32, 8, VAR_LAZYF_MIRROR>;
  tab[2][8] = (const void*)&sw_block_kernel<W32, 9, VAR_LAZYF_MIRROR>;
  tab[2][9] = (const void*)&sw_block_kernel<W32, 10, VAR_LAZYF_MIRROR>;
  tab[2][10] = (const void*)&sw_block_kernel<W32, 11, VAR_LAZYF_MIRROR>;
  tab[2][11] = (const void*)&sw_block_kernel<W32, 12, VAR_LAZYF_MIRROR>;
  tab[2][12] = (const void*)&sw_block_kernel<W32, 13, VAR_LAZYF_MIRROR>;
  tab[2][13] = (const void*)&sw_block_kernel<W32, 14, VAR_LAZYF_MIRROR>;
  tab[2][14] = (const void*)&sw_block_kernel<W32, 15, VAR_LAZYF_MIRROR>;
  tab[2][15] = (const void*)&sw_block_kernel<W32, 16, VAR_LAZYF_MIRROR>;
}
