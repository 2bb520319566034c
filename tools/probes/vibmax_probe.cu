// Probe: do __vibmax_s16x2's predicates (a >= b per half) survive ptxas fusion into
// VIMNMX.S16x2 with predicate outputs?  Build: nvcc -arch=sm_100a vibmax_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__global__ void k(const uint32_t* a, const uint32_t* b, int n, int* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // mimic the search loop: several words against one key, predicates folded into indices
  uint32_t key = b[i];
  int j0 = 99, j1 = 99;
#pragma unroll
  for (int c = 7; c >= 0; --c) {
    bool ph, pl;
    (void)__vibmax_s16x2(a[i * 8 + c], key, &ph, &pl);
    if (pl) j0 = c;
    if (ph) j1 = c;
  }
  out[2 * i] = j0;
  out[2 * i + 1] = j1;
}
int main() {
  const int n = 1 << 16;
  uint32_t *a, *b; int* o;
  cudaMallocManaged(&a, n * 8 * 4); cudaMallocManaged(&b, n * 4); cudaMallocManaged(&o, n * 8);
  srand(7);
  for (int i = 0; i < n; ++i) {
    uint32_t kk = ((rand() % 64) << 16) | (rand() % 64);
    b[i] = kk;
    for (int c = 0; c < 8; ++c) a[i * 8 + c] = ((rand() % 64) << 16) | (rand() % 64);
    if (i % 3 == 0) a[i * 8 + (i % 8)] = kk;  // exact ties
  }
  k<<<n / 256, 256>>>(a, b, n, o);
  cudaDeviceSynchronize();
  long bad = 0;
  for (int i = 0; i < n; ++i) {
    int e0 = 99, e1 = 99;
    for (int c = 7; c >= 0; --c) {
      if ((int16_t)(a[i * 8 + c] & 0xffff) >= (int16_t)(b[i] & 0xffff)) e0 = c;
      if ((int16_t)(a[i * 8 + c] >> 16) >= (int16_t)(b[i] >> 16)) e1 = c;
    }
    if (o[2 * i] != e0 || o[2 * i + 1] != e1) {
      if (bad < 5) printf("i=%d got (%d,%d) want (%d,%d)\n", i, o[2 * i], o[2 * i + 1], e0, e1);
      ++bad;
    }
  }
  printf("vibmax_probe: %ld / %d mismatches\n", bad, n);
  return bad != 0;
}
