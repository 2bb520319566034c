// Which pipe executes each candidate cell-update instruction?  Issue-rate probe:
// every SM runs 8 warps x 8 independent chains of one instruction kind (or a 1:1
// mix of two), timed with events.  A mix running at ~2x the single-kind rate
// means the two kinds issue to different pipes (ALU vs FMA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe pipe_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
template <int KIND>
__global__ void probe(uint32_t* out, int iters, uint32_t k1, uint32_t k2) {
  uint32_t v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x * 7 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (KIND == 0) v[c] = __viaddmax_s16x2(v[c], k1, k2);            // DPX add-max
      if (KIND == 1) v[c] = __vadd2(v[c], k1);                           // packed add
      if (KIND == 2) v[c] = (c & 1) ? __vadd2(v[c], k1) : __viaddmax_s16x2(v[c], k1, k2);
      if (KIND == 3) v[c] = v[c] * k1 + k2;                              // IMAD
      if (KIND == 4) v[c] = (c & 1) ? v[c] * k1 + k2 : __viaddmax_s16x2(v[c], k1, k2);
      if (KIND == 5) v[c] = __vmaxs2(v[c], k1);                          // packed max
      if (KIND == 6) v[c] = (c & 1) ? __vadd2(v[c], k1) : __vmaxs2(v[c], k2);
      if (KIND == 7) v[c] = __vimax3_s16x2(v[c], k1, k2);                // 3-input max
      if (KIND == 8) v[c] = v[c] + k1;                                   // IADD (32-bit)
      if (KIND == 9) v[c] = (c & 1) ? v[c] + k1 : __viaddmax_s16x2(v[c], k1, k2);
      if (KIND == 10) v[c] = (c % 3 == 0) ? __vadd2(v[c], k1) : __viaddmax_s16x2(v[c], k1, k2);
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= v[c];
  if (s == 0x12345678u) out[threadIdx.x] = s;
}

template <int KIND>
double run(uint32_t* d, int sms) {
  const int iters = 20000;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  probe<KIND><<<sms * 4, 256>>>(d, 100, 3u, 5u);
  cudaEventRecord(a);
  probe<KIND><<<sms * 4, 256>>>(d, iters, 3u, 5u);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double ops = (double)sms * 4 * 256 * iters * CH;
  return ops / (ms * 1e-3);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* d;
  cudaMalloc(&d, 4096);
  const char* names[] = {"viaddmax_s16x2", "vadd2", "vadd2+viaddmax 1:1", "imad", "imad+viaddmax 1:1",
                         "vmaxs2", "vadd2+vmaxs2 1:1", "vimax3_s16x2", "iadd32", "iadd32+viaddmax 1:1",
                         "vadd2+viaddmax 1:2"};
  double r[11];
  r[0] = run<0>(d, sms); r[1] = run<1>(d, sms); r[2] = run<2>(d, sms); r[3] = run<3>(d, sms);
  r[4] = run<4>(d, sms); r[5] = run<5>(d, sms); r[6] = run<6>(d, sms); r[7] = run<7>(d, sms);
  r[8] = run<8>(d, sms); r[9] = run<9>(d, sms); r[10] = run<10>(d, sms);
  for (int k = 0; k < 11; ++k)
    printf("%-24s %8.3f Tinst/s  %6.1f lanes/clk/SM (at %d MHz)\n", names[k], r[k] / 1e12,
           r[k] / sms / (clk * 1e3), clk / 1000);
  return 0;
}
