// Probe: dependent-chain latency (cycles) of the integer ops on the strip pipeline's
// per-column critical path, one warp: 32 dependent ops per loop iteration.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o lat_probe lat_probe.cu
#include <cstdint>
#include <cstdio>

template <int V>
__global__ void chain(int iters, int a, int b, int* out, long long* cyc) {
  int x = threadIdx.x * 13 + a;
  __shared__ int sm[64];
  sm[threadIdx.x] = threadIdx.x;
  sm[32 + threadIdx.x] = 32 + threadIdx.x;
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (V == 0) x = __viaddmax_s32(x, b, a);          // VIADDMNMX
      if (V == 1) x = __viaddmax_s32_relu(x, b, a);     // VIADDMNMX.RELU
      if (V == 2) x = max(x, a + k);                    // VIMNMX / IMNMX
      if (V == 3) x = __vimax3_s32(x, a, b);            // VIMNMX3
      if (V == 4) x = x + b;                            // IADD
      if (V == 5) x = x * b + a;                        // IMAD
      if (V == 6) x = sm[(x & 31)];                     // LDS
      if (V == 7) x = __shfl_xor_sync(~0u, x, 1);       // SHFL
      if (V == 8) x = __vimax_s32_relu(x, a);           // VIMNMX.RELU
      if (V == 9) x = (x > a) ? x : b;                  // ISETP+SEL
    }
    if (V == 10) {  // throughput: 32 independent shuffles per iteration, one warp
      int acc = 0;
#pragma unroll
      for (int k = 0; k < 32; ++k) acc += __shfl_up_sync(~0u, x + k, (k & 7) + 1);
      x = acc;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = x;
}

int main() {
  int* out;
  long long* cyc;
  cudaMalloc(&out, 4096);
  cudaMallocManaged(&cyc, 64);
  const char* names[] = {"VIADDMNMX", "VIADDMNMX.RELU", "IMNMX(max)", "VIMNMX3", "IADD",
                         "IMAD", "LDS", "SHFL", "VIMNMX.RELU", "ISETP+SEL",
                         "SHFL indep. (per shfl)"};
  const int iters = 2000;
  for (int v = 0; v < 11; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (v) {
        case 0: chain<0><<<1, 32>>>(iters, 3, -1, out, cyc); break;
        case 1: chain<1><<<1, 32>>>(iters, 3, -1, out, cyc); break;
        case 2: chain<2><<<1, 32>>>(iters, 3, -1, out, cyc); break;
        case 3: chain<3><<<1, 32>>>(iters, 3, -1, out, cyc); break;
        case 4: chain<4><<<1, 32>>>(iters, 3, -1, out, cyc); break;
        case 5: chain<5><<<1, 32>>>(iters, 3, 3, out, cyc); break;
        case 6: chain<6><<<1, 32>>>(iters, 3, -1, out, cyc); break;
        case 7: chain<7><<<1, 32>>>(iters, 3, -1, out, cyc); break;
        case 8: chain<8><<<1, 32>>>(iters, 3, -1, out, cyc); break;
        case 9: chain<9><<<1, 32>>>(iters, 3, -1, out, cyc); break;
        default: chain<10><<<1, 32>>>(iters, 3, -1, out, cyc); break;
      }
      cudaDeviceSynchronize();
    }
    printf("%-16s %.2f cycles\n", names[v], (double)cyc[0] / (iters * 32.0));
  }
  return 0;
}
