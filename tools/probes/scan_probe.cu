// Probe: latency of the per-column F scan of the strip pipeline (one warp, 32 lanes,
// int32), as a dependent chain of columns: x -> scan -> x' = f(scan) -> ...
//   v0  log2 scan: shift-in + 5 x (SHFL.UP + VIADDMNMX)           (sw_chain.cuh today)
//   v1  radix-4: shift-in + rounds of 3, 3, 1 independent SHFLs
//   v2  radix-8 tree: 7 then 3 independent SHFLs, VIADDMNMX tree (depth 3 + 2)
//   v3  shared memory: STS, 7 LDS window, STS, 3 LDS
//   lat_shfl / lat_dpx / lat_redux: dependent chains of one op
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scan_probe scan_probe.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ int amax(int a, int b, int c) { return __viaddmax_s32(a, b, c); }

template <int V>
__global__ void probe(int iters, int d, int* out, long long* cyc) {
  const int t = threadIdx.x;
  __shared__ int sm[64];
  int x = (t * 7919) & 1023;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    int r;
    if (V == 0) {
      int acc = __shfl_up_sync(~0u, x, 1);
      acc = t ? acc : 0;
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        int y = __shfl_up_sync(~0u, acc, 1 << s);
        acc = __viaddmax_s32_relu(y, -(d << s), acc);
      }
      r = acc;
    } else if (V == 1) {
      int acc = __shfl_up_sync(~0u, x, 1);
      acc = t ? acc : 0;
      int k = 1;
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        int y1 = __shfl_up_sync(~0u, acc, k), y2 = __shfl_up_sync(~0u, acc, 2 * k),
            y3 = __shfl_up_sync(~0u, acc, 3 * k);
        int q = amax(y1, -k * d, acc);
        int q2 = amax(y3, -k * d, y2);
        acc = amax(q2, -2 * k * d, q);
        k *= 4;
      }
      int y = __shfl_up_sync(~0u, acc, 16);
      r = amax(y, -16 * d, acc);
    } else if (V == 2) {
      int a2 = __shfl_up_sync(~0u, x, 2);
      a2 = t >= 2 ? a2 : 0;
      int y1 = __shfl_up_sync(~0u, a2, 1), y2 = __shfl_up_sync(~0u, a2, 2),
          y3 = __shfl_up_sync(~0u, a2, 3), y4 = __shfl_up_sync(~0u, a2, 4),
          y5 = __shfl_up_sync(~0u, a2, 5), y6 = __shfl_up_sync(~0u, a2, 6),
          y7 = __shfl_up_sync(~0u, a2, 7);
      int q1 = amax(y1, -d, a2), q2 = amax(y3, -d, y2), q3 = amax(y5, -d, y4), q4 = amax(y7, -d, y6);
      int r1 = amax(q2, -2 * d, q1), r2 = amax(q4, -2 * d, q3);
      int w = amax(r2, -4 * d, r1);
      int z1 = __shfl_up_sync(~0u, w, 8), z2 = __shfl_up_sync(~0u, w, 16), z3 = __shfl_up_sync(~0u, w, 24);
      int p = amax(z1, -8 * d, w), p2 = amax(z3, -8 * d, z2);
      r = amax(p2, -16 * d, p);
    } else if (V == 3) {
      sm[32 + t] = x;
      sm[t] = 0;
      __syncwarp();
      int acc = 0;
#pragma unroll
      for (int k = 2; k <= 8; ++k) acc = max(acc, sm[32 + t - k] - (k - 2) * d);
      __syncwarp();
      sm[32 + t] = acc;
      __syncwarp();
      int z1 = sm[32 + t - 8], z2 = sm[32 + t - 16], z3 = sm[32 + t - 24];
      int p = amax(z1, -8 * d, acc), p2 = amax(z3, -8 * d, z2);
      r = amax(p2, -16 * d, p);
      __syncwarp();
    } else if (V == 4) {
      r = __shfl_up_sync(~0u, x, 1);
    } else if (V == 5) {
      r = __viaddmax_s32_relu(x, -d, x ^ 5);
    } else {
      r = __reduce_max_sync(~0u, x) ^ t;
    }
    x = (r & 1023) ^ t;
  }
  long long t1 = clock64();
  if (t == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * 32 + t] = x;
}

int main() {
  int* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 64 * 32 * 4);
  cudaMallocManaged(&cyc, 148 * 64 * 8);
  const int iters = 20000;
  const char* names[] = {"v0 log2", "v1 radix4", "v2 radix8", "v3 smem", "lat shfl", "lat dpx",
                         "lat redux"};
  for (int v = 0; v < 7; ++v) {
    for (int blocks : {1, 148 * 8}) {
      for (int rep = 0; rep < 2; ++rep) {
        switch (v) {
          case 0: probe<0><<<blocks, 32>>>(iters, 3, out, cyc); break;
          case 1: probe<1><<<blocks, 32>>>(iters, 3, out, cyc); break;
          case 2: probe<2><<<blocks, 32>>>(iters, 3, out, cyc); break;
          case 3: probe<3><<<blocks, 32>>>(iters, 3, out, cyc); break;
          case 4: probe<4><<<blocks, 32>>>(iters, 3, out, cyc); break;
          case 5: probe<5><<<blocks, 32>>>(iters, 3, out, cyc); break;
          default: probe<6><<<blocks, 32>>>(iters, 3, out, cyc); break;
        }
        cudaDeviceSynchronize();
      }
      printf("%-10s blocks=%4d  %.1f cycles per column\n", names[v], blocks,
             (double)cyc[0] / iters);
    }
  }
  return 0;
}
