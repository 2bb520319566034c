// sw_pack.cu -- 2-bit packed DNA input (four residues per byte, residue k of a byte in
// bits 2k..2k+1) expanded to the one-byte codes the alignment kernels read.
//
// The reference encodes residues one code per element (Alphabet.encode,
// src/scoring.py:45-46; int16 arrays across its compiled boundary,
// src/_compiled.py:583,592).  Short-read batches are copy-bound on the host link at one
// byte per residue (config 3: 7.55 GB per batch); the packed form carries a quarter of
// that, and this kernel restores the codes on the device at HBM speed.
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/swscan_b200.h"

namespace swb {

// one thread per packed byte: 4 codes, one 32-bit store (n_res is the residue count;
// the last byte may be partial)
__global__ void sw_unpack2_kernel(const uint8_t* __restrict__ packed, int64_t n_res,
                                  uint8_t* __restrict__ codes) {
  const int64_t n_bytes = (n_res + 3) >> 2;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n_bytes;
       b += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = packed[b];
    const uint32_t w = (v & 3u) | ((v & 0xcu) << 6) | ((v & 0x30u) << 12) | ((v & 0xc0u) << 18);
    const int64_t r = b << 2;
    if (r + 4 <= n_res && ((reinterpret_cast<uintptr_t>(codes) & 3u) == 0)) {
      *reinterpret_cast<uint32_t*>(codes + r) = w;
    } else {
      for (int k = 0; k < 4 && r + k < n_res; ++k) codes[r + k] = (uint8_t)((w >> (8 * k)) & 0xffu);
    }
  }
}

}  // namespace swb

extern "C" int32_t swb_unpack2_launch(const uint8_t* d_packed, int64_t n_res, uint8_t* d_codes,
                                      sw_stream_t stream) {
  if (n_res <= 0) return 0;
  const int64_t n_bytes = (n_res + 3) >> 2;
  int64_t blocks = (n_bytes + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  swb::sw_unpack2_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(d_packed, n_res, d_codes);
  return (int32_t)cudaGetLastError();
}
