// sw_chain.cuh -- long single pairs: a pipeline of query strips.
//
// The query is cut into NB strips of M = P*L positions; strip b is owned by
// one warp-sized CTA (P = 32 lanes in 32-bit, 64 in 16-bit), which streams
// every reference residue (column) through the same striped recurrence and
// Alg. 6 scan as the single-warp kernels (sw_kernels.cuh).  The only coupling
// between strips is one boundary value pair per column, produced by strip b-1
// and consumed by strip b:
//   F_out[i]  -- the true vertical-gap value leaving strip b-1 in column i,
//                folded into strip b's carry: carry[l] = max(carry_local[l],
//                F_in - l*L*ge)  (one DPX op);
//   H_last[i] -- the corrected H of strip b-1's last cell in column i, the
//                diagonal input of strip b's first cell in column i+1.
// Boundary values move in tiles of K columns through a ring buffer in global
// memory (L2) with release/acquire progress counters and back-pressure; all
// strips are co-resident (cooperative launch), strip b runs one tile behind
// strip b-1.  The per-strip best (score, first column, first query position)
// is reduced by the last strip to finish.
#pragma once
#include "sw_kernels.cuh"

namespace swb {

#ifndef SWB_CHAIN_COORDS
#define SWB_CHAIN_COORDS 1
#endif
#ifndef SWB_CHAIN_SLEEP
#define SWB_CHAIN_SLEEP 1
#endif
#ifndef SWB_CHAIN_RADIX
#define SWB_CHAIN_RADIX 1  // 32-bit strips: radix-8 scan on F shifted by two lanes
#endif
#ifndef SWB_CHAIN_BP_ALL
// Back-pressure spin by every lane.  With only the writing lane spinning (divergent),
// the head strip's warp stayed in a degraded issue mode afterwards: ~9x slower columns
// for the rest of the kernel (measured with tools/trace_chain.py).
#define SWB_CHAIN_BP_ALL 1
#endif
constexpr int kChainK = 32;     // columns per handoff tile
#ifndef SWB_CHAIN_RING
#define SWB_CHAIN_RING 32  // tiles per boundary ring (8 -> 32: config 5 wavefront 62.7 -> 59.4 ms, scan 196 -> 192 ms)
#endif
constexpr int kChainRing = SWB_CHAIN_RING;  // tiles in flight per boundary

struct ChainArgs {
  const uint32_t* prof;   // [(A+1)][L][32] words, striped per strip (see sw_chain_profile_kernel)
  int32_t n_sym;
  int32_t m;              // query length
  int32_t nb;             // strips
  const uint8_t* ref;
  int64_t n;              // reference length
  int32_t go, ge, bias, max_sub;
  int32_t early_exit;
  // workspace (zeroed before launch)
  int2* ring;                     // [nb][kChainRing*kChainK] (F_out, H_last)
  unsigned long long* published;  // [nb*16] columns published by strip b (one 128-B line each)
  unsigned long long* consumed;   // [nb*16] columns consumed by strip b (from strip b-1)
  int4* best;                     // [nb] per-strip (score, col, q, 0)
  unsigned int* done;             // [1] ticket
  // outputs
  int32_t* score;
  int32_t* ref_end;
  int32_t* query_end;
  uint8_t* flags;
  // optional timeline (diagnostics): per strip, per tile: [start, ready, end] globaltimer ns
  unsigned long long* trace;
  int32_t trace_tiles;
  int32_t reverse;  // diagnostics: strip b runs on block nb-1-b
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Spin with relaxed loads (an acquire load per iteration would invalidate L1 every
// poll), then one acquire fence once the producer's release is observed.
__device__ __forceinline__ void wait_ge(const unsigned long long* p, unsigned long long want) {
  if (ld_relaxed(p) < want) {
    unsigned ns = 32;
    while (ld_relaxed(p) < want) {
      if (SWB_CHAIN_SLEEP) __nanosleep(ns);
      if (ns < 512) ns <<= 1;
    }
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// Chain profile: strip-major layout prof[b][(A+1)][L][32] so each CTA reads one contiguous slab.
template <class Wd>
__global__ void sw_chain_profile_kernel(const uint8_t* __restrict__ query, int m,
                                        const int8_t* __restrict__ sub, int A, int L, int nb,
                                        int bias, uint32_t* __restrict__ prof) {
  constexpr int P = 32 * Wd::LPW;
  const int words = nb * (A + 1) * L * 32;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
    const int t = w & 31;
    const int j = (w >> 5) % L;
    const int sym = (w / (32 * L)) % (A + 1);
    const int b = w / (32 * L * (A + 1));
    int v[2] = {0, 0};
#pragma unroll
    for (int h = 0; h < Wd::LPW; ++h) {
      const int q = b * P * L + (h * 32 + t) * L + j;
      if (sym == A) v[h] = Wd::NULLV;
      else if (q >= m) v[h] = -bias;
      else v[h] = sub[sym * A + query[q]];
    }
    prof[w] = Wd::pack(v[0], v[1]);
  }
}

template <class Wd, int L, int VAR>
__global__ void __launch_bounds__(32) sw_chain_kernel(const ChainArgs a) {
  static_assert(VAR == VAR_SCAN, "the strip pipeline implements the scan kernel");
  constexpr int T = 32;
  constexpr int P = T * Wd::LPW;
  constexpr int STEPS = ceil_log2(P);
  constexpr int RING = kChainRing * kChainK;
  const int t = threadIdx.x;
  const int b = a.reverse ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x;
  const int nb = a.nb;
  const uint32_t gmask = 0xffffffffu;
  const int A = a.n_sym;

  // profile slab of this strip -> shared memory
  extern __shared__ uint32_t smem[];
  {
    const int words = (A + 1) * L * 32;
    const uint32_t* src = a.prof + (size_t)b * words;
    for (int w = t; w < words; w += 32) smem[w] = __ldg(src + w);
    __syncwarp();
  }
  const uint32_t* prof_t = smem + t;
  // per-tile staging: incoming (F_in, H_last, residue) per column, outgoing (F_out, H_last)
  int4* tile_in = reinterpret_cast<int4*>(smem + (A + 1) * L * 32);
  int2* tile_out = reinterpret_cast<int2*>(tile_in + kChainK);
  if (a.trace && t == 0) {  // diagnostics: SM of this strip, after the timeline
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    a.trace[(size_t)64 * a.trace_tiles * 4 + b] = smid;  // tools/trace_chain.py reserves 64 strips
  }

  uint32_t sel[6];
#pragma unroll
  for (int s = 0; s < 6; ++s) sel[s] = Wd::shift_sel(t, 1 << s);
  // scan-step selectors: lanes with no source keep their own value (harmless under
  // max(relu(x - K*d), x)), which drops the zero-select from the 32-bit steps
  uint32_t ssel[6];
#pragma unroll
  for (int s = 0; s < 6; ++s) ssel[s] = Wd::scan_sel(t, 1 << s);
  // first scan shift: lane 0 (thread 0, low half) receives the strip's incoming F,
  // so the scan itself applies the lane * L * ge decay
  const uint32_t sel_in = Wd::inject_sel(t);
  const int cl = Wd::CLAMP;
  const int go = a.go, ge = a.ge;
  const uint32_t NGO = Wd::splat(-min(go, cl));
  const uint32_t NGE = Wd::splat(-min(ge, cl));
  const uint32_t NWRAP = Wd::splat(-(int)min((int64_t)(L - 1) * ge, (int64_t)cl));
  const uint32_t NLD = Wd::splat(-(int)min((int64_t)L * ge, (int64_t)cl));
  uint32_t NJ[L];
#pragma unroll
  for (int c = 0; c < L; ++c) NJ[c] = Wd::splat(-(int)min((int64_t)c * ge, (int64_t)cl));
  uint32_t NKD[STEPS];
#pragma unroll
  for (int s = 0; s < STEPS; ++s)
    NKD[s] = Wd::splat(-(int)min((int64_t)(1 << s) * L * (int64_t)ge, (int64_t)cl));

  uint32_t H[L], E[L];
#pragma unroll
  for (int c = 0; c < L; ++c) { H[c] = 0u; E[c] = 0u; }
  uint32_t carry = 0u, wnext = 0u;
  int gb = 0;                      // best of all earlier columns in this strip
  int bv = 0, bcol = -1, bq = -1;  // this thread's first-maximum record
  const int64_t n = a.n;
  const int64_t qbase = (int64_t)b * P * L;
  int hd_prev = 0;  // H_last of strip b-1 for the previous column

  int2* ring_in = a.ring + (size_t)(b > 0 ? b - 1 : 0) * RING;
  int2* ring_out = a.ring + (size_t)b * RING;
  // Handoff without flags or fences (as sw_wave_kernel): one 64-bit word per column
  // (F_out | tag << 31, H_last), tag = parity of the ring generation, flipped so the
  // zeroed ring never validates; tiles are loaded one tile ahead and validated when
  // used; back-pressure polls the consumer's relaxed progress counter only when the
  // last observed value is insufficient.
  unsigned long long* ring_out64 = reinterpret_cast<unsigned long long*>(ring_out);
  const unsigned long long* ring_in64 = reinterpret_cast<const unsigned long long*>(ring_in);
  auto tag_of = [](int64_t c) -> unsigned { return (((unsigned)(c / RING)) & 1u) ^ 1u; };
  auto load_raw = [&](int64_t c0) -> unsigned long long {
    return (c0 + t < n && t < kChainK) ? ld_relaxed(ring_in64 + ((c0 + t) % RING)) : 0ull;
  };
  unsigned long long raw_next = b > 0 ? load_raw(0) : 0ull;
  unsigned long long cons_seen = 0;

  for (int64_t t0 = 0; t0 < n; t0 += kChainK) {
    const int kc = (int)min((int64_t)kChainK, n - t0);
    const int64_t tile = t0 / kChainK;
    unsigned long long* tr = (a.trace && tile < a.trace_tiles && t == 0)
                                 ? a.trace + ((size_t)b * a.trace_tiles + tile) * 4 : nullptr;
    unsigned long long* tr31 = (a.trace && tile < a.trace_tiles && t == T - 1)
                                   ? a.trace + ((size_t)b * a.trace_tiles + tile) * 4 : nullptr;
    if (tr) tr[0] = gtimer();
    // ---- incoming boundary tile (loaded last tile; validate, then load the next) ----
    int fin_l = 0, hl_l = 0;
    if (b > 0) {
      const unsigned want = tag_of(t0);
      const bool mine = t < kc;
      unsigned long long raw = raw_next;
      while (!__all_sync(gmask, !mine || (unsigned)((raw >> 31) & 1u) == want)) {
        if (SWB_CHAIN_SLEEP) __nanosleep(32);
        raw = load_raw(t0);
      }
      if (mine) {
        fin_l = (int)((uint32_t)raw & 0x7fffffffu);
        hl_l = (int)(raw >> 32);
      }
      if (t == 0)  // the tile's loads returned (their values are in registers): relaxed
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(a.consumed + (size_t)b * 16),
                     "l"((unsigned long long)(t0 + kc)) : "memory");
      raw_next = load_raw(t0 + kChainK);
    }
    // ---- back-pressure before producing this tile ----
    if (b + 1 < nb && t0 >= RING) {
      const unsigned long long need = (unsigned long long)(t0 - RING + kc);
      if (cons_seen < need) {
        wait_ge(a.consumed + (size_t)(b + 1) * 16, need);
        cons_seen = ld_relaxed(a.consumed + (size_t)(b + 1) * 16);
      }
    }
    if (tr31) tr31[3] = gtimer();
    __syncwarp();
    if (tr) tr[1] = gtimer();
    // stage this tile's per-column inputs in shared memory: each column then reads
    // them with one broadcast load instead of three shuffles
    tile_in[t] = make_int4(fin_l, hl_l, t < kc ? (int)__ldg(a.ref + t0 + t) : 0, 0);
    __syncwarp();

    // profile words of the tile's first column; each column then loads the next
    // column's words before its own work, so the two dependent shared-memory loads
    // (residue, then profile row) leave the column's critical path
    uint32_t Sc[L];
    {
      const uint32_t* pr0 = prof_t + tile_in[0].z * (L * 32);
#pragma unroll
      for (int c = 0; c < L; ++c) Sc[c] = pr0[c * 32];
    }
    for (int col_k = 0; col_k < kc; ++col_k) {
      const int64_t i = t0 + col_k;
      const int4 tin = tile_in[col_k];
      uint32_t Sn[L];
      {
        const uint32_t* pr1 = prof_t + tile_in[min(col_k + 1, kc - 1)].z * (L * 32);
#pragma unroll
        for (int c = 0; c < L; ++c) Sn[c] = pr1[c * 32];
      }
      const int fin = tin.x;
      const int hlk = tin.y;
      // diagonal for the strip's first cell: corrected H of strip b-1, column i-1
      uint32_t vh;
      if constexpr (Wd::LPW == 1 && SWB_CHAIN_RADIX) {
        vh = wnext;  // already the lane-shifted wrap (lane 0: strip b-1's value)
      } else {
        vh = Wd::template shift<T, 1>(wnext, t, gmask, sel[0]);
        if (t == 0) {  // lane 0 (low half of thread 0) takes the previous strip's value
          constexpr uint32_t keep = Wd::LPW == 2 ? 0xffff0000u : 0u;
          vh = (vh & keep) | (Wd::pack(hd_prev, 0) & ~keep);
        }
      }
      hd_prev = hlk;
      uint32_t F = 0u;
      constexpr int kCh = 8, kNch = (L + kCh - 1) / kCh;
      uint32_t cmk[kNch];
#pragma unroll
      for (int ch = 0; ch < kNch; ++ch) cmk[ch] = 0u;
#pragma unroll
      for (int c = 0; c < L; ++c) {
        const uint32_t S = Sc[c];
        const uint32_t u = Wd::addmax(vh, S, E[c]);
        const uint32_t Hn = Wd::vmax(u, F);
        const uint32_t Xu = Wd::add(u, NGO);
        E[c] = Wd::addmax_relu(E[c], NGE, Xu);
        F = Wd::addmax_relu(F, NGE, Xu);
        cmk[c / kCh] = Wd::vmax(cmk[c / kCh], u);
        vh = Wd::addmax(carry, NJ[c], H[c]);
        H[c] = Hn;
      }
      // end coordinates: as sw_striped_kernel, gated on the strip's running best
      // (a strip-local bound is weaker than the global one, so no event is lost)
      uint32_t cm = cmk[0];
#pragma unroll
      for (int k = 1; k < kNch; ++k) cm = Wd::vmax(cm, cmk[k]);
      const int cmx = Wd::hmax(cm);
      if (SWB_CHAIN_COORDS && cmx > gb) {
#pragma unroll
        for (int h = 0; h < Wd::LPW; ++h) {
          const int cv = Wd::get(cm, h);
          if (cv > gb && cv > bv) {
            int kk = 0;
#pragma unroll
            for (int k = kNch - 1; k >= 0; --k)
              if (Wd::get(cmk[k], h) >= cv) kk = k;
            int jj = 0;
#pragma unroll
            for (int k = 0; k < kNch; ++k) {
              if (k == kk) {
#pragma unroll
                for (int c = (k + 1) * kCh - 1; c >= k * kCh; --c)
                  if (c < L && Wd::get(H[c], h) >= cv) jj = c;
              }
            }
            bv = cv;
            bcol = (int)i;
            bq = (int)(qbase + (h * T + t) * L + jj);
          }
        }
      }
      {
        int g = max(gb, cmx);
        g = __reduce_max_sync(gmask, g);  // one REDUX for the strip-wide best
        gb = g;
      }
      if constexpr (Wd::LPW == 1 && SWB_CHAIN_RADIX) {
        // 32-bit strips: Alg. 6's scan as a radix-8 weighted max-plus prefix (two
        // rounds of independent shuffles instead of five dependent ones), run on F
        // shifted by TWO lanes so it yields G[l] = carry[l-1] directly:
        //   carry[l] = max(F[l-1], G[l] - L*ge)            (the lane's carry)
        //   wrap[l]  = max(H[l-1][L-1], G[l] - (L-1)*ge)   (next column's word-0 diagonal)
        // -- the wrap no longer waits for a shuffle of the finished carry.
        // Lanes below a shuffle distance receive their own value, which the max-plus
        // step leaves unchanged (every value is >= 0).
        const int d = min(L * ge, cl);
        const int f = (int)F;
        int f1 = __shfl_up_sync(gmask, f, 1);
        int f2 = __shfl_up_sync(gmask, f, 2);
        int hs = __shfl_up_sync(gmask, (int)H[L - 1], 1);
        f1 = t == 0 ? fin : f1;               // lane 0: the F entering the strip
        f2 = t == 1 ? fin : (t == 0 ? 0 : f2);
        hs = t == 0 ? hlk : hs;               // lane 0: strip b-1's corrected last H
        int y1 = __shfl_up_sync(gmask, f2, 1), y2 = __shfl_up_sync(gmask, f2, 2),
            y3 = __shfl_up_sync(gmask, f2, 3), y4 = __shfl_up_sync(gmask, f2, 4),
            y5 = __shfl_up_sync(gmask, f2, 5), y6 = __shfl_up_sync(gmask, f2, 6),
            y7 = __shfl_up_sync(gmask, f2, 7);
        const int q1 = __viaddmax_s32(y1, -d, f2), q2 = __viaddmax_s32(y3, -d, y2);
        const int q3 = __viaddmax_s32(y5, -d, y4), q4 = __viaddmax_s32(y7, -d, y6);
        const int r1 = __viaddmax_s32(q2, -2 * d, q1), r2 = __viaddmax_s32(q4, -2 * d, q3);
        const int w8 = __viaddmax_s32(r2, -4 * d, r1);  // window of 8 lanes
        const int z1 = __shfl_up_sync(gmask, w8, 8), z2 = __shfl_up_sync(gmask, w8, 16),
                  z3 = __shfl_up_sync(gmask, w8, 24);
        const int p1 = __viaddmax_s32(z1, -8 * d, w8), p2 = __viaddmax_s32(z3, -8 * d, z2);
        const int g = __viaddmax_s32(p2, -16 * d, p1);  // carry[l-1]
        carry = (uint32_t)__viaddmax_s32(g, -d, f1);
        wnext = (uint32_t)__viaddmax_s32(g, -(int)min((int64_t)(L - 1) * ge, (int64_t)cl), hs);
        const uint32_t fo = Wd::addmax(carry, NLD, F);  // true F leaving each lane
        if (t == T - 1) {
          // the boundary H of this column: lane 31's corrected last word
          const int hlast = __viaddmax_s32((int)carry, -(int)min((int64_t)(L - 1) * ge,
                                                                 (int64_t)cl), (int)H[L - 1]);
          tile_out[col_k] = make_int2((int)fo, hlast);
        }
#pragma unroll
        for (int c = 0; c < L; ++c) Sc[c] = Sn[c];
        continue;
      }
      // Alg. 6 scan inside the strip, then fold in the strip's incoming F
      uint32_t acc = Wd::template shift_in<T>(F, Wd::splat(fin), t, gmask, sel_in);
#pragma unroll
      for (int s = 0; s < STEPS; ++s) {
        // K = 1 << s, dispatched statically
        if (s == 0) acc = Wd::addmax_relu(Wd::template scan_shift<T, 1>(acc, t, gmask, ssel[0]), NKD[0], acc);
        if (s == 1) acc = Wd::addmax_relu(Wd::template scan_shift<T, 2>(acc, t, gmask, ssel[1]), NKD[1], acc);
        if (s == 2) acc = Wd::addmax_relu(Wd::template scan_shift<T, 4>(acc, t, gmask, ssel[2]), NKD[2], acc);
        if (s == 3) acc = Wd::addmax_relu(Wd::template scan_shift<T, 8>(acc, t, gmask, ssel[3]), NKD[3], acc);
        if (s == 4) acc = Wd::addmax_relu(Wd::template scan_shift<T, 16>(acc, t, gmask, ssel[4]), NKD[4], acc);
        if constexpr (Wd::LPW == 2)
          if (s == 5) acc = Wd::addmax_relu(Wd::template scan_shift<T, 32>(acc, t, gmask, ssel[5]), NKD[5], acc);
      }
      carry = acc;  // includes the incoming F decayed by lane * L * ge
      wnext = Wd::addmax(carry, NWRAP, H[L - 1]);       // corrected H of the last word
      const uint32_t fo = Wd::addmax(carry, NLD, F);    // true F leaving each lane
      // the strip's last lane (thread 31, top half) holds this column's boundary
      // pair; stage it so the tile leaves in one coalesced store
      if (t == T - 1) tile_out[col_k] = make_int2(Wd::get(fo, Wd::LPW - 1), Wd::get(wnext, Wd::LPW - 1));
#pragma unroll
      for (int c = 0; c < L; ++c) Sc[c] = Sn[c];
    }
    __syncwarp();
    if (b + 1 < nb && t < kc) {
      const int2 e = tile_out[t];
      __stcg(ring_out64 + ((t0 + t) % RING), ((unsigned long long)(uint32_t)e.y << 32) |
                                                 (uint32_t)e.x | ((unsigned long long)tag_of(t0) << 31));
    }
    if (tr) tr[2] = gtimer();
  }

  // ---- per-strip best, then the last strip to finish reduces ----
  int best = bv, col = bcol, q = bq;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const int ob = __shfl_xor_sync(gmask, best, off);
    const int oc = __shfl_xor_sync(gmask, col, off);
    const int oq = __shfl_xor_sync(gmask, q, off);
    if (ob > best || (ob == best && (oc < col || (oc == col && oq < q)))) {
      best = ob; col = oc; q = oq;
    }
  }
  if (t == 0) {
    a.best[b] = make_int4(best, col, q, 0);
    __threadfence();
    const unsigned ticket = atomicAdd(a.done, 1u);
    if (ticket == (unsigned)nb - 1) {
      __threadfence();
      for (int s = 0; s < nb; ++s) {
        const int4 r = __ldcg(a.best + s);
        if (r.x > best || (r.x == best && (r.y < col || (r.y == col && r.z < q)))) {
          best = r.x; col = r.y; q = r.z;
        }
      }
      uint8_t fl = 0;
      if constexpr (Wd::LPW == 2) {
        if (best >= 32767 - a.max_sub) fl |= FLAG_RESCUE;
      }
      if (best > 65535 - a.bias) fl |= FLAG_REF_OVERFLOW;
      if (best == 0) { col = -1; q = -1; }
      a.score[0] = best;
      if (a.ref_end) a.ref_end[0] = col;
      if (a.query_end) a.query_end[0] = q;
      if (a.flags) a.flags[0] = fl;
    }
  }
}

}  // namespace swb
