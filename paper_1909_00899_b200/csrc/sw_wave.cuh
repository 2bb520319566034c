// sw_wave.cuh -- long single pairs: the strip pipeline with an intra-strip wavefront.
//
// Same strips, ring buffer, progress counters and final reduction as the scan
// strip pipeline (sw_chain.cuh); only the schedule inside a strip differs.
// Lane l of strip b owns the L consecutive query rows b*32L + l*L + [0, L) and,
// at step s, processes reference column i = s - l: the F leaving its last row
// and the H of its last row reach lane l+1 by one shuffle at the next step,
// so F flows down the strip row by row and no scan is needed.  Each step's
// dependency chain is one shuffle plus one VIADDMNMX per row (the F chain);
// a scan strip pays ~7 dependent shuffles per column instead.
//
// Cell update (E and F opened from u, the corner argument of DESIGN.md §1):
//   u  = max(diag + S, E)        Hn = max(u, F)
//   Xu = u - go                  E  = max(E - ge, Xu, 0)     F = max(F - ge, Xu, 0)
// 32-bit lanes (one cell per lane per instruction); scores and end coordinates
// equal the scan kernels' (tests/test_gpu_parity.py).
#pragma once
#include "sw_chain.cuh"

namespace swb {

// One wavefront step of one lane: column i = s - lane of its L rows.  CHECKED
// handles the fill/drain tiles (columns outside [0, n)); interior tiles skip
// every bounds test.  Branch-free: the only control flow is the unrolled loop.
#ifndef SWB_WAVE_SLEEP_NS
#define SWB_WAVE_SLEEP_NS 32  // poll interval cap: a strip waits on its neighbour every 32 steps
#endif
// Progress wait with a short, fixed poll interval: the strips run in lock-step, so
// an exponential backoff would overshoot the producer's release by up to a tile.
__device__ __forceinline__ void wait_ge_tight(const unsigned long long* p, unsigned long long want) {
  while (ld_relaxed(p) < want) {
    if (SWB_WAVE_SLEEP_NS > 0) __nanosleep(SWB_WAVE_SLEEP_NS);
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

__host__ __device__ constexpr int wave_lp(int L) { return L <= 1 ? 1 : L <= 2 ? 2 : L <= 4 ? 4 : 8; }

template <int L>
struct WaveLane {
  uint32_t H[L], E[L], Sn[L];
  uint32_t h_bot, f_bot, hab_prev;
  int tkey;             // this step tile's best key (see wave_step)
  int bkey, thr, bcol;  // first-maximum record: key, column
};

template <int L, bool CHECKED>
__device__ __forceinline__ void wave_step(WaveLane<L>& w, const int s, const int k, const int lane,
                                          const int n, const int A, const uint8_t* sref,
                                          const uint32_t* sprof, const int2* tile_in,
                                          int2* tlo, int2* thi, const bool handoff,
                                          const uint32_t NGO, const uint32_t NGE) {
  using Wd = W32;
  const int i = s - lane;
  uint32_t S[L];
#pragma unroll
  for (int j = 0; j < L; ++j) S[j] = w.Sn[j];
  {  // prefetch the scores of column i + 1 (off the F chain)
    const int c = i + 1;
    const int sym = (!CHECKED || (c >= 0 && c < n)) ? (int)sref[c & 127] : A;
    const uint32_t* pr = sprof + (sym * 32 + lane) * L;
    if constexpr (L % 4 == 0) {
#pragma unroll
      for (int q = 0; q < L / 4; ++q) {
        const uint4 v = *reinterpret_cast<const uint4*>(pr + 4 * q);
        w.Sn[4 * q] = v.x; w.Sn[4 * q + 1] = v.y; w.Sn[4 * q + 2] = v.z; w.Sn[4 * q + 3] = v.w;
      }
    } else if constexpr (L == 2) {
      const uint2 v = *reinterpret_cast<const uint2*>(pr);
      w.Sn[0] = v.x; w.Sn[1] = v.y;
    } else {
#pragma unroll
      for (int j = 0; j < L; ++j) w.Sn[j] = pr[j];
    }
  }
  // inputs: the lane above (its previous step) or, for lane 0, strip b-1's column s
  const int2 in = tile_in[k];
  const uint32_t sh = __shfl_up_sync(0xffffffffu, w.h_bot, 1);
  const uint32_t sf = __shfl_up_sync(0xffffffffu, w.f_bot, 1);
  const uint32_t up_h = lane == 0 ? (uint32_t)in.y : sh;
  uint32_t F = lane == 0 ? (uint32_t)in.x : sf;
  uint32_t diag = w.hab_prev;
  w.hab_prev = up_h;
  uint32_t um[L];
#pragma unroll
  for (int j = 0; j < L; ++j) {
    const uint32_t u = Wd::addmax(diag, S[j], w.E[j]);
    diag = w.H[j];
    const uint32_t Xu = Wd::add(u, NGO);
    w.E[j] = Wd::addmax_relu(w.E[j], NGE, Xu);
    w.H[j] = Wd::vmax(u, F);
    F = Wd::addmax_relu(F, NGE, Xu);
    um[j] = u;
  }
  w.h_bot = w.H[L - 1];
  w.f_bot = F;
  // first maximum of this lane (a best cell is a diagonal cell, observed as u): the
  // step tile keeps one max over keys u * 32LP + (31 - k) * LP + (LP - 1 - j), so the
  // largest key holds the tile's largest value at its first step (column) and first
  // row; tile_record folds it in at the tile end.  Pad rows score the null
  // residue and columns outside [0, n) see only E values below an earlier u, so
  // neither can hold a first maximum.
  constexpr int LP = wave_lp(L);
#pragma unroll
  for (int j = 0; j < L; ++j)
    w.tkey = max(w.tkey, (int)um[j] * (32 * LP) + ((31 - k) * LP + (LP - 1 - j)));
  // lane 31 parks column i = s - 31 for strip b+1: steps k < 31 finish column tile
  // t0/32 - 1 (tlo), step 31 starts column tile t0/32 (thi)
  if (handoff && lane == 31 && (!CHECKED || (i >= 0 && i < n)))
    (k < 31 ? tlo : thi)[(k + 1) & 31] = make_int2((int)F, (int)w.H[L - 1]);
}

template <int L>
__global__ void __launch_bounds__(32) sw_wave_kernel(const ChainArgs a) {
  constexpr int RING = kChainRing * kChainK;
  constexpr int K = kChainK;  // columns per handoff tile (= lanes per strip)
  static_assert(K == 32, "one handoff tile per 32 steps");
  const int lane = threadIdx.x;
  const int b = (int)blockIdx.x;
  const int nb = a.nb;
  const int A = a.n_sym;
  const int n = (int)a.n;  // < 2^31 (host-checked)

  // profile: chain layout [b][sym][j][lane] -> shared [sym][lane][j] (a lane's L words
  // are contiguous: one LDS.128 per 4 rows; lanes of a quarter warp hit distinct banks)
  extern __shared__ uint32_t smem[];
  uint32_t* sprof = smem;
  {
    const int words = (A + 1) * L * 32;
    const uint32_t* src = a.prof + (size_t)b * words;
    for (int w = lane; w < words; w += 32) {
      const int tl = w & 31, j = (w >> 5) % L, sym = w / (32 * L);
      // pad rows (q >= m) take the null residue here: below the query they cannot
      // reach a real cell, and this way they never hold a maximum either
      const int q = b * 32 * L + tl * L + j;
      sprof[(sym * 32 + tl) * L + j] = q < a.m ? __ldg(src + w) : (uint32_t)W32::NULLV;
    }
  }
  uint8_t* sref = reinterpret_cast<uint8_t*>(sprof + (A + 1) * L * 32);  // column ring, 128 B
  int2* tile_in = reinterpret_cast<int2*>(sref + 128);                   // 32 x (F_in, H_in)
  int2* tile_out = tile_in + K;  // 2 x 32 (F_out, H_last), by column-tile parity

  // reference residues: column c lives at sref[c & 127]; columns [0, 64) now, then
  // one tile ahead (columns [t0 + 32, t0 + 64) at the start of step tile t0)
  sref[lane] = lane < n ? __ldg(a.ref + lane) : (uint8_t)A;
  sref[32 + lane] = 32 + lane < n ? __ldg(a.ref + 32 + lane) : (uint8_t)A;
  __syncwarp();

  const int cl = W32::CLAMP;
  const uint32_t NGO = (uint32_t)-min(a.go, cl), NGE = (uint32_t)-min(a.ge, cl);
  WaveLane<L> w;
#pragma unroll
  for (int j = 0; j < L; ++j) { w.H[j] = 0u; w.E[j] = 0u; }
  w.h_bot = w.f_bot = w.hab_prev = 0u;
  constexpr int LP = wave_lp(L);
  constexpr int KB = 32 * LP;  // key units per score point
  w.bkey = 0; w.thr = KB - 1; w.bcol = -1; w.tkey = 0;
  // a tile's best key beats the record only with a strictly larger value
  // (thr = record key | (KB - 1)); its column is t0 + (31 - step) - lane
  auto tile_record = [&](int t0) {
    if (w.tkey > w.thr) {
      w.bkey = w.tkey;
      w.thr = w.tkey | (KB - 1);
      w.bcol = t0 + (31 - ((w.tkey / LP) & 31)) - lane;
    }
    w.tkey = 0;
  };
  const int qbase = b * 32 * L + lane * L;

  int2* ring_in = a.ring + (size_t)(b > 0 ? b - 1 : 0) * RING;
  int2* ring_out = a.ring + (size_t)b * RING;
  const int steps = n + 31;
  const bool handoff = b + 1 < nb;

  // Handoff without flags or fences: a ring entry is one 64-bit word (F | tag << 31,
  // H) written by a single store, and the tag is the parity of the ring generation
  // (c / RING), flipped so that the zeroed ring never reads as valid.  The consumer
  // prefetches a tile one tile ahead and, when it needs it, checks every entry's
  // tag (re-reading until the producer's stores have landed); back-pressure uses the
  // consumer's progress counter, written relaxed once the tile's loads returned and
  // polled only when the last observed value is insufficient.
  unsigned long long* ring_out64 = reinterpret_cast<unsigned long long*>(ring_out);
  const unsigned long long* ring_in64 = reinterpret_cast<const unsigned long long*>(ring_in);
  auto tag_of = [](int c) -> unsigned { return (((unsigned)(c / RING)) & 1u) ^ 1u; };
  unsigned long long cons_seen = 0;  // last observed progress of strip b+1
  // store columns [c0, c0 + kc) of an outgoing tile
  auto store_tile = [&](int c0, int kc, const int2* buf) {
    if (c0 >= RING) {
      const unsigned long long need = (unsigned long long)(c0 - RING + kc);
      if (cons_seen < need) {
        wait_ge_tight(a.consumed + (size_t)(b + 1) * 16, need);
        cons_seen = ld_relaxed(a.consumed + (size_t)(b + 1) * 16);
      }
    }
    __syncwarp();
    if (lane < kc) {
      const int2 e = buf[lane];
      const unsigned long long word = ((unsigned long long)(uint32_t)e.y << 32) |
                                      (uint32_t)e.x | ((unsigned long long)tag_of(c0) << 31);
      __stcg(ring_out64 + ((c0 + lane) % RING), word);
    }
  };
  // incoming columns [c0, c0 + 32) of strip b-1: issue the loads (checked later)
  auto load_raw = [&](int c0) -> unsigned long long {
    return (c0 + lane < n) ? ld_relaxed(ring_in64 + ((c0 + lane) % RING)) : 0ull;
  };
  // validate (re-reading until every entry carries this generation's tag) and unpack
  auto take_tile = [&](int c0, unsigned long long raw) -> int2 {
    if (c0 >= n) return make_int2(0, 0);
    const unsigned want = tag_of(c0);
    const bool mine = c0 + lane < n;
    while (!__all_sync(0xffffffffu, !mine || (unsigned)((raw >> 31) & 1u) == want)) {
      if (SWB_WAVE_SLEEP_NS > 0) __nanosleep(SWB_WAVE_SLEEP_NS);
      raw = load_raw(c0);
    }
    if (!mine) return make_int2(0, 0);
    return make_int2((int)((uint32_t)raw & 0x7fffffffu), (int)(raw >> 32));
  };
  unsigned long long raw_next = b > 0 ? load_raw(0) : 0ull;

  {  // scores of step 0 (lane 0: column 0; other lanes idle)
    const int sym = lane == 0 ? (int)sref[0] : A;
    const uint32_t* pr = sprof + (sym * 32 + lane) * L;
#pragma unroll
    for (int j = 0; j < L; ++j) w.Sn[j] = pr[j];
  }

  for (int t0 = 0; t0 < steps; t0 += 32) {
    // ---- step tile [t0, t0 + 32): boundary work ----
    if (t0 > 0) {  // residues of columns [t0 + 32, t0 + 64)
      const int c = t0 + 32 + lane;
      sref[c & 127] = c < n ? __ldg(a.ref + c) : (uint8_t)A;
    }
    if (handoff && t0 >= 64) store_tile(t0 - 64, 32, tile_out + ((t0 >> 5) & 1) * K);  // tile t0/32 - 2
    // strip b-1's columns [t0, t0 + 32): loaded last tile; load the next
    if (b > 0) {
      tile_in[lane] = take_tile(t0, raw_next);
      __syncwarp();
      if (lane == 0 && t0 < n)  // those ring slots are read: relaxed is enough
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(a.consumed + (size_t)b * 16),
                     "l"((unsigned long long)min(t0 + K, n)) : "memory");
      raw_next = load_raw(t0 + K);
    } else {
      tile_in[lane] = make_int2(0, 0);
    }
    __syncwarp();
    // outgoing: lane 31 covers columns t0 - 31 .. t0 here, the tail of column tile
    // t0/32 - 1 (buffer parity (t0/32 - 1) & 1) and the head of column tile t0/32;
    // wave_step indexes [0, 32) = the former, [32, 64) = the latter
    int2* tlo = tile_out + ((((t0 >> 5) - 1) & 1) * K);
    int2* thi = tile_out + (((t0 >> 5) & 1) * K);
    const bool interior = t0 >= 32 && t0 + 32 < n;  // every lane's columns i, i+1 in [0, n)
    if (interior) {
#pragma unroll
      for (int k = 0; k < 32; ++k)
        wave_step<L, false>(w, t0 + k, k, lane, n, A, sref, sprof, tile_in, tlo,
                            thi, handoff, NGO, NGE);
    } else {
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (t0 + k < steps)
          wave_step<L, true>(w, t0 + k, k, lane, n, A, sref, sprof, tile_in, tlo,
                             thi, handoff, NGO, NGE);
    }
    tile_record(t0);
  }
  // the last (partial) outgoing tiles
  if (handoff) {
    const int tend = (steps + 31) & ~31;  // first step tile not entered
    for (int c0 = (tend >= 64 ? tend - 64 : 0); c0 < n; c0 += 32)
      store_tile(c0, min(K, n - c0), tile_out + ((c0 >> 5) & 1) * K);
  }
  const int bv = w.bkey / KB;
  int bcol = bv > 0 ? w.bcol : -1, bq = bv > 0 ? qbase + (LP - 1 - (w.bkey & (LP - 1))) : -1;
  const uint32_t full = 0xffffffffu;

  // ---- per-strip best, then the last strip to finish reduces ----
  int best = bv, col = bcol, q = bq;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const int ob = __shfl_xor_sync(full, best, off);
    const int oc = __shfl_xor_sync(full, col, off);
    const int oq = __shfl_xor_sync(full, q, off);
    if (ob > best || (ob == best && (oc < col || (oc == col && oq < q)))) {
      best = ob; col = oc; q = oq;
    }
  }
  if (lane == 0) {
    a.best[b] = make_int4(best, col, q, 0);
    __threadfence();
    const unsigned ticket = atomicAdd(a.done, 1u);
    if (ticket == (unsigned)nb - 1) {
      __threadfence();
      for (int k = 0; k < nb; ++k) {
        const int4 r = __ldcg(a.best + k);
        if (r.x > best || (r.x == best && (r.y < col || (r.y == col && r.z < q)))) {
          best = r.x; col = r.y; q = r.z;
        }
      }
      uint8_t fl = 0;
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
