// sw_wave.cuh -- long single pairs: the strip pipeline with an intra-strip wavefront.
//
// Same strips, ring buffer, progress counters and final reduction as the scan
// strip pipeline (sw_chain.cuh); only the schedule inside a strip differs.
// Lane l of strip b owns the L consecutive query rows b*32L + l*L + [0, L) and,
// at step s, processes the KC reference columns of super-column B = s - l,
// columns B*KC + [0, KC): the F leaving its last row and that row's H reach
// lane l+1 by KC shuffles at the next step, so F flows down the strip row by
// row and no scan is needed.  A step is an L x KC tile: KC > 1 amortises the
// shuffles and the per-step bookkeeping over KC columns, but a column still
// waits on its left neighbour through E (u -> Xu -> E -> u'), so only KC = 2 at
// L = 1 pays (measured, tools/wave_sweep.py; wave_geo in sw_capi.cu picks).
//
// Cell update (E and F opened from u, the corner argument of DESIGN.md §1):
//   u  = max(diag + S, E)        Hn = max(u, F)
//   Xu = u - go                  E  = max(E - ge, Xu, 0)     F = max(F - ge, Xu, 0)
// 32-bit lanes (one cell per lane per instruction); scores and end coordinates
// equal the scan kernels' (tests/test_gpu_parity.py).
#pragma once
#include "sw_chain.cuh"

namespace swb {

#ifndef SWB_WAVE_UNR
#define SWB_WAVE_UNR 0  // steps unrolled per loop iteration (0: by tile size, see UNR)
#endif
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

template <int L, int KC>
struct WaveLane {
  uint32_t H[L], E[L], Sn[KC][L];
  uint32_t h_bot[KC], f_bot[KC], hab_prev;
  int rv, rcol, rrow;  // first-maximum record of this lane: value, column, row
};

// One wavefront step of one lane: super-column B = s - lane, i.e. columns B*KC + r.
// CHECKED handles the fill/drain tiles (columns outside [0, n)); interior tiles skip
// every bounds test.  Columns outside [0, n) score the null residue, so their u is
// an E value, below an earlier u of the same row: they never beat the record.
template <int L, int KC, bool CHECKED>
__device__ __forceinline__ void wave_step(WaveLane<L, KC>& w, const int s, const int k, const int lane,
                                          const int n, const int A, const uint8_t* sref,
                                          const uint32_t* sprof, const int2* tile_in,
                                          int2* tlo, int2* thi, const bool handoff,
                                          const uint32_t NGO, const uint32_t NGE, const int qbase,
                                          const uint32_t (&NJG)[L + 1]) {
  using Wd = W32;
  constexpr int RMASK = 128 * KC - 1;  // residue ring: 4 handoff tiles of columns
  const int B = s - lane;
  uint32_t S[KC][L];
#pragma unroll
  for (int r = 0; r < KC; ++r)
#pragma unroll
    for (int j = 0; j < L; ++j) S[r][j] = w.Sn[r][j];
#pragma unroll
  for (int r = 0; r < KC; ++r) {  // prefetch the scores of super-column B + 1 (off the F chain)
    const int c = (B + 1) * KC + r;
    const int sym = (!CHECKED || (c >= 0 && c < n)) ? (int)sref[c & RMASK] : A;
    const uint32_t* pr = sprof + (sym * 32 + lane) * L;
    if constexpr (L % 4 == 0) {
#pragma unroll
      for (int q = 0; q < L / 4; ++q) {
        const uint4 v = *reinterpret_cast<const uint4*>(pr + 4 * q);
        w.Sn[r][4 * q] = v.x; w.Sn[r][4 * q + 1] = v.y; w.Sn[r][4 * q + 2] = v.z; w.Sn[r][4 * q + 3] = v.w;
      }
    } else if constexpr (L == 2) {
      const uint2 v = *reinterpret_cast<const uint2*>(pr);
      w.Sn[r][0] = v.x; w.Sn[r][1] = v.y;
    } else {
#pragma unroll
      for (int j = 0; j < L; ++j) w.Sn[r][j] = pr[j];
    }
  }
  // inputs: the lane above (its previous step) or, for lane 0, strip b-1's columns
  uint32_t up_h[KC], fin[KC];
#pragma unroll
  for (int r = 0; r < KC; ++r) {
    const int2 in = tile_in[k * KC + r];
    const uint32_t sh = __shfl_up_sync(0xffffffffu, w.h_bot[r], 1);
    const uint32_t sf = __shfl_up_sync(0xffffffffu, w.f_bot[r], 1);
    up_h[r] = lane == 0 ? (uint32_t)in.y : sh;
    fin[r] = lane == 0 ? (uint32_t)in.x : sf;
  }
  uint32_t um[KC][L];
#pragma unroll
  for (int r = 0; r < KC; ++r) {
    if constexpr (L <= 2) {  // short lanes: the plain F chain (fewer instructions)
      uint32_t diag = r == 0 ? w.hab_prev : up_h[r - 1];
      uint32_t F = fin[r];
#pragma unroll
      for (int j = 0; j < L; ++j) {
        const uint32_t u = Wd::addmax(diag, S[r][j], w.E[j]);
        diag = w.H[j];
        const uint32_t Xu = Wd::add(u, NGO);
        w.E[j] = Wd::addmax_relu(w.E[j], NGE, Xu);
        w.H[j] = Wd::vmax(u, F);
        F = Wd::addmax_relu(F, NGE, Xu);
        um[r][j] = u;
      }
      w.h_bot[r] = w.H[L - 1];
      w.f_bot[r] = F;
      continue;
    }
    // Everything but the incoming F first: u, E and the lane-local F prefix
    // B_j = max(B_{j-1} - ge, Xu_j, 0) do not depend on the lane above, so they
    // overlap the shuffle; then F_j = max(F_in - j*ge, B_{j-1}) is one op per row
    // and the lane-to-lane path per step is the shuffle plus two DPX ops (instead
    // of the shuffle plus an L-long F chain; config 5 at L = 8: 154 -> 100 ms).
    uint32_t B[L];
#pragma unroll
    for (int j = 0; j < L; ++j) {
      const uint32_t diag = j == 0 ? (r == 0 ? w.hab_prev : up_h[r - 1]) : w.H[j - 1];
      const uint32_t u = Wd::addmax(diag, S[r][j], w.E[j]);
      um[r][j] = u;
    }
#pragma unroll
    for (int j = 0; j < L; ++j) {
      const uint32_t Xu = Wd::add(um[r][j], NGO);
      w.E[j] = Wd::addmax_relu(w.E[j], NGE, Xu);
      B[j] = j == 0 ? Wd::addmax_relu(Xu, 0u, 0u) : Wd::addmax_relu(B[j - 1], NGE, Xu);
    }
    const uint32_t F = fin[r];
#pragma unroll
    for (int j = 0; j < L; ++j)
      w.H[j] = Wd::vmax(um[r][j], j == 0 ? F : Wd::addmax(F, NJG[j], B[j - 1]));
    w.h_bot[r] = w.H[L - 1];
    w.f_bot[r] = Wd::addmax(F, NJG[L], B[L - 1]);
  }
  w.hab_prev = up_h[KC - 1];
  // first maximum of this lane (a best cell is a diagonal cell, observed as u): the
  // step's maximum, then -- only when it beats the record -- its first cell in
  // (column, row) order.  Pad rows score the null residue: never a maximum.
  int ms = (int)um[0][0];
#pragma unroll
  for (int r = 0; r < KC; ++r)
#pragma unroll
    for (int j = 0; j < L; ++j)
      if (r | j) ms = max(ms, (int)um[r][j]);
  if (ms > w.rv) {
    int rr = KC - 1, jj = L - 1;
#pragma unroll
    for (int r = KC - 1; r >= 0; --r)
#pragma unroll
      for (int j = L - 1; j >= 0; --j)
        if ((int)um[r][j] == ms) { rr = r; jj = j; }
    w.rv = ms;
    w.rcol = B * KC + rr;
    w.rrow = qbase + jj;
  }
  // lane 31 parks super-column s - 31 for strip b+1: steps k < 31 finish handoff
  // tile t0/32 - 1 (tlo), step 31 starts handoff tile t0/32 (thi)
  if (handoff && lane == 31) {
    int2* dst = (k < 31 ? tlo : thi) + ((k + 1) & 31) * KC;
#pragma unroll
    for (int r = 0; r < KC; ++r) {
      const int c = B * KC + r;
      if (!CHECKED || (c >= 0 && c < n)) dst[r] = make_int2((int)w.f_bot[r], (int)w.h_bot[r]);
    }
  }
}

// GE > 0: gap-extend penalty known at compile time (decays as immediate operands)
template <int L, int KC, int GE = 0>
__global__ void __launch_bounds__(32) sw_wave_kernel(const ChainArgs a) {
  constexpr int TS = kChainK;        // steps (super-columns) per handoff tile
  constexpr int TC = TS * KC;        // columns per handoff tile
  constexpr int RING = kChainRing * TC;
  constexpr int RMASK = 128 * KC - 1;
  static_assert(TS == 32, "one handoff tile per 32 steps");
  static_assert((KC & (KC - 1)) == 0, "KC: power of two");
  // steps unrolled per loop iteration: the unrolled tile loop must stay inside the
  // instruction cache (KC * L cells per step; full unrolling at KC * L = 16 is ~8k
  // instructions per variant and ran 3x slower)
  constexpr int UNR = SWB_WAVE_UNR > 0 ? SWB_WAVE_UNR : (KC * L <= 4 ? 32 : KC * L <= 8 ? 8 : 4);
  const int lane = threadIdx.x;
  const int b = (int)blockIdx.x;
  const int nb = a.nb;
  const int A = a.n_sym;
  const int n = (int)a.n;  // < 2^30 (host-checked)
  const int nsc = (n + KC - 1) / KC;  // super-columns

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
  uint8_t* sref = reinterpret_cast<uint8_t*>(sprof + (A + 1) * L * 32);  // column ring, 128*KC B
  int2* tile_in = reinterpret_cast<int2*>(sref + 128 * KC);               // TC x (F_in, H_in)
  int2* tile_out = tile_in + TC;  // 2 x TC (F_out, H_last), by handoff-tile parity

  // reference residues: column c lives at sref[c & RMASK]; super-columns [0, 64)
  // now, then one tile ahead (super-columns [t0 + 32, t0 + 64) at step tile t0)
#pragma unroll
  for (int o = lane; o < 2 * TC; o += 32) sref[o] = o < n ? __ldg(a.ref + o) : (uint8_t)A;
  __syncwarp();

  const int cl = W32::CLAMP;
  const int ge_ = GE > 0 ? GE : a.ge;
  const uint32_t NGO = (uint32_t)-min(a.go, cl), NGE = (uint32_t)-min(ge_, cl);
  uint32_t NJG[L + 1];  // -j * ge (clamped): decay of the incoming F at row j
#pragma unroll
  for (int j = 0; j <= L; ++j) NJG[j] = (uint32_t)-(int)min((int64_t)j * ge_, (int64_t)cl);
  WaveLane<L, KC> w;
#pragma unroll
  for (int j = 0; j < L; ++j) { w.H[j] = 0u; w.E[j] = 0u; }
#pragma unroll
  for (int r = 0; r < KC; ++r) { w.h_bot[r] = 0u; w.f_bot[r] = 0u; }
  w.hab_prev = 0u;
  w.rv = 0; w.rcol = -1; w.rrow = -1;
  const int qbase = b * 32 * L + lane * L;

  int2* ring_in = a.ring + (size_t)(b > 0 ? b - 1 : 0) * RING;
  int2* ring_out = a.ring + (size_t)b * RING;
  const int steps = nsc + 31;
  const bool handoff = b + 1 < nb;

  // Handoff without flags or fences: a ring entry is one 64-bit word (F | tag << 31,
  // H) written by a single store, and the tag is the parity of the ring generation
  // (c / RING), flipped so that the zeroed ring never reads as valid.  The consumer
  // prefetches a tile one tile ahead and, when it needs it, checks every entry's
  // tag (re-reading until the producer's stores have landed); back-pressure uses the
  // consumer's progress counter, written relaxed once the tile's loads returned and
  // polled only when the last observed value is insufficient.  Units: columns.
  unsigned long long* ring_out64 = reinterpret_cast<unsigned long long*>(ring_out);
  const unsigned long long* ring_in64 = reinterpret_cast<const unsigned long long*>(ring_in);
  auto tag_of = [](int c) -> unsigned { return (((unsigned)(c / RING)) & 1u) ^ 1u; };
  unsigned long long cons_seen = 0;  // last observed progress of strip b+1
  // store columns [c0, c0 + kc) of an outgoing tile (c0 a tile start)
  auto store_tile = [&](int c0, int kc, const int2* buf) {
    if (c0 >= RING) {
      const unsigned long long need = (unsigned long long)(c0 - RING + kc);
      if (cons_seen < need) {
        wait_ge_tight(a.consumed + (size_t)(b + 1) * 16, need);
        cons_seen = ld_relaxed(a.consumed + (size_t)(b + 1) * 16);
      }
    }
    __syncwarp();
    const unsigned long long tag = (unsigned long long)tag_of(c0) << 31;
#pragma unroll
    for (int r = 0; r < KC; ++r) {
      const int o = r * 32 + lane;
      if (o < kc) {
        const int2 e = buf[o];
        __stcg(ring_out64 + ((c0 + o) % RING),
               ((unsigned long long)(uint32_t)e.y << 32) | (uint32_t)e.x | tag);
      }
    }
  };
  // incoming columns [c0, c0 + TC) of strip b-1: issue the loads (checked later)
  auto load_raw = [&](int c0, unsigned long long (&raw)[KC]) {
#pragma unroll
    for (int r = 0; r < KC; ++r) {
      const int c = c0 + r * 32 + lane;
      raw[r] = c < n ? ld_relaxed(ring_in64 + (c % RING)) : 0ull;
    }
  };
  // validate (re-reading until every entry carries this generation's tag), unpack
  auto take_tile = [&](int c0, unsigned long long (&raw)[KC]) {
    if (c0 >= n) {
#pragma unroll
      for (int r = 0; r < KC; ++r) tile_in[r * 32 + lane] = make_int2(0, 0);
      return;
    }
    const unsigned want = tag_of(c0);
    for (;;) {
      bool ok = true;
#pragma unroll
      for (int r = 0; r < KC; ++r)
        ok = ok && (c0 + r * 32 + lane >= n || (unsigned)((raw[r] >> 31) & 1u) == want);
      if (__all_sync(0xffffffffu, ok)) break;
      if (SWB_WAVE_SLEEP_NS > 0) __nanosleep(SWB_WAVE_SLEEP_NS);
      load_raw(c0, raw);
    }
#pragma unroll
    for (int r = 0; r < KC; ++r) {
      const bool mine = c0 + r * 32 + lane < n;
      tile_in[r * 32 + lane] = mine ? make_int2((int)((uint32_t)raw[r] & 0x7fffffffu), (int)(raw[r] >> 32))
                                    : make_int2(0, 0);
    }
  };
  unsigned long long raw_next[KC];
#pragma unroll
  for (int r = 0; r < KC; ++r) raw_next[r] = 0ull;
  if (b > 0) load_raw(0, raw_next);

  {  // scores of step 0 (lane 0: super-column 0; other lanes idle)
#pragma unroll
    for (int r = 0; r < KC; ++r) {
      const int sym = (lane == 0 && r < n) ? (int)sref[r] : A;
      const uint32_t* pr = sprof + (sym * 32 + lane) * L;
#pragma unroll
      for (int j = 0; j < L; ++j) w.Sn[r][j] = pr[j];
    }
  }

  for (int t0 = 0; t0 < steps; t0 += TS) {
    // ---- step tile [t0, t0 + 32): boundary work ----
    if (t0 > 0) {  // residues of super-columns [t0 + 32, t0 + 64)
#pragma unroll
      for (int r = 0; r < KC; ++r) {
        const int c = (t0 + 32) * KC + r * 32 + lane;
        sref[c & RMASK] = c < n ? __ldg(a.ref + c) : (uint8_t)A;
      }
    }
    if (handoff && t0 >= 64)  // handoff tile t0/32 - 2
      store_tile((t0 - 64) * KC, TC, tile_out + ((t0 >> 5) & 1) * TC);
    // strip b-1's columns of super-columns [t0, t0 + 32): loaded last tile; load the next
    if (b > 0) {
      take_tile(t0 * KC, raw_next);
      __syncwarp();
      if (lane == 0 && t0 * KC < n)  // those ring slots are read: relaxed is enough
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(a.consumed + (size_t)b * 16),
                     "l"((unsigned long long)min((t0 + TS) * KC, n)) : "memory");
      load_raw((t0 + TS) * KC, raw_next);
    } else {
#pragma unroll
      for (int r = 0; r < KC; ++r) tile_in[r * 32 + lane] = make_int2(0, 0);
    }
    __syncwarp();
    // outgoing: lane 31 covers super-columns t0 - 31 .. t0 here, the tail of handoff
    // tile t0/32 - 1 (buffer parity (t0/32 - 1) & 1) and the head of tile t0/32
    int2* tlo = tile_out + ((((t0 >> 5) - 1) & 1) * TC);
    int2* thi = tile_out + (((t0 >> 5) & 1) * TC);
    const bool interior = t0 >= 32 && (t0 + 33) * KC <= n;  // every lane's columns in [0, n)
    if (interior) {
#pragma unroll (UNR)
      for (int k = 0; k < TS; ++k)
        wave_step<L, KC, false>(w, t0 + k, k, lane, n, A, sref, sprof, tile_in, tlo, thi, handoff,
                                NGO, NGE, qbase, NJG);
    } else {
#pragma unroll (UNR)
      for (int k = 0; k < TS; ++k)
        if (t0 + k < steps)
          wave_step<L, KC, true>(w, t0 + k, k, lane, n, A, sref, sprof, tile_in, tlo, thi, handoff,
                                 NGO, NGE, qbase, NJG);
    }
  }
  // the last (partial) outgoing tiles
  if (handoff) {
    const int tend = (steps + 31) & ~31;  // first step tile not entered
    for (int c0 = (tend >= 64 ? (tend - 64) * KC : 0); c0 < n; c0 += TC)
      store_tile(c0, min(TC, n - c0), tile_out + ((c0 / TC) & 1) * TC);
  }
  const int bv = w.rv;
  int bcol = bv > 0 ? w.rcol : -1, bq = bv > 0 ? w.rrow : -1;
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
