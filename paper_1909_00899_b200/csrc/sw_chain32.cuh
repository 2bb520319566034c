// sw_chain32.cuh -- 32-bit strip pipeline with the scan taken off the word loop's
// critical path ("carry-split" column schedule).
//
// Same strips, ring hand-off, coordinates and final reduction as sw_chain_kernel
// (sw_chain.cuh); what changes is the order of work inside a column.  A strip is
// a dependency chain of n reference columns: column i+1 needs column i's carry
// (the Alg. 6 scan of its F, src/_compiled.py:320-336).  In sw_chain_kernel the
// path from one carry to the next runs through the whole L-word recurrence and
// then the scan.  Here it runs through two instructions and the scan, because the
// F leaving a lane is a max-plus function of the carry:
//
//   u_c = max(vh_c + S_c, E_c),  vh_0 = max(Hs, G - (L-1)ge),  vh_c = max(H'_{c-1}, K - (c-1)ge)
//   F_L = relu(max_c(u_c - go - (L-1-c)ge))
//       = relu(max(A, K + B, G + C))          (exact, integer max-plus algebra)
//   A = max_c(max(H'_{c-1} + S_c, E_c) - go - (L-1-c)ge)   (H'_{-1} = Hs)
//   B = max_{c>=1} S_c - go - (L-2)ge,   C = S_0 - go - 2(L-1)ge
//
// K = carry[l], G = carry[l-1] of the previous column, H' / E / Hs the stored
// values of the previous column (Hs = lane l-1's last H; strip b-1's value at lane
// 0).  A, B, C need only the previous column's stored state and this column's
// profile row, so they are computed while the previous column's scan is in
// flight.  The exact L-word recurrence (stored H, E, end coordinates) still runs
// every column, off the critical path.  The scan is the radix-8 form on F shifted
// by two lanes (G directly, see sw_chain.cuh), so the critical path per column is
//   2 VIADDMNMX -> SHFL -> 7 SHFL + 3-deep max tree -> 3 SHFL + 2-deep tree -> 1 op.
// Word-loop length no longer adds latency, so strips can be taller (fewer strips,
// shorter pipeline fill) up to the SM issue budget.
#pragma once
#include "sw_chain.cuh"

#ifndef SWB_CHAIN32_SMEM_SCAN
#define SWB_CHAIN32_SMEM_SCAN 0  // 1: the radix-8 scan through shared memory instead of shuffles
#endif
#ifndef SWB_CHAIN32_BF_L
#define SWB_CHAIN32_BF_L 8
#endif
#ifndef SWB_CHAIN32_UNROLL
#define SWB_CHAIN32_UNROLL 2  // columns per loop iteration, coordinate instances
#endif
#ifndef SWB_CHAIN32_UNROLL_SO
#define SWB_CHAIN32_UNROLL_SO 4  // score-only instances (config 5: 2 -> 116.7 ms, 4 -> 110.4, 8 -> 128.9)
#endif

namespace swb {

// GE > 0: gap-extend penalty known at compile time, so the lane decays (d, 2d, .. 16d,
// the wrap decay) and the E / F decay are immediate operands (fewer register sources
// on the scan's critical path).
template <int L, bool COORDS = true, int GE = 0>
__global__ void __launch_bounds__(32) sw_chain32_kernel(const ChainArgs a) {
  constexpr int T = 32;
  constexpr int RING = kChainRing * kChainK;
  // strips of up to SWB_CHAIN32_BF_L words per lane track the first maximum without a
  // branch (L compares + 4 selects per column instead of a REDUX and a branch)
  constexpr bool kBranchFree = L <= SWB_CHAIN32_BF_L;
  constexpr int kColUnroll = COORDS ? SWB_CHAIN32_UNROLL : SWB_CHAIN32_UNROLL_SO;
  const int t = threadIdx.x;
  const int b = a.reverse ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x;
  const int nb = a.nb;
  const uint32_t gmask = 0xffffffffu;
  const int A_ = a.n_sym;

  extern __shared__ uint32_t smem[];
  {
    const int words = (A_ + 1) * L * 32;
    const uint32_t* src = a.prof + (size_t)b * words;
    for (int w = t; w < words; w += 32) smem[w] = __ldg(src + w);
    __syncwarp();
  }
  const int* prof_t = reinterpret_cast<const int*>(smem) + t;
  // per-tile staging: (F_in, H_last, residue) per column + the next tile's first residue
  int4* tile_in = reinterpret_cast<int4*>(smem + (A_ + 1) * L * 32);
  int2* tile_out = reinterpret_cast<int2*>(tile_in + kChainK + 1);
  // per (residue, lane): (B, C) of the F_L formula -- they depend on the profile row only
  int2* bc_tab = reinterpret_cast<int2*>(tile_out + kChainK);
  // shared-memory scan buffers (SWB_CHAIN32_SMEM_SCAN): [column parity][round][64],
  // the lower 32 entries of every buffer stay zero
  int* sbuf = reinterpret_cast<int*>(bc_tab + (A_ + 1) * 32);
  for (int k = t; k < 256; k += 32) sbuf[k] = 0;

  const int CL = W32::CLAMP;
  const int go = min(a.go, CL), ge = GE > 0 ? GE : min(a.ge, CL);
  const int d = min(L * ge, CL);                       // decay per lane
  const int dw = (int)min((int64_t)(L - 1) * ge, (int64_t)CL);  // wrap decay
  const int kB = (int)min((int64_t)go + (int64_t)(L >= 2 ? L - 2 : 0) * ge, (int64_t)CL);
  const int kC = (int)min((int64_t)go + 2 * (int64_t)(L - 1) * ge, (int64_t)CL);
  int kA[L];  // go + (L-1-c) ge
#pragma unroll
  for (int c = 0; c < L; ++c) kA[c] = (int)min((int64_t)go + (int64_t)(L - 1 - c) * ge, (int64_t)CL);
  const int nullsym = A_;
  const int keep1 = t >= 1 ? -1 : 0, keep2 = t >= 2 ? -1 : 0;
  for (int sym = 0; sym <= A_; ++sym) {
    const int* row = prof_t + sym * (L * 32);
    int sm = -(1 << 29);
#pragma unroll
    for (int c = 1; c < L; ++c) sm = max(sm, row[c * 32]);
    bc_tab[sym * 32 + t] = make_int2(L >= 2 ? sm - kB : -(1 << 29), row[0] - kC);
  }
  __syncwarp();

  int H[L], E[L];
#pragma unroll
  for (int c = 0; c < L; ++c) { H[c] = 0; E[c] = 0; }
  int K = 0, G = 0, Hs = 0;  // previous column: carry[l], carry[l-1], lane l-1's last H
  int gb = 0;                      // best of all earlier columns in this strip
  int bv = 0, bcol = -1, bq = -1;  // this thread's first-maximum record
  const int64_t n = a.n;
  const int64_t qbase = (int64_t)b * T * L;

  // A of the next column from its profile row and the current stored state
  auto a_of = [&](const int (&S)[L], int hs) -> int {
    int acc = __viaddmax_s32(hs, S[0], E[0]) - kA[0];
#pragma unroll
    for (int c = 1; c < L; ++c) acc = max(acc, __viaddmax_s32(H[c - 1], S[c], E[c]) - kA[c]);
    return acc;
  };

  int2* ring_in = a.ring + (size_t)(b > 0 ? b - 1 : 0) * RING;
  int2* ring_out = a.ring + (size_t)b * RING;
  unsigned long long* ring_out64 = reinterpret_cast<unsigned long long*>(ring_out);
  const unsigned long long* ring_in64 = reinterpret_cast<const unsigned long long*>(ring_in);
  auto tag_of = [](int64_t c) -> unsigned { return (((unsigned)(c / RING)) & 1u) ^ 1u; };
  auto load_raw = [&](int64_t c0) -> unsigned long long {
    return (c0 + t < n && t < kChainK) ? ld_relaxed(ring_in64 + ((c0 + t) % RING)) : 0ull;
  };
  unsigned long long raw_next = b > 0 ? load_raw(0) : 0ull;
  unsigned long long cons_seen = 0;

  // column 0's profile row and A, B, C (all stored state is zero)
  int Sc[L];
  int Acur, Bcur, Ccur;
  {
    const int sym0 = (int)__ldg(a.ref);
    const int* pr0 = prof_t + sym0 * (L * 32);
#pragma unroll
    for (int c = 0; c < L; ++c) Sc[c] = pr0[c * 32];
    Acur = a_of(Sc, 0);
    const int2 bc = bc_tab[sym0 * 32 + t];
    Bcur = bc.x;
    Ccur = bc.y;
  }
  // residues two tiles ahead: res1 = the next tile's, res2 = the one after (clamped
  // loads, masked when staged, so no instruction waits on a load issued this tile)
  auto ld_res = [&](int64_t c) -> int { return (int)__ldg(a.ref + min(c, n - 1)); };
  int res1 = ld_res(t), res2 = ld_res(kChainK + t);
  // Start two tiles behind strip b-1: the boundary tile prefetched at the start of a
  // tile is then already written when it is loaded (one tile behind, every prefetch
  // found the entries stale and the validation paid a full L2 round trip per tile).
  if (b > 0 && n > kChainK) {
    const int64_t c1 = kChainK + t;
    const unsigned want = tag_of(kChainK);
    while (!__all_sync(gmask, c1 >= n || (unsigned)((ld_relaxed(ring_in64 + (c1 % RING)) >> 31) &
                                                    1u) == want))
      __nanosleep(64);
  }

  for (int64_t t0 = 0; t0 < n; t0 += kChainK) {
    const int kc = (int)min((int64_t)kChainK, n - t0);
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
      if (t == 0)
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
    __syncwarp();
    const int res_here = res1;
    res1 = res2;
    res2 = ld_res(t0 + 2 * kChainK + t);
    tile_in[t] = make_int4(fin_l, hl_l, t < kc ? res_here : nullsym, 0);
    // the residue after this tile (the next tile's first): the last column prepares
    // the next column's A, B, C from it
    const int first_next = __shfl_sync(gmask, res1, 0);
    if (t == 0) tile_in[kChainK] = make_int4(0, 0, t0 + kc < n ? first_next : nullsym, 0);
    __syncwarp();

    int2 fh = *reinterpret_cast<const int2*>(&tile_in[0]);  // (F_in, H_last) of column t0
#pragma unroll kColUnroll
    for (int col_k = 0; col_k < kc; ++col_k) {
      const int64_t i = t0 + col_k;
      const int fin = fh.x, hlk = fh.y;
      // next column's inputs (off the critical path)
      const int nk = col_k + 1 < kc ? col_k + 1 : kChainK;
      const int4 tn = tile_in[nk];
      fh = make_int2(tn.x, tn.y);
      int Sn[L];
      {
        const int* pr1 = prof_t + tn.z * (L * 32);
#pragma unroll
        for (int c = 0; c < L; ++c) Sn[c] = pr1[c * 32];
      }
      const int2 bcn = bc_tab[tn.z * 32 + t];

      // ---- critical path: F leaving each lane, the radix-8 scan, the carry ----
      const int FL = __viaddmax_s32_relu(G, Ccur, __viaddmax_s32(K, Bcur, Acur));
#if SWB_CHAIN32_SMEM_SCAN
      // the same radix-8 scan through shared memory: one store of F (and of the F
      // entering the strip, at slot 31), a warp barrier, and each lane reads its eight
      // predecessors of the shifted-by-two vector directly (zeros below lane 0), so no
      // shift instruction precedes the window; buffers alternate with the column
      int* b1 = sbuf + (col_k & 1) * 128;
      int* b2 = b1 + 64;
      b1[32 + t] = FL;
      if (t == 0) b1[31] = fin;
      __syncwarp();
      const int* rw = b1 + 30 + t;  // rw[-k] = F shifted by two, lane t - k
      const int f2 = rw[0], y1 = rw[-1], y2 = rw[-2], y3 = rw[-3], y4 = rw[-4], y5 = rw[-5],
                y6 = rw[-6], y7 = rw[-7];
      const int f1 = b1[31 + t];
      const int q1 = __viaddmax_s32(y1, -d, f2), q2 = __viaddmax_s32(y3, -d, y2);
      const int q3 = __viaddmax_s32(y5, -d, y4), q4 = __viaddmax_s32(y7, -d, y6);
      const int w8 = __viaddmax_s32(__viaddmax_s32(q4, -2 * d, q3), -4 * d,
                                    __viaddmax_s32(q2, -2 * d, q1));
      b2[32 + t] = w8;
      __syncwarp();
      const int z1 = b2[24 + t], z2 = b2[16 + t], z3 = b2[8 + t];
#else
      // lane 0 of the shift by one and lane 1 of the shift by two take the F entering
      // the strip, lane 0 of the shift by two nothing: (x & keep) | inject, one LOP3
      const int f1 = (__shfl_up_sync(gmask, FL, 1) & keep1) | (t == 0 ? fin : 0);
      const int f2 = (__shfl_up_sync(gmask, FL, 2) & keep2) | (t == 1 ? fin : 0);
      const int y1 = __shfl_up_sync(gmask, f2, 1), y2 = __shfl_up_sync(gmask, f2, 2),
                y3 = __shfl_up_sync(gmask, f2, 3), y4 = __shfl_up_sync(gmask, f2, 4),
                y5 = __shfl_up_sync(gmask, f2, 5), y6 = __shfl_up_sync(gmask, f2, 6),
                y7 = __shfl_up_sync(gmask, f2, 7);
      const int q1 = __viaddmax_s32(y1, -d, f2), q2 = __viaddmax_s32(y3, -d, y2);
      const int q3 = __viaddmax_s32(y5, -d, y4), q4 = __viaddmax_s32(y7, -d, y6);
      const int w8 = __viaddmax_s32(__viaddmax_s32(q4, -2 * d, q3), -4 * d,
                                    __viaddmax_s32(q2, -2 * d, q1));
      const int z1 = __shfl_up_sync(gmask, w8, 8), z2 = __shfl_up_sync(gmask, w8, 16),
                z3 = __shfl_up_sync(gmask, w8, 24);
#endif
      const int gn = __viaddmax_s32(__viaddmax_s32(z3, -8 * d, z2), -16 * d,
                                    __viaddmax_s32(z1, -8 * d, w8));  // carry[l-1]
      const int Kn = __viaddmax_s32(gn, -d, f1);                       // carry[l]

      // ---- the exact recurrence of this column (stored H, E; coordinates) ----
      int vh = __viaddmax_s32(G, -dw, Hs);
      int F = 0;
      constexpr int kCh = 8, kNch = (L + kCh - 1) / kCh;
      int cmk[kNch];
#pragma unroll
      for (int ch = 0; ch < kNch; ++ch) cmk[ch] = 0;
#pragma unroll
      for (int c = 0; c < L; ++c) {
        const int u = __viaddmax_s32(vh, Sc[c], E[c]);
        const int Hn = max(u, F);
        const int Xu = u - go;
        E[c] = __viaddmax_s32_relu(E[c], -ge, Xu);
        F = __viaddmax_s32_relu(F, -ge, Xu);
        cmk[c / kCh] = max(cmk[c / kCh], u);
        vh = __viaddmax_s32(K, -(int)min((int64_t)c * ge, (int64_t)CL), H[c]);
        H[c] = Hn;
      }
      // F == FL (same max-plus value); the boundary leaving lane 31 uses it
      int cm = cmk[0];
#pragma unroll
      for (int k = 1; k < kNch; ++k) cm = max(cm, cmk[k]);
      int gb_prev = gb;
      if constexpr (!COORDS) {
        bv = max(bv, cm);  // score-only launch: the running maximum is all it needs
      } else if constexpr (kBranchFree) {
        // each lane keeps its own first maximum without a branch: the first column
        // where its maximum grows, and in it the first word reaching the new value
        // (a cell reaching the best is a diagonal cell, stored H == u); the strip
        // and pipeline reductions pick (score desc, column asc, row asc) at the end
        int jj = L - 1;
#pragma unroll
        for (int c = L - 2; c >= 0; --c) jj = H[c] >= cm ? c : jj;
        const bool up = cm > bv;
        bv = up ? cm : bv;
        bcol = up ? (int)i : bcol;
        bq = up ? (int)(qbase + t * L) + jj : bq;
      } else {
        gb = __reduce_max_sync(gmask, max(gb, cm));  // the strip's best of all columns so far
      }

      // ---- next column's A, B, C from this column's stored state ----
      int hsn = __shfl_up_sync(gmask, H[L - 1], 1);
      hsn = t == 0 ? hlk : hsn;  // lane 0: strip b-1's corrected last H of this column
      Acur = a_of(Sn, hsn);
      Bcur = bcn.x;
      Ccur = bcn.y;
      if (t == T - 1) {
        const int fo = __viaddmax_s32(Kn, -d, F);          // true F leaving the strip
        const int hlast = __viaddmax_s32(Kn, -dw, H[L - 1]);  // its corrected last H
        tile_out[col_k] = make_int2(fo, hlast);
      }
      K = Kn;
      G = gn;
      Hs = hsn;
#pragma unroll
      for (int c = 0; c < L; ++c) Sc[c] = Sn[c];
      // end coordinates (rare: the strip's best improved in this lane) -- the only
      // branch of the column, placed after everything the next column needs so the
      // scheduler can interleave the scan with the recurrence above
      if (COORDS && !kBranchFree && SWB_CHAIN_COORDS && cm > gb_prev && cm > bv) {
        int kk = 0;
#pragma unroll
        for (int k = kNch - 1; k >= 0; --k)
          if (cmk[k] >= cm) kk = k;
        int jj = 0;
#pragma unroll
        for (int k = 0; k < kNch; ++k) {
          if (k == kk) {
#pragma unroll
            for (int c = (k + 1) * kCh - 1; c >= k * kCh; --c)
              if (c < L && H[c] >= cm) jj = c;
          }
        }
        bv = cm;
        bcol = (int)i;
        bq = (int)(qbase + t * L + jj);
      }
    }
    __syncwarp();
    if (b + 1 < nb && t < kc) {
      const int2 e = tile_out[t];
      __stcg(ring_out64 + ((t0 + t) % RING), ((unsigned long long)(uint32_t)e.y << 32) |
                                                 (uint32_t)e.x | ((unsigned long long)tag_of(t0) << 31));
    }
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
