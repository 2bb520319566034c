// sw_block.cuh -- one alignment per CTA, or per thread-block cluster: the paper's
// F scan at high stripe counts, warp shuffle -> block -> cluster (DSMEM).
//
// Layout: the reference's striping (src/profile.py:37-81) with P = p lanes;
// lane l owns query positions [l*L, l*L + L), L = ceil(m / P).  Global thread
// g = rank * NT + tid (rank = CTA rank in the cluster, NT threads per CTA) holds
// lanes 2g (low half) and 2g + 1 (high half) with 16-bit scores, lane g with
// 32-bit scores -- adjacent lanes in one register, so a one-lane shift is a
// single SHFL.UP + PRMT and the cross-thread scan is a scan over threads.
//
// Per reference residue (column, src/_compiled.py:247-340):
//   1. the L-word recurrence (sw_kernels.cuh), diagonal input of the thread's
//      first lane from the previous thread's corrected last H (wrap);
//   2. VAR_SCAN: Alg. 6's weighted max-plus scan of the column's F over all P
//      lanes, as an exclusive scan over threads with per-thread decay D:
//        A_g   = F leaving thread g's last lane, inclusive of its own lanes
//        warp  : 5 SHFL.UP + VIADDMNMX.RELU steps -> warp-exclusive prefix
//        block : lane 31 of each warp publishes (aggregate, its prefix, ...) to
//                shared memory; one bar.sync; every warp combines the
//                aggregates of the warps before it with one REDUX.MAX
//        cluster: the CTA's inclusive aggregate and the corrected H of its last
//                lane go to CTA rank+1 through distributed shared memory (one
//                64-bit remote store per column into a tagged ring), folded into
//                that CTA's block combine by the same REDUX.  CTA r only needs
//                CTA r-1's column i before finishing its own column i, so the
//                CTAs run as a pipeline, each one hop (~200 cycles) behind.
//      The carry is applied when the next column reads H (deferred correction).
//   2'. VAR_LAZYF / VAR_LAZYF_MIRROR (single CTA): Farrar's passes with the
//      reference's early exit (src/_compiled.py:189-217); each pass shifts F one
//      lane across the whole block and votes with one __syncthreads_or.
#pragma once
#include "sw_kernels.cuh"

namespace swb {

constexpr int kBlockRing = 128;     // columns in flight between neighbouring CTAs
constexpr int kBlockMaxThreads = 1024;

struct BlockArgs {
  const uint8_t* query;   // [m] codes
  const int8_t* sub;      // [A][A]
  int32_t n_sym, m, seg_len;
  const uint8_t* ref;
  int64_t n;
  int32_t go, ge, bias, max_sub;
  int32_t early_exit;     // lazy-F: the reference's early exit (1) or all P passes (0)
  int32_t coords;         // locate end coordinates
  int32_t* score;
  int32_t* ref_end;
  int32_t* query_end;
  uint8_t* flags;
  int32_t* col_passes;    // lazy-F: per-column passes (nullable)
  int64_t* pass_stats;    // lazy-F: [2] total passes, early-exit columns (nullable)
};

__device__ __forceinline__ int relu_sub(int x, int d) { return __viaddmax_s32_relu(x, -d, 0); }

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void st_cluster_u64(uint32_t local_addr, unsigned rank, unsigned long long v) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_addr), "r"(rank));
  asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(ra), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_local_u64(uint32_t addr) {
  unsigned long long v;
  asm volatile("ld.relaxed.cluster.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <class Wd, int L, int VAR>
__global__ void __launch_bounds__(L <= 4 ? 1024 : (L <= 8 ? 512 : 256), 1) sw_block_kernel(const BlockArgs a) {
  constexpr int LPW = Wd::LPW;
  constexpr bool SCAN = VAR == VAR_SCAN;
  const int NT = blockDim.x, NW = NT >> 5;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  unsigned rank, CL;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(CL));
  const int A = a.n_sym;
  const int m = a.m;
  const int64_t n = a.n;
  constexpr uint32_t FULL = 0xffffffffu;

  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* prof_s = smem;                                           // [(A+1)][L][NT]
  int4* agg = reinterpret_cast<int4*>(smem + (A + 1) * L * NT);      // [2][32] warp publications
  unsigned long long* ring = reinterpret_cast<unsigned long long*>(agg + 64);  // [kBlockRing] from CTA rank-1
  unsigned long long* cons = ring + kBlockRing;                      // [1] progress of CTA rank+1
  int4* red = reinterpret_cast<int4*>(cons + 2);                     // [32] final reduction; [CL] on rank 0

  // ---- this CTA's slab of the striped profile, built in place ----
  {
    const int words = (A + 1) * L * NT;
    for (int k = tid; k < words; k += NT) {
      const int t = k % NT, j = (k / NT) % L, sym = k / (NT * L);
      const int g = (int)rank * NT + t;
      int v[2] = {0, 0};
#pragma unroll
      for (int h = 0; h < LPW; ++h) {
        const int q = (LPW * g + h) * L + j;
        if (sym == A) v[h] = Wd::NULLV;
        else if (q >= m) v[h] = -a.bias;  // reference pad: profile 0 == -bias
        else v[h] = a.sub[sym * A + a.query[q]];
      }
      prof_s[k] = Wd::pack(v[0], v[1]);
    }
    for (int k = tid; k < kBlockRing + 2; k += NT) ring[k] = 0ull;  // ring + cons
  }
  // every CTA's ring is zeroed before any neighbour may write into it
  if (CL > 1) cluster_sync_all(); else __syncthreads();

  // ---- constants ----
  const int cl = Wd::CLAMP;
  const int go = a.go, ge = a.ge;
  const uint32_t NGO = Wd::splat(-min(go, cl));
  const uint32_t NGE = Wd::splat(-min(ge, cl));
  const uint32_t NWRAP = Wd::splat(-(int)min((int64_t)(L - 1) * ge, (int64_t)cl));
  uint32_t NJ[L];
#pragma unroll
  for (int c = 0; c < L; ++c) NJ[c] = Wd::splat(-(int)min((int64_t)c * ge, (int64_t)cl));
  // scalar scan decays (32-bit arithmetic for both widths): d per lane, D per thread
  constexpr int64_t kDecCap = 1 << 29;
  const int64_t d64 = (int64_t)L * ge, D64 = LPW * d64;
  auto dec = [&](int64_t k) -> int { return (int)min(k * D64, kDecCap); };
  const int d = (int)min(d64, kDecCap), D = dec(1);
  const int wrap_dec = (int)min((int64_t)(L - 1) * ge, kDecCap);
  int NK[5];
#pragma unroll
  for (int s = 0; s < 5; ++s) NK[s] = -dec(1 << s);
  const int dl = dec(lane);                                   // lane's distance from its warp start
  const int dk1 = lane < w ? dec((int64_t)(w - 1 - lane) * 32) : 0;      // warp `lane` -> end of warp w-1
  const int dk2 = lane < w - 1 ? dec((int64_t)(w - 2 - lane) * 32) : 0;  // warp `lane` -> end of warp w-2
  const int dc1 = dec((int64_t)w * 32);                       // previous CTA's end -> end of warp w-1
  const int dc2 = w > 0 ? dec((int64_t)(w - 1) * 32) : 0;     // previous CTA's end -> end of warp w-2
  const int d31 = dec(31);
  const uint32_t ring_base = smem_addr(ring);
  const uint32_t cons_addr = smem_addr(cons);
  const int g = (int)rank * NT + tid;
  const bool last_thread_global = (rank + 1 == CL) && (tid == NT - 1);

  uint32_t H[L], E[L];
#pragma unroll
  for (int c = 0; c < L; ++c) { H[c] = 0u; E[c] = 0u; }
  uint32_t carry = 0u, wcorr = 0u;
  int wb = 0;                       // lane 0: corrected last H of the previous thread (wrap input)
  int gb = 0;                       // warp's running best of all earlier columns
  int bv = 0, bcol = -1, bq = -1;   // this thread's first-maximum record
  constexpr int kCh = 8, kNch = (L + kCh - 1) / kCh;
  uint32_t cmk[kNch];
#pragma unroll
  for (int k = 0; k < kNch; ++k) cmk[k] = 0u;
  int64_t tot_passes = 0, breaks = 0;
  int par = 0;                       // parity of the shared-memory publication slots
  unsigned cons_seen = 0;  // last observed progress of CTA rank+1
  const int P = (int)CL * NT * LPW;
  int nxt = n > 0 ? (int)__ldg(a.ref) : 0;

  const int n32 = (int)n;  // host guarantees n < 2^31
  for (int i = 0; i < n32; ++i) {
    const int sym = nxt;
    nxt = (i + 1 < n32) ? (int)__ldg(a.ref + i + 1) : 0;
    const uint32_t* pr = prof_s + sym * (L * NT) + tid;
    // diagonal input of each lane: the previous lane's corrected last H (shift by one lane)
    uint32_t r = __shfl_up_sync(FULL, wcorr, 1);
    if (lane == 0) r = LPW == 2 ? ((uint32_t)wb << 16) : (uint32_t)wb;
    uint32_t vh = LPW == 2 ? prmt(r, wcorr, 0x5432u) : r;  // {r.hi, wcorr.lo}
    uint32_t F = 0u;
#pragma unroll
    for (int c = 0; c < L; ++c) {
      const uint32_t S = pr[c * NT];
      const uint32_t u = Wd::addmax(vh, S, E[c]);
      const uint32_t Hn = Wd::vmax(u, F);
      const uint32_t Xu = Wd::add(u, NGO);
      if constexpr (VAR == VAR_LAZYF_MIRROR) E[c] = Wd::addmax_relu(E[c], NGE, Wd::add(Hn, NGO));
      else E[c] = Wd::addmax_relu(E[c], NGE, Xu);
      F = Wd::addmax_relu(F, NGE, Xu);
      cmk[c / kCh] = Wd::vmax(cmk[c / kCh], u);
      if constexpr (SCAN) vh = Wd::addmax(carry, NJ[c], H[c]);
      else vh = H[c];
      H[c] = Hn;
    }

    // ---- end coordinates (as sw_striped_kernel), gated on the warp's running best ----
    if (a.coords) {
      uint32_t cm = cmk[0];
#pragma unroll
      for (int k = 1; k < kNch; ++k) cm = Wd::vmax(cm, cmk[k]);
      const int cmx = Wd::hmax(cm);
      if (cmx > gb) {
#pragma unroll
        for (int h = 0; h < LPW; ++h) {
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
            bcol = i;
            bq = (LPW * g + h) * L + jj;
          }
        }
      }
      gb = __reduce_max_sync(FULL, max(gb, cmx));
    }

    if constexpr (SCAN) {
      // ---- Alg. 6 scan over all P lanes: warp shuffle, block, cluster ----
      const int xlo = Wd::get(F, 0);
      const int Ag = LPW == 2 ? __viaddmax_s32_relu(xlo, -d, Wd::get(F, 1)) : xlo;  // thread-inclusive
      int acc = __shfl_up_sync(FULL, Ag, 1);
      if (lane == 0) acc = 0;
#pragma unroll
      for (int s = 0; s < 5; ++s) {  // lanes below K read their own value: max(x, relu(x - K*D)) = x
        const int o = __shfl_up_sync(FULL, acc, 1 << s);
        acc = __viaddmax_s32_relu(o, NK[s], acc);
      }
      const int wex = acc;  // warp-exclusive prefix
      if (lane == 31)
        agg[par * 32 + w] = make_int4(__viaddmax_s32_relu(wex, -D, Ag), wex, xlo, Wd::get(H[L - 1], LPW - 1));
      __syncthreads();
      int cin = 0, win = 0;
      if (rank > 0) {
        // the previous CTA's column-i boundary (inclusive F prefix, corrected last H)
        const unsigned want = (((unsigned)i / kBlockRing) & 1u) ^ 1u;
        const uint32_t addr = ring_base + ((unsigned)i % kBlockRing) * 8u;
        unsigned long long v = ld_local_u64(addr);
        while ((((unsigned)(v >> 31)) & 1u) != want || (((unsigned)(v >> 63)) & 1u) != want)
          v = ld_local_u64(addr);
        cin = (int)((uint32_t)v & 0x7fffffffu);
        win = (int)((uint32_t)(v >> 32) & 0x7fffffffu);
        if (tid == 0 && ((unsigned)i % (kBlockRing / 4)) == kBlockRing / 4 - 1)
          st_cluster_u64(cons_addr, rank - 1, (unsigned long long)(i + 1));
      }
      const int ak = lane < w ? agg[par * 32 + lane].x : 0;
      int v1 = relu_sub(ak, dk1), v2 = lane < w - 1 ? relu_sub(ak, dk2) : 0;
      if (lane == 31) { v1 = relu_sub(cin, dc1); v2 = relu_sub(cin, dc2); }
      const int pin = __reduce_max_sync(FULL, v1);   // inclusive prefix at the end of warp w-1
      const int pin1 = __reduce_max_sync(FULL, v2);  // ... at the end of warp w-2
      const int bex = max(wex, relu_sub(pin, dl));    // thread-exclusive prefix (all lanes before)
      if constexpr (LPW == 2) carry = Wd::pack(bex, __viaddmax_s32_relu(bex, -d, xlo));
      else carry = (uint32_t)bex;
      wcorr = Wd::addmax(carry, NWRAP, H[L - 1]);
      if (lane == 0) {
        if (w == 0) {
          wb = win;
        } else {  // previous warp's last thread, from its publication
          const int4 pv = agg[par * 32 + w - 1];
          const int bp = max(pv.y, relu_sub(pin1, d31));
          const int cp = LPW == 2 ? __viaddmax_s32_relu(bp, -d, pv.z) : bp;
          wb = __viaddmax_s32_relu(cp, -wrap_dec, pv.w);
        }
      }
      // the CTA's boundary for CTA rank+1: inclusive prefix and corrected last H
      if (rank + 1 < CL && w == NW - 1) {
        if (cons_seen + kBlockRing <= (unsigned)i) {
          const unsigned need = (unsigned)i - kBlockRing + 1;
          unsigned c = (unsigned)ld_local_u64(cons_addr);
          while (c < need) c = (unsigned)ld_local_u64(cons_addr);
          cons_seen = c;
        }
        if (lane == 31) {
          const unsigned tag = (((unsigned)i / kBlockRing) & 1u) ^ 1u;
          const uint32_t so = (uint32_t)__viaddmax_s32_relu(bex, -D, Ag) | (tag << 31);
          const uint32_t wo = (uint32_t)Wd::get(wcorr, LPW - 1) | (tag << 31);
          st_cluster_u64(ring_base + ((unsigned)i % kBlockRing) * 8u, rank + 1,
                         ((unsigned long long)wo << 32) | so);
        }
      }
      par ^= 1;
    } else {
      // ---- lazy-F (single CTA): one block-wide shift + vote per pass ----
      int2* lz = reinterpret_cast<int2*>(agg);
      uint32_t vf = F;
      int passes = 0;
      for (int it = 0;; ++it) {
        if (lane == 31) lz[par * 32 + w] = make_int2(Wd::get(vf, LPW - 1), Wd::get(H[L - 1], LPW - 1));
        // the shifted F is all zero iff every lane but the global last one is zero
        bool nz = vf != 0u;
        if (last_thread_global) nz = LPW == 2 ? Wd::get(vf, 0) != 0 : false;
        const int any = __syncthreads_or(a.early_exit ? (int)nz : 1);
        const int2 prev = (lane == 0 && w > 0) ? lz[par * 32 + w - 1] : make_int2(0, 0);
        par ^= 1;
        if (!any || it == P) {  // H final: the wrap input is the previous thread's last H
          wcorr = H[L - 1];
          if (lane == 0) wb = prev.y;
          break;
        }
        uint32_t rr = __shfl_up_sync(FULL, vf, 1);
        if (lane == 0) rr = LPW == 2 ? ((uint32_t)prev.x << 16) : (uint32_t)prev.x;
        vf = LPW == 2 ? prmt(rr, vf, 0x5432u) : rr;
#pragma unroll
        for (int c = 0; c < L; ++c) {
          H[c] = Wd::vmax(H[c], vf);
          vf = Wd::addmax_relu(vf, NGE, NGE);
        }
        ++passes;
      }
      if (tid == 0) {
        if (a.col_passes) a.col_passes[i] = passes;
        tot_passes += passes;
        breaks += (a.early_exit && passes < P) ? 1 : 0;
      }
    }
  }

  // ---- reduce (best desc, ref_end asc, query_end asc): warp, CTA, cluster ----
  int sc;
  {
    uint32_t cm = cmk[0];
#pragma unroll
    for (int k = 1; k < kNch; ++k) cm = Wd::vmax(cm, cmk[k]);
    sc = Wd::hmax(cm);
  }
  int best = bv, col = bcol, q = bq;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    sc = max(sc, __shfl_xor_sync(FULL, sc, off));
    const int ob = __shfl_xor_sync(FULL, best, off);
    const int oc = __shfl_xor_sync(FULL, col, off);
    const int oq = __shfl_xor_sync(FULL, q, off);
    if (ob > best || (ob == best && (oc < col || (oc == col && oq < q)))) { best = ob; col = oc; q = oq; }
  }
  __syncthreads();  // publication slots are reused below
  int4* wred = reinterpret_cast<int4*>(agg);
  if (lane == 0) wred[w] = make_int4(best, col, q, sc);
  __syncthreads();
  if (w == 0) {
    int4 v = lane < NW ? wred[lane] : make_int4(0, -1, -1, 0);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const int ob = __shfl_xor_sync(FULL, v.x, off), oc = __shfl_xor_sync(FULL, v.y, off);
      const int oq = __shfl_xor_sync(FULL, v.z, off), os = __shfl_xor_sync(FULL, v.w, off);
      v.w = max(v.w, os);
      if (ob > v.x || (ob == v.x && (oc < v.y || (oc == v.y && oq < v.z)))) { v.x = ob; v.y = oc; v.z = oq; }
    }
    if (lane == 0) {
      if (CL > 1) {  // to rank 0's shared memory
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_addr(red + rank)), "r"(0));
        asm volatile("st.shared::cluster.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(ra), "r"(v.x), "r"(v.y),
                     "r"(v.z), "r"(v.w) : "memory");
      } else {
        red[0] = v;
      }
    }
  }
  if (CL > 1) cluster_sync_all(); else __syncthreads();
  if (rank == 0 && tid == 0) {
    int4 v = red[0];
    for (unsigned s = 1; s < CL; ++s) {
      const int4 o = red[s];
      v.w = max(v.w, o.w);
      if (o.x > v.x || (o.x == v.x && (o.y < v.y || (o.y == v.y && o.z < v.z)))) { v.x = o.x; v.y = o.y; v.z = o.z; }
    }
    const int score = v.w;
    uint8_t fl = 0;
    if constexpr (LPW == 2) {
      if (score >= 32767 - a.max_sub) fl |= FLAG_RESCUE;
    }
    if (score > 65535 - a.bias) fl |= FLAG_REF_OVERFLOW;
    int rc = v.y, rq = v.z;
    if (score == 0 || !a.coords) { rc = -1; rq = -1; }
    a.score[0] = score;
    if (a.ref_end) a.ref_end[0] = rc;
    if (a.query_end) a.query_end[0] = rq;
    if (a.flags) a.flags[0] = fl;
    if (a.pass_stats) { a.pass_stats[0] = tot_passes; a.pass_stats[1] = breaks; }
  }
}

}  // namespace swb
