// sw_kernels.cuh -- B200 (sm_100a) striped Smith-Waterman with the max-plus F scan.
//
// One alignment is owned by a *group* of T threads (T = 1..32, a power of two;
// several groups share a warp).  The query is striped exactly as the reference
// does it (src/profile.py:37-72, stripe_index :75-81): P virtual lanes, lane l
// owns query positions [l*L, l*L + L), L = ceil(m / P).  With 16-bit scores a
// 32-bit register packs two lanes (thread t holds lane t in the low half and
// lane T+t in the high half, P = 2T) and every cell update is one DPX
// instruction on both halves; with 32-bit scores P = T.
//
// Per reference residue (a "column", src/_compiled.py:247-340) a thread runs
// its L words serially (the intra-lane F chain is ONE dependent DPX op per
// word), then the cross-lane F dependency is resolved
//   * VAR_SCAN  -- by the paper's Alg. 6: a log2(P)-step weighted max-plus scan
//                  of the column's F (warp shuffles), applied lazily when the
//                  next column reads H (the deferred correction),
//   * VAR_LAZYF -- by Farrar's lazy-F loop with the reference's early exit
//                  (src/_compiled.py:189-217), a group vote per pass.
// VAR_LAZYF_MIRROR additionally reproduces the reference's E recurrence bit
// for bit so per-column pass counts equal the reference's (parity mode).
//
// Cell update per packed word (F chain = the single dependent op on F):
//   u  = max(vh + S, E)          diagonal / horizontal gap (E >= 0, so u >= 0)
//   Hn = max(u, F)               stored H (before cross-lane correction)
//   Xu = u - go
//   E  = max(E - ge, Xu, 0)      (MIRROR: max(E - ge, Hn - go, 0))
//   F  = max(F - ge, Xu, 0)      == reference F' (F - go <= F - ge)
//   cm = max(cm, u)              column max for score / end coordinates
//   vh = max(carry - j*ge, Hold) deferred correction (VAR_SCAN)
// E excludes F-derived H in the fast mode: a vertical->horizontal gap corner
// costs the same as the horizontal->vertical one the recurrence keeps, so H is
// exact (the same argument the reference makes for never revisiting E after a
// correction); the parity tests check it against the oracle.
//
// Runtime segment length: words are kept in registers H[0..LMAX), E[0..LMAX);
// a column enters a fall-through switch at word `first = LMAX - L`, so word c
// holds segment position j = c - first and the last word is always LMAX-1.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace swb {

enum Variant : int { VAR_SCAN = 0, VAR_LAZYF = 1, VAR_LAZYF_MIRROR = 2 };

// result flag bits (per alignment)
enum : uint8_t {
  FLAG_REF_OVERFLOW = 1,  // the reference uint16 kernels would saturate (exact > 65535 - bias)
  FLAG_RESCUE = 2,        // 16-bit run may have wrapped: re-run in 32 bits
  FLAG_RESCUED = 4,       // score/coords come from the 32-bit re-run
  FLAG_FEED_TIMEOUT = 8,  // streamed input never arrived (results invalid)
};

constexpr int kMaxSym = 32;  // alphabet size limit of the device path (plus one null row)
constexpr int kPairSubWords = kMaxSym * kMaxSym / 4;  // pairs mode: the int8 matrix staged in shared memory

__device__ __forceinline__ int ld_acquire_s32(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

__device__ __forceinline__ uint32_t w4(const uint4& v, int k) {
  return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}

// ---- word policies -------------------------------------------------------
#ifndef SWB_IMAD_SHIFT
#define SWB_IMAD_SHIFT 1  // lane shifts: multiply by 1 / 65536 (IMAD, FMA pipe) instead of PRMT (ALU pipe)
#endif
__device__ __forceinline__ uint32_t mul_lo(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

struct W16 {
  static constexpr int LPW = 2;
  static constexpr int NULLV = -16384;   // null-residue row (beyond a target's end)
  static constexpr int CLAMP = 32767;    // decay constants are clamped to the score range
  __host__ __device__ static constexpr uint32_t splat(int v) {
    return (uint32_t)(v & 0xffff) * 0x10001u;
  }
  __device__ static __forceinline__ uint32_t add(uint32_t a, uint32_t b) { return __vadd2(a, b); }
  __device__ static __forceinline__ uint32_t vmax(uint32_t a, uint32_t b) { return __vmaxs2(a, b); }
  __device__ static __forceinline__ uint32_t addmax(uint32_t a, uint32_t b, uint32_t c) {
    return __viaddmax_s16x2(a, b, c);
  }
  __device__ static __forceinline__ uint32_t addmax_relu(uint32_t a, uint32_t b, uint32_t c) {
    return __viaddmax_s16x2_relu(a, b, c);
  }
  __device__ static __forceinline__ int get(uint32_t v, int h) {
    return h ? (int)(int16_t)(v >> 16) : (int)(int16_t)(v & 0xffffu);
  }
  __device__ static __forceinline__ uint32_t pack(int lo, int hi) {
    return (uint32_t)(lo & 0xffff) | ((uint32_t)hi << 16);
  }
  __device__ static __forceinline__ int hmax(uint32_t v) { return max(get(v, 0), get(v, 1)); }
  // shift up by K virtual lanes inside a group of T threads: out[l] = v[l-K], 0 for l < K.
  // `sel` is this thread's PRMT selector for K (identity when t >= K).
  template <int T, int K>
  __device__ static __forceinline__ uint32_t shift(uint32_t v, int t, uint32_t gmask, uint32_t sel) {
    if constexpr (K == T) {
      return v << 16;
    } else {
      uint32_t r = __shfl_sync(gmask, v, (t - K) & (T - 1), T);
#if SWB_IMAD_SHIFT
      // the cell update saturates the ALU pipe; r * 65536 == r << 16 runs on the FMA pipe
      return mul_lo(r, sel);
#else
      return prmt(r, 0u, sel);
#endif
    }
  }
  // the same with the source lane precomputed (kept in a register by the caller)
  template <int T, int K>
  __device__ static __forceinline__ uint32_t shift_from(uint32_t v, int src, uint32_t gmask, uint32_t sel) {
    if constexpr (K == T) {
      return v << 16;
    } else {
      uint32_t r = __shfl_sync(gmask, v, src, T);
#if SWB_IMAD_SHIFT
      return mul_lo(r, sel);
#else
      return prmt(r, 0u, sel);
#endif
    }
  }
  __device__ static __forceinline__ uint32_t shift_sel(int t, int k) {
#if SWB_IMAD_SHIFT
    return t >= k ? 1u : 0x10000u;
#else
    return t >= k ? 0x3210u : 0x1044u;  // r<<16: bytes {0,0,r0,r1}
#endif
  }
  // scan shift: like shift, but source-less lanes keep their own value (bytes {v0,v1,r0,r1})
  template <int T, int K>
  __device__ static __forceinline__ uint32_t scan_shift(uint32_t v, int t, uint32_t gmask, uint32_t sel) {
    if constexpr (K == T) {
      return prmt(v, v, 0x1010u);  // {v.lo, v.lo}: low half keeps itself
    } else {
      uint32_t r = __shfl_sync(gmask, v, (t - K) & (T - 1), T);
      return prmt(r, v, sel);
    }
  }
  __device__ static __forceinline__ uint32_t scan_sel(int t, int k) {
    return t >= k ? 0x3210u : 0x1054u;
  }
  // shift by one lane with `in` entering lane 0 (thread 0, low half)
  template <int T>
  __device__ static __forceinline__ uint32_t shift_in(uint32_t v, uint32_t in, int t, uint32_t gmask,
                                                      uint32_t sel) {
    uint32_t r = __shfl_sync(gmask, v, (t - 1) & (T - 1), T);
    return prmt(r, in, sel);
  }
  __device__ static __forceinline__ uint32_t inject_sel(int t) { return t ? 0x3210u : 0x1054u; }
};

struct W32 {
  static constexpr int LPW = 1;
  static constexpr int NULLV = -(1 << 28);
  static constexpr int CLAMP = 1 << 29;
  __host__ __device__ static constexpr uint32_t splat(int v) { return (uint32_t)v; }
  __device__ static __forceinline__ uint32_t add(uint32_t a, uint32_t b) {
    return (uint32_t)((int)a + (int)b);
  }
  __device__ static __forceinline__ uint32_t vmax(uint32_t a, uint32_t b) {
    return (uint32_t)max((int)a, (int)b);
  }
  __device__ static __forceinline__ uint32_t addmax(uint32_t a, uint32_t b, uint32_t c) {
    return (uint32_t)__viaddmax_s32((int)a, (int)b, (int)c);
  }
  __device__ static __forceinline__ uint32_t addmax_relu(uint32_t a, uint32_t b, uint32_t c) {
    return (uint32_t)__viaddmax_s32_relu((int)a, (int)b, (int)c);
  }
  __device__ static __forceinline__ int get(uint32_t v, int) { return (int)v; }
  __device__ static __forceinline__ uint32_t pack(int lo, int) { return (uint32_t)lo; }
  __device__ static __forceinline__ int hmax(uint32_t v) { return (int)v; }
  template <int T, int K>
  __device__ static __forceinline__ uint32_t shift(uint32_t v, int t, uint32_t gmask, uint32_t) {
    static_assert(K < T, "32-bit lanes shift inside the group");
    uint32_t r = __shfl_sync(gmask, v, (t - K) & (T - 1), T);
    return t >= K ? r : 0u;
  }
  __device__ static __forceinline__ uint32_t shift_sel(int, int) { return 0u; }
  // scan shift: lanes t < K receive their own value (harmless in the max-plus step)
  template <int T, int K>
  __device__ static __forceinline__ uint32_t scan_shift(uint32_t v, int, uint32_t gmask, uint32_t) {
    static_assert(K < T, "32-bit lanes shift inside the group");
    return __shfl_up_sync(gmask, v, K, T);
  }
  __device__ static __forceinline__ uint32_t scan_sel(int, int) { return 0u; }
  template <int T>
  __device__ static __forceinline__ uint32_t shift_in(uint32_t v, uint32_t in, int t, uint32_t gmask,
                                                      uint32_t) {
    const uint32_t r = __shfl_up_sync(gmask, v, 1, T);
    return t ? r : in;
  }
  __device__ static __forceinline__ uint32_t inject_sel(int) { return 0u; }
};

__host__ __device__ constexpr int ceil_log2(int p) {
  int s = 0;
  while ((1 << s) < p) ++s;
  return s == 0 ? 1 : s;  // _scan_steps, src/_compiled.py:39-46
}

template <class Wd, int T>
struct Geo {
  static constexpr int P = T * Wd::LPW;  // virtual lanes per alignment
  static constexpr int STEPS = ceil_log2(P);
};

// ---- kernel arguments -----------------------------------------------------
struct SwArgs {
  // job description
  int64_t n_jobs;
  const int32_t* order;      // job slot -> job id (nullable: identity)
  int32_t mode;              // 0 = one shared query profile (DB), 1 = per-job query (pairs)
  int32_t early_exit;        // lazy-F: reference early exit (1) or all P passes (0)
  int32_t n_sym;             // alphabet size A (profile rows 0..A-1, row A = null residue)
  int32_t shared_L;          // DB mode: segment length of the shared profile
  int32_t shared_m;          // DB mode: query length
  const uint32_t* prof;      // DB mode: global profile [(A+1)][L][T] words
  // targets (reference sequences)
  const uint8_t* tgt;
  const int64_t* t_start;    // [n_jobs] start of job's target in tgt
  const int32_t* t_len;      // [n_jobs]
  // queries (pairs mode)
  const uint8_t* qry;
  const int64_t* q_start;
  const int32_t* q_len;
  // scoring
  const int8_t* sub;         // pairs mode shared matrix [A][A] (nullable when per-pair 4x4)
  const int32_t* pp_match;   // pairs mode per-job 4x4 match/mismatch/go/ge (nullable)
  const int32_t* pp_mismatch;
  const int32_t* pp_go;
  const int32_t* pp_ge;
  int32_t go, ge;            // uniform gaps
  int32_t bias;              // uniform bias (pairs mode with shared matrix / DB mode)
  int32_t max_sub;           // uniform max(0, max S)
  // outputs, indexed by job id
  int32_t* score;
  int32_t* ref_end;
  int32_t* query_end;
  uint8_t* flags;
  int32_t* col_passes;       // optional: per-column correction passes (job 0 only)
  int64_t* pass_stats;       // optional [n_jobs][2]: total lazy-F passes, early-exit columns
  const int64_t* n_jobs_dev; // optional device-side job count (overrides n_jobs; rescue launches)
  int32_t pair_stride;       // pairs mode: words per group profile slice ((A+1)*Lmax*T)
  int32_t* coord_floor;       // optional: locate end coordinates only for scores >= *floor
  int64_t floor_sample;       // > 0: raise *coord_floor to the floor_k-th best exact score
  int32_t floor_k;            //      of the first floor_sample jobs once they complete
  unsigned long long* task_ctr; // optional zeroed counters: [0] task claims, [1] sample tasks done
  uint32_t* floor_hist;       // zeroed [kFloorBins] histogram of the sample's scores
  const int32_t* arrived;     // streamed input: chunk c readable once arrived[c] >= epoch
  int64_t arrive_jobs;        // jobs per chunk
  int32_t arrive_epoch;
  int64_t arrive_timeout_ns;  // a chunk later than this aborts the feed (FLAG_FEED_TIMEOUT)
};
constexpr int kFloorBins = 4096;  // sample-score histogram bins (scores >= 4095 share the top bin)

// ---- the striped kernel -----------------------------------------------------
#define SWB_REP32(X)                                                                     \
  X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) \
  X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29)  \
  X(30) X(31)

#ifndef SWB_EXACT_MINB
#define SWB_EXACT_MINB 3  // CTAs of 128 threads per SM the exact kernels are register-capped for
#endif
#ifndef SWB_EXACT_LONG_BLOCK
#define SWB_EXACT_LONG_BLOCK 128  // threads per CTA of the database kernels over 32 words
#endif
#ifndef SWB_EXACT_LONG_MINB
#define SWB_EXACT_LONG_MINB 2  // the same for segments over 32 words
#endif
#ifndef SWB_OWN_GATE
#define SWB_OWN_GATE 1
#endif
#ifndef SWB_PACKED_GATE
#define SWB_PACKED_GATE 0  // measured slower (config 2 kernel 28.21 -> 28.53 ms, config 3 with coordinates 190 -> 201 ms)
#endif
#ifndef SWB_FUSE3
#define SWB_FUSE3 1  // 3-input deferred correction (see FUSE3 in the kernel)
#endif
#ifndef SWB_IMM_DECAY
#define SWB_IMM_DECAY 1
#endif
#ifndef SWB_MINB5_L
#define SWB_MINB5_L 0  // exact instances up to this many words register-capped for 5 CTAs per SM (19: config 3 126.0 -> 132.4 ms, off)
#endif
#ifndef SWB_BF_SNAP
#define SWB_BF_SNAP 0  // branch-free end-coordinate snapshots for segments of <= 32 words (config 3: coordinates 156.1 -> 150.6 ms but score-only 126.0 -> 127.3 ms: off)
#endif
#ifndef SWB_PIN_SHIFT
#define SWB_PIN_SHIFT 1
#endif
#ifndef SWB_PREF_D
#define SWB_PREF_D 0  // residue prefetch distance in columns (segments of <= 32 words); 0: the unroll factor
#endif
#ifndef SWB_PREF_D_LONG
#define SWB_PREF_D_LONG 1  // the same for longer segments (a column outlasts the load)
#endif
#ifndef SWB_RADIX_SCAN
#define SWB_RADIX_SCAN 0  // (measured: config 3 score-only 126.1 -> 128.5 ms, config 2 +0.2 %) T = 4: one round of independent shuffles + a max tree instead of 3 dependent steps
#endif
#ifndef SWB_FUSE3_CHAIN
#define SWB_FUSE3_CHAIN 4  // carry - j*ge: this many interleaved running adds down the words
#endif
#ifndef SWB_FUSE3_UNROLL
#define SWB_FUSE3_UNROLL 2
#endif
#ifndef SWB_FUSE3_MAXL
#define SWB_FUSE3_MAXL 32  // longest segment using it (3 state words per query word)
#endif
#ifndef SWB_FUSE3_PARTIAL
#define SWB_FUSE3_PARTIAL 38  // longer segments: the first N words use it (register budget)
#endif
#ifndef SWB_FUSE3_REGS
#define SWB_FUSE3_REGS 156  // state-word budget (2 per word + 1 per fused word)
#endif
#ifndef SWB_FUSE3_PARTIAL_UNROLL
#define SWB_FUSE3_PARTIAL_UNROLL 2
#endif
#ifndef SWB_COL_UNROLL
#define SWB_COL_UNROLL 1  // reference columns per loop iteration (unroll factor)
#endif
#ifndef SWB_COL_UNROLL_SHORT
#define SWB_COL_UNROLL_SHORT 1  // the same for exact instances of <= SWB_SHORT_L words
#endif
#ifndef SWB_SHORT_L
#define SWB_SHORT_L 24
#endif
#define SWB_PRAGMA(x) _Pragma(#x)
#define SWB_UNROLL(n) SWB_PRAGMA(unroll n)

template <class Wd, int T, int LMAX, int VAR, bool EXACT = false, int GE = 0>
__global__ void __launch_bounds__(EXACT ? (LMAX > 32 ? SWB_EXACT_LONG_BLOCK : 128) : 256,
                                  EXACT ? (LMAX > 32 ? SWB_EXACT_LONG_MINB
                                                     : LMAX <= SWB_MINB5_L ? 5 : SWB_EXACT_MINB) : 1)
sw_striped_kernel(const SwArgs a) {
  // GE > 0: gap-extend penalty known at compile time, so every decay constant
  // (j*ge, k*L*ge) is an immediate operand of VIADDMNMX instead of a register.
  // EXACT: LMAX is the segment length itself (uniform-L launches); the word
  // loop is straight-line code the scheduler can software-pipeline.
  static_assert(LMAX >= 1 && (LMAX <= 32 || (EXACT && LMAX <= 64)), "LMAX");
  static_assert(T >= 1 && T <= 32 && (T & (T - 1)) == 0, "T");
  static_assert(Wd::LPW == 2 || T >= 2, "32-bit lanes need T >= 2");
  constexpr int P = Geo<Wd, T>::P;
  constexpr int STEPS = Geo<Wd, T>::STEPS;
  constexpr int G = 32 / T;
  constexpr bool VEC = EXACT;          // vectorised [sym][L/4][T][4] profile layout
  constexpr int LP4 = (LMAX + 3) / 4;
  // With T = 4 a (sym, j4) block is 16 words = half the banks, and the two groups
  // of a quarter-warp LDS.128 phase read different symbols: blocks are placed at
  // 32-word granularity with the group parity selecting the half, so the phase
  // never conflicts (DB mode: two copies; pairs mode: two groups interleaved).
  // T = 2 likewise with GRP = 4 quarters (four groups per quarter-warp phase).
  constexpr int GRP = (VEC && T <= 4) ? 32 / (4 * T) : 1;
  constexpr bool DUP = GRP > 1;
  constexpr int BW = DUP ? 32 : T * 4;  // words per (sym, j4) block

  // FUSE3 (exact scan instances with a compile-time gap extend): the stored H of a
  // word, max(u, F), is only ever read by the next column's deferred correction
  // max(carry - j*ge, H).  Keeping u and the F that entered the word instead turns
  // those two ALU-pipe maxima into one 3-input maximum,
  //   vh = max3(carry - j*ge, u_old, F_old)            VIMNMX3  (ALU pipe)
  //   cj = cj - ge  (carry - j*ge, running down the words)  VIADD (FMA-lite pipe)
  // i.e. 4.5 ALU-pipe instructions per packed word instead of 5.5 (the ALU pipe is
  // the bound; the adds issue beside it), at the price of a third state word.
  constexpr bool FUSE3 = SWB_FUSE3 && VAR == VAR_SCAN && EXACT && GE > 0 && LMAX <= SWB_FUSE3_MAXL;
  // two columns per iteration let the register allocator rename u / F into the state
  // words instead of copying them (one IMAD.MOV per word and column otherwise)
  // longer segments fuse only their first KF words: a fused word keeps three state
  // registers (u, entering F, E), so 2*LMAX + KF stays inside the register file
  // (measured on config 2, L = 58: 24 / 30 / 36 / 42 / 57 fused words -> 27.77 / 27.48 /
  // 27.57 / 29.20 / 28.87 ms against 28.40 ms unfused; with two max accumulators
  // 30 / 34 / 36 / 38 / 40 -> 26.08 / 26.10 / 25.97 / 25.75 / 26.04 ms)
  constexpr int kFuseBudget = SWB_FUSE3_REGS - (T >= 16 ? 20 : 0) - 2 * LMAX -
                              (LMAX > 58 ? 2 * (LMAX - 58) + 4 : 0);  // (no spills up to 64 words)
  constexpr int kFuseWords = kFuseBudget < SWB_FUSE3_PARTIAL ? (kFuseBudget < 0 ? 0 : kFuseBudget) : SWB_FUSE3_PARTIAL;
  constexpr int KF = FUSE3 ? LMAX
                     : (SWB_FUSE3 && VAR == VAR_SCAN && EXACT && GE > 0) ? (kFuseWords < LMAX ? kFuseWords : LMAX - 1)
                                                                         : 0;  // words in the fused form
  // (wide groups with short segments are the single-pair shapes, one warp's latency:
  // config 1 at 16 stripes x 10 words runs 2.11 ms with two columns per iteration,
  // 1.91 ms with one)
  constexpr int kColUnroll = FUSE3 ? ((T >= 8 && LMAX <= 16) ? 1 : SWB_FUSE3_UNROLL) : KF > 0 ? SWB_FUSE3_PARTIAL_UNROLL
                                   : (EXACT && LMAX <= SWB_SHORT_L) ? SWB_COL_UNROLL_SHORT : SWB_COL_UNROLL;

  // a queue as deep as the unroll factor rotates by register renaming (no moves)
  // (runtime-L instances also serve single pairs, where one warp waits out every load: 4 ahead)
  constexpr int kPref = LMAX <= 32 ? (SWB_PREF_D > 0 ? SWB_PREF_D : EXACT ? kColUnroll : 4) : SWB_PREF_D_LONG;

  extern __shared__ uint32_t smem[];

  const int lane = threadIdx.x & 31;
  const int t = lane & (T - 1);
  const int gw = lane / T;
  const uint32_t gmask = (T == 32) ? 0xffffffffu : (((1u << T) - 1u) << (gw * T));
  const int warp_in_block = threadIdx.x >> 5;
  const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_in_block;
  const int64_t n_warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t n_jobs = a.n_jobs_dev ? *a.n_jobs_dev : a.n_jobs;
  const int64_t n_tasks = (n_jobs + G - 1) / G;
  const int A = a.n_sym;
  if ((int64_t)blockIdx.x * (blockDim.x >> 5) >= n_tasks) return;  // nothing for this block

  // shift selectors for K = 1, 2, 4, ... (16-bit packing only)
  uint32_t sel[6];
#pragma unroll
  for (int s = 0; s < 6; ++s) sel[s] = Wd::shift_sel(t, 1 << s);

  // Source lanes of the shifts.  With the exact kernels at the register limit ptxas
  // rebuilt these and the selectors from SR_TID inside the column loop (S2R + in-order
  // wait every iteration); pinned, they stay in registers.
  int srcl[6];
#pragma unroll
  for (int s = 0; s < 6; ++s) srcl[s] = (t - (1 << s)) & (T - 1);
  constexpr bool kPinShift = SWB_PIN_SHIFT && Wd::LPW == 2 && EXACT;
  if constexpr (kPinShift) {
#pragma unroll
    for (int s = 0; s < 6; ++s)
      if ((1 << s) < T) asm volatile("" : "+r"(sel[s]), "+r"(srcl[s]));
  }
#define SWB_SHIFT(K, S, v, mask)                                                   \
  (kPinShift ? W16::template shift_from<T, (K)>((v), srcl[S], (mask), sel[S])      \
             : Wd::template shift<T, (K)>((v), t, (mask), sel[S]))

  // radix scan (T = 4): selectors of the shifts by 3, 5, 6 and 7 lanes (multipliers)
  const uint32_t rsel3 = t >= 3 ? 1u : 0x10000u;
  const uint32_t hsel[2] = {t >= 1 ? 0x10000u : 0u, t >= 2 ? 0x10000u : 0u};
  const uint32_t hsel3 = t >= 3 ? 0x10000u : 0u;
  (void)rsel3; (void)hsel; (void)hsel3;

  // per-job constants
  int L = 0, first = 0, m = 0;
  uint32_t NGO = 0, NGE = 0, NWRAP = 0;
  uint32_t NJ[LMAX];
  uint32_t NKD[STEPS];
  int bias = a.bias, max_sub = a.max_sub;

  auto set_gaps = [&](int go, int ge_rt, int L_rt) {
    const int ge = GE > 0 ? GE : ge_rt;
    // exact instances: the segment length is LMAX (host-guaranteed), so with a
    // compile-time ge every decay is an immediate operand, not a register
    const int L_ = EXACT ? LMAX : L_rt;
    const int cl = Wd::CLAMP;
    NGO = Wd::splat(-min(go, cl));
    NGE = Wd::splat(-min(ge, cl));
    NWRAP = Wd::splat(-(int)min((int64_t)(L_ - 1) * ge, (int64_t)cl));
#pragma unroll
    for (int c = 0; c < LMAX; ++c) {
      int64_t j = c - (LMAX - L_);
      NJ[c] = Wd::splat(-(int)min((j < 0 ? 0 : j) * (int64_t)ge, (int64_t)cl));
    }
#pragma unroll
    for (int s = 0; s < STEPS; ++s)
      NKD[s] = Wd::splat(-(int)min((int64_t)(1 << s) * L_ * (int64_t)ge, (int64_t)cl));
  };

  const uint32_t* prof_base;  // this thread's profile column (word 0 of row 0)
  int LT;                     // words per profile row
  if (a.mode == 0) {
    // DB mode: one profile for the whole launch, staged in shared memory.
    L = EXACT ? LMAX : a.shared_L;
    m = a.shared_m;
    first = LMAX - L;
    LT = L * T;
    if constexpr (VEC) {
      // [(A+1)][L/4][copy][T][4]: a thread's 4 consecutive words are one 16-byte
      // LDS; a group reads 4*T contiguous words of its symbol row.
      const int words = (A + 1) * LP4 * BW;
      for (int w = threadIdx.x; w < words; w += blockDim.x) {
        const int k = w & 3, tt = (w >> 2) % T, j4 = (w / BW) % LP4, sym = w / (BW * LP4);
        const int j = 4 * j4 + k;
        smem[w] = j < L ? __ldg(a.prof + (sym * L + j) * T + tt) : 0u;
      }
      LT = LP4 * BW;
    } else {
      const int words = (A + 1) * LT;
      const uint4* src = reinterpret_cast<const uint4*>(a.prof);
      uint4* dst = reinterpret_cast<uint4*>(smem);
      for (int w = threadIdx.x; w < (words >> 2); w += blockDim.x) dst[w] = __ldg(src + w);
      for (int w = (words & ~3) + threadIdx.x; w < words; w += blockDim.x) smem[w] = __ldg(a.prof + w);
    }
    __syncthreads();
    set_gaps(a.go, a.ge, L);
    prof_base = VEC ? smem + 4 * t + (DUP ? 4 * T * (gw & (GRP - 1)) : 0) : smem + t - first * T;
  } else {
    LT = 0;
    prof_base = nullptr;
  }
  // pairs mode: the substitution matrix (int8 [A][A]) in the first kPairSubWords words,
  // then each group owns a slice of (A+1)*LMAX*T words
  uint32_t* const pbase = smem + (a.mode == 1 ? kPairSubWords : 0);
  const int8_t* const subs = reinterpret_cast<const int8_t*>(smem);
  // Exact pairs-mode instances keep ONE null-residue row per CTA behind the slices
  // (instead of one per group: 20 % less shared memory, a fifth CTA per SM for
  // 150-residue reads).  A slice unit is A rows of LP4*BW words, so from unit u the
  // shared row is row (units - u) * A: the thread's null symbol is that row index and
  // the row address needs no select.
  const int units = (int)(blockDim.x / T) / GRP;
  const int unit = ((int)(threadIdx.x >> 5) * G + gw) / GRP;
  if (a.mode == 1) {
    if (a.sub != nullptr) {
      int8_t* dst = reinterpret_cast<int8_t*>(smem);
      for (int w = threadIdx.x; w < A * A; w += blockDim.x) dst[w] = a.sub[w];
    }
    if constexpr (VEC) {
      uint32_t* nullrow = pbase + (size_t)units * GRP * (size_t)a.pair_stride;
      for (int w = threadIdx.x; w < LP4 * BW; w += blockDim.x)
        nullrow[w] = Wd::pack(Wd::NULLV, Wd::NULLV);
    }
    __syncthreads();
  }
  uint32_t* gslice =
      DUP ? pbase + (size_t)((threadIdx.x >> 5) * G + (gw & ~(GRP - 1))) * (size_t)a.pair_stride +
                4 * T * (gw & (GRP - 1))
          : pbase + (size_t)((threadIdx.x >> 5) * G + gw) * (size_t)a.pair_stride;

  // Coordinate floor (database top-k): end coordinates are located only for
  // alignments scoring >= *coord_floor, so the per-column gate compares against
  // the floor and the thread's own best -- no group reduction per column. A floor
  // of 0 (not yet raised by the sample) keeps the group-wide gate.
  // (exact scan instances only: the database-search kernels; elsewhere the floor
  // code would cost registers and every alignment gets its coordinates)
  const bool has_floor = EXACT && VAR == VAR_SCAN && a.coord_floor != nullptr;
  const bool no_coords = a.ref_end == nullptr && a.query_end == nullptr;
  const int64_t fs_tasks = (has_floor && a.task_ctr) ? min((a.floor_sample + G - 1) / G, n_tasks) : 0;
#ifndef SWB_KCH
#define SWB_KCH 0  // 0: by segment length (see kCh)
#endif
  // chunk of the running column maxima (a position search scans one chunk):
  // 16 words for the long exact segments (fewer maxima to combine per column)
  // End coordinates: a thread whose column maximum beats the alignment's best so
  // far stores the column's words (its snapshot) to shared memory -- LMAX
  // STS.32 -- and the first word reaching the final best is located once, from
  // the last snapshot, when the alignment ends (the best only grows, so the last
  // snapshot holds the column of the final best). Searching in registers at every
  // improvement (planted reads improve on most columns) cost the warp ~70 issue
  // slots per improving column; SWB_SNAP=0 restores it (chunked column maxima).
#ifndef SWB_SNAP
#define SWB_SNAP 1
#endif
  constexpr bool SNAP = SWB_SNAP;
  constexpr int SNW = LMAX | 1;  // snapshot words per thread (odd: rows spread over the banks)
  // (chunked column maxima also with SNAP: independent accumulators, short chains)
  constexpr int kCh = SWB_KCH > 0 ? SWB_KCH : (EXACT && LMAX > 32 ? 32 : 8);  // (config 2: 8 / 16 / 20 / 32 / 64 words per accumulator: 26.77 / 26.66 / 26.17 / 26.09 / 26.30 ms)
  constexpr int kNch = (LMAX + kCh - 1) / kCh;
  // end-coordinate snapshots: SNW words per thread after the profile / the slices
  const int prof_w = a.mode == 0 ? (VEC ? (A + 1) * LP4 * BW : (A + 1) * L * T)
                                 : (int)(blockDim.x / T) * a.pair_stride + (VEC ? LP4 * BW : 0);
  uint32_t* const snap = pbase + (prof_w + 3) / 4 * 4 + threadIdx.x * SNW;
  (void)snap;

  // Task claiming: with a counter, warps take the next task (in length-descending
  // order) when they finish one -- longest-first greedy, so the warps end together
  // instead of the static stride leaving the warps that drew the longest targets
  // of every round running alone at the end. The next claim is issued at the top
  // of each task so the atomic's latency hides behind the alignment.
  auto claim = [&]() -> int64_t {
    unsigned long long v = 0;
    if (lane == 0) v = atomicAdd(a.task_ctr, 1ull);
    return (int64_t)v;
  };
  int64_t task = a.task_ctr ? (int64_t)__shfl_sync(0xffffffffu, (unsigned long long)claim(), 0)
                            : warp_global;
  while (task < n_tasks) {
    const int64_t pref = a.task_ctr ? claim() : task + n_warps;
    const int64_t slot = task * G + gw;
    const bool valid = slot < n_jobs;
    const int64_t job = valid ? (a.order ? (int64_t)a.order[slot] : slot) : 0;
    // Streamed input: wait until the chunk holding this task's jobs has arrived
    // (chunks arrive in order, so the latest chunk needed is the only one to check).
    // Target data is read through L2 (ld.cg) so no L1 line fetched before its
    // chunk arrived can be reused.
    // (every lane waits for its own job's chunk: no warp collective here, which
    // would raise the register allocation of the whole kernel)
    // A chunk that has not arrived after arrive_timeout_ns (globaltimer) -- e.g. the
    // copy engine never ran concurrently with this kernel (profilers, serialised
    // launches) -- raises the launch's abort word (task_ctr[2]); every waiting or
    // later task then gives up at once and reports FLAG_FEED_TIMEOUT, and the host
    // re-runs exactly those jobs once the copies are done (search_streamed): the
    // feed can be slow, never wrong.
    bool feed_ok = true;
    if (a.arrived && valid) {
      const int32_t* flag = a.arrived + job / a.arrive_jobs;
      if (ld_acquire_s32(flag) < a.arrive_epoch) {
        volatile unsigned long long* abort_w = a.task_ctr + 2;
        const uint64_t t0 = globaltimer_ns();
        while (ld_acquire_s32(flag) < a.arrive_epoch) {
          __nanosleep(512);
          if (*abort_w != 0ull) { feed_ok = false; break; }
          if (globaltimer_ns() - t0 > (uint64_t)a.arrive_timeout_ns) {
            atomicExch(a.task_ctr + 2, 1ull);
            feed_ok = false;
            break;
          }
        }
      }
    }
    const int len = (valid && feed_ok) ? __ldcg(a.t_len + job) : 0;
    const uint8_t* tp = a.tgt + ((valid && feed_ok) ? __ldcg(a.t_start + job) : 0);
    // keep the pointer itself in registers: left to itself ptxas re-adds the base from
    // the constant bank every column (LDC + 3-input add), and the in-order wait on that
    // LDC costs a single-warp launch ~50 cycles per column
    asm volatile("" : "+l"(tp));

    if (a.mode == 1) {
      // ---- per-job query profile (pairs mode) ----
      m = valid ? a.q_len[job] : 0;
      L = (m + P - 1) / P;
      if (L < 1) L = 1;
      first = LMAX - L;
      int go = a.go, ge = a.ge;
      int mt = 0, mm = 0;
      const bool pp = a.pp_match != nullptr;
      if (pp && valid) {
        mt = a.pp_match[job]; mm = a.pp_mismatch[job]; go = a.pp_go[job]; ge = a.pp_ge[job];
        bias = max(0, -min(mt, mm));
        max_sub = max(0, max(mt, mm));
      }
      set_gaps(go, ge, L);
      const uint8_t* qp = a.qry + (valid ? a.q_start[job] : 0);
      LT = L * T;
      if constexpr (VEC) {
        // Four word positions at a time: the thread's 8 query residues (two halves) are
        // read once, then every symbol's four words are filled from them with the
        // matrix in shared memory and stored as one 128-bit word -- the query is not
        // re-read per symbol and no global load sits inside the symbol loop.
        for (int j4 = 0; j4 < LP4; ++j4) {
          uint32_t cl = 0u, ch = 0u;  // 4 residue codes per half, 0xff = pad
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int j = 4 * j4 + k;
            const int q0 = t * L + j, q1 = (T + t) * L + j;
            const uint32_t c0 = (j < L && q0 < m) ? (uint32_t)qp[q0] : 0xffu;
            const uint32_t c1 = (Wd::LPW == 2 && j < L && q1 < m) ? (uint32_t)qp[q1] : 0xffu;
            cl |= c0 << (8 * k);
            ch |= c1 << (8 * k);
          }
          for (int sym = 0; sym < A; ++sym) {  // (the null row is shared, see above)
            const int8_t* srow = subs + sym * A;
            uint32_t wv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              int v[2] = {0, 0};
#pragma unroll
              for (int h = 0; h < Wd::LPW; ++h) {
                const int qs = (int)(((h ? ch : cl) >> (8 * k)) & 0xffu);
                int sv;
                if (qs == 0xff) sv = -bias;  // reference pad: profile 0 == -bias (src/profile.py:60-63)
                else sv = pp ? (qs == sym ? mt : mm) : (int)srow[qs & 31];
                v[h] = sv;
              }
              wv[k] = Wd::pack(v[0], v[1]);
            }
            *reinterpret_cast<uint4*>(gslice + (sym * LP4 + j4) * BW + t * 4) =
                make_uint4(wv[0], wv[1], wv[2], wv[3]);
          }
        }
      } else {
        for (int sym = 0; sym <= A; ++sym) {
          for (int j = 0; j < L; ++j) {
            int v[2];
#pragma unroll
            for (int h = 0; h < Wd::LPW; ++h) {
              const int q = (h * T + t) * L + j;
              int sv;
              if (sym == A) sv = Wd::NULLV;
              else if (q >= m) sv = -bias;  // reference pad: profile 0 == -bias (src/profile.py:60-63)
              else {
                const int qs = qp[q];
                sv = pp ? (qs == sym ? mt : mm) : (int)subs[sym * A + qs];
              }
              v[h] = sv;
            }
            gslice[(sym * L + j) * T + t] = Wd::pack(v[0], v[1]);
          }
        }
      }
      if constexpr (VEC) LT = LP4 * BW;
      prof_base = VEC ? gslice + 4 * t : gslice + t - first * T;
    }
    const int maxlen = __reduce_max_sync(0xffffffffu, len);

    // ---- alignment state ----
    uint32_t H[LMAX], E[LMAX];
#pragma unroll
    for (int c = 0; c < LMAX; ++c) { H[c] = 0u; E[c] = 0u; }
    uint32_t Fs[KF > 0 ? KF : 1];  // fused words: the F entering the word (H[] then holds u)
#pragma unroll
    for (int c = 0; c < (KF > 0 ? KF : 1); ++c) Fs[c] = 0u;
    uint32_t carry = 0u;
    int64_t tot_passes = 0, breaks = 0;  // lazy-F statistics (reference op counters)
    // best of all earlier columns: group-wide, or (floor mode) own best and floor - 1;
    // the floor is re-read per task, as a sample-complete warp may have raised it
    int floor_v = 0;
    if (has_floor) {
      if (lane == 0) floor_v = *(volatile const int32_t*)a.coord_floor;
      floor_v = __shfl_sync(0xffffffffu, floor_v, 0);
    }
    // per-thread gate (own best): no group reduction per column; with snapshots a
    // thread records its own first maximum and the group reduction at the end
    // picks the alignment's (SWB_OWN_GATE)
    const bool floor_mode = floor_v > 0 || (SNAP && SWB_OWN_GATE);
    // score-only launches (no coordinate outputs) never search: the gate never opens
    int gb = no_coords ? 0x7fffffff : floor_mode ? floor_v - 1 : 0;
    // packed copy of the per-thread gate level (each half: floor - 1 and the half's own best)
    constexpr bool kPackedGate = SWB_PACKED_GATE && SNAP && SWB_OWN_GATE;
    uint32_t gbp = Wd::splat(min(max(gb, 0), Wd::LPW == 2 ? 32767 : 0x7fffffff));
    (void)gbp;
    int bv = 0, bcol = -1, bq = -1;   // this thread's first-maximum record
    int bh = 0;                       // SNAP: the half (lane) holding bv
    // running maxima of u per chunk of kCh words (never reset: a chunk reaches a
    // value above gb only in the column that first produces it)
    uint32_t cmk[kNch];
#pragma unroll
    for (int k = 0; k < kNch; ++k) cmk[k] = 0u;
    const int nullsym = (VEC && a.mode == 1) ? (units - unit) * A : A;
    // residues are fetched kPref columns ahead (a byte queue in registers): with short
    // segments a column is shorter than an L2 round trip, and the profile row address
    // (sym * LT) stalled on the load issued one column earlier (long-scoreboard stalls)
    int nq[kPref];
#pragma unroll
    for (int d = 0; d < kPref; ++d) nq[d] = (d < len) ? (int)__ldcg(tp + d) : nullsym;

#pragma unroll kColUnroll
    for (int i = 0; i < maxlen; ++i) {
      const int sym = nq[0];
#pragma unroll
      for (int d = 0; d + 1 < kPref; ++d) nq[d] = nq[d + 1];
      nq[kPref - 1] = (i + kPref < len) ? (int)__ldcg(tp + i + kPref) : nullsym;
      const uint32_t* pr = prof_base + sym * LT;
      uint4 S4[VEC ? LP4 : 1];
      if constexpr (VEC) {
#pragma unroll
        for (int k = 0; k < LP4; ++k) S4[k] = *reinterpret_cast<const uint4*>(pr + k * BW);
      }

      // scan path: the whole warp is converged here, so shuffles take the full
      // mask (width T keeps the data inside the group) and skip the runtime
      // convergence checks a sub-warp mask costs; lazy-F passes diverge per group.
      constexpr bool kConverged = VAR == VAR_SCAN;
      const uint32_t cmask = kConverged ? 0xffffffffu : gmask;
      uint32_t w = H[LMAX - 1];
      if constexpr (FUSE3) w = Wd::vmax(Wd::vmax(Wd::add(carry, NWRAP), w), Fs[LMAX - 1]);
      else if constexpr (VAR == VAR_SCAN) w = Wd::addmax(carry, NWRAP, w);
      uint32_t vh = SWB_SHIFT(1, 0, w, cmask);
      uint32_t F = 0u;
      // fused words: carry - j*ge for the word being read, as kCjS interleaved running
      // adds (each value feeds a maximum and the next add, which keeps ptxas from folding
      // the add back into a VIADDMNMX; one chain would put L dependent adds behind the scan)
      constexpr int kCjS = SWB_FUSE3_CHAIN;
      const uint32_t NSGE = Wd::splat(-(GE > 0 ? GE : 1) * kCjS);
      uint32_t cjs[kCjS];
#pragma unroll
      for (int k = 0; k < kCjS; ++k) cjs[k] = (k == 0 || KF == 0) ? carry : Wd::add(carry, NJ[k < LMAX ? k : 0]);

      // max(x - ge, y, 0): the E / F decay
      // (compile-time ge: a fresh single-use constant per call, so ptxas folds it into the
      // instruction as an immediate instead of holding it in a register -- a third
      // register source can collide in the register-file banks)
      auto decay_relu = [&](uint32_t x, uint32_t y) -> uint32_t {
        if constexpr (GE > 0 && SWB_IMM_DECAY) {
          uint32_t k;
          asm volatile("mov.b32 %0, %1;" : "=r"(k) : "n"(Wd::splat(-GE)));
          return Wd::addmax_relu(x, k, y);
        } else {
          return Wd::addmax_relu(x, NGE, y);
        }
      };
#define SWB_WORD_BODY(C)                                                   \
  if ((C) < KF) {                                                          \
    const uint32_t S = w4(S4[VEC ? (C) / 4 : 0], (C) & 3);                 \
    const uint32_t u = Wd::addmax(vh, S, E[C]);                            \
    const uint32_t Xu = Wd::add(u, NGO);                                   \
    E[C] = decay_relu(E[C], Xu);                                           \
    vh = Wd::vmax(Wd::vmax(cjs[(C) % kCjS], H[C]), Fs[C]);                  \
    cjs[(C) % kCjS] = Wd::add(cjs[(C) % kCjS], NSGE);                      \
    H[C] = u;                                                              \
    Fs[C] = F;                                                             \
    F = decay_relu(F, Xu);                                                 \
    cmk[(C) / kCh] = Wd::vmax(cmk[(C) / kCh], u);                          \
  } else {                                                                 \
    const uint32_t S = VEC ? w4(S4[VEC ? (C) / 4 : 0], (C) & 3) : pr[(C) * T]; \
    const uint32_t u = Wd::addmax(vh, S, E[C]);                            \
    const uint32_t Hn = Wd::vmax(u, F);                                    \
    const uint32_t Xu = Wd::add(u, NGO);                                   \
    if constexpr (VAR == VAR_LAZYF_MIRROR)                                 \
      E[C] = Wd::addmax_relu(E[C], NGE, Wd::add(Hn, NGO));                 \
    else                                                                   \
      E[C] = decay_relu(E[C], Xu);                                         \
    F = decay_relu(F, Xu);                                                 \
    cmk[(C) / kCh] = Wd::vmax(cmk[(C) / kCh], u);                          \
    if constexpr (VAR == VAR_SCAN) vh = Wd::addmax(carry, NJ[C], H[C]);    \
    else vh = H[C];                                                        \
    H[C] = Hn;                                                             \
  }
#define SWB_WORD(C)                                                        \
  case C:                                                                  \
    if constexpr ((C) < LMAX) SWB_WORD_BODY(C)                             \
    [[fallthrough]];

      if constexpr (EXACT) {
#pragma unroll
        for (int c = 0; c < LMAX; ++c) SWB_WORD_BODY(c)
      } else {
        switch (first) {
          SWB_REP32(SWB_WORD)
          default: break;
        }
      }
#undef SWB_WORD
#undef SWB_WORD_BODY

      // ---- end coordinates --------------------------------------------------
      // The first cell (reference-major order) reaching the final best must
      // exceed every value of the earlier columns, so only columns whose max
      // beats the group's running best `gb` need the position search (rare:
      // the alignment's best grows a few dozen times, not per lane-column).
      // A cell attaining the best is a diagonal cell, so its stored H equals
      // u; the first word with H >= cm is the first such cell in the lane.
      // score-only launches (no coordinate outputs: a launch-uniform branch) skip the
      // gate entirely -- the chunk maxima already hold the score. Segments of up to
      // 32 words only (pair batches): for the long database segments the extra
      // branch cost more than the gate it skips (config 2 kernel -3 %).
      if (!(LMAX <= 32 && no_coords)) {
        uint32_t cm = cmk[0];
#pragma unroll
        for (int k = 1; k < kNch; ++k) cm = Wd::vmax(cm, cmk[k]);
        // packed gate: the running maxima never decrease, so a column raises a half's
        // best exactly when max(cm, gbp) != gbp -- one packed max and one compare on
        // the common path instead of unpack + scalar max + compare + scalar max
        bool gate_open = true;
        if constexpr (kPackedGate) {
          const uint32_t g2 = Wd::vmax(cm, gbp);
          gate_open = g2 != gbp;
          gbp = g2;
        }
        if (gate_open) {
        const int cmx = Wd::hmax(cm);
        if constexpr (SNAP && SWB_BF_SNAP && LMAX <= 32 && Wd::LPW == 2) {
          // short segments (pair batches): on planted reads some thread of the warp improves
          // in almost every column, so the snapshot runs branch-free -- selects for the
          // record and LMAX predicated stores instead of a divergent region
          const int lo = Wd::get(cm, 0), hi = Wd::get(cm, 1);
          const bool up = cmx > gb && cmx > bv;
          bv = up ? cmx : bv;
          bcol = up ? i : bcol;
          bh = up ? (hi > lo ? 1 : 0) : bh;
          const uint32_t sa = (uint32_t)__cvta_generic_to_shared(snap);
#pragma unroll
          for (int c = 0; c < LMAX; ++c)
            asm volatile("{.reg .pred q; setp.ne.u32 q, %2, 0; @q st.shared.b32 [%0], %1;}" ::"r"(sa + 4 * c),
                         "r"(H[c]), "r"((uint32_t)up) : "memory");
        } else if (SNAP && cmx > gb) {
          bool now = false;
#pragma unroll
          for (int h = 0; h < Wd::LPW; ++h) {
            const int cv = Wd::get(cm, h);
            if (cv > gb && cv > bv) { bv = cv; bcol = i; bh = h; now = true; }
          }
          if (now) {
            // one STS.32 per word at immediate offsets (odd row stride: few bank
            // conflicts); a 128-bit store would need H in aligned register quads,
            // which costs ~45 moves per column
#pragma unroll
            for (int c = 0; c < LMAX; ++c) snap[c] = H[c];
          }
        } else if (!SNAP && cmx > gb) {
#pragma unroll
          for (int h = 0; h < Wd::LPW; ++h) {
            const int cv = Wd::get(cm, h);
            if (cv > gb && cv > bv) {
              // the first chunk reaching cv holds the first cell reaching it
              int kk = 0;
#pragma unroll
              for (int k = kNch - 1; k >= 0; --k)
                if (Wd::get(cmk[k], h) >= cv) kk = k;
              int jj;
              if constexpr (EXACT) {
                // gather the chunk's words without branching on kk, then search them
                int jo = kCh;
#pragma unroll
                for (int j = kCh - 1; j >= 0; --j) {
                  uint32_t w = 0u;
#pragma unroll
                  for (int k = 0; k < kNch; ++k)
                    if (k * kCh + j < LMAX) w = (k == kk) ? H[k * kCh + j] : w;
                  if (Wd::get(w, h) >= cv) jo = j;  // unused / padding words hold 0 < cv
                }
                jj = kk * kCh + jo;
              } else {
                jj = first;
#pragma unroll
                for (int k = 0; k < kNch; ++k) {
                  if (k == kk) {
#pragma unroll
                    for (int c = (k + 1) * kCh - 1; c >= k * kCh; --c)
                      if (c < LMAX && c >= first && Wd::get(H[c], h) >= cv) jj = c;
                  }
                }
              }
              bv = cv;
              bcol = i;
              bq = (h * T + t) * L + (jj - first);
            }
          }
        }
        if (floor_mode) {
          gb = max(gb, cmx);
        } else {
          int g = max(gb, cmx);
#pragma unroll
          for (int off = T / 2; off >= 1; off >>= 1) g = max(g, __shfl_xor_sync(cmask, g, off, T));
          gb = g;
        }
        }
      }

      // ---- cross-lane F dependency ----
      if constexpr (VAR == VAR_SCAN && SWB_RADIX_SCAN && T == 4 && Wd::LPW == 2 && SWB_IMAD_SHIFT) {
        // 8 stripes in 4 threads: the same weighted scan (src/_compiled.py:320-336) as one
        // round of three independent shuffles of F itself instead of three dependent
        // shuffle steps: carry[l] = relu(max_{k=1..7} F[l-k] - (k-1) d), the seven shifted
        // copies (k and k+4 lanes from each shuffle, k = 4 from the word itself) combined
        // by a depth-3 tree -- three more maxima per column, half the latency from F to
        // the carry every word of the next column waits for.
        const uint32_t r1 = __shfl_sync(cmask, F, (t - 1) & 3, 4);
        const uint32_t r2 = __shfl_sync(cmask, F, (t - 2) & 3, 4);
        const uint32_t r3 = __shfl_sync(cmask, F, (t - 3) & 3, 4);
        const uint32_t s1 = mul_lo(r1, sel[0]), s5 = mul_lo(r1, hsel[0]);  // shifts by 1 and 5 lanes
        const uint32_t s2 = mul_lo(r2, sel[1]), s6 = mul_lo(r2, hsel[1]);  // 2 and 6
        const uint32_t s3 = mul_lo(r3, rsel3), s7 = mul_lo(r3, hsel3);     // 3 and 7
        const uint32_t s4 = F << 16;                                        // 4
        const uint32_t t1 = Wd::addmax(s2, NKD[0], s1);
        const uint32_t t2 = Wd::addmax(s4, NKD[0], s3);
        const uint32_t t3 = Wd::addmax(s6, NKD[0], s5);
        const uint32_t u1 = Wd::addmax(t2, NKD[1], t1);
        const uint32_t u2 = Wd::addmax(s7, NKD[1], t3);
        carry = Wd::addmax_relu(u2, NKD[2], u1);
      } else if constexpr (VAR == VAR_SCAN) {
        uint32_t acc = SWB_SHIFT(1, 0, F, cmask);
        // Alg. 6 weighted max-scan, k = 1, 2, 4, ... (src/_compiled.py:320-336)
#define SWB_STEP(S)                                                                         \
  if constexpr ((S) < STEPS) {                                                             \
    acc = Wd::addmax_relu(SWB_SHIFT((1 << (S)), S, acc, cmask), NKD[S], acc);                \
  }
        SWB_STEP(0) SWB_STEP(1) SWB_STEP(2) SWB_STEP(3) SWB_STEP(4) SWB_STEP(5)
#undef SWB_STEP
        carry = acc;
      } else {
        // lazy-F (src/_compiled.py:189-217): shift, optional all-zero exit, correct, repeat
        uint32_t vf = F;
        int passes = 0;
        for (int it = 0; it < P; ++it) {
          vf = Wd::template shift<T, 1>(vf, t, gmask, sel[0]);
          if (a.early_exit) {
            if ((__ballot_sync(gmask, vf != 0u) & gmask) == 0u) break;
          }
#define SWB_FIX_BODY(C)                      \
  {                                          \
    H[C] = Wd::vmax(H[C], vf);               \
    vf = Wd::addmax_relu(vf, NGE, NGE);      \
  }
#define SWB_FIX(C)                           \
  case C:                                    \
    if constexpr ((C) < LMAX) SWB_FIX_BODY(C) \
    [[fallthrough]];
          if constexpr (EXACT) {
#pragma unroll
            for (int c = 0; c < LMAX; ++c) SWB_FIX_BODY(c)
          } else {
            switch (first) {
              SWB_REP32(SWB_FIX)
              default: break;
            }
          }
#undef SWB_FIX
#undef SWB_FIX_BODY
          ++passes;
        }
        if (a.col_passes != nullptr && job == 0 && valid && t == 0 && i < len)
          a.col_passes[i] = passes;
        if (i < len) {
          tot_passes += passes;
          breaks += (a.early_exit && passes < P) ? 1 : 0;
        }
      }
    }

    if (SNAP && bcol >= 0) {
      // the first word of the snapshot column reaching bv (a diagonal cell: H == u)
      int jj = LMAX - 1;
      for (int c = LMAX - 1; c >= first; --c)
        if (Wd::get(snap[c], bh) >= bv) jj = c;
      bq = (bh * T + t) * L + (jj - first);
    }
    // ---- reduce (best desc, ref_end asc, query_end asc) over the group ----
    int best = bv, col = bcol, q = bq;
    int sc;  // the score: the running maximum (equals best unless the floor skipped it)
    {
      uint32_t cm = cmk[0];
#pragma unroll
      for (int k = 1; k < kNch; ++k) cm = Wd::vmax(cm, cmk[k]);
      sc = Wd::hmax(cm);
    }
#pragma unroll
    for (int off = T / 2; off >= 1; off >>= 1) {
      sc = max(sc, __shfl_xor_sync(gmask, sc, off, T));
      const int ob = __shfl_xor_sync(gmask, best, off, T);
      const int oc = __shfl_xor_sync(gmask, col, off, T);
      const int oq = __shfl_xor_sync(gmask, q, off, T);
      if (ob > best || (ob == best && (oc < col || (oc == col && oq < q)))) {
        best = ob; col = oc; q = oq;
      }
    }
    if (valid && t == 0) {
      uint8_t fl = 0;
      if constexpr (Wd::LPW == 2) {
        if (sc >= 32767 - max_sub) fl |= FLAG_RESCUE;
      }
      if (sc > 65535 - bias) fl |= FLAG_REF_OVERFLOW;
      // device-counted 32-bit launches are the overflow rescue passes (a 16-bit
      // device-counted launch re-runs jobs whose streamed input timed out)
      if (a.n_jobs_dev && Wd::LPW == 1) fl |= FLAG_RESCUED;
      if (!feed_ok) fl |= FLAG_FEED_TIMEOUT;
      if (sc == 0) { col = -1; q = -1; }
      else if (best != sc) { col = -2; q = -2; }  // below the coordinate floor: not located
      a.score[job] = sc;
      if (a.pass_stats) {
        a.pass_stats[2 * job] = tot_passes;
        a.pass_stats[2 * job + 1] = breaks;
      }
      if (a.ref_end) a.ref_end[job] = col;
      if (a.query_end) a.query_end[job] = q;
      if (a.flags) a.flags[job] = fl;
      if (task < fs_tasks)  // sample histogram (16-bit rescue candidates count as 0)
        atomicAdd(a.floor_hist + min((fl & FLAG_RESCUE) ? 0 : sc, kFloorBins - 1), 1u);
    }
    if (task < fs_tasks) {
      // the warp completing the last sample task sets the floor: the floor_k-th best
      // exact score of the sample (capped at kFloorBins-1), a lower bound of the
      // final k-th best, so every possible top-k hit is located
      __threadfence();
      __syncwarp();
      unsigned long long done = 0;
      if (lane == 0) done = atomicAdd(a.task_ctr + 1, 1ull);
      done = __shfl_sync(0xffffffffu, done, 0);
      if ((int64_t)done == fs_tasks - 1) {
        __threadfence();
        // one lane scans the histogram from the top, 32 bins per step (warp
        // collectives here would raise the register allocation of the whole kernel)
        int floor_v = 0;
        if (lane == 0) {
          const uint4* h4 = reinterpret_cast<const uint4*>(a.floor_hist);
          int acc = 0;
          for (int q = kFloorBins / 4 - 8; q >= 0; q -= 8) {
            uint4 v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = __ldcg(h4 + q + j);
            int tot = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) tot += (int)(v[j].x + v[j].y + v[j].z + v[j].w);
            if (acc + tot >= a.floor_k) {
              int f = -1;  // the highest bin at which the count from the top reaches k
#pragma unroll
              for (int j = 7; j >= 0; --j) {
                const int c[4] = {(int)v[j].x, (int)v[j].y, (int)v[j].z, (int)v[j].w};
#pragma unroll
                for (int e = 3; e >= 0; --e) {
                  acc += c[e];
                  if (acc >= a.floor_k && f < 0) f = 4 * (q + j) + e;
                }
              }
              floor_v = f;
              break;
            }
            acc += tot;
          }
        }
        if (lane == 0) atomicMax(a.coord_floor, floor_v);
      }
    }
    task = a.task_ctr ? (int64_t)__shfl_sync(0xffffffffu, (unsigned long long)pref, 0) : pref;
  }
}

// ---- DB-mode profile builder: prof[(A+1)][L][T] words ------------------------
// word (a, j, t) packs lanes t and T+t (16-bit) or lane t (32-bit):
// S[a][query[l*L + j]] for in-range positions, -bias for pads (the reference's
// profile value 0 minus the bias, src/profile.py:54-64), NULLV for the null row.
template <class Wd, int T>
__global__ void sw_profile_kernel(const uint8_t* __restrict__ query, int m, const int8_t* __restrict__ sub,
                                  int A, int L, int bias, uint32_t* __restrict__ prof) {
  const int words = (A + 1) * L * T;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
    const int t = w % T;
    const int j = (w / T) % L;
    const int sym = w / (T * L);
    int v[2] = {0, 0};
#pragma unroll
    for (int h = 0; h < Wd::LPW; ++h) {
      const int q = (h * T + t) * L + j;
      if (sym == A) v[h] = Wd::NULLV;
      else if (q >= m) v[h] = -bias;
      else v[h] = sub[sym * A + query[q]];
    }
    prof[w] = Wd::pack(v[0], v[1]);
  }
}

// ---- device weighted max-scan (unit-test entry for the scan device function) ----
// f: [n][P] uint16 lanes -> out: [n][P], one group of T threads per vector,
// bit-equal to _weighted_max_scan_c (src/_compiled.py:448-460).
template <class Wd, int T>
__global__ void sw_scan_test_kernel(const uint16_t* __restrict__ f, const int32_t* __restrict__ d,
                                    int n, uint16_t* __restrict__ out) {
  constexpr int P = Geo<Wd, T>::P;
  constexpr int STEPS = Geo<Wd, T>::STEPS;
  constexpr int G = 32 / T;
  const int lane = threadIdx.x & 31, t = lane & (T - 1), gw = lane / T;
  const uint32_t gmask = (T == 32) ? 0xffffffffu : (((1u << T) - 1u) << (gw * T));
  const int vec = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * G + gw;
  const bool ok = vec < n;
  const int v = ok ? vec : 0;
  uint32_t sel[6];
#pragma unroll
  for (int s = 0; s < 6; ++s) sel[s] = Wd::shift_sel(t, 1 << s);
  // values are uint16 in the reference; the device scan runs on the signed
  // representation with every decay clamped to the score range.
  const int lo = f[(size_t)v * P + t];
  const int hi = (Wd::LPW == 2) ? f[(size_t)v * P + T + t] : 0;
  uint32_t acc = Wd::pack(lo, hi);
  acc = Wd::template shift<T, 1>(acc, t, gmask, sel[0]);
  const int64_t dd = d[v];
#define SWB_TSTEP(S)                                                                        \
  if constexpr ((S) < STEPS) {                                                             \
    const uint32_t nk = Wd::splat(-(int)min((int64_t)(1 << (S)) * dd, (int64_t)Wd::CLAMP)); \
    acc = Wd::addmax_relu(Wd::template shift<T, (1 << (S))>(acc, t, gmask, sel[S]), nk, acc); \
  }
  SWB_TSTEP(0) SWB_TSTEP(1) SWB_TSTEP(2) SWB_TSTEP(3) SWB_TSTEP(4) SWB_TSTEP(5)
#undef SWB_TSTEP
  if (ok) {
    out[(size_t)v * P + t] = (uint16_t)Wd::get(acc, 0);
    if (Wd::LPW == 2) out[(size_t)v * P + T + t] = (uint16_t)Wd::get(acc, 1);
  }
}

}  // namespace swb

namespace swb {
// gather ids of jobs whose flags intersect `mask` (rescue list)
__global__ void sw_collect_kernel(const uint8_t* __restrict__ flags, int64_t n, uint8_t mask,
                                  int32_t* __restrict__ list, unsigned long long* __restrict__ count);
}  // namespace swb

namespace swb {
// gather ids of jobs whose flags intersect `mask` (rescue list); count is a device int64
__global__ void sw_collect_kernel(const uint8_t* __restrict__ flags, int64_t n, uint8_t mask,
                                  int32_t* __restrict__ list, unsigned long long* __restrict__ count);

// kernel table: [width 0=16,1=32][variant 0..2][log2 T 0..5][lmax idx 0..2]
constexpr int kNumT = 6;
constexpr int kNumLmax = 3;
constexpr int kLmaxSet[kNumLmax] = {8, 16, 32};
using KernelTable = const void* [kNumT][kNumLmax];
}  // namespace swb

void swb_fill_w16_scan(swb::KernelTable& t);
void swb_fill_w16_lazyf(swb::KernelTable& t);
void swb_fill_w16_mirror(swb::KernelTable& t);
void swb_fill_w32_scan(swb::KernelTable& t);
void swb_fill_w32_lazyf(swb::KernelTable& t);
void swb_fill_w32_mirror(swb::KernelTable& t);

// exact-L instances (uniform segment length): [ge specialisation 0=runtime,1,2][log2 T][L]
namespace swb {
constexpr int kNumGe = 3;
constexpr int kExactLmax = 64;
using ExactTable = const void* [kNumGe][kNumT][kExactLmax + 1];
}
#define SWB_X_DECL(T, GE, PART) void swb_fill_exact_t##T##_g##GE##_##PART(swb::ExactTable& t);
SWB_X_DECL(8, 0, a) SWB_X_DECL(8, 0, b) SWB_X_DECL(8, 1, a) SWB_X_DECL(8, 1, b)
SWB_X_DECL(8, 2, a) SWB_X_DECL(8, 2, b) SWB_X_DECL(16, 0, b) SWB_X_DECL(16, 1, b)
SWB_X_DECL(16, 2, b) SWB_X_DECL(32, 0, b) SWB_X_DECL(32, 1, b) SWB_X_DECL(32, 2, b) SWB_X_DECL(4, 0, b) SWB_X_DECL(4, 1, b) SWB_X_DECL(4, 2, b)
SWB_X_DECL(4, 0, a) SWB_X_DECL(4, 1, a) SWB_X_DECL(4, 2, a)
SWB_X_DECL(4, 0, c) SWB_X_DECL(4, 1, c) SWB_X_DECL(4, 2, c)
SWB_X_DECL(4, 0, d) SWB_X_DECL(4, 1, d) SWB_X_DECL(4, 2, d)
SWB_X_DECL(4, 0, e) SWB_X_DECL(4, 1, e) SWB_X_DECL(4, 2, e)
SWB_X_DECL(4, 0, f) SWB_X_DECL(4, 1, f) SWB_X_DECL(4, 2, f)
SWB_X_DECL(16, 0, c) SWB_X_DECL(16, 1, c) SWB_X_DECL(16, 2, c)
SWB_X_DECL(32, 0, c) SWB_X_DECL(32, 1, c) SWB_X_DECL(32, 2, c)
SWB_X_DECL(2, 0, c) SWB_X_DECL(2, 1, c) SWB_X_DECL(2, 2, c)
#undef SWB_X_DECL
void swb_fill_chain(const void* (&tab)[2][6], const void* (&ptab)[2], const void* (&so)[6]);
void swb_fill_chain_g1(const void* (&tab)[6], const void* (&so)[6]);
void swb_fill_wave(const void* (&tab)[4][4]);
void swb_fill_wave_g1(const void* (&tab)[4][4]);
void swb_fill_block16(const void* (&tab)[3][16]);
void swb_fill_block32(const void* (&tab)[3][16]);
