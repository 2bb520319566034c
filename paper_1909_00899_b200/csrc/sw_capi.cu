// sw_capi.cu -- extern "C" entry points of libswscan_b200.so (see include/swscan_b200.h).
//
// Host-side responsibilities: choose the striped layout, pick the kernel
// instance from the table, size the persistent grid from the occupancy API,
// and launch on the caller's stream.  No allocation, no synchronisation.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <utility>

#include "sw_chain.cuh"
#include "sw_block.cuh"
#include "../../include/swscan_b200.h"

using namespace swb;

#ifndef SWB_CHAIN_SPLIT_SO
#define SWB_CHAIN_SPLIT_SO 1
#endif

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(SW_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

KernelTable g_tab[2][3];
ExactTable g_exact;  // 16-bit scan, exact segment length
const void* g_chain[2][6];  // strip pipeline [width][L = 1, 2, 4, 8, 16, 32]
const void* g_chain_so[6];  // 32-bit score-only strips [L]
#ifndef SWB_CHAIN_GE1
#define SWB_CHAIN_GE1 1  // 32-bit strips: instances with gap extend 1 as a compile-time constant
#endif
const void* g_chain_g1[6];     // 32-bit strips, gap extend 1 as a compile-time constant
const void* g_chain_so_g1[6];
const void* g_chain_prof[2];
const void* g_wave[4][4];  // [L = 1, 2, 4, 8][KC = 1, 2, 4, 8]
const void* g_wave_g1[4][4];  // the same with gap extend 1 as a compile-time constant
const void* g_block[2][3][16];  // block / cluster scan [width][variant][L-1]  // strip pipeline, intra-strip wavefront [L = 1, 2, 4, 8]
std::once_flag g_once;

void init_tables() {
  std::memset(g_tab, 0, sizeof g_tab);
  std::memset(g_exact, 0, sizeof g_exact);
  swb_fill_exact_t8_g0_a(g_exact); swb_fill_exact_t8_g0_b(g_exact);
  swb_fill_exact_t8_g1_a(g_exact); swb_fill_exact_t8_g1_b(g_exact);
  swb_fill_exact_t8_g2_a(g_exact); swb_fill_exact_t8_g2_b(g_exact);
  swb_fill_exact_t16_g0_b(g_exact); swb_fill_exact_t16_g1_b(g_exact); swb_fill_exact_t16_g2_b(g_exact);
  swb_fill_exact_t32_g0_b(g_exact); swb_fill_exact_t32_g1_b(g_exact); swb_fill_exact_t32_g2_b(g_exact);
  // 33..64 words at 32/64 stripes: database queries up to 4,096 residues
  swb_fill_exact_t16_g0_c(g_exact); swb_fill_exact_t16_g1_c(g_exact); swb_fill_exact_t16_g2_c(g_exact);
  swb_fill_exact_t32_g0_c(g_exact); swb_fill_exact_t32_g1_c(g_exact); swb_fill_exact_t32_g2_c(g_exact);
  swb_fill_exact_t4_g0_b(g_exact); swb_fill_exact_t4_g1_b(g_exact); swb_fill_exact_t4_g2_b(g_exact);
  swb_fill_exact_t4_g0_a(g_exact); swb_fill_exact_t4_g1_a(g_exact); swb_fill_exact_t4_g2_a(g_exact);
  swb_fill_exact_t4_g0_c(g_exact); swb_fill_exact_t4_g1_c(g_exact); swb_fill_exact_t4_g2_c(g_exact);
  swb_fill_exact_t4_g0_d(g_exact); swb_fill_exact_t4_g1_d(g_exact); swb_fill_exact_t4_g2_d(g_exact);
  swb_fill_exact_t4_g0_e(g_exact); swb_fill_exact_t4_g1_e(g_exact); swb_fill_exact_t4_g2_e(g_exact);
  swb_fill_exact_t4_g0_f(g_exact); swb_fill_exact_t4_g1_f(g_exact); swb_fill_exact_t4_g2_f(g_exact);
  // T = 2 (4 stripes): 33..40 words, pair batches of ~150-residue reads at lanes = 4
  swb_fill_exact_t2_g0_c(g_exact); swb_fill_exact_t2_g1_c(g_exact); swb_fill_exact_t2_g2_c(g_exact);
  swb_fill_chain(g_chain, g_chain_prof, g_chain_so);
  swb_fill_chain_g1(g_chain_g1, g_chain_so_g1);
  swb_fill_wave(g_wave);
  swb_fill_wave_g1(g_wave_g1);
  swb_fill_block16(g_block[0]);
  swb_fill_block32(g_block[1]);
  swb_fill_w16_scan(g_tab[0][VAR_SCAN]);
  swb_fill_w16_lazyf(g_tab[0][VAR_LAZYF]);
  swb_fill_w16_mirror(g_tab[0][VAR_LAZYF_MIRROR]);
  swb_fill_w32_scan(g_tab[1][VAR_SCAN]);
  swb_fill_w32_lazyf(g_tab[1][VAR_LAZYF]);
  swb_fill_w32_mirror(g_tab[1][VAR_LAZYF_MIRROR]);
}

int ilog2(int x) {
  int s = 0;
  while ((1 << s) < x) ++s;
  return s;
}

bool pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

// ---- block / cluster kernel geometry ----
struct BlockGeo {
  int lanes, nt, cl, L;
  size_t smem;
};
int block_max_threads(int L) { return L <= 4 ? 1024 : (L <= 8 ? 512 : 256); }
size_t block_smem(int A, int L, int nt) {
  return (size_t)(A + 1) * L * nt * 4 + 64 * 16 + (kBlockRing + 2) * 8 + 32 * 16;
}
constexpr size_t kMaxDynSmem = 227 * 1024;
// layout for `lanes` stripes (a power of two): CTAs per cluster doubled until a CTA
// fits the thread and shared-memory limits; lazy-F needs a single CTA
bool block_geo_for(int width, bool scan, int64_t m, int A, int lanes, BlockGeo* g) {
  const int lpw = width == 16 ? 2 : 1;
  if (!pow2(lanes) || lanes < 32 * lpw) return false;
  const int64_t L = (m + lanes - 1) / lanes;
  if (L < 1 || L > 16) return false;
  const int T = lanes / lpw;
  int cl = 1;
  while (cl <= 16 && (T / cl > block_max_threads((int)L) || block_smem(A, (int)L, T / cl) > kMaxDynSmem)) cl *= 2;
  if (cl > 16 || T / cl < 32 || (!scan && cl > 1)) return false;
  g->lanes = lanes; g->nt = T / cl; g->cl = cl; g->L = (int)L;
  g->smem = block_smem(A, (int)L, g->nt);
  return true;
}
// lanes = 0: scan -- the fewest stripes with segments of <= 4 words (more threads cost
// the per-column scan little; longer segments cost every column), else <= 16;
// lazy-F -- the fewest stripes that fit one CTA (every pass shifts F by one lane)
bool block_geo(int width, bool scan, int64_t m, int A, int lanes, BlockGeo* g) {
  if (lanes) return block_geo_for(width, scan, m, A, lanes, g);
  const int lpw = width == 16 ? 2 : 1;
  for (int lmax : {4, 16})
    for (int p = 32 * lpw; p <= 16 * 1024 * lpw; p *= 2)
      if ((m + p - 1) / p <= (scan ? lmax : 16) && block_geo_for(width, scan, m, A, p, g)) return true;
  return false;
}

int lmax_index(int L) {
  for (int i = 0; i < kNumLmax; ++i)
    if (L <= kLmaxSet[i]) return i;
  return -1;
}

// kernel id -> (variant, early_exit)
bool decode_kernel(int kernel, int* var, int* early_exit) {
  switch (kernel) {
    case SW_KERNEL_LAZYF: *var = VAR_LAZYF; *early_exit = 1; return true;
    case SW_KERNEL_LAZYF_NOEXIT: *var = VAR_LAZYF; *early_exit = 0; return true;
    case SW_KERNEL_SCAN: *var = VAR_SCAN; *early_exit = 0; return true;
    case SW_KERNEL_LAZYF_MIRROR: *var = VAR_LAZYF_MIRROR; *early_exit = 1; return true;
    case SW_KERNEL_LAZYF_NOEXIT_MIRROR: *var = VAR_LAZYF_MIRROR; *early_exit = 0; return true;
    default: return false;
  }
}

// Layout choice.  The throughput layout keeps L near the register budget so
// the per-column shuffle/scan overhead (~log2 P shuffles) is amortised over
// many cells; `lanes` > 0 reproduces the reference's VectorSpec(p) exactly.
int plan(int m, int n_sym, int width, int lanes, sw_plan_t* out) {
  if (width != 16 && width != 32) return fail(SW_EINVAL, "width must be 16 or 32, got %d", width);
  if (m < 0) return fail(SW_EINVAL, "query length must be >= 0");
  if (n_sym < 1 || n_sym > kMaxSym) return fail(SW_ENOTSUP, "alphabet size %d outside 1..%d", n_sym, kMaxSym);
  const int lpw = width == 16 ? 2 : 1;
  int P;
  if (lanes > 0) {
    if (!pow2(lanes)) return fail(SW_EINVAL, "lanes must be a power of two, got %d", lanes);
    if (lanes / lpw < (width == 32 ? 2 : 1) || lanes / lpw > 32)
      return fail(SW_ENOTSUP, "lanes %d outside the warp kernels' range for width %d", lanes, width);
    P = lanes;
  } else {
    // smallest P whose segment fits 32 register words (longer segments amortise the
    // per-column scan): 8 stripes (4 threads, 8 alignments per warp) in 16-bit,
    // measured +16 % over 16 stripes on config 3 (150-residue reads).
    // Segments beyond the runtime-L kernels' 32 words exist only as exact 16-bit
    // scan instances (register-resident, 2 CTAs/SM); the auto layout takes them
    // when they exist (SWB_PLAN_MAX_L caps the segment length for experiments).
    std::call_once(g_once, init_tables);
    int cap = kExactLmax;
    if (const char* e = getenv("SWB_PLAN_MAX_L")) cap = atoi(e);
    P = 32 * lpw;
    for (int PP = 8; PP <= 32 * lpw; PP *= 2) {
      const int LL = (m + PP - 1) / PP;
      if (LL <= kLmaxSet[kNumLmax - 1] && LL <= cap) { P = PP; break; }
      if (width == 16 && LL <= cap && LL <= kExactLmax && g_exact[0][ilog2(PP / lpw)][LL]) {
        P = PP;
        break;
      }
    }
  }
  const int T = P / lpw;
  int L = (m + P - 1) / P;
  if (L < 1) L = 1;
  int li = lmax_index(L);
  if (li < 0 && !(L <= kExactLmax && width == 16 && g_exact[0][ilog2(T)][L]))
    return fail(SW_ENOTSUP, "query length %d needs %d words per lane at %d lanes (max %d)", m, L, P,
                kLmaxSet[kNumLmax - 1]);
  out->width = width;
  out->lanes = P;
  out->threads = T;
  out->seg_len = L;
  out->lmax = li >= 0 ? kLmaxSet[li] : L;  // lmax > 32: exact-instance-only plan
  out->m = m;
  out->n_sym = n_sym;
  out->prof_words = (n_sym + 1) * L * T;
  return SW_OK;
}

// Task counters for dynamic task claiming (SwArgs::task_ctr: [0] task claims,
// [1] sample tasks done, [2] streamed-input abort word) and the coordinate-floor
// sample histogram: one slot = a 128-byte counter line + kFloorBins words.  Every
// (device, stream) pair owns its own slot, allocated on first use: launches on one
// stream run in order (each zeroes the slot on that stream before it runs), and
// launches on different streams never share a slot, however many are in flight.
// (A stream handle that is destroyed and re-created while its last launch still
// runs would share the slot; destroy streams only after their work completed.)
constexpr size_t kSlotBytes = 128 + kFloorBins * 4;
constexpr int64_t kDefaultArriveTimeoutNs = 2000000000ll;  // 2 s per chunk wait
std::mutex g_ctr_mu;
std::map<std::pair<int, cudaStream_t>, char*> g_ctr_slots;

cudaError_t task_counter(cudaStream_t stream, bool hist, unsigned long long** out,
                         uint32_t** hist_out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  char* slot = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ctr_mu);
    auto it = g_ctr_slots.find({dev, stream});
    if (it == g_ctr_slots.end()) {
      e = cudaMalloc((void**)&slot, kSlotBytes);
      if (e != cudaSuccess) return e;
      g_ctr_slots[{dev, stream}] = slot;
    } else {
      slot = it->second;
    }
  }
  e = cudaMemsetAsync(slot, 0, hist ? kSlotBytes : 128, stream);
  *out = (unsigned long long*)slot;
  *hist_out = (uint32_t*)(slot + 128);
  return e;
}

int launch(const void* fn, const SwArgs& args_in, size_t smem, int block, int64_t n_tasks_hint,
           cudaStream_t stream) {
  cudaError_t e;
  SwArgs args = args_in;
  e = task_counter(stream, args.floor_sample > 0, &args.task_ctr, &args.floor_hist);
  if (e != cudaSuccess) return cuda_fail(e, "task counter");
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(smem)");
  }
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, block, smem);
  if (e != cudaSuccess) return cuda_fail(e, "occupancy");
  if (occ < 1) return fail(SW_ENOTSUP, "kernel does not fit on an SM (smem %zu B)", smem);
  int64_t grid = (int64_t)sms * occ;
  const int64_t warps_per_block = block / 32;
  if (n_tasks_hint > 0) {
    const int64_t need = (n_tasks_hint + warps_per_block - 1) / warps_per_block;
    if (need < grid) grid = need;
  }
  if (grid < 1) grid = 1;
  void* params[] = {(void*)&args};
  e = cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(block), params, smem, stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernel(sw_striped_kernel)");
  return SW_OK;
}

}  // namespace

namespace swb {
__global__ void sw_collect_kernel(const uint8_t* __restrict__ flags, int64_t n, uint8_t mask,
                                  int32_t* __restrict__ list, unsigned long long* __restrict__ count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool hit = (flags[i] & mask) != 0;
    const unsigned ballot = __ballot_sync(__activemask(), hit);
    if (ballot == 0) continue;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(ballot) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(count, (unsigned long long)__popc(ballot));
    base = __shfl_sync(__activemask(), base, leader);
    if (hit) list[base + __popc(ballot & ((1u << lane) - 1u))] = (int32_t)i;
  }
}
}  // namespace swb

namespace swb {
// DPX issue-rate probe: 8 independent dependency chains per thread so the
// measurement is throughput- (not latency-) bound.  kind 0: VIADDMNMX.S16x2
// only; kind 1: the cell-update mix of sw_striped_kernel (per word: 2 ADDMNMX.RELU,
// 2 ADDMNMX, 1 IMNMX, 1 IADD.16x2; 6 instructions).
__global__ void sw_dpx_probe_kernel(int kind, int64_t iters, uint32_t* out) {
  uint32_t x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 2654435761u + k;
  const uint32_t b = 0xfffefffeu, c = 0x00030003u;
  if (kind == 0) {
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = __viaddmax_s16x2(x[k], b, c);
    }
  } else {
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        uint32_t u = __viaddmax_s16x2(x[k], b, x[k + 1]);
        uint32_t h = __vmaxs2(u, x[k]);
        uint32_t xu = __vadd2(u, b);
        x[k + 1] = __viaddmax_s16x2_relu(x[k + 1], c, xu);
        x[k] = __viaddmax_s16x2_relu(h, b, xu);
        x[k + 1] = __viaddmax_s16x2(x[k + 1], c, h);
      }
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) r ^= x[k];
  if (r == 0x12345678u) out[threadIdx.x] = r;  // keep the chains live
}
}  // namespace swb

extern "C" {

int32_t sw_version(void) { return 1; }

int64_t sw_dpx_probe(int32_t kind, int64_t iters, uint32_t* d_scratch, sw_stream_t stream) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int block = 256, grid = sms * 8;
  sw_dpx_probe_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(kind, iters, d_scratch);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "sw_dpx_probe_kernel");
  const int64_t per_iter = kind == 0 ? 8 : 24;  // DPX instructions per thread per iteration
  return (int64_t)grid * block * iters * per_iter;
}

const char* sw_last_error(void) { return g_err; }

int32_t sw_plan_query(int32_t m, int32_t n_sym, int32_t width, int32_t lanes, sw_plan_t* out) {
  if (!out) return fail(SW_EINVAL, "out is NULL");
  return plan(m, n_sym, width, lanes, out);
}

int32_t sw_profile_build(const sw_plan_t* p, const uint8_t* d_query, const int8_t* d_sub,
                         int32_t bias, uint32_t* d_prof, sw_stream_t stream) {
  if (!p || !d_prof || !d_sub || (p->m > 0 && !d_query)) return fail(SW_EINVAL, "NULL argument");
  const int words = p->prof_words;
  const int block = 256;
  const int grid = (words + block - 1) / block;
  cudaStream_t s = (cudaStream_t)stream;
  const int T = p->threads;
  if (p->width == 16) {
    switch (T) {
#define CASE(TT) case TT: sw_profile_kernel<W16, TT><<<grid, block, 0, s>>>(d_query, p->m, d_sub, p->n_sym, p->seg_len, bias, d_prof); break;
      CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32)
#undef CASE
      default: return fail(SW_EINVAL, "bad plan threads %d", T);
    }
  } else {
    switch (T) {
#define CASE(TT) case TT: sw_profile_kernel<W32, TT><<<grid, block, 0, s>>>(d_query, p->m, d_sub, p->n_sym, p->seg_len, bias, d_prof); break;
      CASE(2) CASE(4) CASE(8) CASE(16) CASE(32)
#undef CASE
      default: return fail(SW_EINVAL, "bad plan threads %d", T);
    }
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SW_OK : cuda_fail(e, "sw_profile_kernel");
}

int32_t sw_db_align(const sw_plan_t* p, const uint32_t* d_prof, int32_t kernel, int32_t gap_open,
                    int32_t gap_extend, int32_t bias, int32_t max_sub, const uint8_t* d_tgt,
                    const int64_t* d_start, const int32_t* d_len, const int32_t* d_order, int64_t n,
                    const int64_t* d_n_jobs, int32_t* d_score, int32_t* d_ref_end,
                    int32_t* d_query_end, uint8_t* d_flags, int32_t* d_col_passes,
                    int64_t* d_pass_stats, const sw_db_opts_t* opts, sw_stream_t stream) {
  std::call_once(g_once, init_tables);
  if (!p || !d_prof || !d_tgt || !d_start || !d_len || !d_score)
    return fail(SW_EINVAL, "NULL argument");
  if (n < 0) return fail(SW_EINVAL, "n < 0");
  if (!(gap_open >= gap_extend && gap_extend >= 1))
    return fail(SW_EINVAL, "require gap_open >= gap_extend >= 1");
  if (n == 0 && !d_n_jobs) return SW_OK;
  int var, early;
  if (!decode_kernel(kernel, &var, &early)) return fail(SW_EINVAL, "unknown kernel %d", kernel);
  const int wi = p->width == 16 ? 0 : 1;
  const int li = lmax_index(p->lmax);
  if (li >= 0 && kLmaxSet[li] != p->lmax) return fail(SW_EINVAL, "bad plan lmax %d", p->lmax);
  if (li < 0 && !(wi == 0 && var == VAR_SCAN))
    return fail(SW_ENOTSUP, "segment length %d only has exact 16-bit scan kernels", p->seg_len);
  const void* fn = nullptr;
  int block = 256;
  if (wi == 0 && var == VAR_SCAN) {
    const int gi = (gap_extend == 1 || gap_extend == 2) ? gap_extend : 0;
    fn = g_exact[gi][ilog2(p->threads)][p->seg_len];
    if (fn) block = p->seg_len > 32 ? SWB_EXACT_LONG_BLOCK : 128;
  }
  if (!fn && li >= 0) fn = g_tab[wi][var][ilog2(p->threads)][li];
  if (!fn) return fail(SW_ENOTSUP, "no kernel for width %d, threads %d", p->width, p->threads);
  SwArgs a;
  std::memset(&a, 0, sizeof a);
  a.n_jobs = n;
  a.n_jobs_dev = d_n_jobs;
  a.order = d_order;
  a.mode = 0;
  a.early_exit = early;
  a.n_sym = p->n_sym;
  a.shared_L = p->seg_len;
  a.shared_m = p->m;
  a.prof = d_prof;
  a.tgt = d_tgt;
  a.t_start = d_start;
  a.t_len = d_len;
  a.go = gap_open;
  a.ge = gap_extend;
  a.bias = bias;
  a.max_sub = max_sub;
  a.score = d_score;
  a.ref_end = d_ref_end;
  a.query_end = d_query_end;
  a.flags = d_flags;
  a.col_passes = d_col_passes;
  a.pass_stats = d_pass_stats;
  if (opts) {
    if (opts->floor_sample > 0 && (!opts->d_coord_floor || opts->floor_k < 1))
      return fail(SW_EINVAL, "floor_sample needs d_coord_floor and floor_k >= 1");
    if (opts->arrive_epoch > 0 && (!opts->d_arrived || opts->arrive_jobs < 1))
      return fail(SW_EINVAL, "arrive_epoch needs d_arrived and arrive_jobs >= 1");
    a.coord_floor = opts->d_coord_floor;
    a.floor_sample = opts->floor_sample;
    a.floor_k = opts->floor_k;
    if (opts->arrive_epoch > 0) {
      a.arrived = opts->d_arrived;
      a.arrive_jobs = opts->arrive_jobs;
      a.arrive_epoch = opts->arrive_epoch;
      a.arrive_timeout_ns =
          opts->arrive_timeout_ns > 0 ? opts->arrive_timeout_ns : kDefaultArriveTimeoutNs;
    }
  }
  // exact instances stage the profile as [sym][ceil(L/4)][T][4]
  // (T = 4: two copies at 32-word block granularity, see DUP in sw_kernels.cuh)
  const size_t prof_bytes = block != 256 ? (size_t)(p->n_sym + 1) * ((p->seg_len + 3) / 4 * 4) * p->threads *
                                               4 * (p->threads <= 4 ? 8 / p->threads : 1)
                                         : (size_t)p->prof_words * 4;
  // + the end-coordinate snapshots (SWB_SNAP): LMAX words per thread, only when
  // coordinates are requested (score-only launches keep their occupancy)
  const int lmax_k = block != 256 ? p->seg_len : p->lmax;
  const bool snap = SWB_SNAP && (d_ref_end || d_query_end);
  const size_t smem = (prof_bytes + 15) / 16 * 16 + (snap ? (size_t)block * (lmax_k | 1) * 4 : 0);
  const int G = 32 / p->threads;
  const int64_t tasks = d_n_jobs ? 0 : (n + G - 1) / G;
  return launch(fn, a, smem, block, tasks, (cudaStream_t)stream);
}

int32_t sw_pairs_align(int32_t width, int32_t lanes, int32_t kernel, const uint8_t* d_qry,
                       const int64_t* d_qstart, const int32_t* d_qlen, const uint8_t* d_tgt,
                       const int64_t* d_tstart, const int32_t* d_tlen, const int32_t* d_order,
                       int64_t n, const int64_t* d_n_jobs, int32_t min_qlen, int32_t max_qlen,
                       const int8_t* d_sub,
                       int32_t n_sym, int32_t gap_open, int32_t gap_extend, int32_t bias,
                       int32_t max_sub, const int32_t* d_match, const int32_t* d_mismatch,
                       const int32_t* d_go, const int32_t* d_ge, int32_t* d_score,
                       int32_t* d_ref_end, int32_t* d_query_end, uint8_t* d_flags,
                       int32_t* d_col_passes, int64_t* d_pass_stats, sw_stream_t stream) {
  std::call_once(g_once, init_tables);
  if (!d_qry || !d_qstart || !d_qlen || !d_tgt || !d_tstart || !d_tlen || !d_score)
    return fail(SW_EINVAL, "NULL argument");
  const bool per_pair = d_sub == nullptr;
  if (per_pair && (!d_match || !d_mismatch || !d_go || !d_ge))
    return fail(SW_EINVAL, "per-pair schemes need d_match, d_mismatch, d_go and d_ge");
  if (per_pair) n_sym = 4;
  if (!per_pair && !(gap_open >= gap_extend && gap_extend >= 1))
    return fail(SW_EINVAL, "require gap_open >= gap_extend >= 1");
  if (n < 0) return fail(SW_EINVAL, "n < 0");
  if (n == 0 && !d_n_jobs) return SW_OK;
  int var, early;
  if (!decode_kernel(kernel, &var, &early)) return fail(SW_EINVAL, "unknown kernel %d", kernel);
  sw_plan_t p;
  int rc = plan(max_qlen, n_sym, width, lanes, &p);
  if (rc) return rc;
  if (lmax_index(p.lmax) < 0) {
    // long segments exist only as exact scan instances: other kernels and mixed
    // segment lengths take the smallest stripe count with <= 32 words instead
    const bool uniform = min_qlen > 0 && (min_qlen + p.lanes - 1) / p.lanes == p.seg_len;
    if (var != VAR_SCAN || !uniform || per_pair) {
      int P = 8;
      while ((max_qlen + P - 1) / P > kLmaxSet[kNumLmax - 1]) P *= 2;
      rc = plan(max_qlen, n_sym, width, P, &p);
      if (rc) return rc;
    }
  }
  const int wi = width == 16 ? 0 : 1;
  const void* fn = nullptr;
  // every query of the batch has the same segment length: exact-L instance
  const bool uniform_L = min_qlen > 0 && (min_qlen + p.lanes - 1) / p.lanes == p.seg_len;
  int max_block = 256;
  if (wi == 0 && var == VAR_SCAN && uniform_L && !per_pair) {
    const int gi = (gap_extend == 1 || gap_extend == 2) ? gap_extend : 0;
    fn = g_exact[gi][ilog2(p.threads)][p.seg_len];
    if (fn) max_block = 128;
  }
  if (!fn && lmax_index(p.lmax) >= 0) fn = g_tab[wi][var][ilog2(p.threads)][lmax_index(p.lmax)];
  if (!fn) return fail(SW_ENOTSUP, "no kernel for width %d, threads %d", width, p.threads);
  SwArgs a;
  std::memset(&a, 0, sizeof a);
  a.n_jobs = n;
  a.n_jobs_dev = d_n_jobs;
  a.order = d_order;
  a.mode = 1;
  a.early_exit = early;
  a.n_sym = n_sym;
  a.tgt = d_tgt;
  a.t_start = d_tstart;
  a.t_len = d_tlen;
  a.qry = d_qry;
  a.q_start = d_qstart;
  a.q_len = d_qlen;
  a.sub = d_sub;
  a.pp_match = per_pair ? d_match : nullptr;
  a.pp_mismatch = per_pair ? d_mismatch : nullptr;
  a.pp_go = per_pair ? d_go : nullptr;
  a.pp_ge = per_pair ? d_ge : nullptr;
  a.go = gap_open;
  a.ge = gap_extend;
  a.bias = bias;
  a.max_sub = max_sub;
  a.score = d_score;
  a.ref_end = d_ref_end;
  a.query_end = d_query_end;
  a.flags = d_flags;
  a.col_passes = d_col_passes;
  a.pass_stats = d_pass_stats;
  const bool vec = max_block == 128;  // exact instance: vectorised profile layout
  const int lslice = vec ? (p.seg_len + 3) / 4 * 4 : p.seg_len;
  // exact instances: A rows per group slice + one shared null-residue row per CTA
  const int rows = vec ? n_sym : n_sym + 1;
  a.pair_stride = rows * lslice * p.threads;
  // block size: as many warps as the per-group profile slices allow (<= 256 threads)
  int block = max_block;
  // slice bytes / T, + the end-coordinate snapshot of the thread (SWB_SNAP)
  const int lmax_k = vec ? p.seg_len : p.lmax;
  const bool snap = SWB_SNAP && (d_ref_end || d_query_end);  // score-only: no snapshots
  const size_t per_thread =
      (size_t)rows * lslice * 4 + (snap ? (size_t)(lmax_k | 1) * 4 : 0);
  while (block > 32 && per_thread * block > 110 * 1024) block >>= 1;
  // + the staged matrix, + the shared null row ([ceil(L/4)][32 or 4T] words)
  const size_t null_bytes = vec ? (size_t)(lslice / 4) * (p.threads <= 4 ? 32 : p.threads * 4) * 4 : 0;
  const size_t smem = per_thread * block + kPairSubWords * 4 + null_bytes;
  if (smem > 227 * 1024) return fail(SW_ENOTSUP, "pair profile slice too large (%zu B)", smem);
  const int G = 32 / p.threads;
  const int64_t tasks = d_n_jobs ? 0 : (n + G - 1) / G;
  return launch(fn, a, smem, block, tasks, (cudaStream_t)stream);
}

// strip-pipeline geometry: per-column latency model t(L) ~ 190 + 5 L cycles,
// total ~ (n + nb*K) * t(L); prefer the smallest total.
struct ChainGeo {
  int li, L, nb;
  int ki = 0, KC = 1;  // wavefront: columns per step (index into 1, 2, 4, 8)
  size_t prof_words, ring_bytes, total;
};

static ChainGeo chain_geo(int64_t m, int64_t n, int n_sym, int width) {
  const int lpw = width == 16 ? 2 : 1;
  static const int Ls[6] = {1, 2, 4, 8, 16, 32};
  ChainGeo g{};
  double best = 1e300;
  // measured per-column latency (cycles, 32-bit, B200) of one strip alone and of a
  // strip in a full pipeline (~3.5 strips per SM); tools/chain_latency.py
  static const double lat_alone16[6] = {315, 323, 356, 404, 486, 670};
  static const double lat_loaded16[6] = {380, 366, 386, 431, 511, 700};
  // 32-bit carry-split strips (sw_chain32.cuh), profiles/r02j_chain_latency.txt
  static const double lat_alone32[6] = {215, 209, 211, 277, 386, 670};
  static const double lat_loaded32[6] = {240, 232, 240, 312, 448, 700};
  const double* lat_alone = width == 32 ? lat_alone32 : lat_alone16;
  const double* lat_loaded = width == 32 ? lat_loaded32 : lat_loaded16;
  for (int li = 0; li < 6; ++li) {
    const int L = Ls[li];
    const int64_t rows = 32LL * lpw * L;
    const int64_t nb = (m + rows - 1) / rows;
    const double load = nb >= 518 ? 1.0 : (double)nb / 518.0;
    const double lat = lat_alone[li] + load * (lat_loaded[li] - lat_alone[li]);
    // every strip must be co-resident (cooperative launch): keep well inside
    // 148 SMs x 16 one-warp CTAs unless no strip height fits
    // a strip trails by ~2 tiles (32-bit: ~3, it starts two tiles behind, sw_chain32.cuh)
    double cost = (double)(n + nb * (width == 32 ? 3 : 2) * kChainK) * lat;
    if (nb > 148 * 16 && li < 5) cost *= 1e6;
    if (cost < best) {
      best = cost;
      g.li = li; g.L = L; g.nb = (int)(nb < 1 ? 1 : nb);
    }
  }
  if (const char* force = getenv("SWB_CHAIN_L")) {  // debugging / tuning override
    const int L = atoi(force);
    for (int li = 0; li < 6; ++li)
      if (Ls[li] == L) {
        const int64_t rows = 32LL * lpw * L;
        g.li = li; g.L = L; g.nb = (int)((m + rows - 1) / rows);
      }
  }
  g.prof_words = (size_t)g.nb * (n_sym + 1) * g.L * 32;
  g.ring_bytes = (size_t)g.nb * kChainRing * kChainK * sizeof(int2);
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  g.total = al(g.prof_words * 4) + al(g.ring_bytes) + al(g.nb * 128) * 2 + al(g.nb * 16) + 256;
  return g;
}

// Wavefront strips (32-bit): per-step latency (cycles) of one strip alone and in a
// full pipeline; total ~ (n + 4K * nb) * t(L) (a strip trails the one above by ~4
// tiles).  Measured with tools/chain_latency.py --kernel wavefront.
static ChainGeo wave_geo(int64_t m, int64_t n, int n_sym) {
  static const int Ls[4] = {1, 2, 4, 8};
  static const double lat_alone[4] = {84, 83, 96, 205};
  static const double lat_loaded[4] = {226, 166, 138, 260};
  ChainGeo g{};
  double best = 1e300;
  int force = 0;
  if (const char* f = getenv("SWB_WAVE_L")) force = atoi(f);
  for (int li = 0; li < 4; ++li) {
    const int L = Ls[li];
    const int64_t rows = 32LL * L;
    const int64_t nb = (m + rows - 1) / rows;
    const double load = nb >= 518 ? 1.0 : (double)nb / 518.0;
    const double lat = lat_alone[li] + load * (lat_loaded[li] - lat_alone[li]);
    double cost = (double)(n + nb * 4 * kChainK) * lat;  // a strip trails by ~4 tiles
    if (nb > 148 * 16 && li < 3) cost *= 1e6;
    if (force) cost = (L == force) ? 0.0 : 1e300;
    if (cost < best) {
      best = cost;
      g.li = li; g.L = L; g.nb = (int)(nb < 1 ? 1 : nb);
    }
  }
  // Columns per step (tools/wave_sweep.py, B200): two columns per step at one row
  // per lane win while the 1-row strips fit one warp per SM sub-partition (config 1
  // 0.52 -> 0.38 ms, config 4 5.0 -> 3.7 ms); beyond that taller strips at one
  // column per step do (config 5: L = 4, KC = 1, 62 ms; KC = 2 / 4: 79 / 64 ms).
  int kc = 1;
  if (!force && (m + 31) / 32 <= 148 * 4) {
    g.li = 0; g.L = 1; g.nb = (int)((m + 31) / 32);
    kc = 2;
  }
  if (const char* f = getenv("SWB_WAVE_KC")) kc = atoi(f);
  g.ki = kc >= 8 ? 3 : kc >= 4 ? 2 : kc >= 2 ? 1 : 0;
  g.KC = 1 << g.ki;
  g.prof_words = (size_t)g.nb * (n_sym + 1) * g.L * 32;
  g.ring_bytes = (size_t)g.nb * kChainRing * kChainK * g.KC * sizeof(int2);
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  g.total = al(g.prof_words * 4) + al(g.ring_bytes) + al(g.nb * 128) * 2 + al(g.nb * 16) + 256;
  return g;
}

int64_t sw_long_workspace_bytes(int64_t m, int64_t n, int32_t n_sym, int32_t width) {
  if ((width != 16 && width != 32) || n_sym < 1 || n_sym > kMaxSym || m < 1)
    return fail(SW_EINVAL, "bad long-pair shape");
  // enough for either schedule (scan strips or wavefront strips)
  const size_t c = chain_geo(m, n, n_sym, width).total, w = wave_geo(m, n, n_sym).total;
  return (int64_t)(c > w ? c : w);
}

int32_t sw_align_long(int32_t width, int32_t kernel, const uint8_t* d_query, int64_t m,
                      const uint8_t* d_ref, int64_t n, const int8_t* d_sub, int32_t n_sym,
                      int32_t gap_open, int32_t gap_extend, int32_t bias, int32_t max_sub,
                      void* d_workspace, int64_t workspace_bytes, int32_t* d_score,
                      int32_t* d_ref_end, int32_t* d_query_end, uint8_t* d_flags,
                      sw_stream_t stream) {
  std::call_once(g_once, init_tables);
  if (!d_query || !d_ref || !d_sub || !d_workspace || !d_score) return fail(SW_EINVAL, "NULL argument");
  if (width != 16 && width != 32) return fail(SW_EINVAL, "width must be 16 or 32");
  if (kernel != SW_KERNEL_SCAN && kernel != SW_KERNEL_WAVEFRONT)
    return fail(SW_ENOTSUP, "the strip pipeline runs the scan or wavefront kernel");
  const bool wave = kernel == SW_KERNEL_WAVEFRONT;
  if (wave) width = 32;  // the wavefront strips compute in 32-bit lanes
  if (wave && (m > (1LL << 30) || n > (1LL << 30))) return fail(SW_ENOTSUP, "wavefront: sequences up to 2^30");
  if (wave && (double)(m < n ? m : n) * (max_sub > 0 ? max_sub : 1) >= (double)(1 << 23))
    return fail(SW_ENOTSUP, "wavefront: scores must stay below 2^23 (use the scan kernel)");
  if (!(gap_open >= gap_extend && gap_extend >= 1)) return fail(SW_EINVAL, "require gap_open >= gap_extend >= 1");
  if (m < 1 || n < 1) return fail(SW_EINVAL, "empty sequence");
  if (n_sym < 1 || n_sym > kMaxSym) return fail(SW_ENOTSUP, "alphabet size %d", n_sym);
  const ChainGeo g = wave ? wave_geo(m, n, n_sym) : chain_geo(m, n, n_sym, width);
  if ((size_t)workspace_bytes < g.total) return fail(SW_EINVAL, "workspace too small (%zu B needed)", g.total);
  const int wi = width == 16 ? 0 : 1;
  cudaStream_t s = (cudaStream_t)stream;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  char* ws = (char*)d_workspace;
  uint32_t* prof = (uint32_t*)ws;
  ws += al(g.prof_words * 4);
  int2* ring = (int2*)ws;
  ws += al(g.ring_bytes);
  // zeroed per launch: the ring (its entries are validated by a generation tag, which
  // must not match stale data), counters, bests, ticket
  char* zero_begin = (char*)ring;
  unsigned long long* published = (unsigned long long*)ws;  // one 128-B line per strip
  ws += al(g.nb * 128);
  unsigned long long* consumed = (unsigned long long*)ws;
  ws += al(g.nb * 128);
  int4* best = (int4*)ws;
  ws += al(g.nb * 16);
  unsigned int* done = (unsigned int*)ws;
  ws += 256;
  cudaError_t e = cudaMemsetAsync(zero_begin, 0, (size_t)(ws - zero_begin), s);
  if (e != cudaSuccess) return cuda_fail(e, "memset chain workspace");
  {
    int A = n_sym, L = g.L, nb = g.nb, mm = (int)m;
    void* pargs[] = {(void*)&d_query, (void*)&mm, (void*)&d_sub, (void*)&A, (void*)&L,
                     (void*)&nb, (void*)&bias, (void*)&prof};
    const int words = (int)g.prof_words;
    e = cudaLaunchKernel(g_chain_prof[wi], dim3((words + 255) / 256), dim3(256), pargs, 0, s);
    if (e != cudaSuccess) return cuda_fail(e, "sw_chain_profile_kernel");
  }
  ChainArgs a;
  std::memset(&a, 0, sizeof a);
  a.prof = prof;
  a.n_sym = n_sym;
  a.m = (int)m;
  a.nb = g.nb;
  a.ref = d_ref;
  a.n = n;
  a.go = gap_open;
  a.ge = gap_extend;
  a.bias = bias;
  a.max_sub = max_sub;
  a.ring = ring;
  a.published = published;
  a.consumed = consumed;
  a.best = best;
  a.done = done;
  a.score = d_score;
  a.ref_end = d_ref_end;
  a.query_end = d_query_end;
  a.flags = d_flags;
  if (const char* tp = getenv("SWB_CHAIN_TRACE_PTR")) {  // diagnostics timeline
    a.trace = (unsigned long long*)strtoull(tp, nullptr, 0);
    a.trace_tiles = atoi(getenv("SWB_CHAIN_TRACE_TILES"));
    a.reverse = getenv("SWB_CHAIN_REVERSE") != nullptr;
  }
  // score-only launches (no coordinate outputs) of the 32-bit strips skip the
  // end-coordinate tracking
  const bool score_only = !d_ref_end && !d_query_end;
  const bool g1 = wi == 1 && gap_extend == 1 && SWB_CHAIN_GE1 && !getenv("SWB_CHAIN_NO_GE1");
  const void* fn = wave ? (gap_extend == 1 && SWB_CHAIN_GE1 && !getenv("SWB_CHAIN_NO_GE1") ? g_wave_g1[g.li][g.ki]
                                                                                             : g_wave[g.li][g.ki])
                        : (wi == 1 && score_only && SWB_CHAIN_SPLIT_SO
                               ? (g1 ? g_chain_so_g1[g.li] : g_chain_so[g.li])
                               : (g1 ? g_chain_g1[g.li] : g_chain[wi][g.li]));
  const size_t smem = wave ? (size_t)(n_sym + 1) * g.L * 32 * 4 + 128 * g.KC + 3 * kChainK * g.KC * 8  // residues, tile_in, 2 x tile_out
                           : (size_t)(n_sym + 1) * g.L * 32 * 4 + (kChainK + 1) * 16 + kChainK * 8
                                 + (width == 32 ? (size_t)(n_sym + 1) * 32 * 8 + 1024 : 0);  // + tile staging, (B, C) table, scan buffers
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(chain smem)");
  }
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 32, smem);
  if (e != cudaSuccess) return cuda_fail(e, "chain occupancy");
  if ((int64_t)occ * sms < g.nb)
    return fail(SW_ENOTSUP, "%d query strips cannot be co-resident (%d per SM x %d SMs)", g.nb, occ, sms);
  void* params[] = {(void*)&a};
  e = cudaLaunchCooperativeKernel(fn, dim3(g.nb), dim3(32), params, smem, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchCooperativeKernel(sw_chain_kernel)");
  return SW_OK;
}

int32_t sw_block_plan(int32_t width, int32_t kernel, int64_t m, int32_t n_sym, int32_t lanes,
                      int32_t* out) {
  if (!out) return fail(SW_EINVAL, "NULL argument");
  if (width != 16 && width != 32) return fail(SW_EINVAL, "width must be 16 or 32");
  if (kernel < SW_KERNEL_LAZYF || kernel > SW_KERNEL_LAZYF_NOEXIT_MIRROR) return fail(SW_EINVAL, "kernel %d", kernel);
  if (m < 1) return fail(SW_EINVAL, "empty query");
  if (n_sym < 1 || n_sym > kMaxSym) return fail(SW_ENOTSUP, "alphabet size %d", n_sym);
  BlockGeo g;
  if (!block_geo(width, kernel == SW_KERNEL_SCAN, m, n_sym, lanes, &g))
    return fail(SW_ENOTSUP, "no block layout for m=%lld lanes=%d width=%d kernel=%d", (long long)m, lanes,
                width, kernel);
  out[0] = g.lanes; out[1] = g.nt; out[2] = g.cl; out[3] = g.L;
  return SW_OK;
}

int32_t sw_align_block(int32_t width, int32_t kernel, int32_t lanes, const uint8_t* d_query,
                       int64_t m, const uint8_t* d_ref, int64_t n, const int8_t* d_sub,
                       int32_t n_sym, int32_t gap_open, int32_t gap_extend, int32_t bias,
                       int32_t max_sub, int32_t coords, int32_t* d_score, int32_t* d_ref_end,
                       int32_t* d_query_end, uint8_t* d_flags, int32_t* d_col_passes,
                       int64_t* d_pass_stats, sw_stream_t stream) {
  std::call_once(g_once, init_tables);
  if (!d_query || !d_ref || !d_sub || !d_score) return fail(SW_EINVAL, "NULL argument");
  int32_t geo[4];
  int32_t rc = sw_block_plan(width, kernel, m, n_sym, lanes, geo);
  if (rc != SW_OK) return rc;
  if (!(gap_open >= gap_extend && gap_extend >= 1)) return fail(SW_EINVAL, "require gap_open >= gap_extend >= 1");
  if (n < 1) return fail(SW_EINVAL, "empty reference");
  if (n > (1LL << 31) - 2) return fail(SW_ENOTSUP, "reference longer than 2^31");
  BlockGeo g;
  block_geo(width, kernel == SW_KERNEL_SCAN, m, n_sym, lanes, &g);
  const int var = kernel == SW_KERNEL_SCAN ? VAR_SCAN
                  : (kernel == SW_KERNEL_LAZYF_MIRROR || kernel == SW_KERNEL_LAZYF_NOEXIT_MIRROR) ? VAR_LAZYF_MIRROR
                                                                                                   : VAR_LAZYF;
  const void* fn = g_block[width == 16 ? 0 : 1][var][g.L - 1];
  BlockArgs a;
  std::memset(&a, 0, sizeof a);
  a.query = d_query; a.sub = d_sub; a.n_sym = n_sym; a.m = (int)m; a.seg_len = g.L;
  a.ref = d_ref; a.n = n; a.go = gap_open; a.ge = gap_extend; a.bias = bias; a.max_sub = max_sub;
  a.early_exit = (kernel == SW_KERNEL_LAZYF || kernel == SW_KERNEL_LAZYF_MIRROR) ? 1 : 0;
  a.coords = coords ? 1 : 0;
  a.score = d_score; a.ref_end = d_ref_end; a.query_end = d_query_end; a.flags = d_flags;
  a.col_passes = d_col_passes; a.pass_stats = d_pass_stats;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(block smem)");
  if (g.cl > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(non-portable cluster)");
  }
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof cfg);
  cfg.gridDim = dim3(g.cl);
  cfg.blockDim = dim3(g.nt);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = g.cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* params[] = {(void*)&a};
  e = cudaLaunchKernelExC(&cfg, fn, params);
  if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernelEx(sw_block_kernel)");
  return SW_OK;
}

int32_t sw_collect_flagged(const uint8_t* d_flags, int64_t n, uint8_t mask, int32_t* d_list,
                           int64_t* d_count, sw_stream_t stream) {
  if (!d_flags || !d_list || !d_count) return fail(SW_EINVAL, "NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(d_count, 0, sizeof(int64_t), s);
  if (e != cudaSuccess) return cuda_fail(e, "memset count");
  if (n == 0) return SW_OK;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  sw_collect_kernel<<<blocks, 256, 0, s>>>(d_flags, n, mask, d_list, (unsigned long long*)d_count);
  e = cudaGetLastError();
  return e == cudaSuccess ? SW_OK : cuda_fail(e, "sw_collect_kernel");
}

int32_t swb_unpack2_launch(const uint8_t* d_packed, int64_t n_res, uint8_t* d_codes,
                           sw_stream_t stream);

int32_t sw_unpack_2bit(const uint8_t* d_packed, int64_t n_res, uint8_t* d_codes,
                       sw_stream_t stream) {
  if (n_res < 0) return fail(SW_EINVAL, "n_res < 0");
  if (n_res > 0 && (!d_packed || !d_codes)) return fail(SW_EINVAL, "NULL argument");
  const int32_t rc = swb_unpack2_launch(d_packed, n_res, d_codes, stream);
  return rc == 0 ? SW_OK : cuda_fail((cudaError_t)rc, "sw_unpack2_kernel");
}

int32_t swb_topk_launch(const int32_t* d_score, const int64_t* d_ids, const int32_t* d_ref_end,
                        const int32_t* d_query_end, int64_t n, int32_t k, int64_t* d_records,
                        void* d_work, sw_stream_t stream, const char** err);

int32_t sw_topk(const int32_t* d_score, const int64_t* d_ids, const int32_t* d_ref_end,
                const int32_t* d_query_end, int64_t n, int32_t k, int64_t* d_records,
                void* d_work, sw_stream_t stream) {
  if (!d_score || !d_records || !d_work) return fail(SW_EINVAL, "NULL argument");
  if (n < 0) return fail(SW_EINVAL, "n < 0");
  if (k < 1 || k > 1024) return fail(SW_ENOTSUP, "top-k supports 1 <= k <= 1024, got %d", k);
  const char* what = "";
  const int32_t rc = swb_topk_launch(d_score, d_ids, d_ref_end, d_query_end, n, k, d_records,
                                     d_work, stream, &what);
  return rc == 0 ? SW_OK : cuda_fail((cudaError_t)rc, what);
}

int32_t sw_scan_lanes(int32_t width, int32_t lanes, const uint16_t* d_f, const int32_t* d_d,
                      int32_t n, uint16_t* d_out, sw_stream_t stream) {
  if (!d_f || !d_d || !d_out) return fail(SW_EINVAL, "NULL argument");
  if (n <= 0) return SW_OK;
  const int lpw = width == 16 ? 2 : (width == 32 ? 1 : 0);
  if (!lpw || !pow2(lanes)) return fail(SW_EINVAL, "bad width/lanes");
  const int T = lanes / lpw;
  if (T < (lpw == 1 ? 2 : 1) || T > 32) return fail(SW_ENOTSUP, "lanes %d unsupported", lanes);
  const int G = 32 / T;
  const int warps = (n + G - 1) / G;
  const int block = 128;
  const int grid = (warps + 3) / 4;
  cudaStream_t s = (cudaStream_t)stream;
  if (lpw == 2) {
    switch (T) {
#define CASE(TT) case TT: sw_scan_test_kernel<W16, TT><<<grid, block, 0, s>>>(d_f, d_d, n, d_out); break;
      CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32)
#undef CASE
    }
  } else {
    switch (T) {
#define CASE(TT) case TT: sw_scan_test_kernel<W32, TT><<<grid, block, 0, s>>>(d_f, d_d, n, d_out); break;
      CASE(2) CASE(4) CASE(8) CASE(16) CASE(32)
#undef CASE
    }
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SW_OK : cuda_fail(e, "sw_scan_test_kernel");
}

}  // extern "C"
