/*
 * swscan_b200.h -- C ABI of the B200-native striped Smith-Waterman library
 * (libswscan_b200.so).  Plain pointers and sizes only; every device pointer is
 * caller-owned CUDA memory, every call is asynchronous on `stream`.
 *
 * Each entry point replaces one operator of the reference package
 * (/root/reference/pkg/src/swscan); the reference interface is cited beside it.
 * Return value: 0 on success, a negative SW_E* code on error (message in
 * sw_last_error()).  Score overflow is a per-alignment flag, never an error
 * (reference: src/vectors.py:145-154).
 *
 * Scores are exact. End coordinates are the 0-based (ref_end, query_end) of
 * the first cell reaching the best score in the reference's scalar loop order
 * (reference residue outer, query position inner; src/_compiled.py:83-114);
 * (-1, -1) for score 0.  See DESIGN.md "End coordinates".
 */
#ifndef SWSCAN_B200_H
#define SWSCAN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sw_stream_t; /* == cudaStream_t */

enum {
  SW_OK = 0,
  SW_EINVAL = -1,   /* bad argument (reference: ValueError / ProfileMismatch) */
  SW_ECUDA = -2,    /* CUDA launch / runtime failure */
  SW_ENOTSUP = -3,  /* shape outside the compiled kernel set */
};

/* kernels: the reference's _KERNEL_IDS {"lazyf": 0, "lazyf-noexit": 1, "scan": 2}
 * (src/_compiled.py:576) plus the parity-mode lazy-F that mirrors the
 * reference's E recurrence so per-column pass counts match bit for bit. */
enum {
  SW_KERNEL_LAZYF = 0,
  SW_KERNEL_LAZYF_NOEXIT = 1,
  SW_KERNEL_SCAN = 2,
  SW_KERNEL_LAZYF_MIRROR = 3,
  SW_KERNEL_LAZYF_NOEXIT_MIRROR = 4,
  SW_KERNEL_WAVEFRONT = 5, /* sw_align_long only: strips with an intra-strip wavefront */
};

/* per-alignment flag bits */
enum {
  SW_FLAG_REF_OVERFLOW = 1, /* reference uint16 kernels would saturate: exact > 65535 - bias */
  SW_FLAG_RESCUE = 2,       /* 16-bit run hit the wrap guard (internal; cleared by rescue) */
  SW_FLAG_RESCUED = 4,      /* result comes from the 32-bit re-run */
  SW_FLAG_FEED_TIMEOUT = 8, /* streamed input (sw_db_opts_t.d_arrived) never arrived */
};

/* Striped layout chosen for one query (reference: VectorSpec(lanes) +
 * QueryProfile.seg_len, src/vectors.py:21-36, src/profile.py:26-51). */
typedef struct sw_plan {
  int32_t width;      /* score bits: 16 (two lanes per register) or 32 */
  int32_t lanes;      /* P: stripes per alignment (reference p) */
  int32_t threads;    /* T: threads per alignment (P/2 for 16-bit, P for 32-bit) */
  int32_t seg_len;    /* L = ceil(m / P) */
  int32_t lmax;       /* register words per thread of the kernel instance (>= L) */
  int32_t m;          /* query length */
  int32_t n_sym;      /* alphabet size A */
  int32_t prof_words; /* 32-bit words of the device profile: (A+1) * L * T */
} sw_plan_t;

int32_t sw_version(void);
const char* sw_last_error(void);

/* Choose (P, T, L) for a query of length m.  lanes = 0 picks the throughput
 * layout; lanes = p reproduces the reference layout for VectorSpec(p).
 * Reference: build_profile_arrays(query, scheme, p), src/_compiled.py:579-585. */
int32_t sw_plan_query(int32_t m, int32_t n_sym, int32_t width, int32_t lanes, sw_plan_t* out);

/* Build the striped device profile (reference _build_profile_c,
 * src/_compiled.py:59-73; build_profile src/profile.py:37-72).
 * d_query: uint8 codes [m]; d_sub: int8 [n_sym][n_sym]; d_prof: prof_words. */
int32_t sw_profile_build(const sw_plan_t* plan, const uint8_t* d_query, const int8_t* d_sub,
                         int32_t bias, uint32_t* d_prof, sw_stream_t stream);

/* One prebuilt query profile against n targets (database search form).
 * Reference: align_prebuilt(kernel, prof, bias, ref, scheme), src/_compiled.py:588-607,
 * applied to every target.  Targets: d_tgt bytes, target j = d_tgt[d_start[j] ..
 * d_start[j] + d_len[j]).  d_order (nullable): processing order of job ids
 * (length-sorted, descending, for load balance).  d_n_jobs (nullable): device
 * job count overriding n: a re-run pass that runs without a host sync (the
 * 32-bit overflow rescue, whose results are marked SW_FLAG_RESCUED, or a 16-bit
 * re-run of jobs whose streamed input timed out).
 * Outputs are indexed by job id; d_ref_end/d_query_end/d_flags/d_col_passes/d_pass_stats
 * nullable.  d_col_passes (lazy-F kernels): per-column correction passes of job 0.
 * d_pass_stats (lazy-F kernels): int64 [n][2] = (total correction passes, columns that
 * took the early exit) per alignment -- with the reference layout and a *_MIRROR
 * kernel these reproduce the reference's OpCounters exactly (src/vectors.py:61-95).
 * opts (nullable): database-search controls, see sw_db_opts_t. */
typedef struct sw_db_opts {
  /* d_coord_floor (nullable device int32): end coordinates are located only for
   * alignments scoring >= *d_coord_floor (others report ref_end = query_end = -2;
   * scores are always exact).  A database search passes a lower bound of its top-k
   * threshold so that only candidate hits pay for the position search.  Applied by
   * the exact 16-bit scan instances; other kernels locate every alignment. */
  int32_t* d_coord_floor;
  /* floor_sample > 0: the kernel itself raises *d_coord_floor (a valid floor at
   * launch, e.g. 0) to the floor_k-th best exact score of the first floor_sample
   * jobs in processing order once they complete -- a lower bound of the final
   * top-floor_k threshold, found without a second launch. */
  int64_t floor_sample;
  int32_t floor_k;
  /* Streamed input: arrive_epoch > 0 makes every task wait until the chunk holding
   * its jobs has arrived: jobs [c * arrive_jobs, (c + 1) * arrive_jobs) (ids before
   * d_order) are readable once d_arrived[c] >= arrive_epoch.  The caller copies
   * chunk c (residues, starts, lengths) and then the flag on one copy stream, so
   * one launch overlaps the whole host-to-device transfer.  A task whose chunk
   * has not arrived after arrive_timeout_ns (0 = 2 s) aborts the feed: it and every
   * job not yet started report score 0 with SW_FLAG_FEED_TIMEOUT (no hang, no
   * unflagged result).  The caller re-runs the flagged jobs once its copies are
   * done (sw_collect_flagged(mask = SW_FLAG_FEED_TIMEOUT) + a device-counted
   * sw_db_align); the Python layer does this in search_streamed. */
  int32_t arrive_epoch;
  const int32_t* d_arrived;
  int64_t arrive_jobs;
  int64_t arrive_timeout_ns;
} sw_db_opts_t;

int32_t sw_db_align(const sw_plan_t* plan, const uint32_t* d_prof, int32_t kernel,
                    int32_t gap_open, int32_t gap_extend, int32_t bias, int32_t max_sub,
                    const uint8_t* d_tgt, const int64_t* d_start, const int32_t* d_len,
                    const int32_t* d_order, int64_t n, const int64_t* d_n_jobs,
                    int32_t* d_score, int32_t* d_ref_end, int32_t* d_query_end, uint8_t* d_flags,
                    int32_t* d_col_passes, int64_t* d_pass_stats, const sw_db_opts_t* opts,
                    sw_stream_t stream);

/* n independent (query_k, target_k) pairs.  Reference: batch_align(kernel_id, p,
 * flat_q, q_off, flat_r, r_off, match_a, mis_a, go_a, ge_a), src/_compiled.py:504-529.
 * Scoring: a shared d_sub [n_sym][n_sym] with gap_open/gap_extend, or (d_sub NULL)
 * per-pair 4x4 match/mismatch schemes d_match/d_mismatch/d_go/d_ge like batch_align.
 * lanes = 0 picks the throughput layout; min_qlen/max_qlen bound the query lengths
 * (min_qlen = 0 if unknown; equal segment lengths select the exact-length kernels). */
int32_t sw_pairs_align(int32_t width, int32_t lanes, int32_t kernel, const uint8_t* d_qry,
                       const int64_t* d_qstart, const int32_t* d_qlen, const uint8_t* d_tgt,
                       const int64_t* d_tstart, const int32_t* d_tlen, const int32_t* d_order,
                       int64_t n, const int64_t* d_n_jobs, int32_t min_qlen, int32_t max_qlen,
                       const int8_t* d_sub,
                       int32_t n_sym, int32_t gap_open, int32_t gap_extend, int32_t bias,
                       int32_t max_sub, const int32_t* d_match, const int32_t* d_mismatch,
                       const int32_t* d_go, const int32_t* d_ge, int32_t* d_score,
                       int32_t* d_ref_end, int32_t* d_query_end, uint8_t* d_flags,
                       int32_t* d_col_passes, int64_t* d_pass_stats, sw_stream_t stream);

/* Long single pairs (query beyond the warp kernels' 2048 16-bit / 1024 32-bit
 * positions, e.g. config 4/5): a pipeline of query strips, one warp-sized CTA
 * per strip, streaming every reference column and passing the strip boundary
 * (F out, corrected last H) to the next strip through an L2 ring buffer.
 * Reference: align_pair("scan", p, query, ref, scheme), src/_compiled.py:610-615,
 * for a single pair.  Scan kernel only.  Outputs are single values (device).
 * d_workspace: sw_long_workspace_bytes(m, n, n_sym, width) bytes of device memory. */
int64_t sw_long_workspace_bytes(int64_t m, int64_t n, int32_t n_sym, int32_t width);
int32_t sw_align_long(int32_t width, int32_t kernel, const uint8_t* d_query, int64_t m,
                      const uint8_t* d_ref, int64_t n, const int8_t* d_sub, int32_t n_sym,
                      int32_t gap_open, int32_t gap_extend, int32_t bias, int32_t max_sub,
                      void* d_workspace, int64_t workspace_bytes, int32_t* d_score,
                      int32_t* d_ref_end, int32_t* d_query_end, uint8_t* d_flags,
                      sw_stream_t stream);

/* One alignment across a CTA or a thread-block cluster at high stripe counts: the
 * reference layout VectorSpec(p) for p beyond one warp (up to 32,768 16-bit /
 * 16,384 32-bit stripes), with Alg. 6's F scan resolved warp shuffle -> block
 * (shared memory + one bar.sync per column) -> cluster (distributed shared memory,
 * CTAs pipelined along the query).  Reference: align_pair(kernel, p, query, ref,
 * scheme) / align_prebuilt, src/_compiled.py:588-615, for p the reference accepts
 * (power of two).  Lazy-F kernels (SW_KERNEL_LAZYF*) run on one CTA (p <= 2,048
 * 16-bit / 1,024 32-bit), one block-wide vote per pass; d_col_passes (int32 [n])
 * and d_pass_stats (int64 [2]: total passes, early-exit columns) are nullable.
 * lanes = 0 chooses the layout.  sw_block_plan reports it: out[4] = {lanes,
 * threads per CTA, CTAs per cluster, seg_len}.  coords = 0 skips the end-coordinate
 * search (ref_end = query_end = -1). */
int32_t sw_block_plan(int32_t width, int32_t kernel, int64_t m, int32_t n_sym, int32_t lanes,
                      int32_t* out);
int32_t sw_align_block(int32_t width, int32_t kernel, int32_t lanes, const uint8_t* d_query,
                       int64_t m, const uint8_t* d_ref, int64_t n, const int8_t* d_sub,
                       int32_t n_sym, int32_t gap_open, int32_t gap_extend, int32_t bias,
                       int32_t max_sub, int32_t coords, int32_t* d_score, int32_t* d_ref_end,
                       int32_t* d_query_end, uint8_t* d_flags, int32_t* d_col_passes,
                       int64_t* d_pass_stats, sw_stream_t stream);

/* Gather the ids of alignments whose flags intersect `mask` into d_list and
 * their count into *d_count (device int64).  Used to re-run 16-bit overflow
 * suspects in 32 bits without a host round trip. */
int32_t sw_collect_flagged(const uint8_t* d_flags, int64_t n, uint8_t mask, int32_t* d_list,
                           int64_t* d_count, sw_stream_t stream);

/* Top-k of a database search on the device (BASELINE.json config 2's top-100 merge;
 * the reference has no database driver, its runner aligns pairs,
 * src/runner.py:141-153).  d_records: int64 [k][4] = (score, target id, ref_end,
 * query_end), score descending, then target id ascending; rows past min(k, n) are
 * -1.  d_ids (nullable: the index itself) maps an alignment to its global target id
 * (< 2^32); d_ref_end / d_query_end nullable (-1).  d_work: sw_topk_workspace()
 * bytes of device scratch.  1 <= k <= 1024.  Three small launches on `stream`
 * (score histogram + threshold, compaction, one-CTA sort); mass ties beyond the
 * 4,096 candidates the sort holds take an exact single-CTA radix select. */
int64_t sw_topk_workspace(void);
int32_t sw_topk(const int32_t* d_score, const int64_t* d_ids, const int32_t* d_ref_end,
                const int32_t* d_query_end, int64_t n, int32_t k, int64_t* d_records,
                void* d_work, sw_stream_t stream);

/* Expand 2-bit packed DNA (four residues per byte, residue k of a byte in bits
 * 2k..2k+1) to one-byte codes on the device: d_codes[0 .. n_res).  The reference
 * carries one code per element (Alphabet.encode, src/scoring.py:45-46); the packed
 * form is an input format for host links that bound short-read batches.  d_codes
 * 4-byte aligned for the fast path. */
int32_t sw_unpack_2bit(const uint8_t* d_packed, int64_t n_res, uint8_t* d_codes,
                       sw_stream_t stream);

/* Device weighted max-plus scan over P lanes (reference weighted_max_scan /
 * _weighted_max_scan_c, src/kernels.py:177-201, src/_compiled.py:448-460):
 * d_f, d_out: uint16 [n][lanes]; d_d: decay per vector.  Values must fit the
 * signed lane width (< 32768 for width 16). */
int32_t sw_scan_lanes(int32_t width, int32_t lanes, const uint16_t* d_f, const int32_t* d_d,
                      int32_t n, uint16_t* d_out, sw_stream_t stream);

/* Diagnostics: launch the DPX issue-rate probe (kind 0: VIADDMNMX.S16x2 only;
 * kind 1: the cell-update instruction mix) on every SM; returns the number of
 * per-thread DPX instructions it executes (time it with events on `stream`),
 * or a negative SW_E* code.  d_scratch: >= 256 words.  Used for the roofline
 * denominator; no reference counterpart. */
int64_t sw_dpx_probe(int32_t kind, int64_t iters, uint32_t* d_scratch, sw_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* SWSCAN_B200_H */
