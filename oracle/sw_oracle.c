/*
 * sw_oracle.c -- CPU restatement of the reference `swscan` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package may link or call
 * this file; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs load it, as the checker or as the timed CPU baseline.
 *
 * Every function restates one reference function, cited file:line against
 * /root/reference/pkg/src/swscan/ (the reference is Python + numba; there is no
 * compiled reference to build).  Arithmetic follows the
 * reference exactly: unsigned 16-bit saturating lanes with the profile bias
 * trick for the striped kernels, exact int64 for the scalar Gotoh oracle.
 * The restatement is pinned against golden vectors produced by the reference
 * itself (tests/golden/make_golden.py).
 *
 * Additions beyond the reference (documented in DESIGN.md, contract A10):
 *   - swo_scalar() also returns end coordinates: the FIRST cell reaching the
 *     best score in the reference loop order of _sw_scalar_c (reference
 *     residue i outer, query position q inner, strict '>'), as 0-based
 *     (ref_end, query_end); (-1, -1) when the score is 0.
 *   - OpenMP batch drivers (the reference's batch drivers are serial loops).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define U16MAX 0xFFFF

enum { SHIFTS = 0, SAT_ADDS, SAT_SUBS, MAXES, LOADS, STORES, PASSES };

/* _clamp_u16  src/_compiled.py:32-36 */
static inline int64_t clamp_u16(int64_t x) { return x > U16MAX ? (int64_t)U16MAX : x; }

/* _scan_steps  src/_compiled.py:39-46 */
int32_t swo_scan_steps(int64_t p) {
    int32_t s = 0;
    while (((int64_t)1 << s) < p) s++;
    return s == 0 ? 1 : s;
}

/* _bias_of  src/_compiled.py:49-56  (bias = max(0, -min S), src/scoring.py:90-92) */
int64_t swo_bias(const int8_t *sub, int32_t n_sym) {
    int64_t lo = 0;
    for (int32_t i = 0; i < n_sym * n_sym; i++)
        if ((int64_t)sub[i] < lo) lo = sub[i];
    return -lo;
}

/* _build_profile_c  src/_compiled.py:59-73 ; build_profile src/profile.py:37-72
 * prof[a][j][l] = bias + S[a][query[l*L + j]] for l*L+j < m, else 0. */
int64_t swo_build_profile(const uint8_t *query, int64_t m, const int8_t *sub, int32_t n_sym,
                          int64_t p, uint16_t *prof) {
    int64_t L = (m + p - 1) / p;
    int64_t bias = swo_bias(sub, n_sym);
    memset(prof, 0, sizeof(uint16_t) * (size_t)(n_sym * L * p));
    for (int32_t a = 0; a < n_sym; a++)
        for (int64_t l = 0; l < p; l++)
            for (int64_t j = 0; j < L; j++) {
                int64_t q = l * L + j;
                if (q < m)
                    prof[((int64_t)a * L + j) * p + l] =
                        (uint16_t)(bias + (int64_t)sub[a * n_sym + query[q]]);
            }
    return bias;
}

/* _sw_scalar_c  src/_compiled.py:76-115 (pure form: sw_scalar src/oracle.py:31-71).
 * Exact Gotoh recurrences over int64, rows = reference residues, columns = query.
 * Extension: first-max end coordinates (strict '>' in the same loop order). */
int64_t swo_scalar(const uint8_t *query, int64_t m, const uint8_t *ref, int64_t n,
                   const int8_t *sub, int32_t n_sym, int64_t go, int64_t ge,
                   int32_t *ref_end, int32_t *query_end) {
    int64_t *h = (int64_t *)calloc((size_t)(m + 1), sizeof(int64_t));
    int64_t *e = (int64_t *)calloc((size_t)(m + 1), sizeof(int64_t));
    int64_t best = 0;
    int64_t bi = -1, bq = -1;
    for (int64_t i = 0; i < n; i++) {
        const int8_t *row = sub + (int64_t)ref[i] * n_sym;
        int64_t diag = h[0];
        int64_t f = 0, hq_prev = 0;
        for (int64_t q = 1; q <= m; q++) {
            int64_t ev = e[q] - ge, t = h[q] - go;
            if (t > ev) ev = t;
            if (ev < 0) ev = 0;
            int64_t fv = f - ge;
            t = hq_prev - go;
            if (t > fv) fv = t;
            if (fv < 0) fv = 0;
            int64_t hv = diag + (int64_t)row[query[q - 1]];
            if (ev > hv) hv = ev;
            if (fv > hv) hv = fv;
            if (hv < 0) hv = 0;
            diag = h[q];
            h[q] = hv;
            e[q] = ev;
            f = fv;
            hq_prev = hv;
            if (hv > best) { best = hv; bi = i; bq = q - 1; }
        }
    }
    free(h);
    free(e);
    if (ref_end) *ref_end = (int32_t)bi;
    if (query_end) *query_end = (int32_t)bq;
    return best;
}

/* _align_lazyf_c  src/_compiled.py:118-223 (pure form: align_lazyf src/kernels.py:110-174).
 * prof is [n_sym][L][p] uint16; counters int64[7]; col_passes int64[n] (nullable). */
int64_t swo_align_lazyf(const uint16_t *prof, int64_t L, int64_t p, const uint8_t *ref, int64_t n,
                        int64_t bias, int64_t go_raw, int64_t ge_raw, int32_t early_exit,
                        uint8_t *saturated_out, int64_t *counters, int64_t *col_passes) {
    int64_t go = clamp_u16(go_raw), ge = clamp_u16(ge_raw);
    size_t plane = (size_t)(L * p);
    uint16_t *buf = (uint16_t *)calloc(3 * plane + 3 * (size_t)p, sizeof(uint16_t));
    uint16_t *hs = buf, *hl = buf + plane, *ea = buf + 2 * plane;
    uint16_t *vh = buf + 3 * plane, *vf = vh + p, *vmax = vf + p;
    int64_t cnt[7] = {0};
    int saturated = 0;
    for (int64_t i = 0; i < n; i++) {
        const uint16_t *row = prof + (int64_t)ref[i] * L * p;
        cnt[LOADS] += 1;
        cnt[SHIFTS] += 1;
        for (int64_t l = p - 1; l > 0; l--) vh[l] = hs[(L - 1) * p + l - 1];
        vh[0] = 0;
        { uint16_t *t = hl; hl = hs; hs = t; }
        for (int64_t l = 0; l < p; l++) vf[l] = 0;
        for (int64_t j = 0; j < L; j++) {
            cnt[LOADS] += 3; cnt[STORES] += 2; cnt[SAT_ADDS] += 1; cnt[SAT_SUBS] += 4; cnt[MAXES] += 5;
            for (int64_t l = 0; l < p; l++) {
                int64_t h = (int64_t)vh[l] + (int64_t)row[j * p + l];
                if (h > U16MAX) { h = U16MAX; saturated = 1; }
                h -= bias;
                if (h < 0) h = 0;
                if (h > (int64_t)vmax[l]) vmax[l] = (uint16_t)h;
                int64_t e = ea[j * p + l], t = h;
                if (e > t) t = e;
                int64_t fc = vf[l];
                if (fc > t) t = fc;
                hs[j * p + l] = (uint16_t)t;
                int64_t hgo = t - go;
                if (hgo < 0) hgo = 0;
                int64_t e2 = e - ge;
                if (e2 < 0) e2 = 0;
                if (hgo > e2) e2 = hgo;
                ea[j * p + l] = (uint16_t)e2;
                int64_t f2 = fc - ge;
                if (f2 < 0) f2 = 0;
                if (hgo > f2) f2 = hgo;
                vf[l] = (uint16_t)f2;
                vh[l] = hl[j * p + l];
            }
        }
        int64_t passes = 0;
        for (int64_t it = 0; it < p; it++) {
            cnt[SHIFTS] += 1;
            for (int64_t l = p - 1; l > 0; l--) vf[l] = vf[l - 1];
            vf[0] = 0;
            if (early_exit) {
                uint16_t mx = 0;
                for (int64_t l = 0; l < p; l++) if (vf[l] > mx) mx = vf[l];
                if (mx == 0) break;
            }
            for (int64_t j = 0; j < L; j++) {
                cnt[LOADS] += 1; cnt[MAXES] += 1; cnt[STORES] += 1; cnt[SAT_SUBS] += 1;
                for (int64_t l = 0; l < p; l++) {
                    uint16_t fv = vf[l];
                    if (fv > hs[j * p + l]) hs[j * p + l] = fv;
                    int64_t d = (int64_t)fv - ge;
                    if (d < 0) d = 0;
                    vf[l] = (uint16_t)d;
                }
            }
            passes++;
            cnt[PASSES] += 1;
        }
        if (col_passes) col_passes[i] = passes;
    }
    int64_t score = 0;
    for (int64_t l = 0; l < p; l++) if ((int64_t)vmax[l] > score) score = vmax[l];
    free(buf);
    if (saturated_out) *saturated_out = (uint8_t)saturated;
    if (counters) memcpy(counters, cnt, sizeof cnt);
    return score;
}

/* _align_scan_c  src/_compiled.py:226-342 (pure form: align_scan src/kernels.py:204-264). */
int64_t swo_align_scan(const uint16_t *prof, int64_t L, int64_t p, const uint8_t *ref, int64_t n,
                       int64_t bias, int64_t go_raw, int64_t ge_raw,
                       uint8_t *saturated_out, int64_t *counters, int64_t *col_passes) {
    int64_t go = clamp_u16(go_raw), ge = clamp_u16(ge_raw);
    int64_t d_scan = clamp_u16(L * ge_raw);
    int64_t d_wrap = clamp_u16((L - 1) * ge_raw);
    int32_t steps = swo_scan_steps(p);
    size_t plane = (size_t)(L * p);
    uint16_t *buf = (uint16_t *)calloc(3 * plane + 5 * (size_t)p, sizeof(uint16_t));
    uint16_t *hs = buf, *hl = buf + plane, *ea = buf + 2 * plane;
    uint16_t *vh = buf + 3 * plane, *vf = vh + p, *vfj = vf + p, *carry = vfj + p, *vmax = carry + p;
    int64_t cnt[7] = {0};
    int saturated = 0;
    for (int64_t i = 0; i < n; i++) {
        const uint16_t *row = prof + (int64_t)ref[i] * L * p;
        cnt[LOADS] += 1; cnt[SAT_SUBS] += 1; cnt[MAXES] += 1; cnt[SHIFTS] += 1;
        for (int64_t l = p - 1; l > 0; l--) {
            int64_t x = hs[(L - 1) * p + l - 1];
            int64_t y = (int64_t)carry[l - 1] - d_wrap;
            if (y < 0) y = 0;
            if (y > x) x = y;
            vh[l] = (uint16_t)x;
        }
        vh[0] = 0;
        { uint16_t *t = hl; hl = hs; hs = t; }
        for (int64_t l = 0; l < p; l++) { vf[l] = 0; vfj[l] = carry[l]; }
        for (int64_t j = 0; j < L; j++) {
            cnt[LOADS] += 3; cnt[STORES] += 2; cnt[SAT_ADDS] += 1; cnt[SAT_SUBS] += 5; cnt[MAXES] += 6;
            for (int64_t l = 0; l < p; l++) {
                int64_t h = (int64_t)vh[l] + (int64_t)row[j * p + l];
                if (h > U16MAX) { h = U16MAX; saturated = 1; }
                h -= bias;
                if (h < 0) h = 0;
                if (h > (int64_t)vmax[l]) vmax[l] = (uint16_t)h;
                int64_t e = ea[j * p + l], t = h;
                if (e > t) t = e;
                int64_t fc = vf[l];
                if (fc > t) t = fc;
                hs[j * p + l] = (uint16_t)t;
                int64_t hgo = t - go;
                if (hgo < 0) hgo = 0;
                int64_t e2 = e - ge;
                if (e2 < 0) e2 = 0;
                if (hgo > e2) e2 = hgo;
                ea[j * p + l] = (uint16_t)e2;
                int64_t f2 = fc - ge;
                if (f2 < 0) f2 = 0;
                if (hgo > f2) f2 = hgo;
                vf[l] = (uint16_t)f2;
                int64_t h2 = hl[j * p + l], fj = vfj[l];
                if (fj > h2) h2 = fj;
                vh[l] = (uint16_t)h2;
                fj -= ge;
                if (fj < 0) fj = 0;
                vfj[l] = (uint16_t)fj;
            }
        }
        cnt[SHIFTS] += 1;
        for (int64_t l = p - 1; l > 0; l--) carry[l] = vf[l - 1];
        carry[0] = 0;
        for (int32_t s = 0; s < steps; s++) {
            int64_t k = (int64_t)1 << s;
            int64_t dd = clamp_u16(k * d_scan);
            cnt[SHIFTS] += 1; cnt[SAT_SUBS] += 1; cnt[MAXES] += 1; cnt[PASSES] += 1;
            for (int64_t l = p - 1; l > k - 1; l--) {
                int64_t v = (int64_t)carry[l - k] - dd;
                if (v > (int64_t)carry[l]) carry[l] = (uint16_t)v;
            }
        }
        if (col_passes) col_passes[i] = steps;
    }
    int64_t score = 0;
    for (int64_t l = 0; l < p; l++) if ((int64_t)vmax[l] > score) score = vmax[l];
    free(buf);
    if (saturated_out) *saturated_out = (uint8_t)saturated;
    if (counters) memcpy(counters, cnt, sizeof cnt);
    return score;
}

/* _scan_sequential_c  src/_compiled.py:431-445 (pure: scan_sequential src/oracle.py:107-123) */
void swo_scan_sequential(const uint16_t *f, int64_t p, int64_t d_raw, uint16_t *acc) {
    int64_t d = clamp_u16(d_raw);
    uint16_t *cur = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)p);
    memcpy(cur, f, sizeof(uint16_t) * (size_t)p);
    memset(acc, 0, sizeof(uint16_t) * (size_t)p);
    for (int64_t it = 0; it < p; it++) {
        for (int64_t l = p - 1; l > 0; l--) cur[l] = cur[l - 1];
        cur[0] = 0;
        for (int64_t l = 0; l < p; l++) {
            if (cur[l] > acc[l]) acc[l] = cur[l];
            int64_t t = (int64_t)cur[l] - d;
            cur[l] = (uint16_t)(t < 0 ? 0 : t);
        }
    }
    free(cur);
}

/* _weighted_max_scan_c  src/_compiled.py:448-460 (pure: _weighted_scan_on src/kernels.py:177-185) */
void swo_weighted_max_scan(const uint16_t *f, int64_t p, int64_t d_raw, uint16_t *acc) {
    memset(acc, 0, sizeof(uint16_t) * (size_t)p);
    for (int64_t l = 1; l < p; l++) acc[l] = f[l - 1];
    int32_t steps = swo_scan_steps(p);
    for (int32_t s = 0; s < steps; s++) {
        int64_t k = (int64_t)1 << s;
        int64_t dd = clamp_u16(k * d_raw);
        for (int64_t l = p - 1; l > k - 1; l--) {
            int64_t v = (int64_t)acc[l - k] - dd;
            if (v > (int64_t)acc[l]) acc[l] = (uint16_t)v;
        }
    }
}

/* ---- batch drivers (OpenMP; the reference's batch_oracle_scores / batch_align,
 *      src/_compiled.py:491-529, are serial numba loops) ---- */

/* _fill_sub4  src/_compiled.py:483-488 */
static void fill_sub4(int8_t *sub, int64_t match, int64_t mismatch) {
    for (int a = 0; a < 4; a++) {
        for (int b = 0; b < 4; b++) sub[a * 4 + b] = (int8_t)mismatch;
        sub[a * 4 + a] = (int8_t)match;
    }
}

/* Pairwise scalar oracle.  Either `sub` (shared n_sym x n_sym matrix; go/ge
 * scalars) or, when sub == NULL, per-pair 4x4 match/mismatch schemes like
 * batch_oracle_scores (src/_compiled.py:491-501). */
void swo_batch_scalar(int64_t npairs, const uint8_t *flat_q, const int64_t *q_off,
                      const uint8_t *flat_r, const int64_t *r_off, const int8_t *sub,
                      int32_t n_sym, int64_t go, int64_t ge, const int64_t *match_a,
                      const int64_t *mis_a, const int64_t *go_a, const int64_t *ge_a,
                      int64_t *score, int32_t *ref_end, int32_t *query_end, int32_t nthreads) {
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t t = 0; t < npairs; t++) {
        int8_t sub4[16];
        const int8_t *s = sub;
        int32_t ns = n_sym;
        int64_t g_o = go, g_e = ge;
        if (!sub) {
            fill_sub4(sub4, match_a[t], mis_a[t]);
            s = sub4; ns = 4; g_o = go_a[t]; g_e = ge_a[t];
        }
        int32_t ri, qi;
        score[t] = swo_scalar(flat_q + q_off[t], q_off[t + 1] - q_off[t], flat_r + r_off[t],
                              r_off[t + 1] - r_off[t], s, ns, g_o, g_e, &ri, &qi);
        if (ref_end) ref_end[t] = ri;
        if (query_end) query_end[t] = qi;
    }
}

/* One query against many targets with the scalar oracle (database search form). */
void swo_db_scalar(const uint8_t *query, int64_t m, int64_t ntargets, const uint8_t *flat_r,
                   const int64_t *r_off, const int8_t *sub, int32_t n_sym, int64_t go, int64_t ge,
                   int64_t *score, int32_t *ref_end, int32_t *query_end, int32_t nthreads) {
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t t = 0; t < ntargets; t++) {
        int32_t ri, qi;
        score[t] = swo_scalar(query, m, flat_r + r_off[t], r_off[t + 1] - r_off[t], sub, n_sym,
                              go, ge, &ri, &qi);
        if (ref_end) ref_end[t] = ri;
        if (query_end) query_end[t] = qi;
    }
}

/* batch_align  src/_compiled.py:504-529 generalised: kernel_id 0 = lazy-F with
 * early exit, 1 = lazy-F full, 2 = scan; shared matrix or per-pair 4x4 schemes.
 * The profile is rebuilt per pair exactly as the reference does (:518). */
void swo_batch_striped(int32_t kernel_id, int64_t p, int64_t npairs, const uint8_t *flat_q,
                       const int64_t *q_off, const uint8_t *flat_r, const int64_t *r_off,
                       const int8_t *sub, int32_t n_sym, int64_t go, int64_t ge,
                       const int64_t *match_a, const int64_t *mis_a, const int64_t *go_a,
                       const int64_t *ge_a, int64_t *score, uint8_t *overflow, int64_t *counters,
                       int32_t nthreads) {
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t t = 0; t < npairs; t++) {
        int8_t sub4[16];
        const int8_t *s = sub;
        int32_t ns = n_sym;
        int64_t g_o = go, g_e = ge;
        if (!sub) {
            fill_sub4(sub4, match_a[t], mis_a[t]);
            s = sub4; ns = 4; g_o = go_a[t]; g_e = ge_a[t];
        }
        int64_t m = q_off[t + 1] - q_off[t];
        int64_t L = (m + p - 1) / p;
        uint16_t *prof = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)(ns * L * p + 1));
        int64_t bias = swo_build_profile(flat_q + q_off[t], m, s, ns, p, prof);
        uint8_t sat = 0;
        int64_t cnt[7];
        const uint8_t *r = flat_r + r_off[t];
        int64_t n = r_off[t + 1] - r_off[t];
        if (kernel_id == 2)
            score[t] = swo_align_scan(prof, L, p, r, n, bias, g_o, g_e, &sat, cnt, NULL);
        else
            score[t] = swo_align_lazyf(prof, L, p, r, n, bias, g_o, g_e, kernel_id == 0, &sat, cnt,
                                       NULL);
        if (overflow) overflow[t] = sat;
        if (counters) memcpy(counters + 7 * t, cnt, sizeof cnt);
        free(prof);
    }
}

/* One query profile against many targets with a striped reference kernel
 * (the reference's align_prebuilt, src/_compiled.py:588-607, in a loop). */
void swo_db_striped(int32_t kernel_id, const uint16_t *prof, int64_t L, int64_t p, int64_t bias,
                    int64_t ntargets, const uint8_t *flat_r, const int64_t *r_off, int64_t go,
                    int64_t ge, int64_t *score, uint8_t *overflow, int32_t nthreads) {
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t t = 0; t < ntargets; t++) {
        uint8_t sat = 0;
        const uint8_t *r = flat_r + r_off[t];
        int64_t n = r_off[t + 1] - r_off[t];
        if (kernel_id == 2)
            score[t] = swo_align_scan(prof, L, p, r, n, bias, go, ge, &sat, NULL, NULL);
        else
            score[t] = swo_align_lazyf(prof, L, p, r, n, bias, go, ge, kernel_id == 0, &sat, NULL,
                                       NULL);
        if (overflow) overflow[t] = sat;
    }
}

/* ---- start coordinates (extension: SURVEY 8(f) item 4; the reference lists
 *      traceback as a non-goal) ----
 * Given the score and first-max end cell of an optimal local alignment, the
 * start is found by an anchored Gotoh DP over the reversed prefixes (reversed
 * reference index i' = ref_end - i outer, reversed query index q' = query_end - q
 * inner) whose only start is the end pair itself: no clamping at 0, boundary
 * -inf except the virtual origin.  The first cell in that loop order whose
 * anchored score equals `score` is the alignment's first aligned pair, i.e. the
 * start of the optimal alignment ending at the end cell that is shortest in the
 * reference, ties to the largest query start.  Such a cell is a diagonal cell
 * (a gap cell is strictly below its predecessor).  Returns 0, or -1 when no
 * anchored alignment reaches `score` (inconsistent inputs). */
int32_t swo_start_coords(const uint8_t *query, const uint8_t *ref, const int8_t *sub,
                         int32_t n_sym, int64_t go, int64_t ge, int64_t score, int32_t ref_end,
                         int32_t query_end, int32_t *ref_start, int32_t *query_start) {
    *ref_start = -1;
    *query_start = -1;
    if (score <= 0 || ref_end < 0 || query_end < 0) return score <= 0 ? 0 : -1;
    const int64_t NEG = -((int64_t)1 << 60);
    const int64_t mq = (int64_t)query_end + 1, nr = (int64_t)ref_end + 1;
    int64_t *h = (int64_t *)malloc((size_t)(mq + 1) * sizeof(int64_t));  /* h[k]: q' = k-1 */
    int64_t *e = (int64_t *)malloc((size_t)(mq + 1) * sizeof(int64_t));
    for (int64_t k = 0; k <= mq; k++) { h[k] = NEG; e[k] = NEG; }
    h[0] = 0; /* row i' = -1: the virtual origin, diagonal of (0, 0) */
    int32_t rc = -1;
    for (int64_t ip = 0; ip < nr && rc < 0; ip++) {
        const int8_t *row = sub + (int64_t)ref[ref_end - ip] * n_sym;
        int64_t diag = h[0];
        h[0] = NEG; /* column q' = -1 for rows i' >= 0 */
        int64_t f = NEG, hleft = NEG;
        for (int64_t k = 1; k <= mq; k++) {
            int64_t ev = e[k] - ge, t = h[k] - go;
            if (t > ev) ev = t;
            int64_t fv = f - ge;
            t = hleft - go;
            if (t > fv) fv = t;
            int64_t u = diag + (int64_t)row[query[query_end - (k - 1)]];
            int64_t hv = u;
            if (ev > hv) hv = ev;
            if (fv > hv) hv = fv;
            diag = h[k];
            h[k] = hv;
            e[k] = ev;
            f = fv;
            hleft = hv;
            if (hv == score) {
                *ref_start = (int32_t)(ref_end - ip);
                *query_start = (int32_t)(query_end - (k - 1));
                rc = 0;
                break;
            }
        }
    }
    free(h);
    free(e);
    return rc;
}

/* Batch form: pair t = (query t, target t) of CSR inputs with its hit. */
void swo_batch_starts(int64_t npairs, const uint8_t *flat_q, const int64_t *q_off,
                      const uint8_t *flat_r, const int64_t *r_off, const int8_t *sub,
                      int32_t n_sym, int64_t go, int64_t ge, const int64_t *score,
                      const int32_t *ref_end, const int32_t *query_end, int32_t *ref_start,
                      int32_t *query_start, int32_t nthreads) {
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t t = 0; t < npairs; t++)
        swo_start_coords(flat_q + q_off[t], flat_r + r_off[t], sub, n_sym, go, ge, score[t],
                         ref_end[t], query_end[t], ref_start + t, query_start + t);
}
