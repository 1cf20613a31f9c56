/*
 * oracle/s2o_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, fp64, single-threaded restatement of the reference S2O hot path
 * (/root/reference/proj). It is the CHECKER for the CUDA product path: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * The product library (paper_2602_22575_b200/lib/libs2o_cuda.so) never links
 * or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 * (a) the golden vectors frozen in the reference's own unit tests
 *     (tests/test_plan.cpp, tests/test_kernel.cpp, tests/test_tensor.cpp,
 *      tests/test_attention.cpp) re-expressed in tests/golden/, and
 * (b) the compiled reference itself (oracle/_ref/libs2o_ref.so, built from
 *     the unmodified sources by oracle/Makefile) on randomized inputs,
 * requiring bit-identical plans/traces and outputs.
 *
 * Flat layouts are identical to oracle/ref_capi.cpp:
 *   tensors fp32 [Z,H,L,D]; q_perm int64 [Z*H][N][S]; kv_perm int64 packed
 *   per (z,h) with segment n at S*n*(n-1)/2; trace int64 [Z*H][N][ceil(S/b_m)];
 *   pass buffers fp64 acc [Z,H,L,D], ell/m [Z,H,L].
 *
 * Compile with -ffp-contract=off (no FMA contraction) so every fp64
 * expression rounds exactly like the reference build (x86-64 baseline ISA).
 */
#include <math.h>
#include <float.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[160];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }

/* kNegInfSentinel: proj/include/s2o/tensor.hpp:86-87 */
static const double kSentinel = (double)(-FLT_MAX);

/* std::max(a, b) == (a < b) ? b : a -- keeps NaN semantics of the reference */
static double std_max(double a, double b) { return (a < b) ? b : a; }

/* ---------------------------------------------------------------- segments */
/* SegmentConfig::for_sequence proj/src/plan.cpp:35-44 */
typedef struct {
    int64_t seg_len, seg_count, last_len;
} seg_cfg;

static int seg_for_sequence(int64_t l, int64_t s, seg_cfg* out) {
    if (s < 1 || s > l) return fail(1, "segment length must satisfy 1 <= S <= L");
    out->seg_len = s;
    out->seg_count = (l + s - 1) / s;
    out->last_len = l - (out->seg_count - 1) * s;
    return 0;
}
static int64_t seg_len_of(const seg_cfg* c, int64_t n) {
    return (n + 1 == c->seg_count) ? c->last_len : c->seg_len;
}
static int64_t kv_packed_per_head(const seg_cfg* c) {
    return c->seg_len * c->seg_count * (c->seg_count - 1) / 2;
}

/* dot_f proj/src/plan.cpp:14-20, dot_qk proj/src/attention.cpp:14-20 */
static double dot_f(const float* a, const float* b, int64_t d) {
    double acc = 0.0;
    for (int64_t i = 0; i < d; ++i) acc += (double)a[i] * (double)b[i];
    return acc;
}

/* ------------------------------------------------------------------ argsort */
/* argsort_desc_stable proj/src/tensor.cpp:43-61: sentinel mapping, then a
 * stable descending sort == total order (key desc, index asc). */
static const double* g_sort_keys;
static int cmp_desc_stable(const void* pa, const void* pb) {
    const int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
    const double ka = g_sort_keys[a], kb = g_sort_keys[b];
    if (ka > kb) return -1;
    if (kb > ka) return 1;
    return (a < b) ? -1 : (a > b);
}

int orc_argsort_desc_stable(const double* scores, int64_t n, int64_t* out) {
    if (n <= 0) return fail(1, "empty score vector");
    double* keys = (double*)malloc((size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        const double s = scores[i];
        keys[i] = (isnan(s) || s < kSentinel) ? kSentinel : s;
        out[i] = i;
    }
    g_sort_keys = keys;
    qsort(out, (size_t)n, sizeof(int64_t), cmp_desc_stable);
    free(keys);
    return 0;
}

/* mean_pool_rows proj/src/tensor.cpp:63-84: fp64 row-sequential sum, x (1/len) */
static void mean_pool_rows(const float* t, int64_t d, int64_t row_begin, int64_t row_end,
                           float* out) {
    double* acc = (double*)calloc((size_t)d, sizeof(double));
    for (int64_t r = row_begin; r < row_end; ++r) {
        const float* src = t + r * d;
        for (int64_t i = 0; i < d; ++i) acc[i] += (double)src[i];
    }
    const double inv = 1.0 / (double)(row_end - row_begin);
    for (int64_t i = 0; i < d; ++i) out[i] = (float)(acc[i] * inv);
    free(acc);
}

/* segment_representatives proj/src/plan.cpp:46-67 */
int orc_segment_representatives(const float* q, const float* k, int64_t z, int64_t h, int64_t l,
                                int64_t d, int64_t seg_len, float* q_mean, float* k_mean) {
    seg_cfg seg = {0, 0, 0};
    int rc = seg_for_sequence(l, seg_len, &seg);
    if (rc) return rc;
    for (int64_t zh = 0; zh < z * h; ++zh) {
        for (int64_t n = 0; n < seg.seg_count; ++n) {
            const int64_t lo = n * seg.seg_len, hi = lo + seg_len_of(&seg, n);
            mean_pool_rows(q + zh * l * d, d, lo, hi, q_mean + (zh * seg.seg_count + n) * d);
            mean_pool_rows(k + zh * l * d, d, lo, hi, k_mean + (zh * seg.seg_count + n) * d);
        }
    }
    return 0;
}

/* build_plan proj/src/plan.cpp:140-162 with rank_queries (:69-101) and
 * rank_prefix_keys (:103-138); guide = k_mean[z,h,segment 0] (:145-151). */
int orc_build_plan(const float* q, const float* k, int64_t z, int64_t h, int64_t l, int64_t d,
                   int64_t seg_len, int64_t* q_perm, int64_t* kv_perm, int64_t* cost2) {
    seg_cfg seg = {0, 0, 0};
    int rc = seg_for_sequence(l, seg_len, &seg);
    if (rc) return rc;
    const int64_t N = seg.seg_count, S = seg.seg_len;
    float* q_mean = (float*)malloc((size_t)(N * d) * sizeof(float));
    float* guide = (float*)malloc((size_t)d * sizeof(float));
    double* scores = (double*)malloc((size_t)l * sizeof(double));
    int64_t dots = 0;
    for (int64_t zh = 0; zh < z * h; ++zh) {
        const float* qh = q + zh * l * d;
        const float* kh = k + zh * l * d;
        for (int64_t n = 0; n < N; ++n) {
            const int64_t lo = n * S, hi = lo + seg_len_of(&seg, n);
            mean_pool_rows(qh, d, lo, hi, q_mean + n * d);
        }
        mean_pool_rows(kh, d, 0, seg_len_of(&seg, 0), guide);
        int64_t slice_dots = 0;
        /* rank_queries: s_Q = Q row . guide, per-segment argsort (segment-local ids) */
        for (int64_t n = 0; n < N; ++n) {
            const int64_t len = seg_len_of(&seg, n);
            for (int64_t s = 0; s < len; ++s) scores[s] = dot_f(qh + (n * S + s) * d, guide, d);
            slice_dots += len;
            if (q_perm) orc_argsort_desc_stable(scores, len, q_perm + (zh * N + n) * S);
        }
        /* rank_prefix_keys: s_K = q_mean[n] . K[t], t < nS, absolute ids */
        for (int64_t n = 1; n < N; ++n) {
            const int64_t prefix = n * S;
            for (int64_t t = 0; t < prefix; ++t) scores[t] = dot_f(q_mean + n * d, kh + t * d, d);
            slice_dots += prefix;
            if (kv_perm)
                orc_argsort_desc_stable(scores, prefix,
                                        kv_perm + zh * kv_packed_per_head(&seg) + S * n * (n - 1) / 2);
        }
        dots = slice_dots;
    }
    if (cost2) {
        cost2[0] = dots; /* RankingCost is per slice (plan.hpp:71-76) */
        cost2[1] = dots;
    }
    free(q_mean);
    free(guide);
    free(scores);
    return 0;
}

/* --------------------------------------------------------------- os_update */
/* proj/src/attention.cpp:31-88. states: m[rows], ell[rows], acc[rows*d].
 * q rows / k,v keys are given as row pointers (gathered views). */
static void os_update(int64_t rows, int64_t keys, int64_t d, double* m, double* ell, double* acc,
                      const float* const* q_rows, const float* const* k_rows,
                      const float* const* v_rows, const uint8_t* mask, double* scratch) {
    const double scale = 1.0 / sqrt((double)d);
    for (int64_t r = 0; r < rows; ++r) {
        const uint8_t* mrow = mask ? mask + r * keys : NULL;
        double tile_max = -INFINITY;
        int any = 0;
        for (int64_t j = 0; j < keys; ++j) {
            if (mrow && mrow[j] == 0) continue;
            const double s = dot_f(q_rows[r], k_rows[j], d) * scale;
            scratch[j] = s;
            tile_max = std_max(tile_max, s);
            any = 1;
        }
        if (!any) continue;
        const double m_new = std_max(m[r], tile_max);
        const double rescale = exp(m[r] - m_new);
        double ell_new = ell[r] * rescale;
        double* a = acc + r * d;
        for (int64_t i = 0; i < d; ++i) a[i] *= rescale;
        for (int64_t j = 0; j < keys; ++j) {
            if (mrow && mrow[j] == 0) continue;
            const double w = exp(scratch[j] - m_new);
            ell_new += w;
            const float* vr = v_rows[j];
            for (int64_t i = 0; i < d; ++i) a[i] += w * (double)vr[i];
        }
        m[r] = m_new;
        ell[r] = ell_new;
    }
}

/* early_stop_check proj/src/kernel.cpp:220-234 */
int orc_early_stop_check(const double* prev, const double* nw, int64_t n, double tau, int* stop) {
    if (n <= 0) return fail(1, "normalizer vectors must align");
    double max_gain = -INFINITY;
    for (int64_t r = 0; r < n; ++r) {
        if (prev[r] <= 0.0) return fail(1, "uninitialized state");
        max_gain = std_max(max_gain, (nw[r] - prev[r]) / prev[r]);
    }
    *stop = max_gain < tau;
    return 0;
}

/* KernelConfig::validate proj/src/kernel.cpp:166-182 */
static int validate_cfg(int64_t l, int64_t seg_len, double tau, int64_t b_m, int64_t b_n,
                        int q_reorder, int fused, int64_t local_window) {
    if (seg_len < 1 || seg_len > l) return fail(1, "segment length must satisfy 1 <= S <= L");
    if (!(tau >= 0.0)) return fail(1, "tau must be >= 0");
    if (b_m < 1 || b_n < 1) return fail(1, "tile sizes must be >= 1");
    if (local_window > seg_len) return fail(1, "local window must satisfy W <= S");
    if (fused && q_reorder) return fail(1, "fused variant requires q_reorder = false");
    return 0;
}

typedef struct {
    int64_t d, cap;
    double *m, *ell, *acc;    /* committed state */
    double *cm, *cell, *cacc; /* candidate */
    double *prev, *nw, *scratch;
    const float **qr, **kr, **vr;
    uint8_t* mask;
} tile_ws;

static void ws_init(tile_ws* w, int64_t b_m, int64_t b_n, int64_t d) {
    w->d = d;
    w->cap = b_m;
    w->m = malloc((size_t)b_m * sizeof(double));
    w->ell = malloc((size_t)b_m * sizeof(double));
    w->acc = malloc((size_t)(b_m * d) * sizeof(double));
    w->cm = malloc((size_t)b_m * sizeof(double));
    w->cell = malloc((size_t)b_m * sizeof(double));
    w->cacc = malloc((size_t)(b_m * d) * sizeof(double));
    w->prev = malloc((size_t)b_m * sizeof(double));
    w->nw = malloc((size_t)b_m * sizeof(double));
    w->scratch = malloc((size_t)b_n * sizeof(double));
    w->qr = malloc((size_t)b_m * sizeof(float*));
    w->kr = malloc((size_t)b_n * sizeof(float*));
    w->vr = malloc((size_t)b_n * sizeof(float*));
    w->mask = malloc((size_t)(b_m * b_n));
}
static void ws_free(tile_ws* w) {
    free(w->m); free(w->ell); free(w->acc); free(w->cm); free(w->cell); free(w->cacc);
    free(w->prev); free(w->nw); free(w->scratch); free(w->qr); free(w->kr); free(w->vr);
    free(w->mask);
}
static void ws_reset_state(tile_ws* w, int64_t rows) {
    for (int64_t r = 0; r < rows; ++r) {
        w->m[r] = -INFINITY;
        w->ell[r] = 0.0;
    }
    memset(w->acc, 0, (size_t)(rows * w->d) * sizeof(double));
}

/* segment_causal_tile proj/src/kernel.cpp:36-71 */
static void segment_causal_tile(tile_ws* w, const float* q, const float* k, const float* v,
                                int64_t d, int64_t seg_begin, int64_t seg_rows, int64_t tile_begin,
                                int64_t tile_rows, int64_t b_n) {
    for (int64_t r = 0; r < tile_rows; ++r) w->qr[r] = q + (seg_begin + tile_begin + r) * d;
    const int64_t last_row = tile_begin + tile_rows - 1;
    for (int64_t k0 = 0; k0 <= last_row && k0 < seg_rows; k0 += b_n) {
        const int64_t kn = (b_n < seg_rows - k0) ? b_n : seg_rows - k0;
        for (int64_t j = 0; j < kn; ++j) {
            w->kr[j] = k + (seg_begin + k0 + j) * d;
            w->vr[j] = v + (seg_begin + k0 + j) * d;
        }
        if (k0 + kn - 1 <= tile_begin) {
            os_update(tile_rows, kn, d, w->m, w->ell, w->acc, w->qr, w->kr, w->vr, NULL, w->scratch);
        } else {
            for (int64_t r = 0; r < tile_rows; ++r)
                for (int64_t j = 0; j < kn; ++j) w->mask[r * kn + j] = (k0 + j <= tile_begin + r);
            os_update(tile_rows, kn, d, w->m, w->ell, w->acc, w->qr, w->kr, w->vr, w->mask,
                      w->scratch);
        }
    }
}

/* traverse_prefix proj/src/kernel.cpp:86-122; q rows already in w->qr */
static int traverse_prefix(tile_ws* w, int64_t rows, const float* k, const float* v, int64_t d,
                           const int64_t* kv, int64_t kv_len, int64_t b_n, double tau,
                           int64_t* pair_accum, int64_t* committed_out) {
    int64_t committed = 0;
    for (int64_t c0 = 0; c0 < kv_len; c0 += b_n) {
        const int64_t cn = (b_n < kv_len - c0) ? b_n : kv_len - c0;
        for (int64_t j = 0; j < cn; ++j) {
            w->kr[j] = k + kv[c0 + j] * d;
            w->vr[j] = v + kv[c0 + j] * d;
        }
        memcpy(w->cm, w->m, (size_t)rows * sizeof(double));
        memcpy(w->cell, w->ell, (size_t)rows * sizeof(double));
        memcpy(w->cacc, w->acc, (size_t)(rows * d) * sizeof(double));
        os_update(rows, cn, d, w->cm, w->cell, w->cacc, w->qr, w->kr, w->vr, NULL, w->scratch);
        for (int64_t r = 0; r < rows; ++r) {
            w->prev[r] = w->ell[r] * exp(w->m[r] - w->cm[r]);
            w->nw[r] = w->cell[r];
        }
        int stop = 0;
        int rc = orc_early_stop_check(w->prev, w->nw, rows, tau, &stop);
        if (rc) return rc;
        if (stop) break;
        memcpy(w->m, w->cm, (size_t)rows * sizeof(double));
        memcpy(w->ell, w->cell, (size_t)rows * sizeof(double));
        memcpy(w->acc, w->cacc, (size_t)(rows * d) * sizeof(double));
        ++committed;
        *pair_accum += rows * cn;
    }
    *committed_out = committed;
    return 0;
}

/* finalize_rows proj/src/kernel.cpp:149-162 */
static int finalize_rows(tile_ws* w, int64_t rows, const int64_t* global_rows, int64_t d,
                         float* out) {
    for (int64_t r = 0; r < rows; ++r) {
        if (w->ell[r] == 0.0) return fail(4, "uncovered query row");
        float* o = out + global_rows[r] * d;
        for (int64_t i = 0; i < d; ++i) o[i] = (float)(w->acc[r * d + i] / w->ell[r]);
    }
    return 0;
}

/* pass1_dense_init proj/src/kernel.cpp:184-218 */
int orc_pass1(const float* q, const float* k, const float* v, int64_t z, int64_t h, int64_t l,
              int64_t d, int64_t seg_len, double tau, int64_t b_m, int64_t b_n, int q_reorder,
              int fused, int64_t local_window, double* acc, double* ell, double* m) {
    int rc = validate_cfg(l, seg_len, tau, b_m, b_n, q_reorder, fused, local_window);
    if (rc) return rc;
    seg_cfg seg = {0, 0, 0};
    seg_for_sequence(l, seg_len, &seg);
    tile_ws w;
    ws_init(&w, b_m, b_n, d);
    for (int64_t zh = 0; zh < z * h; ++zh) {
        const float *qh = q + zh * l * d, *kh = k + zh * l * d, *vh = v + zh * l * d;
        for (int64_t n = 0; n < seg.seg_count; ++n) {
            const int64_t sb = n * seg.seg_len, rows = seg_len_of(&seg, n);
            for (int64_t t0 = 0; t0 < rows; t0 += b_m) {
                const int64_t tn = (b_m < rows - t0) ? b_m : rows - t0;
                ws_reset_state(&w, tn);
                segment_causal_tile(&w, qh, kh, vh, d, sb, rows, t0, tn, b_n);
                for (int64_t r = 0; r < tn; ++r) {
                    const int64_t slot = zh * l + sb + t0 + r;
                    ell[slot] = w.ell[r];
                    m[slot] = w.m[r];
                    memcpy(acc + slot * d, w.acc + r * d, (size_t)d * sizeof(double));
                }
            }
        }
    }
    ws_free(&w);
    return 0;
}

static int64_t pass1_pair_count(const seg_cfg* seg) {
    int64_t total = 0;
    for (int64_t n = 0; n < seg->seg_count; ++n) {
        const int64_t len = seg_len_of(seg, n);
        total += len * (len + 1) / 2;
    }
    return total;
}

/* pass2_sparse proj/src/kernel.cpp:236-298 (fused=0) and
 * fused_single_pass proj/src/kernel.cpp:300-349 (fused=1) */
static int run_pass2(int is_fused, const float* q, const float* k, const float* v, int64_t z,
                     int64_t h, int64_t l, int64_t d, int64_t seg_len, double tau, int64_t b_m,
                     int64_t b_n, int q_reorder, const double* acc, const double* ell,
                     const double* m, const int64_t* q_perm, const int64_t* kv_perm, float* out,
                     int64_t* processed, int64_t* pass1_pairs, int64_t* pass2_pairs) {
    seg_cfg seg = {0, 0, 0};
    seg_for_sequence(l, seg_len, &seg);
    const int64_t N = seg.seg_count, S = seg.seg_len, T = (S + b_m - 1) / b_m;
    tile_ws w;
    ws_init(&w, b_m, b_n, d);
    int64_t* grow = malloc((size_t)b_m * sizeof(int64_t));
    int rc = 0;
    for (int64_t zh = 0; zh < z * h && !rc; ++zh) {
        const float *qh = q + zh * l * d, *kh = k + zh * l * d, *vh = v + zh * l * d;
        int64_t p2 = 0;
        for (int64_t n = 0; n < N && !rc; ++n) {
            const int64_t sb = n * S, rows = seg_len_of(&seg, n);
            const int64_t* qp = q_perm + (zh * N + n) * S;
            const int64_t* kv = kv_perm + zh * kv_packed_per_head(&seg) + S * n * (n - 1) / 2;
            int64_t tile = 0;
            for (int64_t t0 = 0; t0 < rows && !rc; t0 += b_m, ++tile) {
                const int64_t tn = (b_m < rows - t0) ? b_m : rows - t0;
                if (is_fused) {
                    ws_reset_state(&w, tn);
                    segment_causal_tile(&w, qh, kh, vh, d, sb, rows, t0, tn, b_n);
                    for (int64_t r = 0; r < tn; ++r) grow[r] = sb + t0 + r;
                } else {
                    for (int64_t r = 0; r < tn; ++r) {
                        grow[r] = sb + (q_reorder ? qp[t0 + r] : t0 + r);
                        const int64_t slot = zh * l + grow[r];
                        w.m[r] = m[slot];
                        w.ell[r] = ell[slot];
                        memcpy(w.acc + r * d, acc + slot * d, (size_t)d * sizeof(double));
                    }
                }
                for (int64_t r = 0; r < tn; ++r) w.qr[r] = qh + grow[r] * d;
                int64_t committed = 0;
                rc = traverse_prefix(&w, tn, kh, vh, d, kv, n * S, b_n, tau, &p2, &committed);
                if (rc) break;
                processed[(zh * N + n) * T + tile] = committed;
                rc = finalize_rows(&w, tn, grow, d, out + zh * l * d);
            }
            for (; tile < T; ++tile) processed[(zh * N + n) * T + tile] = 0;
        }
        pass1_pairs[zh] = pass1_pair_count(&seg);
        pass2_pairs[zh] = p2;
    }
    free(grow);
    ws_free(&w);
    return rc;
}

int orc_pass2(const float* q, const float* k, const float* v, int64_t z, int64_t h, int64_t l,
              int64_t d, int64_t seg_len, double tau, int64_t b_m, int64_t b_n, int q_reorder,
              int fused, int64_t local_window, const double* acc, const double* ell,
              const double* m, const int64_t* q_perm, const int64_t* kv_perm, float* out,
              int64_t* processed, int64_t* pass1_pairs, int64_t* pass2_pairs) {
    int rc = validate_cfg(l, seg_len, tau, b_m, b_n, q_reorder, fused, local_window);
    if (rc) return rc;
    return run_pass2(0, q, k, v, z, h, l, d, seg_len, tau, b_m, b_n, q_reorder, acc, ell, m,
                     q_perm, kv_perm, out, processed, pass1_pairs, pass2_pairs);
}

int orc_fused(const float* q, const float* k, const float* v, int64_t z, int64_t h, int64_t l,
              int64_t d, int64_t seg_len, double tau, int64_t b_m, int64_t b_n, int q_reorder,
              int fused, int64_t local_window, const int64_t* q_perm, const int64_t* kv_perm,
              float* out, int64_t* processed, int64_t* pass1_pairs, int64_t* pass2_pairs) {
    if (!fused || q_reorder) return fail(1, "fused variant requires fused = true, q_reorder = false");
    int rc = validate_cfg(l, seg_len, tau, b_m, b_n, q_reorder, fused, local_window);
    if (rc) return rc;
    return run_pass2(1, q, k, v, z, h, l, d, seg_len, tau, b_m, b_n, 0, NULL, NULL, NULL, q_perm,
                     kv_perm, out, processed, pass1_pairs, pass2_pairs);
}

/* s2o_attention proj/src/kernel.cpp:351-369 */
int orc_attention(const float* q, const float* k, const float* v, int64_t z, int64_t h, int64_t l,
                  int64_t d, int64_t seg_len, double tau, int64_t b_m, int64_t b_n, int q_reorder,
                  int fused, int64_t local_window, float* out, int64_t* q_perm, int64_t* kv_perm,
                  int64_t* processed, int64_t* pass1_pairs, int64_t* pass2_pairs, int64_t* cost2) {
    int rc = validate_cfg(l, seg_len, tau, b_m, b_n, q_reorder, fused, local_window);
    if (rc) return rc;
    rc = orc_build_plan(q, k, z, h, l, d, seg_len, q_perm, kv_perm, cost2);
    if (rc) return rc;
    if (fused)
        return orc_fused(q, k, v, z, h, l, d, seg_len, tau, b_m, b_n, q_reorder, fused,
                         local_window, q_perm, kv_perm, out, processed, pass1_pairs, pass2_pairs);
    const size_t rows = (size_t)(z * h * l);
    double* acc = malloc(rows * (size_t)d * sizeof(double));
    double* ell = malloc(rows * sizeof(double));
    double* m = malloc(rows * sizeof(double));
    rc = orc_pass1(q, k, v, z, h, l, d, seg_len, tau, b_m, b_n, q_reorder, fused, local_window, acc,
                   ell, m);
    if (!rc)
        rc = orc_pass2(q, k, v, z, h, l, d, seg_len, tau, b_m, b_n, q_reorder, fused, local_window,
                       acc, ell, m, q_perm, kv_perm, out, processed, pass1_pairs, pass2_pairs);
    free(acc);
    free(ell);
    free(m);
    return rc;
}

/* dense_causal_attention proj/src/attention.cpp:90-125 (the MSE reference).
 * rows [row_begin, row_end) only, so tests can spot-check long sequences. */
int orc_dense_causal_rows(const float* q, const float* k, const float* v, int64_t z, int64_t h,
                          int64_t l, int64_t d, int64_t row_begin, int64_t row_end, float* out) {
    const double scale = 1.0 / sqrt((double)d);
    double* scores = malloc((size_t)l * sizeof(double));
    double* acc = malloc((size_t)d * sizeof(double));
    for (int64_t zh = 0; zh < z * h; ++zh) {
        const float *qh = q + zh * l * d, *kh = k + zh * l * d, *vh = v + zh * l * d;
        for (int64_t i = row_begin; i < row_end; ++i) {
            double row_max = -INFINITY;
            for (int64_t j = 0; j <= i; ++j) {
                scores[j] = dot_f(qh + i * d, kh + j * d, d) * scale;
                row_max = std_max(row_max, scores[j]);
            }
            double denom = 0.0;
            memset(acc, 0, (size_t)d * sizeof(double));
            for (int64_t j = 0; j <= i; ++j) {
                const double w = exp(scores[j] - row_max);
                denom += w;
                for (int64_t t = 0; t < d; ++t) acc[t] += w * (double)vh[j * d + t];
            }
            float* o = out + (zh * (row_end - row_begin) + (i - row_begin)) * d;
            for (int64_t t = 0; t < d; ++t) o[t] = (float)(acc[t] / denom);
        }
    }
    free(scores);
    free(acc);
    return 0;
}

/* Softmax-weighted value sum over an explicit visible key set:
 * proj/tests/oracles.hpp:30-54 (masked_softmax_row). */
int orc_masked_softmax_row(const float* q_row, const float* k, const float* v, int64_t d,
                           const int64_t* visible, int64_t nvis, double* out) {
    const double scale = 1.0 / sqrt((double)d);
    double* s = malloc((size_t)(nvis > 0 ? nvis : 1) * sizeof(double));
    double mx = -INFINITY;
    for (int64_t t = 0; t < nvis; ++t) {
        s[t] = dot_f(q_row, k + visible[t] * d, d) * scale;
        mx = std_max(mx, s[t]);
    }
    double denom = 0.0;
    for (int64_t t = 0; t < nvis; ++t) {
        s[t] = exp(s[t] - mx);
        denom += s[t];
    }
    for (int64_t i = 0; i < d; ++i) out[i] = 0.0;
    for (int64_t t = 0; t < nvis; ++t)
        for (int64_t i = 0; i < d; ++i) out[i] += s[t] / denom * (double)v[visible[t] * d + i];
    free(s);
    return 0;
}

/* Stop-decision evidence, the restatement of ref_tile_gains (ref_capi.cpp):
 * max_r (new - prev) / prev for each of the first nchunks kv_perm chunks of ONE query tile with
 * every chunk committed (traverse_prefix proj/src/kernel.cpp:86-122 without the break); each
 * row's pass-1 state is its own segment_causal_tile scan (kernel.cpp:36-71). rows: segment-local
 * rows of the tile; qh/kh/vh one head [L, D]; kv_seg: kv_perm[n] (n*S absolute ids). */
int orc_tile_gains(const float* qh, const float* kh, const float* vh, int64_t l, int64_t d, int64_t seg_len,
                   int64_t b_n, const int64_t* rows, int64_t tn, int64_t n, const int64_t* kv_seg,
                   int64_t nchunks, double* gains) {
    tile_ws w;
    ws_init(&w, tn, b_n, d);
    ws_reset_state(&w, tn);
    const int64_t sb = n * seg_len, kv_len = n * seg_len;
    const int64_t seg_rows = (seg_len < l - sb) ? seg_len : l - sb;
    for (int64_t r = 0; r < tn; ++r) {
        const int64_t rr = rows[r];
        const float* qr[1] = {qh + (sb + rr) * d};
        for (int64_t k0 = 0; k0 <= rr && k0 < seg_rows; k0 += b_n) {
            const int64_t kn = (b_n < seg_rows - k0) ? b_n : seg_rows - k0;
            for (int64_t j = 0; j < kn; ++j) {
                w.kr[j] = kh + (sb + k0 + j) * d;
                w.vr[j] = vh + (sb + k0 + j) * d;
                w.mask[j] = (k0 + j <= rr);
            }
            os_update(1, kn, d, w.m + r, w.ell + r, w.acc + r * d, qr, w.kr, w.vr,
                      (k0 + kn - 1 <= rr) ? NULL : w.mask, w.scratch);
        }
        w.qr[r] = qh + (sb + rr) * d;
    }
    for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t c0 = c * b_n;
        if (c0 >= kv_len) {
            gains[c] = NAN;
            continue;
        }
        const int64_t cn = (b_n < kv_len - c0) ? b_n : kv_len - c0;
        for (int64_t j = 0; j < cn; ++j) {
            w.kr[j] = kh + kv_seg[c0 + j] * d;
            w.vr[j] = vh + kv_seg[c0 + j] * d;
        }
        memcpy(w.cm, w.m, (size_t)tn * sizeof(double));
        memcpy(w.cell, w.ell, (size_t)tn * sizeof(double));
        memcpy(w.cacc, w.acc, (size_t)(tn * d) * sizeof(double));
        os_update(tn, cn, d, w.cm, w.cell, w.cacc, w.qr, w.kr, w.vr, NULL, w.scratch);
        double max_gain = -INFINITY;
        for (int64_t r = 0; r < tn; ++r) {
            const double prev = w.ell[r] * exp(w.m[r] - w.cm[r]);
            max_gain = std_max(max_gain, (w.cell[r] - prev) / prev);
        }
        gains[c] = max_gain;
        memcpy(w.m, w.cm, (size_t)tn * sizeof(double));
        memcpy(w.ell, w.cell, (size_t)tn * sizeof(double));
        memcpy(w.acc, w.cacc, (size_t)(tn * d) * sizeof(double));
    }
    ws_free(&w);
    return 0;
}
