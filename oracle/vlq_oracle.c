/*
 * vlq_oracle.c -- CPU restatement of the reference VLQ-ADC hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.  The
 * product (paper_1901_00275_b200/, libvlqgpu.so) never links or calls it.
 *
 * It restates, in plain C with IEEE fp32 and no FMA contraction
 * (-ffp-contract=off), the arithmetic of the reference implementation at
 * /root/reference/proj (see Appendix A of SURVEY.md).  Each function cites the
 * reference lines it follows.  Parity of this restatement is pinned against
 * the reference itself (oracle/_ref, built from the reference sources by
 * oracle/Makefile) and against golden vectors in tests/golden/.
 *
 * Index layout (same SoA layout the GPU engine uses on device):
 *   centroids[k*dim], nbr[k*n], elen[k*n], pq[m*256*dsub], t2[m*256],
 *   t3[k*m*256], list_off[k*n+1] (u64), ids[N] (u32), codes[N*m], lambdas[N].
 * Cell c = i*n + j (proj/include/vlq/index.hpp:62-64).
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>
#include <unistd.h>

#define KSUB 256u

typedef struct {
    uint32_t dim, k, n, m;
    int clamp;
    float lo, hi;
    const float* centroids;
    const uint32_t* nbr;
    const float* elen;
    const float* pq;
    const float* t2;
    const float* t3;
    const uint64_t* list_off;
    const uint32_t* ids;
    const uint8_t* codes;
    const uint8_t* lambdas;
} vo_index;

static __thread char g_err[256];

const char* vo_last_error(void) { return g_err; }

static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return -1;
}

/* ---- numeric primitives: proj/src/vecset.cpp:22-45 ---------------------- */
static float vo_sqdist(const float* a, const float* b, size_t d) {
    float acc = 0.0f;
    for (size_t i = 0; i < d; i++) {
        float diff = a[i] - b[i];
        acc += diff * diff;
    }
    return acc;
}

static float vo_sqnorm(const float* a, size_t d) {
    float acc = 0.0f;
    for (size_t i = 0; i < d; i++) acc += a[i] * a[i];
    return acc;
}

static float vo_dot(const float* a, const float* b, size_t d) {
    float acc = 0.0f;
    for (size_t i = 0; i < d; i++) acc += a[i] * b[i];
    return acc;
}

/* ---- line quantization: proj/src/line_quant.cpp:9-22 -------------------- */
static float clampf_std(float v, float lo, float hi) { /* std::clamp semantics */
    return (v < lo) ? lo : ((hi < v) ? hi : v);
}

static int vo_line_lambda(float a, float b, float c, float* out) {
    if (!(c > 0)) return fail("line_lambda: degenerate edge (c == 0)");
    *out = 0.5f * (a + c - b) / c;
    return 0;
}

static float vo_line_sqdist(float a, float b, float c, float lambda) {
    return (1.0f - lambda) * a + (lambda * lambda - lambda) * c + lambda * b;
}

/* ---- lambda byte quantizer: proj/src/index.cpp:12-21 -------------------- */
uint8_t vo_quantize_lambda(float lambda, float lo, float hi) {
    float clamped = clampf_std(lambda, lo, hi);
    float step = (hi - lo) / 256.0f;
    int level = (int)((clamped - lo) / step);
    if (level < 0) level = 0;
    if (level > 255) level = 255;
    return (uint8_t)level;
}

float vo_dequantize_lambda(uint8_t b, float lo, float hi) {
    return lo + ((float)b + 0.5f) * (hi - lo) / 256.0f;
}

/* ---- tables: proj/src/pq.cpp:11-18 (t2), proj/src/index.cpp:54-74 (t3) -- */
int vo_compute_t2(const float* pq, uint32_t dim, uint32_t m, float* t2) {
    if (m == 0 || dim % m) return fail("compute_t2: m must divide dim");
    uint32_t dsub = dim / m;
    for (uint32_t p = 0; p < m; p++)
        for (uint32_t j = 0; j < KSUB; j++)
            t2[(size_t)p * KSUB + j] = vo_sqnorm(pq + ((size_t)p * KSUB + j) * dsub, dsub);
    return 0;
}

int vo_compute_t3(const float* centroids, uint32_t k, uint32_t dim, const float* pq, uint32_t m,
                  float* t3) {
    if (m == 0 || dim % m) return fail("compute_t3: dimension mismatch");
    uint32_t dsub = dim / m;
    for (int64_t i = 0; i < (int64_t)k; i++)
        for (uint32_t p = 0; p < m; p++) {
            const float* slice = centroids + (size_t)i * dim + (size_t)p * dsub;
            float* dst = t3 + ((size_t)i * m + p) * KSUB;
            for (uint32_t j = 0; j < KSUB; j++)
                dst[j] = vo_dot(slice, pq + ((size_t)p * KSUB + j) * dsub, dsub);
        }
    return 0;
}

/* ---- total-order keys ----------------------------------------------------
 * The reference comparators are (dist, id) (search.cpp:28-33, 126-129) and
 * (dist, centroid_id, edge_rank) == (dist, cell id) (search.cpp:63-71).  All
 * compare floats with < / ==, so -0 == +0; the key canonicalises -0 to +0
 * and maps the float to an order-preserving u32 in the high word.           */
static inline uint64_t fkey(float f, uint32_t idx) {
    uint32_t u;
    if (f == 0.0f) f = 0.0f;
    memcpy(&u, &f, 4);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ((uint64_t)u << 32) | idx;
}

static inline float key_float(uint64_t key) {
    uint32_t u = (uint32_t)(key >> 32);
    u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return (x > y) - (x < y);
}

static void swap64(uint64_t* a, uint64_t* b) {
    uint64_t t = *a;
    *a = *b;
    *b = t;
}

/* Moves the `keep` smallest keys of v[0..len) to the front, sorted
 * ascending (equivalent to std::partial_sort under a total order). */
static void select_smallest(uint64_t* v, size_t len, size_t keep) {
    if (keep > len) keep = len;
    if (keep == 0) return;
    if (keep < len) { /* Hoare quickselect for position keep-1 on [lo, hi] */
        int64_t lo = 0, hi = (int64_t)len - 1, target = (int64_t)keep - 1;
        while (lo < hi) {
            uint64_t pivot = v[lo + (hi - lo) / 2];
            int64_t i = lo - 1, j = hi + 1;
            for (;;) {
                do i++; while (v[i] < pivot);
                do j--; while (v[j] > pivot);
                if (i >= j) break;
                swap64(&v[i], &v[j]);
            }
            if (target <= j) hi = j;
            else lo = j + 1;
        }
    }
    qsort(v, keep, sizeof(uint64_t), cmp_u64);
}

/* ---- QueryParams::w2: proj/include/vlq/search.hpp:16-20 ------------------ */
uint32_t vo_w2(uint32_t w1, float alpha, uint32_t n) {
    uint32_t full = w1 * n;
    uint32_t w = (uint32_t)((double)alpha * full);
    return w == 0 ? 1 : (w > full ? full : w);
}

/* ---- adc_distance: proj/src/search.cpp:92-120 ---------------------------- */
static float vo_adc(const vo_index* ix, const uint8_t* code, uint8_t lambda_byte, uint32_t i,
                    uint32_t j, const float* ws, const float* t5) {
    uint32_t s = ix->nbr[(size_t)i * ix->n + j];
    float lam = vo_dequantize_lambda(lambda_byte, ix->lo, ix->hi);
    float d = vo_line_sqdist(ws[i], ws[s], ix->elen[(size_t)i * ix->n + j], lam);
    float sum2 = 0, sum3 = 0, sum4 = 0, sum5 = 0;
    for (uint32_t p = 0; p < ix->m; p++) {
        uint8_t c = code[p];
        sum2 += ix->t2[(size_t)p * KSUB + c];
        sum3 += ix->t3[((size_t)i * ix->m + p) * KSUB + c];
        sum4 += ix->t3[((size_t)s * ix->m + p) * KSUB + c];
        sum5 += t5[(size_t)p * KSUB + c];
    }
    return d + sum2 + 2.0f * (1.0f - lam) * sum3 + 2.0f * lam * sum4 - 2.0f * sum5;
}

/* ---- search_query: proj/src/search.cpp:142-167 (+ stages :11-140) ------- */
typedef struct {
    float* ws;      /* k   (QueryWorkspace::centroid_sqdists) */
    float* t5;      /* m*256 (QueryWorkspace::t5) */
    uint64_t* keys; /* max(k, w1*n) */
    uint64_t* cand; /* candidates (growable) */
    size_t cand_cap;
} vo_scratch;

/* top_in (nullable): the query's top-w1 regions from an earlier
 * first-level pass (the staged / query-split search); top_out (nullable)
 * receives them; out_ids == NULL stops after the first level.
 * sel_out / ab_out (nullable): the w2 selected cells of second_level_rank
 * and their (a, b) = (ws[i], ws[nbr]) (the select-split hand-off; with
 * out_ids == NULL the search stops there).  sel_in / ab_in (nullable): start
 * from such a selection -- first_level_scan and second_level_rank are
 * skipped and ws holds ONLY the handed-over a and b values, which proves the
 * hand-off carries everything the later stages read. */
static int search_one(const vo_index* ix, const float* y, uint32_t w1, uint32_t w2, uint32_t topk,
                      vo_scratch* s, int64_t* out_ids, float* out_d, uint64_t* scanned,
                      const uint32_t* top_in, uint32_t* top_out, const uint32_t* sel_in, const float* ab_in,
                      uint32_t* sel_out, float* ab_out) {
    const uint32_t k = ix->k, n = ix->n, m = ix->m, dim = ix->dim, dsub = dim / m;
    if (sel_in) {
        for (uint32_t i = 0; i < k; i++) s->ws[i] = NAN;
        for (uint32_t r = 0; r < w2; r++) {
            const uint32_t cell = sel_in[r];
            s->keys[r] = cell;
            s->ws[cell / n] = ab_in[2 * (size_t)r];
            s->ws[ix->nbr[cell]] = ab_in[2 * (size_t)r + 1];
        }
        goto term5;
    }
    /* first_level_scan (search.cpp:11-36) */
    for (uint32_t i = 0; i < k; i++) {
        s->ws[i] = vo_sqdist(y, ix->centroids + (size_t)i * dim, dim);
        s->keys[i] = fkey(s->ws[i], i);
    }
    uint32_t* top = (uint32_t*)malloc(sizeof(uint32_t) * w1);
    if (top_in) {
        memcpy(top, top_in, sizeof(uint32_t) * w1);
    } else {
        select_smallest(s->keys, k, w1);
        for (uint32_t r = 0; r < w1; r++) top[r] = (uint32_t)s->keys[r];
    }
    if (top_out) memcpy(top_out, top, sizeof(uint32_t) * w1);
    if (!out_ids && !sel_out) {
        free(top);
        return 0;
    }
    /* second_level_rank (search.cpp:38-78) */
    size_t total = (size_t)w1 * n;
    for (uint32_t r = 0; r < w1; r++) {
        uint32_t i = top[r];
        float a = s->ws[i];
        for (uint32_t j = 0; j < n; j++) {
            float b = s->ws[ix->nbr[(size_t)i * n + j]];
            float c = ix->elen[(size_t)i * n + j];
            float lam;
            if (vo_line_lambda(a, b, c, &lam)) {
                free(top);
                return -1;
            }
            lam = clampf_std(lam, 0.0f, 1.0f);
            s->keys[(size_t)r * n + j] = fkey(vo_line_sqdist(a, b, c, lam), i * n + j);
        }
    }
    free(top);
    select_smallest(s->keys, total, w2);
    if (sel_out) {
        for (uint32_t r = 0; r < w2; r++) {
            const uint32_t cell = (uint32_t)s->keys[r];
            sel_out[r] = cell;
            ab_out[2 * (size_t)r] = s->ws[cell / n];
            ab_out[2 * (size_t)r + 1] = s->ws[ix->nbr[cell]];
        }
        if (!out_ids) return 0;
    }
term5:
    /* query_term5 (search.cpp:80-90) */
    for (uint32_t p = 0; p < m; p++)
        for (uint32_t j = 0; j < KSUB; j++)
            s->t5[(size_t)p * KSUB + j] = vo_dot(y + (size_t)p * dsub, ix->pq + ((size_t)p * KSUB + j) * dsub, dsub);
    /* scan loop (search.cpp:154-162) */
    size_t nc = 0;
    for (uint32_t r = 0; r < w2; r++) {
        uint32_t cell = (uint32_t)s->keys[r];
        uint32_t i = cell / n, j = cell % n;
        uint64_t b0 = ix->list_off[cell], b1 = ix->list_off[cell + 1];
        if (nc + (b1 - b0) > s->cand_cap) {
            size_t cap = s->cand_cap ? s->cand_cap : 1024;
            while (cap < nc + (b1 - b0)) cap *= 2;
            s->cand = (uint64_t*)realloc(s->cand, cap * sizeof(uint64_t));
            s->cand_cap = cap;
        }
        for (uint64_t e = b0; e < b1; e++) {
            float d = vo_adc(ix, ix->codes + e * m, ix->lambdas[e], i, j, s->ws, s->t5);
            s->cand[nc++] = fkey(d, ix->ids[e]);
        }
    }
    *scanned = nc;
    /* select_topk (search.cpp:122-140) + padding (bindings.cpp:116-124) */
    select_smallest(s->cand, nc, topk);
    for (uint32_t r = 0; r < topk; r++) {
        if (r < nc) {
            out_ids[r] = (int64_t)(uint32_t)s->cand[r];
            out_d[r] = key_float(s->cand[r]);
        } else {
            out_ids[r] = -1;
            out_d[r] = INFINITY;
        }
    }
    return 0;
}

/* Minimal thread fan-out (the reference's parallel_for, proj/src/parallel.cpp:
 * 26-72): workers pull fixed chunks; results are independent of the thread
 * count because every item is computed independently. */
typedef struct {
    int64_t n, chunk;
    int64_t next;
    pthread_mutex_t mu;
    int err;
    char errmsg[256];
    void* ctx;
    int (*fn)(void* ctx, void* scratch, int64_t i);
    void* (*make_scratch)(void* ctx);
    void (*free_scratch)(void* scratch);
} par_job;

static void* par_worker(void* arg) {
    par_job* job = (par_job*)arg;
    void* scratch = job->make_scratch(job->ctx);
    for (;;) {
        pthread_mutex_lock(&job->mu);
        int64_t b = job->next;
        job->next += job->chunk;
        int stop = job->err;
        pthread_mutex_unlock(&job->mu);
        if (stop || b >= job->n) break;
        int64_t e = b + job->chunk < job->n ? b + job->chunk : job->n;
        for (int64_t i = b; i < e; i++) {
            if (job->fn(job->ctx, scratch, i)) {
                pthread_mutex_lock(&job->mu);
                if (!job->err) {
                    job->err = 1;
                    snprintf(job->errmsg, sizeof job->errmsg, "%s", g_err);
                }
                pthread_mutex_unlock(&job->mu);
                break;
            }
        }
    }
    job->free_scratch(scratch);
    return NULL;
}

static int par_for(int64_t n, int64_t chunk, int nthreads, void* ctx,
                   int (*fn)(void*, void*, int64_t), void* (*mk)(void*), void (*fr)(void*)) {
    par_job job;
    memset(&job, 0, sizeof job);
    job.n = n;
    job.chunk = chunk;
    job.ctx = ctx;
    job.fn = fn;
    job.make_scratch = mk;
    job.free_scratch = fr;
    pthread_mutex_init(&job.mu, NULL);
    if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    int started = 0;
    for (int t = 1; t < nthreads; t++)
        if (pthread_create(&th[started], NULL, par_worker, &job) == 0) started++;
    par_worker(&job);
    for (int t = 0; t < started; t++) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&job.mu);
    if (job.err) return fail(job.errmsg);
    return 0;
}

typedef struct {
    const vo_index* ix;
    const float* queries;
    uint32_t w1, w2, topk;
    int64_t* out_ids;
    float* out_dists;
    uint64_t* out_scanned;
    const uint32_t* top_in;
    uint32_t* top_out;
    const uint32_t* sel_in; /* select-split hand-off: [nq, w2] cells + [nq, w2, 2] (a, b) */
    const float* ab_in;
    uint32_t* sel_out;
    float* ab_out;
} search_ctx;

static void* search_scratch(void* c) {
    search_ctx* ctx = (search_ctx*)c;
    vo_scratch* s = (vo_scratch*)calloc(1, sizeof(vo_scratch));
    size_t keys_len = (size_t)ctx->w1 * ctx->ix->n > ctx->ix->k ? (size_t)ctx->w1 * ctx->ix->n : ctx->ix->k;
    s->ws = (float*)malloc(sizeof(float) * ctx->ix->k);
    s->t5 = (float*)malloc(sizeof(float) * ctx->ix->m * KSUB);
    s->keys = (uint64_t*)malloc(sizeof(uint64_t) * keys_len);
    return s;
}

static void search_scratch_free(void* p) {
    vo_scratch* s = (vo_scratch*)p;
    free(s->ws);
    free(s->t5);
    free(s->keys);
    free(s->cand);
    free(s);
}

static int search_item(void* c, void* scratch, int64_t q) {
    search_ctx* ctx = (search_ctx*)c;
    return search_one(ctx->ix, ctx->queries + (size_t)q * ctx->ix->dim, ctx->w1, ctx->w2, ctx->topk,
                      (vo_scratch*)scratch, ctx->out_ids ? ctx->out_ids + (size_t)q * ctx->topk : NULL,
                      ctx->out_dists ? ctx->out_dists + (size_t)q * ctx->topk : NULL,
                      ctx->out_scanned ? ctx->out_scanned + q : NULL,
                      ctx->top_in ? ctx->top_in + (size_t)q * ctx->w1 : NULL,
                      ctx->top_out ? ctx->top_out + (size_t)q * ctx->w1 : NULL,
                      ctx->sel_in ? ctx->sel_in + (size_t)q * ctx->w2 : NULL,
                      ctx->ab_in ? ctx->ab_in + (size_t)q * ctx->w2 * 2 : NULL,
                      ctx->sel_out ? ctx->sel_out + (size_t)q * ctx->w2 : NULL,
                      ctx->ab_out ? ctx->ab_out + (size_t)q * ctx->w2 * 2 : NULL);
}

/* search_batch (search.cpp:169-191); per-query scanned counts returned
 * individually so callers can compute roofline bytes per query. */
int vo_search(const vo_index* ix, const float* queries, uint64_t nq, uint32_t w1, float alpha,
              uint32_t topk, int64_t* out_ids, float* out_dists, uint64_t* out_scanned,
              int nthreads) {
    if (w1 == 0 || w1 > ix->k) return fail("first_level_scan: need 0 < w1 <= k");
    search_ctx ctx = {ix, queries, w1, vo_w2(w1, alpha, ix->n), topk, out_ids, out_dists, out_scanned, NULL, NULL,
                      NULL, NULL, NULL, NULL};
    return par_for((int64_t)nq, 4, nthreads, &ctx, search_item, search_scratch, search_scratch_free);
}

/* The same search split at the first-level boundary (the GPU engine's
 * vlq_engine_search_coarse_device / _fine_device): vo_first_level writes
 * the exact top-w1 of every query, vo_search_from_top runs
 * second_level_rank .. select_topk from given top-w1 lists. */
int vo_first_level(const vo_index* ix, const float* queries, uint64_t nq, uint32_t w1, uint32_t* top_out,
                   int nthreads) {
    if (w1 == 0 || w1 > ix->k) return fail("first_level_scan: need 0 < w1 <= k");
    search_ctx ctx = {ix, queries, w1, 1, 0, NULL, NULL, NULL, NULL, top_out, NULL, NULL, NULL, NULL};
    return par_for((int64_t)nq, 4, nthreads, &ctx, search_item, search_scratch, search_scratch_free);
}

int vo_search_from_top(const vo_index* ix, const float* queries, uint64_t nq, uint32_t w1, float alpha,
                       uint32_t topk, const uint32_t* top_in, int64_t* out_ids, float* out_dists,
                       uint64_t* out_scanned, int nthreads) {
    if (w1 == 0 || w1 > ix->k) return fail("first_level_scan: need 0 < w1 <= k");
    search_ctx ctx = {ix, queries, w1, vo_w2(w1, alpha, ix->n), topk, out_ids, out_dists, out_scanned, top_in, NULL,
                      NULL, NULL, NULL, NULL};
    return par_for((int64_t)nq, 4, nthreads, &ctx, search_item, search_scratch, search_scratch_free);
}

/* The search split after second_level_rank (the GPU engine's
 * vlq_engine_search_select_device / _fine_sel_device): vo_select writes the
 * w2 selected cells and their (a, b) of every query, vo_search_from_sel runs
 * query_term5 .. select_topk from such a selection. */
int vo_select(const vo_index* ix, const float* queries, uint64_t nq, uint32_t w1, float alpha, uint32_t* sel_out,
              float* ab_out, int nthreads) {
    if (w1 == 0 || w1 > ix->k) return fail("first_level_scan: need 0 < w1 <= k");
    search_ctx ctx = {ix, queries, w1, vo_w2(w1, alpha, ix->n), 0, NULL, NULL, NULL, NULL, NULL,
                      NULL, NULL, sel_out, ab_out};
    return par_for((int64_t)nq, 4, nthreads, &ctx, search_item, search_scratch, search_scratch_free);
}

int vo_search_from_sel(const vo_index* ix, const float* queries, uint64_t nq, uint32_t w1, float alpha,
                       uint32_t topk, const uint32_t* sel_in, const float* ab_in, int64_t* out_ids, float* out_dists,
                       uint64_t* out_scanned, int nthreads) {
    if (w1 == 0 || w1 > ix->k) return fail("first_level_scan: need 0 < w1 <= k");
    search_ctx ctx = {ix, queries, w1, vo_w2(w1, alpha, ix->n), topk, out_ids, out_dists, out_scanned, NULL, NULL,
                      sel_in, ab_in, NULL, NULL};
    return par_for((int64_t)nq, 4, nthreads, &ctx, search_item, search_scratch, search_scratch_free);
}

/* ---- add path per point ---------------------------------------------------
 * assign_point (index.cpp:86-106) -> assign_edge (line_quant.cpp:24-49) ->
 * residual at the exact lambda (index.cpp:181-184) -> pq_encode
 * (pq.cpp:52-67) -> quantize_lambda (index.cpp:12-17).  Outputs the cell,
 * the exact lambda, the PQ code and the lambda byte of every point; the
 * caller buckets by cell in point order (index.cpp:189-200). */
/* row[i] = sqdist(x, c_i) for a group of points: each centroid row is read
 * once for the whole group (the distances themselves keep the reference's
 * sequential order over d); test-infrastructure speed only. */
static void dist_rows(const vo_index* ix, const float* xs, uint32_t np, float* rows) {
    const uint32_t k = ix->k, dim = ix->dim;
    float* xt = (float*)malloc(sizeof(float) * dim * 16); /* [d][p] */
    for (uint32_t d = 0; d < dim; d++)
        for (uint32_t p = 0; p < 16; p++) xt[d * 16 + p] = p < np ? xs[(size_t)p * dim + d] : 0.0f;
    for (uint32_t i = 0; i < k; i++) {
        const float* c = ix->centroids + (size_t)i * dim;
        float acc[16] = {0};
        for (uint32_t d = 0; d < dim; d++) {
            const float cd = c[d];
            const float* xd = xt + d * 16;
            for (uint32_t p = 0; p < 16; p++) { /* 16 independent sequential chains */
                const float t = xd[p] - cd;
                acc[p] = acc[p] + t * t;
            }
        }
        for (uint32_t p = 0; p < np; p++) rows[(size_t)p * k + i] = acc[p];
    }
    free(xt);
}

static int assign_one(const vo_index* ix, const float* x, float* row, float* r, uint32_t* cell,
                      float* lam_out, uint8_t* code, int clamp, int row_ready) {
    const uint32_t k = ix->k, n = ix->n, dim = ix->dim, m = ix->m, dsub = dim / m;
    uint32_t best = 0;
    float best_d = FLT_MAX;
    for (uint32_t i = 0; i < k; i++) {
        float d = row_ready ? row[i] : vo_sqdist(x, ix->centroids + (size_t)i * dim, dim);
        row[i] = d;
        if (d < best_d) {
            best_d = d;
            best = i;
        }
    }
    float a = row[best];
    int have = 0;
    uint32_t best_j = 0;
    float best_lam = 0, best_sq = 0;
    for (uint32_t j = 0; j < n; j++) {
        float b = row[ix->nbr[(size_t)best * n + j]];
        float c = ix->elen[(size_t)best * n + j];
        float lam;
        if (vo_line_lambda(a, b, c, &lam)) return -1;
        if (clamp) lam = clampf_std(lam, 0.0f, 1.0f);
        float d = vo_line_sqdist(a, b, c, lam);
        if (!have || d < best_sq) {
            have = 1;
            best_j = j;
            best_lam = lam;
            best_sq = d;
        }
    }
    *cell = best * n + best_j;
    *lam_out = best_lam;
    if (code) {
        const float* ci = ix->centroids + (size_t)best * dim;
        const float* sj = ix->centroids + (size_t)ix->nbr[(size_t)best * n + best_j] * dim;
        for (uint32_t d = 0; d < dim; d++) r[d] = x[d] - ((1.0f - best_lam) * ci[d] + best_lam * sj[d]);
        for (uint32_t p = 0; p < m; p++) {
            uint32_t bj = 0;
            float bd = FLT_MAX;
            for (uint32_t j = 0; j < KSUB; j++) {
                float d = vo_sqdist(r + (size_t)p * dsub, ix->pq + ((size_t)p * KSUB + j) * dsub, dsub);
                if (d < bd) {
                    bd = d;
                    bj = j;
                }
            }
            code[p] = (uint8_t)bj;
        }
    }
    return 0;
}

typedef struct {
    const vo_index* ix;
    const float* base;
    int clamp;
    uint32_t* cells;
    float* lambdas;
    uint8_t* codes;
    uint8_t* lam_bytes;
    int64_t nb;
} assign_ctx;

typedef struct {
    float* row;
    float* r;
} assign_scratch_t;

#define ASSIGN_GROUP 16

static void* assign_scratch(void* c) {
    assign_ctx* ctx = (assign_ctx*)c;
    assign_scratch_t* s = (assign_scratch_t*)malloc(sizeof *s);
    s->row = (float*)malloc(sizeof(float) * ctx->ix->k * ASSIGN_GROUP);
    s->r = (float*)malloc(sizeof(float) * ctx->ix->dim);
    return s;
}

static void assign_scratch_free(void* p) {
    assign_scratch_t* s = (assign_scratch_t*)p;
    free(s->row);
    free(s->r);
    free(s);
}

/* item g = points [g*ASSIGN_GROUP, ...) */
static int assign_item(void* c, void* scratch, int64_t g) {
    assign_ctx* ctx = (assign_ctx*)c;
    assign_scratch_t* s = (assign_scratch_t*)scratch;
    const vo_index* ix = ctx->ix;
    const int64_t p0 = g * ASSIGN_GROUP;
    const uint32_t np = (uint32_t)((ctx->nb - p0) < ASSIGN_GROUP ? (ctx->nb - p0) : ASSIGN_GROUP);
    dist_rows(ix, ctx->base + (size_t)p0 * ix->dim, np, s->row);
    for (uint32_t q = 0; q < np; q++) {
        const int64_t p = p0 + q;
        if (assign_one(ix, ctx->base + (size_t)p * ix->dim, s->row + (size_t)q * ix->k, s->r, ctx->cells + p,
                       ctx->lambdas + p, ctx->codes ? ctx->codes + (size_t)p * ix->m : NULL, ctx->clamp, 1))
            return -1;
        if (ctx->lam_bytes) ctx->lam_bytes[p] = vo_quantize_lambda(ctx->lambdas[p], ix->lo, ix->hi);
    }
    return 0;
}

/* Encodes base[0..nb).  lam_bytes uses the index's (lo, hi) range.  When
 * codes == NULL only (cell, lambda) are produced (observe_lambda_range,
 * index.cpp:110-132, which runs assign_point with clamp = false). */
int vo_assign(const vo_index* ix, const float* base, uint64_t nb, int clamp, uint32_t* cells,
              float* lambdas, uint8_t* codes, uint8_t* lam_bytes, int nthreads) {
    assign_ctx ctx = {ix, base, clamp, cells, lambdas, codes, lam_bytes, (int64_t)nb};
    return par_for(((int64_t)nb + ASSIGN_GROUP - 1) / ASSIGN_GROUP, 4, nthreads, &ctx, assign_item, assign_scratch,
                   assign_scratch_free);
}

/* Direct (non-decomposed) ADC: |y - anchor(lambda) - pq_decode(code)|^2, the
 * reference tests' independent oracle (proj/tests/test_search.cpp:37-56). */
float vo_direct_adc(const vo_index* ix, const float* y, const uint8_t* code, uint8_t lambda_byte,
                    uint32_t i, uint32_t j) {
    uint32_t dim = ix->dim, dsub = dim / ix->m;
    float lam = vo_dequantize_lambda(lambda_byte, ix->lo, ix->hi);
    const float* ci = ix->centroids + (size_t)i * dim;
    const float* sj = ix->centroids + (size_t)ix->nbr[(size_t)i * ix->n + j] * dim;
    float acc = 0;
    for (uint32_t t = 0; t < dim; t++) {
        uint32_t p = t / dsub;
        float approx = ix->pq[((size_t)p * KSUB + code[p]) * dsub + (t % dsub)];
        float diff = y[t] - ((1.0f - lam) * ci[t] + lam * sj[t]) - approx;
        acc += diff * diff;
    }
    return acc;
}

/* Table-decomposed ADC for one entry given full-K centroid distances. */
float vo_adc_distance(const vo_index* ix, const float* ws, const float* t5, const uint8_t* code,
                      uint8_t lambda_byte, uint32_t i, uint32_t j) {
    return vo_adc(ix, code, lambda_byte, i, j, ws, t5);
}

/* Exact per-query tables for tests: full centroid row and t5. */
void vo_query_tables(const vo_index* ix, const float* y, float* ws, float* t5) {
    uint32_t dsub = ix->dim / ix->m;
    for (uint32_t i = 0; i < ix->k; i++) ws[i] = vo_sqdist(y, ix->centroids + (size_t)i * ix->dim, ix->dim);
    for (uint32_t p = 0; p < ix->m; p++)
        for (uint32_t j = 0; j < KSUB; j++)
            t5[(size_t)p * KSUB + j] = vo_dot(y + (size_t)p * dsub, ix->pq + ((size_t)p * KSUB + j) * dsub, dsub);
}

float vo_line_lambda_raw(float a, float b, float c) {
    float l = NAN;
    vo_line_lambda(a, b, c, &l);
    return l;
}
float vo_line_sqdist_raw(float a, float b, float c, float l) { return vo_line_sqdist(a, b, c, l); }
float vo_sqdist_raw(const float* a, const float* b, uint32_t d) { return vo_sqdist(a, b, d); }

/* ==== IVFADC comparison baseline: proj/src/ivf_baseline.cpp ==============
 * Single-level index: K lists of (id, PQ code of x - c_i) with the VLQ
 * model's codebook and PQ (eval.cpp:182).  Lists are returned flattened:
 * list_off[K+1], ids[N] (ascending within a list: point order), codes[N*m]. */

/* build_ivf_baseline (ivf_baseline.cpp:11-51): assign_nearest (strict '<',
 * kmeans.cpp:21-33), residual x - c (fp32 sub), pq_encode (pq.cpp:52-67),
 * then ordered appends.  Serial: the output is batch-independent. */
int vo_ivf_build(const vo_index* ix, const float* base, uint64_t nb, uint64_t* list_off, uint32_t* ids,
                 uint8_t* codes) {
    const uint32_t k = ix->k, dim = ix->dim, m = ix->m, dsub = dim / m;
    uint32_t* assign = (uint32_t*)malloc(sizeof(uint32_t) * (nb ? nb : 1));
    uint8_t* code = (uint8_t*)malloc((size_t)(nb ? nb : 1) * m);
    float* r = (float*)malloc(sizeof(float) * dim);
    for (uint64_t i = 0; i < nb; i++) {
        const float* x = base + i * dim;
        uint32_t best = 0;
        float best_d = FLT_MAX;
        for (uint32_t c = 0; c < k; c++) {
            float d = vo_sqdist(x, ix->centroids + (size_t)c * dim, dim);
            if (d < best_d) {
                best_d = d;
                best = c;
            }
        }
        assign[i] = best;
        const float* ctr = ix->centroids + (size_t)best * dim;
        for (uint32_t d = 0; d < dim; d++) r[d] = x[d] - ctr[d];
        for (uint32_t p = 0; p < m; p++) {
            uint32_t bj = 0;
            float bd = FLT_MAX;
            for (uint32_t j = 0; j < KSUB; j++) {
                float d = vo_sqdist(r + (size_t)p * dsub, ix->pq + ((size_t)p * KSUB + j) * dsub, dsub);
                if (d < bd) {
                    bd = d;
                    bj = j;
                }
            }
            code[i * m + p] = (uint8_t)bj;
        }
    }
    for (uint32_t c = 0; c <= k; c++) list_off[c] = 0;
    for (uint64_t i = 0; i < nb; i++) list_off[assign[i] + 1]++;
    for (uint32_t c = 0; c < k; c++) list_off[c + 1] += list_off[c];
    uint64_t* fill = (uint64_t*)malloc(sizeof(uint64_t) * k);
    for (uint32_t c = 0; c < k; c++) fill[c] = list_off[c];
    for (uint64_t i = 0; i < nb; i++) {
        uint64_t e = fill[assign[i]]++;
        ids[e] = (uint32_t)i;
        memcpy(codes + e * m, code + i * m, m);
    }
    free(fill);
    free(r);
    free(code);
    free(assign);
    return 0;
}

typedef struct {
    const vo_index* ix;
    const uint64_t* off;
    const uint32_t* ids;
    const uint8_t* codes;
    const float* queries;
    uint32_t w, topk;
    int64_t* out_ids;
    float* out_dists;
    uint64_t* out_scanned;
} ivf_ctx;

typedef struct {
    uint64_t* keys;  /* k */
    float* resid;    /* dim */
    float* lut;      /* m*256 */
    uint64_t* cand;
    size_t cand_cap;
} ivf_scratch;

static void* ivf_scratch_new(void* c) {
    ivf_ctx* ctx = (ivf_ctx*)c;
    ivf_scratch* s = (ivf_scratch*)calloc(1, sizeof(ivf_scratch));
    s->keys = (uint64_t*)malloc(sizeof(uint64_t) * ctx->ix->k);
    s->resid = (float*)malloc(sizeof(float) * ctx->ix->dim);
    s->lut = (float*)malloc(sizeof(float) * ctx->ix->m * KSUB);
    return s;
}

static void ivf_scratch_free(void* p) {
    ivf_scratch* s = (ivf_scratch*)p;
    free(s->keys);
    free(s->resid);
    free(s->lut);
    free(s->cand);
    free(s);
}

/* search_ivf_baseline (ivf_baseline.cpp:53-126) for one query */
static int ivf_item(void* c, void* scratch, int64_t q) {
    ivf_ctx* ctx = (ivf_ctx*)c;
    ivf_scratch* s = (ivf_scratch*)scratch;
    const vo_index* ix = ctx->ix;
    const uint32_t k = ix->k, dim = ix->dim, m = ix->m, dsub = dim / m;
    const float* y = ctx->queries + (size_t)q * dim;
    for (uint32_t i = 0; i < k; i++) s->keys[i] = fkey(vo_sqdist(y, ix->centroids + (size_t)i * dim, dim), i);
    select_smallest(s->keys, k, ctx->w);
    size_t nc = 0;
    for (uint32_t r = 0; r < ctx->w; r++) {
        uint32_t region = (uint32_t)s->keys[r];
        uint64_t b0 = ctx->off[region], b1 = ctx->off[region + 1];
        if (b0 == b1) continue;
        const float* ctr = ix->centroids + (size_t)region * dim;
        for (uint32_t d = 0; d < dim; d++) s->resid[d] = y[d] - ctr[d];
        for (uint32_t p = 0; p < m; p++)
            for (uint32_t j = 0; j < KSUB; j++)
                s->lut[(size_t)p * KSUB + j] =
                    vo_sqdist(s->resid + (size_t)p * dsub, ix->pq + ((size_t)p * KSUB + j) * dsub, dsub);
        if (nc + (b1 - b0) > s->cand_cap) {
            size_t cap = s->cand_cap ? s->cand_cap : 1024;
            while (cap < nc + (b1 - b0)) cap *= 2;
            s->cand = (uint64_t*)realloc(s->cand, cap * sizeof(uint64_t));
            s->cand_cap = cap;
        }
        for (uint64_t e = b0; e < b1; e++) {
            float d = 0;
            const uint8_t* code = ctx->codes + e * m;
            for (uint32_t p = 0; p < m; p++) d += s->lut[(size_t)p * KSUB + code[p]];
            s->cand[nc++] = fkey(d, ctx->ids[e]);
        }
    }
    ctx->out_scanned[q] = nc;
    select_smallest(s->cand, nc, ctx->topk);
    for (uint32_t r = 0; r < ctx->topk; r++) {
        int64_t* oi = ctx->out_ids + (size_t)q * ctx->topk;
        float* od = ctx->out_dists + (size_t)q * ctx->topk;
        if (r < nc) {
            oi[r] = (int64_t)(uint32_t)s->cand[r];
            od[r] = key_float(s->cand[r]);
        } else {
            oi[r] = -1;
            od[r] = INFINITY;
        }
    }
    return 0;
}

int vo_ivf_search(const vo_index* ix, const uint64_t* list_off, const uint32_t* ids, const uint8_t* codes,
                  const float* queries, uint64_t nq, uint32_t w, uint32_t topk, int64_t* out_ids, float* out_dists,
                  uint64_t* out_scanned, int nthreads) {
    if (w == 0 || w > ix->k) return fail("search_ivf_baseline: need 0 < w <= k");
    ivf_ctx ctx = {ix, list_off, ids, codes, queries, w, topk, out_ids, out_dists, out_scanned};
    return par_for((int64_t)nq, 4, nthreads, &ctx, ivf_item, ivf_scratch_new, ivf_scratch_free);
}
