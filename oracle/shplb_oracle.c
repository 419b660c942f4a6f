/*
 * TEST INFRASTRUCTURE ONLY — the parity oracle. Never linked into, or called
 * by, the product library (paper_2603_10353_b200/). Only tests/, the smoke()
 * check in __graft_entry__.py and bench.py's cpu_baseline / --impl reference
 * legs load it.
 *
 * A plain-C restatement of the reference's sparse-attention algorithm
 * (headbal, /root/reference/proj), generalised from token granularity to the
 * block granularity the north_star's kernels use. At block size 1 the block
 * rules below reduce exactly to the reference's PerQueryTopK (pinned by
 * tests/test_oracle.py against the compiled reference, oracle/_ref).
 *
 *   scale        1/sqrt(d) computed in double, applied after the dot product
 *                (proj/src/attention.cpp:20,26)
 *   causal mask  key j > query i is -inf, top-left aligned (attention.cpp:28-30)
 *   selection    k largest under (value desc, index asc), returned ascending
 *                (attention.cpp:53-64; tests/oracles.hpp:42-52)
 *   softmax      max-subtracted softmax over the kept set, accumulated in
 *                ascending key order; an all-masked kept set gives a zero row
 *                (attention.cpp:35-49)
 *   budgets      uniform split / max-min shifting (allocator.cpp:72-186)
 *   plan         naive contiguous / round-robin and LPT greedy
 *                (partitioner.cpp:130-183), imbalance (partitioner.cpp:236-266)
 *   metric       barrier = max_d t_d, bubble = 1 - mean/max (simulator.cpp:28-47)
 *
 * Block-level definitions (ours, documented in DESIGN.md §3):
 *   pooled row   P[b][c] = (sum over the block's rows of x[t][c]) / count_b,
 *                in fp32 from the exact bf16 values, in the fixed two-level
 *                order of orc_pool_blocks
 *   block score  s[qb][kb] = fmaf-chain over c = 0..d-1 of Qp[qb][c]*Kp[kb][c]
 *                (fp32, ascending c), then * (float)scale
 *   visibility   key block kb is visible to query block qb iff
 *                kb*bk <= last query row of qb (causal); all blocks otherwise
 *   kept count   min(k_h, visible blocks of qb) — the reference keeps k
 *                entries even when some are -inf (masked); those carry zero
 *                weight, so capping at the visible count is output-identical.
 * fp32 arithmetic here is bit-for-bit the GPU's: this file is compiled with
 * -ffp-contract=off and every fused multiply-add is an explicit fmaf().
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline float bf16_to_f32(uint16_t h) {
    uint32_t u = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return f;
}

/* --- block pooling --------------------------------------------------------- */

/* x: [n][d] bf16 bits; out: [ceil(n/block)][d] fp32 means.
 * Summation order (the GPU estimator's): the block's rows are
 * split into POOL_SPLIT interleaved groups (rows g, g+16, g+32, ...); each
 * group is summed in ascending row order from 0.0f, the 16 group sums are
 * added in ascending group order from 0.0f, and the total is divided by the
 * row count. */
#define POOL_SPLIT 16
void orc_pool_blocks(const uint16_t* x, int64_t n, int32_t d, int32_t block, float* out) {
    const int64_t nb = (n + block - 1) / block;
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t t0 = b * block;
        const int64_t cnt = (n - t0 < block) ? (n - t0) : block;
        for (int32_t c = 0; c < d; ++c) {
            float total = 0.0f;
            for (int64_t g = 0; g < POOL_SPLIT; ++g) {
                float acc = 0.0f;
                for (int64_t t = g; t < cnt; t += POOL_SPLIT)
                    acc = acc + bf16_to_f32(x[(t0 + t) * d + c]);
                total = total + acc;
            }
            out[b * d + c] = total / (float)cnt;
        }
    }
}

float orc_score_scale(int32_t d) { return (float)(1.0 / sqrt((double)d)); }

/* Number of key blocks visible to query block qb (n_q query rows, n_k keys;
 * the causal mask is top-left aligned: query i sees keys 0..i). */
int64_t orc_visible_blocks(int64_t qb, int64_t n_q, int64_t n_k, int32_t bq, int32_t bk,
                           int causal) {
    const int64_t nkb = (n_k + bk - 1) / bk;
    if (!causal) return nkb;
    int64_t last = (qb + 1) * bq;
    if (last > n_q) last = n_q;
    last -= 1;
    int64_t v = last / bk + 1;
    return v < nkb ? v : nkb;
}

/* qp: [nqb][d], kp: [nkb][d] -> scores [nqb][nkb]; masked blocks are -inf. */
void orc_block_scores(const float* qp, const float* kp, int64_t n_q, int64_t n_k, int32_t d,
                      int32_t bq, int32_t bk, int causal, float* scores) {
    const int64_t nqb = (n_q + bq - 1) / bq, nkb = (n_k + bk - 1) / bk;
    const float scale = orc_score_scale(d);
    for (int64_t qb = 0; qb < nqb; ++qb) {
        const int64_t vis = orc_visible_blocks(qb, n_q, n_k, bq, bk, causal);
        for (int64_t kb = 0; kb < nkb; ++kb) {
            float acc = 0.0f;
            for (int32_t c = 0; c < d; ++c) acc = fmaf(qp[qb * d + c], kp[kb * d + c], acc);
            scores[qb * nkb + kb] = kb < vis ? acc * scale : -INFINITY;
        }
    }
}

/* Unmasked scores of m pooled query rows against nkb pooled key rows (the
 * same fmaf chain and scale as orc_block_scores). */
void orc_score_rows(const float* qp, const float* kp, int64_t m, int64_t nkb, int32_t d,
                    float* out) {
    const float scale = orc_score_scale(d);
    for (int64_t r = 0; r < m; ++r)
        for (int64_t kb = 0; kb < nkb; ++kb) {
            float acc = 0.0f;
            for (int32_t c = 0; c < d; ++c) acc = fmaf(qp[r * d + c], kp[kb * d + c], acc);
            out[r * nkb + kb] = acc * scale;
        }
}

/* --- top-k selection ------------------------------------------------------- */

typedef struct {
    float v;
    int32_t i;
} scored;

/* (value desc, index asc), tests/oracles.hpp:45-48. */
static int cmp_desc(const void* a, const void* b) {
    const scored* x = (const scored*)a;
    const scored* y = (const scored*)b;
    if (x->v != y->v) return x->v > y->v ? -1 : 1;
    return (x->i > y->i) - (x->i < y->i);
}

static int cmp_i32(const void* a, const void* b) {
    const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* One head: scores [nqb][nkb]; k_blocks is that head's budget in blocks.
 * idx: [nqb][kmax] ascending block ids (unused tail = -1), cnt: [nqb]. */
void orc_select_topk(const float* scores, int64_t n_q, int64_t n_k, int32_t bq, int32_t bk,
                     int causal, int64_t k_blocks, int64_t kmax, int32_t* idx, int32_t* cnt) {
    const int64_t nqb = (n_q + bq - 1) / bq, nkb = (n_k + bk - 1) / bk;
    scored* buf = (scored*)malloc(sizeof(scored) * (size_t)nkb);
    for (int64_t qb = 0; qb < nqb; ++qb) {
        const int64_t vis = orc_visible_blocks(qb, n_q, n_k, bq, bk, causal);
        const int64_t kk = k_blocks < vis ? k_blocks : vis;
        for (int64_t j = 0; j < vis; ++j) {
            buf[j].v = scores[qb * nkb + j];
            buf[j].i = (int32_t)j;
        }
        qsort(buf, (size_t)vis, sizeof(scored), cmp_desc);
        int32_t* row = idx + qb * kmax;
        for (int64_t j = 0; j < kmax; ++j) row[j] = -1;
        for (int64_t j = 0; j < kk; ++j) row[j] = buf[j].i;
        qsort(row, (size_t)kk, sizeof(int32_t), cmp_i32);
        cnt[qb] = (int32_t)kk;
    }
    free(buf);
}

/* --- ColumnAggregateTopK at block granularity (attention.cpp:66-73,136-148) --
 * One key-block set per head, ranked by the column sums of the block-level
 * attention weights: for every query block qb the softmax of its visible
 * pooled scores, W[qb][kb] = e / Z with e = det_ex2((S - m) * log2 e) and Z the
 * sum of e over kb ascending; c[kb] = sum of W over qb ascending; keep the
 * k_h blocks with the largest c (value desc, index asc). Query block qb then
 * attends to the kept blocks it can see (kept ∩ [0, vis(qb)), ascending); the
 * reference keeps invisible keys too, with zero weight, so this is
 * output-identical. det_ex2 is a fixed fp32 polynomial evaluated with the same
 * IEEE operations here and on the GPU, so the sums — and the decisions — are
 * bit-identical. */
float orc_det_ex2(float x) {
    if (!(x > -126.0f)) return 0.0f;
    const float t = x + 12582912.0f;
    const float j = t - 12582912.0f;
    const float f = x - j;
    float p = fmaf(1.3333558e-3f, f, 9.6181291e-3f);
    p = fmaf(p, f, 5.5504109e-2f);
    p = fmaf(p, f, 2.4022651e-1f);
    p = fmaf(p, f, 6.9314718e-1f);
    p = fmaf(p, f, 1.0f);
    int32_t pb, tb;
    memcpy(&pb, &p, 4);
    memcpy(&tb, &t, 4);
    pb += (int32_t)((uint32_t)tb << 23);
    float r;
    memcpy(&r, &pb, 4);
    return r;
}

void orc_colagg_select(const float* scores, int64_t n_q, int64_t n_k, int32_t bq, int32_t bk,
                       int causal, int64_t k_blocks, int64_t kmax, int32_t* idx, int32_t* cnt) {
    const int64_t nqb = (n_q + bq - 1) / bq, nkb = (n_k + bk - 1) / bk;
    const float log2e = 1.44269504088896340736f;
    float* m = (float*)malloc(sizeof(float) * (size_t)nqb);
    float* z = (float*)malloc(sizeof(float) * (size_t)nqb);
    float* c = (float*)calloc((size_t)nkb, sizeof(float));
    for (int64_t qb = 0; qb < nqb; ++qb) {
        const int64_t vis = orc_visible_blocks(qb, n_q, n_k, bq, bk, causal);
        const float* row = scores + qb * nkb;
        float mx = -INFINITY;
        for (int64_t j = 0; j < vis; ++j) mx = row[j] > mx ? row[j] : mx;
        /* z: 32 strided partial sums (partial l over j = l, l+32, ... ascending), then
         * added in lane order from 0.0f — the GPU's warp-per-row order. */
        float part[32];
        for (int l = 0; l < 32; ++l) {
            part[l] = 0.0f;
            for (int64_t j = l; j < vis; j += 32) part[l] = part[l] + orc_det_ex2((row[j] - mx) * log2e);
        }
        float sum = 0.0f;
        for (int l = 0; l < 32; ++l) sum = sum + part[l];
        m[qb] = mx;
        z[qb] = sum;
    }
    for (int64_t kb = 0; kb < nkb; ++kb) {
        float acc = 0.0f;
        for (int64_t qb = 0; qb < nqb; ++qb) {
            if (kb >= orc_visible_blocks(qb, n_q, n_k, bq, bk, causal)) continue;
            acc = acc + orc_det_ex2((scores[qb * nkb + kb] - m[qb]) * log2e) / z[qb];
        }
        c[kb] = acc;
    }
    const int64_t kk = k_blocks < nkb ? k_blocks : nkb;
    scored* buf = (scored*)malloc(sizeof(scored) * (size_t)nkb);
    for (int64_t j = 0; j < nkb; ++j) {
        buf[j].v = c[j] + 0.0f;  /* -0.0 -> +0.0, as the GPU's order key */
        buf[j].i = (int32_t)j;
    }
    qsort(buf, (size_t)nkb, sizeof(scored), cmp_desc);
    int32_t* kept = (int32_t*)malloc(sizeof(int32_t) * (size_t)(kk > 0 ? kk : 1));
    for (int64_t j = 0; j < kk; ++j) kept[j] = buf[j].i;
    qsort(kept, (size_t)kk, sizeof(int32_t), cmp_i32);
    for (int64_t qb = 0; qb < nqb; ++qb) {
        const int64_t vis = orc_visible_blocks(qb, n_q, n_k, bq, bk, causal);
        int32_t* r = idx + qb * kmax;
        int64_t w = 0;
        for (int64_t j = 0; j < kk; ++j)
            if (kept[j] < vis) r[w++] = kept[j];
        for (int64_t j = w; j < kmax; ++j) r[j] = -1;
        cnt[qb] = (int32_t)w;
    }
    free(kept);
    free(buf);
    free(c);
    free(z);
    free(m);
}

/* Token-granular top-k on an arbitrary score row (value desc, index asc),
 * returned ascending: the reference's top_k_indices (attention.cpp:53-64). */
void orc_topk_row(const double* values, int64_t n, int64_t k, int64_t* out) {
    typedef struct {
        double v;
        int64_t i;
    } sd;
    sd* buf = (sd*)malloc(sizeof(sd) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) {
        buf[j].v = values[j];
        buf[j].i = j;
    }
    /* insertion-free: simple selection by full sort */
    for (int64_t a = 1; a < n; ++a) { /* stable insertion sort, n is small in tests */
        sd key = buf[a];
        int64_t b = a - 1;
        while (b >= 0 && (buf[b].v < key.v || (buf[b].v == key.v && buf[b].i > key.i))) {
            buf[b + 1] = buf[b];
            --b;
        }
        buf[b + 1] = key;
    }
    for (int64_t j = 0; j < k; ++j) out[j] = buf[j].i;
    for (int64_t a = 1; a < k; ++a) {
        int64_t key = out[a], b = a - 1;
        while (b >= 0 && out[b] > key) {
            out[b + 1] = out[b];
            --b;
        }
        out[b + 1] = key;
    }
    free(buf);
}

/* --- attention output on the kept set -------------------------------------- */

/* One q head / its kv head. q: [n_q][d], k/v: [n_k][d] bf16 bits. idx/cnt
 * from orc_select_topk. out: [n_q][d] fp64. Follows softmax_weighted_sum
 * (attention.cpp:35-49) on the kept tokens: the selected blocks' tokens in
 * ascending order, minus causally masked ones. */
void orc_block_sparse_attention(const uint16_t* q, const uint16_t* k, const uint16_t* v,
                                int64_t n_q, int64_t n_k, int32_t d, int32_t bq, int32_t bk,
                                int causal, const int32_t* idx, const int32_t* cnt, int64_t kmax,
                                double* out) {
    const double scale = 1.0 / sqrt((double)d);
    double* s = (double*)malloc(sizeof(double) * (size_t)(kmax * bk));
    int64_t* tok = (int64_t*)malloc(sizeof(int64_t) * (size_t)(kmax * bk));
    double* qrow = (double*)malloc(sizeof(double) * (size_t)d);
    for (int64_t i = 0; i < n_q; ++i) {
        const int64_t qb = i / bq;
        for (int32_t c = 0; c < d; ++c) qrow[c] = (double)bf16_to_f32(q[i * d + c]);
        int64_t m_cnt = 0;
        for (int64_t t = 0; t < cnt[qb]; ++t) {
            const int64_t b = idx[qb * kmax + t];
            for (int64_t j = b * bk; j < (b + 1) * bk && j < n_k; ++j) {
                if (causal && j > i) continue;
                double dot = 0.0;
                for (int32_t c = 0; c < d; ++c) dot += qrow[c] * (double)bf16_to_f32(k[j * d + c]);
                s[m_cnt] = dot * scale;
                tok[m_cnt] = j;
                ++m_cnt;
            }
        }
        double* o = out + i * d;
        for (int32_t c = 0; c < d; ++c) o[c] = 0.0;
        if (m_cnt == 0) continue; /* all masked: zero row (attention.cpp:40-41) */
        double m = -INFINITY;
        for (int64_t t = 0; t < m_cnt; ++t) m = s[t] > m ? s[t] : m;
        double denom = 0.0;
        for (int64_t t = 0; t < m_cnt; ++t) denom += exp(s[t] - m);
        for (int64_t t = 0; t < m_cnt; ++t) {
            const double w = exp(s[t] - m) / denom;
            const uint16_t* vr = v + tok[t] * d;
            for (int32_t c = 0; c < d; ++c) o[c] += w * (double)bf16_to_f32(vr[c]);
        }
    }
    free(s);
    free(tok);
    free(qrow);
}

/* Whole layer (GQA: q head h reads kv head h / (hq/hkv)), per-head budgets in
 * blocks. Parallel over heads with OpenMP (each head is computed serially, so
 * the result is thread-count independent, as the reference's fan-out is:
 * attention.cpp:214-223). q: [hq][n_q][d], k/v: [hkv][n_k][d]; out
 * [hq][n_q][d]. The GPU path is prefill (n_q == n_k); the reference (and so
 * this restatement) also allows n_q != n_k. */
void orc_layer_kind(const uint16_t* q, const uint16_t* k, const uint16_t* v, int32_t hq, int32_t hkv,
                    int64_t n_q, int64_t n_k, int32_t d, int32_t bq, int32_t bk, int causal, int kind,
                    const int64_t* k_blocks, int64_t kmax, float* scores_out, int32_t* idx_out,
                    int32_t* cnt_out, double* out) {
    const int64_t nqb = (n_q + bq - 1) / bq, nkb = (n_k + bk - 1) / bk;
    const int32_t group = hq / hkv;
#pragma omp parallel for schedule(dynamic)
    for (int32_t h = 0; h < hq; ++h) {
        const int32_t g = h / group;
        float* qp = (float*)malloc(sizeof(float) * (size_t)(nqb * d));
        float* kp = (float*)malloc(sizeof(float) * (size_t)(nkb * d));
        orc_pool_blocks(q + (int64_t)h * n_q * d, n_q, d, bq, qp);
        orc_pool_blocks(k + (int64_t)g * n_k * d, n_k, d, bk, kp);
        float* sc = scores_out + (int64_t)h * nqb * nkb;
        orc_block_scores(qp, kp, n_q, n_k, d, bq, bk, causal, sc);
        int32_t* ix = idx_out + (int64_t)h * nqb * kmax;
        int32_t* ct = cnt_out + (int64_t)h * nqb;
        if (kind == 1)
            orc_colagg_select(sc, n_q, n_k, bq, bk, causal, k_blocks[h], kmax, ix, ct);
        else
            orc_select_topk(sc, n_q, n_k, bq, bk, causal, k_blocks[h], kmax, ix, ct);
        if (out) {
            orc_block_sparse_attention(q + (int64_t)h * n_q * d, k + (int64_t)g * n_k * d,
                                       v + (int64_t)g * n_k * d, n_q, n_k, d, bq, bk, causal, ix,
                                       ct, kmax, out + (int64_t)h * n_q * d);
        }
        free(qp);
        free(kp);
    }
}

void orc_layer(const uint16_t* q, const uint16_t* k, const uint16_t* v, int32_t hq, int32_t hkv,
               int64_t n_q, int64_t n_k, int32_t d, int32_t bq, int32_t bk, int causal,
               const int64_t* k_blocks, int64_t kmax, float* scores_out, int32_t* idx_out,
               int32_t* cnt_out, double* out) {
    orc_layer_kind(q, k, v, hq, hkv, n_q, n_k, d, bq, bk, causal, 0, k_blocks, kmax, scores_out, idx_out,
                   cnt_out, out);
}

/* --- budget table (allocator.cpp) ------------------------------------------ */

/* Curve lookup: recovery at the largest sampled budget <= b, 0 below the
 * first sample (profiler.cpp:55-62). */
double orc_recovery_at(const int64_t* pb, const double* pr, int64_t np, int64_t b) {
    double r = 0.0;
    for (int64_t p = 0; p < np; ++p) {
        if (pb[p] > b) break;
        r = pr[p];
    }
    return r;
}

/* Returns 0, or 1 when the total is infeasible (allocator.cpp:53-62). */
int orc_uniform_allocate(int64_t n, int64_t total, int64_t floor, int64_t n_k, int64_t* out) {
    if (n < 1 || total < n * floor || total > n * n_k) return 1;
    const int64_t base = total / n, rem = total % n;
    for (int64_t h = 0; h < n; ++h) out[h] = base + (h < rem ? 1 : 0);
    return 0;
}

/* Max-min budget shifting (allocator.cpp:97-186), restated. offsets: [n+1]. */
int orc_maxmin_allocate(int32_t n, int64_t n_k, const int64_t* offsets, const int64_t* pb,
                        const double* pr, int64_t total, int64_t quantum, int64_t floor,
                        int64_t max_iterations, int64_t* budgets, int64_t* transfers_out,
                        int32_t* hit_cap_out) {
    if (orc_uniform_allocate(n, total, floor, n_k, budgets)) return 1;
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
#define REC(h, b) orc_recovery_at(pb + offsets[h], pr + offsets[h], offsets[(h) + 1] - offsets[h], b)
    for (int32_t h = 0; h < n; ++h) r[h] = REC(h, budgets[h]);
    if (max_iterations == 0) {
        max_iterations = 10 * (int64_t)n * n_k / quantum;
        if (max_iterations < 1) max_iterations = 1;
    }
    int64_t it = 0, transfers = 0;
    for (; it < max_iterations; ++it) {
        int32_t rec = 0;
        for (int32_t h = 1; h < n; ++h)
            if (r[h] < r[rec]) rec = h;
        const double cur_min = r[rec];
        int64_t amount = n_k - budgets[rec];
        if (quantum < amount) amount = quantum;
        if (amount == 0) break;
        int32_t donor = n;
        for (int32_t h = 0; h < n; ++h) {
            if (h == rec) continue;
            if (budgets[h] - amount < floor) continue;
            if (donor == n || r[h] > r[donor]) donor = h;
        }
        if (donor == n) break;
        budgets[donor] -= amount;
        budgets[rec] += amount;
        const double rd = REC(donor, budgets[donor]);
        const double rr = REC(rec, budgets[rec]);
        double new_min = INFINITY;
        for (int32_t h = 0; h < n; ++h) {
            const double rh = h == donor ? rd : h == rec ? rr : r[h];
            if (rh < new_min) new_min = rh;
        }
        if (!(new_min > cur_min)) {
            budgets[donor] += amount;
            budgets[rec] -= amount;
            break;
        }
        r[donor] = rd;
        r[rec] = rr;
        ++transfers;
    }
#undef REC
    if (transfers_out) *transfers_out = transfers;
    if (hit_cap_out) *hit_cap_out = it == max_iterations;
    free(r);
    return 0;
}

/* --- head -> device plan (partitioner.cpp) --------------------------------- */

int orc_naive_assign(int32_t n, int32_t devices, int round_robin, int32_t* dev) {
    if (devices < 1 || devices > n) return 1;
    if (round_robin) {
        for (int32_t h = 0; h < n; ++h) dev[h] = h % devices;
        return 0;
    }
    const int32_t base = n / devices, extra = n % devices;
    int32_t next = 0;
    for (int32_t d = 0; d < devices; ++d) {
        const int32_t c = base + (d < extra ? 1 : 0);
        for (int32_t i = 0; i < c; ++i) dev[next++] = d;
    }
    return 0;
}

/* LPT: heads by (budget desc, index asc); each onto the device minimising
 * (load, device index) — the ordering the reference's min-heap of
 * (load, device) pairs pops (partitioner.cpp:164-183). O(N*D) scan here. */
int orc_greedy_assign(const int64_t* budgets, int32_t n, int32_t devices, int32_t* dev) {
    if (devices < 1 || n < 1) return 1;
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int64_t* load = (int64_t*)calloc((size_t)devices, sizeof(int64_t));
    for (int32_t h = 0; h < n; ++h) order[h] = h;
    for (int32_t a = 1; a < n; ++a) { /* stable insertion sort on budget desc */
        int32_t key = order[a], b = a - 1;
        while (b >= 0 && budgets[order[b]] < budgets[key]) {
            order[b + 1] = order[b];
            --b;
        }
        order[b + 1] = key;
    }
    for (int32_t t = 0; t < n; ++t) {
        int32_t best = 0;
        for (int32_t d = 1; d < devices; ++d)
            if (load[d] < load[best]) best = d;
        dev[order[t]] = best;
        load[best] += budgets[order[t]];
    }
    free(order);
    free(load);
    return 0;
}

/* loads[D], returns imbalance = max * D / total (1 when total == 0). */
double orc_imbalance(const int64_t* budgets, int32_t n, const int32_t* dev, int32_t devices,
                     int64_t* loads, int32_t* argmax) {
    int64_t total = 0;
    for (int32_t d = 0; d < devices; ++d) loads[d] = 0;
    for (int32_t h = 0; h < n; ++h) {
        loads[dev[h]] += budgets[h];
        total += budgets[h];
    }
    int64_t mx = loads[0];
    *argmax = 0;
    for (int32_t d = 1; d < devices; ++d)
        if (loads[d] > mx) {
            mx = loads[d];
            *argmax = d;
        }
    return total == 0 ? 1.0 : (double)mx * (double)devices / (double)total;
}

/* Barrier and bubble over per-device latencies (simulator.cpp:35-45). */
void orc_barrier(const double* lat, int32_t devices, double* barrier, double* bubble) {
    double mx = lat[0], sum = 0.0;
    for (int32_t d = 0; d < devices; ++d) {
        if (lat[d] > mx) mx = lat[d];
        sum += lat[d];
    }
    *barrier = mx;
    *bubble = mx == 0.0 ? 0.0 : 1.0 - (sum / (double)devices) / mx;
}
