/*
 * stripefrac_oracle.c — CPU restatement of the reference's Striped UniFrac
 * hot path, TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this (as the checker / the CPU baseline). The product path never
 * links, loads or calls it.
 *
 * Pinned: tests/test_oracle.py checks it bit-for-bit against the golden
 * vectors in tests/golden/ produced by the reference itself (oracle/_ref,
 * built from /root/reference/proj/src by oracle/Makefile).
 *
 * It consumes the same flattened problem as the C ABI (sf_problem layout:
 * postorder rows, parent rows, lengths, leaf features, CSR table) and follows:
 *   - leaf rows: relative_abundance / presence      table.cpp:208-222
 *   - internal rows: pending fold in postorder       embed.cpp:42-82
 *     (sum for weighted, max/OR for unweighted, starting from 0)
 *   - fp32: rows and lengths computed in fp64, rounded once  embed.hpp:71-84
 *   - update_entry, no FMA (compiled -ffp-contract=off)      kernels.hpp:55-66
 *   - per-slot sequential sum over rows in postorder         kernels.hpp:97-119
 *   - finalize: t == 0 ? 0 : d / t                            kernels.hpp:251-259
 *   - stripe pair (k, (k+s+1) mod n)                         stripes.cpp:23-28
 * Stripe ranges are split over threads with the reference's worker formula
 * (kernels.hpp:302-303).
 *
 * Generalized UniFrac (metric 4, orc_compute_stripes_generalized) is NOT in
 * the reference (common.hpp:19): PARITY UNPINNED. It
 * restates the published definition (Chen et al. 2012, generalized UniFrac
 * d^(a) = sum b (pA+pB)^a |pA-pB|/(pA+pB) / sum b (pA+pB)^a) in the striped
 * form of Striped UniFrac (McDonald et al. 2018, the paper this reference
 * re-implements): over the weighted (relative-abundance) embedding, per row
 *     s = u + v; if (s != 0) { w = pow(s, a) * L; d += w * (|u-v| / s); t += w; }
 * then finalize d / t. a = 1 is weighted normalized UniFrac up to rounding.
 */
#include <limits.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct orc_problem {
  int32_t n_rows;
  const int32_t* parent_row;
  const double* lengths;
  const int32_t* leaf_feature;
  int32_t n_samples;
  int32_t n_features;
  const int64_t* feat_ptr;
  const int32_t* sample_idx;
  const double* counts;
  const double* sample_totals;
} orc_problem;

enum { ORC_UW = 1, ORC_WU = 2, ORC_WN = 3, ORC_GEN = 4 };

/* ---------------------------------------------------------------- rows */
/* Embedding rows [0, E) are produced one at a time in postorder; each row is
 * folded into its parent's pending buffer (embed.cpp:71-79). emit() writes
 * the row into `row` (n doubles). */
typedef struct embedder {
  const orc_problem* p;
  int weighted;
  double** pending; /* [E] pending sums per internal row, NULL until a child lands */
  int32_t cursor;
} embedder;

static int emb_init(embedder* em, const orc_problem* p, int weighted) {
  em->p = p;
  em->weighted = weighted;
  em->cursor = 0;
  em->pending = (double**)calloc((size_t)p->n_rows, sizeof(double*));
  return em->pending ? 0 : -1;
}

static void emb_free(embedder* em) {
  if (!em->pending) return;
  for (int32_t r = 0; r < em->p->n_rows; ++r) free(em->pending[r]);
  free(em->pending);
  em->pending = NULL;
}

static int emb_next(embedder* em, double* row) {
  const orc_problem* p = em->p;
  const int n = p->n_samples;
  const int32_t r = em->cursor++;
  const int32_t f = p->leaf_feature[r];
  if (f >= 0) {
    memset(row, 0, sizeof(double) * (size_t)n);
    for (int64_t e = p->feat_ptr[f]; e < p->feat_ptr[f + 1]; ++e) {
      const int s = p->sample_idx[e];
      const double c = p->counts[e];
      row[s] = em->weighted ? c / p->sample_totals[s] : (c > 0.0 ? 1.0 : 0.0);
    }
  } else {
    if (!em->pending[r]) return -1; /* internal node emitted before its children */
    memcpy(row, em->pending[r], sizeof(double) * (size_t)n);
    free(em->pending[r]);
    em->pending[r] = NULL;
  }
  const int32_t par = p->parent_row[r];
  if (par >= 0) {
    if (!em->pending[par]) {
      em->pending[par] = (double*)calloc((size_t)n, sizeof(double));
      if (!em->pending[par]) return -1;
    }
    double* acc = em->pending[par];
    if (em->weighted) {
      for (int i = 0; i < n; ++i) acc[i] += row[i];
    } else {
      for (int i = 0; i < n; ++i) acc[i] = acc[i] < row[i] ? row[i] : acc[i]; /* cwiseMax */
    }
  }
  return 0;
}

int orc_embed_rows(const orc_problem* p, int weighted, double* out) {
  embedder em;
  if (emb_init(&em, p, weighted)) return -1;
  for (int32_t r = 0; r < p->n_rows; ++r)
    if (emb_next(&em, out + (int64_t)r * p->n_samples)) {
      emb_free(&em);
      return -1;
    }
  emb_free(&em);
  return 0;
}

/* -------------------------------------------------------------- stripes */
#define DEFINE_ACCUM(NAME, REAL, POW)                                                \
  static void NAME(int metric, REAL* dist, REAL* tot, const REAL* emb,               \
                   const REAL* lens, int filled, int n, int s0, int s1, int start,   \
                   REAL alpha) {                                                     \
    for (int s = s0; s < s1; ++s) {                                                  \
      REAL* dm = dist + (int64_t)(s - start) * n;                                    \
      REAL* tt = tot ? tot + (int64_t)(s - start) * n : NULL;                        \
      for (int k = 0; k < n; ++k) {                                                  \
        int l = k + s + 1;                                                           \
        if (l >= n) l -= n;                                                          \
        REAL d = dm[k];                                                              \
        REAL t = tt ? tt[k] : (REAL)0;                                               \
        for (int e = 0; e < filled; ++e) {                                           \
          const REAL u = emb[(int64_t)e * n + k], v = emb[(int64_t)e * n + l];       \
          const REAL L = lens[e];                                                    \
          if (metric == ORC_GEN) {                                                   \
            const REAL sum = u + v;                                                  \
            if (sum != (REAL)0) {                                                    \
              REAL sub = u - v;                                                      \
              if (sub < (REAL)0) sub = -sub;                                         \
              const REAL w = POW(sum, alpha) * L;                                    \
              d += w * (sub / sum);                                                  \
              t += w;                                                                \
            }                                                                        \
            continue;                                                                \
          }                                                                          \
          REAL diff = u - v;                                                         \
          if (diff < (REAL)0) diff = -diff;                                          \
          d += diff * L;                                                             \
          if (metric == ORC_UW)                                                      \
            t += (u > v ? u : v) * L;                                                \
          else if (metric == ORC_WN)                                                 \
            t += (u + v) * L;                                                        \
        }                                                                            \
        dm[k] = d;                                                                   \
        if (tt) tt[k] = t;                                                           \
      }                                                                              \
    }                                                                                \
  }
DEFINE_ACCUM(accum_f64, double, pow)
DEFINE_ACCUM(accum_f32, float, powf)

typedef struct job {
  int metric, prec, filled, n, s0, s1, start;
  double alpha;
  void *dist, *tot;
  const void *emb, *lens;
} job;

static void* run_job(void* arg) {
  const job* j = (const job*)arg;
  if (j->prec == 8)
    accum_f64(j->metric, (double*)j->dist, (double*)j->tot, (const double*)j->emb,
              (const double*)j->lens, j->filled, j->n, j->s0, j->s1, j->start, j->alpha);
  else
    accum_f32(j->metric, (float*)j->dist, (float*)j->tot, (const float*)j->emb,
              (const float*)j->lens, j->filled, j->n, j->s0, j->s1, j->start, (float)j->alpha);
  return NULL;
}

/* Full stripe computation: rows streamed in batches of `batch`, stripes
 * [start, stop) split over `threads` workers per batch. Returns 0 on
 * success. dist/tot: (stop-start) x n of double (prec 8) or float (prec 4);
 * tot may be NULL for WU. */
int orc_compute_stripes_rows(const orc_problem* p, int metric, int prec, int start, int stop,
                             void* dist, void* tot, int finalize, int threads, int batch,
                             int row_limit);
static int compute_rows_alpha(const orc_problem* p, int metric, int prec, int start, int stop,
                              void* dist, void* tot, int finalize, int threads, int batch,
                              int row_limit, double alpha);

/* Generalized UniFrac with exponent alpha (metric 4; parity unpinned). */
int orc_compute_stripes_generalized(const orc_problem* p, double alpha, int prec, int start,
                                    int stop, void* dist, void* tot, int finalize, int threads,
                                    int batch) {
  return compute_rows_alpha(p, ORC_GEN, prec, start, stop, dist, tot, finalize, threads, batch, 0,
                            alpha);
}

int orc_compute_stripes(const orc_problem* p, int metric, int prec, int start, int stop,
                        void* dist, void* tot, int finalize, int threads, int batch) {
  return orc_compute_stripes_rows(p, metric, prec, start, stop, dist, tot, finalize, threads,
                                  batch, 0);
}

/* As orc_compute_stripes, but only the first row_limit postorder rows (0 =
 * all): a bounded sample of the same workload for the CPU baseline. */
int orc_compute_stripes_rows(const orc_problem* p, int metric, int prec, int start, int stop,
                             void* dist, void* tot, int finalize, int threads, int batch,
                             int row_limit) {
  return compute_rows_alpha(p, metric, prec, start, stop, dist, tot, finalize, threads, batch,
                            row_limit, 1.0);
}

static int compute_rows_alpha(const orc_problem* p, int metric, int prec, int start, int stop,
                              void* dist, void* tot, int finalize, int threads, int batch,
                              int row_limit, double alpha) {
  const int n = p->n_samples;
  const int E = row_limit > 0 && row_limit < p->n_rows ? row_limit : p->n_rows;
  const size_t w = prec == 8 ? 8 : 4;
  const int64_t slots = (int64_t)(stop - start) * n;
  if (batch < 1) batch = 64;
  if (threads < 1) threads = 1;
  if (threads > stop - start) threads = stop - start;
  memset(dist, 0, (size_t)slots * w);
  if (tot) memset(tot, 0, (size_t)slots * w);
  const int has_t = metric != ORC_WU;
  void* t_use = has_t ? tot : NULL;

  embedder em;
  if (emb_init(&em, p, metric != ORC_UW)) return -1;
  double* rows64 = (double*)malloc(sizeof(double) * (size_t)batch * (size_t)n);
  float* rows32 = prec == 4 ? (float*)malloc(sizeof(float) * (size_t)batch * (size_t)n) : NULL;
  double* lens64 = (double*)malloc(sizeof(double) * (size_t)batch);
  float* lens32 = (float*)malloc(sizeof(float) * (size_t)batch);
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  job* jobs = (job*)malloc(sizeof(job) * (size_t)threads);
  int rc = 0;
  if (!rows64 || (prec == 4 && !rows32) || !lens64 || !lens32 || !tids || !jobs) rc = -1;
  for (int r0 = 0; rc == 0 && r0 < E; r0 += batch) {
    const int filled = E - r0 < batch ? E - r0 : batch;
    for (int i = 0; i < filled; ++i) {
      if (emb_next(&em, rows64 + (int64_t)i * n)) {
        rc = -1;
        break;
      }
      lens64[i] = p->lengths[r0 + i];
    }
    if (rc) break;
    const void* emb = rows64;
    const void* lens = lens64;
    if (prec == 4) { /* cast_batch: round once */
      for (int64_t i = 0; i < (int64_t)filled * n; ++i) rows32[i] = (float)rows64[i];
      for (int i = 0; i < filled; ++i) lens32[i] = (float)lens64[i];
      emb = rows32;
      lens = lens32;
    }
    const int span = stop - start;
    for (int wk = 0; wk < threads; ++wk) {
      job* j = &jobs[wk];
      j->metric = metric;
      j->alpha = alpha;
      j->prec = prec;
      j->filled = filled;
      j->n = n;
      j->s0 = start + (int)((int64_t)span * wk / threads);
      j->s1 = start + (int)((int64_t)span * (wk + 1) / threads);
      j->start = start;
      j->dist = dist;
      j->tot = t_use;
      j->emb = emb;
      j->lens = lens;
      if (threads == 1)
        run_job(j);
      else
        pthread_create(&tids[wk], NULL, run_job, j);
    }
    if (threads > 1)
      for (int wk = 0; wk < threads; ++wk) pthread_join(tids[wk], NULL);
  }
  if (rc == 0 && finalize && has_t) {
    for (int64_t i = 0; i < slots; ++i) {
      if (prec == 8) {
        const double t = ((double*)tot)[i];
        ((double*)dist)[i] = t == 0.0 ? 0.0 : ((double*)dist)[i] / t;
      } else {
        const float t = ((float*)tot)[i];
        ((float*)dist)[i] = t == 0.0f ? 0.0f : ((float*)dist)[i] / t;
      }
    }
  }
  free(rows64);
  free(rows32);
  free(lens64);
  free(lens32);
  free(tids);
  free(jobs);
  emb_free(&em);
  return rc;
}

/* condense (stripes.cpp:68-129) of one finalized full-range stripe set into
 * an n x n double matrix; returns -1 if an even-n duplicate slot disagrees. */
int orc_condense(int prec, int n, const void* dist, double* out) {
  const int S = n / 2;
  memset(out, 0, sizeof(double) * (size_t)n * (size_t)n);
  for (int s = 0; s < S; ++s)
    for (int k = 0; k < n; ++k) {
      const double v = prec == 8 ? ((const double*)dist)[(int64_t)s * n + k]
                                 : (double)((const float*)dist)[(int64_t)s * n + k];
      int l = k + s + 1;
      if (l >= n) l -= n;
      if (n % 2 == 0 && s == S - 1 && k >= n / 2) {
        if (prec == 8) {
          if (out[(int64_t)k * n + l] != v) return -1;
        } else { /* duplicate_slots_agree, fp32 (stripes.cpp:51-58) */
          const float a = (float)out[(int64_t)k * n + l], b = (float)v;
          const float da = a < b ? b - a : a - b;
          const float fa = a < 0 ? -a : a, fb = b < 0 ? -b : b;
          if (!(da <= 1e-6f * (fa > fb ? fa : fb))) return -1;
        }
        continue;
      }
      out[(int64_t)k * n + l] = v;
      out[(int64_t)l * n + k] = v;
    }
  return 0;
}

/* ============================================================ sparse form
 * orc_sparse_stripes: the same arithmetic as orc_compute_stripes (and so
 * the reference's), without the dense F x n / E x n embedding, for sizes
 * where the reference's leaf_rows_ cannot be built (C5: 273 GB; SURVEY
 * 8(c)). A row where both samples are zero adds exactly +0.0 to d and t
 * (|0-0|*L = 0, max(0,0)*L = 0, (0+0)*L = 0; kernels.hpp:55-66), so each
 * slot's sequential sum over rows in postorder equals the sequential sum
 * over the rows present in either sample, in postorder. Per sample, its
 * present rows are the upward closure of its leaves; weighted values fold
 * the children in ascending row order from 0.0 (embed.cpp:71-79: the
 * pending buffer starts at zero and children arrive in postorder; skipping
 * zero children leaves the bits unchanged), leaf values are c / total
 * (table.cpp:208-215). fp32: values and lengths computed in fp64 and
 * rounded once (embed.hpp:71-84), then fp32 update_entry without FMA.
 * Pinned bitwise to the dense form and the reference goldens in
 * tests/test_oracle.py. */
typedef struct sp_cols {
  int64_t* ptr;  /* [n+1] */
  int32_t* row;  /* present rows of each sample, ascending */
  double* val;   /* their embedding values (fp64) */
} sp_cols;

typedef struct sp_build_job {
  const orc_problem* p;
  int weighted, t, T;
  const int32_t* feat_row;  /* [F] leaf row of each feature */
  const int64_t* sptr;      /* table transposed by sample: [n+1] */
  const int32_t* sfeat;     /* features of each sample */
  const double* scnt;       /* counts */
  int64_t* cnt;             /* [n] present rows per sample (pass 1) */
  sp_cols* cols;            /* pass 2 output */
  int pass;
} sp_build_job;

static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return x < y ? -1 : x > y;
}

static void* sp_build(void* arg) {
  sp_build_job* j = (sp_build_job*)arg;
  const orc_problem* p = j->p;
  const int n = p->n_samples, E = p->n_rows;
  int32_t* stamp = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
  double* val = (double*)malloc(sizeof(double) * (size_t)E);
  int32_t* list = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
  if (!stamp || !val || !list) {
    free(stamp), free(val), free(list);
    return (void*)1;
  }
  for (int32_t r = 0; r < E; ++r) stamp[r] = -1;
  for (int k = j->t; k < n; k += j->T) {
    int32_t m = 0;
    for (int64_t e = j->sptr[k]; e < j->sptr[k + 1]; ++e) {
      int32_t r = j->feat_row[j->sfeat[e]];
      const double c = j->scnt[e];
      if (!(c > 0.0)) continue; /* presence: c > 0 (table.cpp:216-222) */
      stamp[r] = k;
      val[r] = j->weighted ? c / p->sample_totals[k] : 1.0;
      list[m++] = r;
      for (int32_t q = p->parent_row[r]; q >= 0 && stamp[q] != k; q = p->parent_row[q]) {
        stamp[q] = k;
        val[q] = j->weighted ? 0.0 : 1.0;
        list[m++] = q;
      }
    }
    if (j->pass == 1) {
      j->cnt[k] = m;
      continue;
    }
    qsort(list, (size_t)m, sizeof(int32_t), cmp_i32);
    int32_t* orow = j->cols->row + j->cols->ptr[k];
    double* oval = j->cols->val + j->cols->ptr[k];
    for (int32_t i = 0; i < m; ++i) {
      const int32_t r = list[i];
      orow[i] = r;
      oval[i] = val[r]; /* children (smaller rows) were folded into it already */
      const int32_t q = p->parent_row[r];
      if (j->weighted && q >= 0) val[q] += val[r];
    }
  }
  free(stamp);
  free(val);
  free(list);
  return NULL;
}

static int sp_columns(const orc_problem* p, int weighted, int threads, sp_cols* out) {
  const int n = p->n_samples, F = p->n_features, E = p->n_rows;
  const int64_t nnz = p->feat_ptr[F];
  int32_t* feat_row = (int32_t*)malloc(sizeof(int32_t) * (size_t)F);
  int64_t* sptr = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int32_t* sfeat = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
  double* scnt = (double*)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
  int64_t* cnt = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  int rc = (!feat_row || !sptr || !sfeat || !scnt || !cnt) ? -1 : 0;
  if (rc == 0) {
    for (int f = 0; f < F; ++f) feat_row[f] = -1;
    for (int32_t r = 0; r < E; ++r)
      if (p->leaf_feature[r] >= 0) feat_row[p->leaf_feature[r]] = r;
    for (int f = 0; f < F; ++f)
      if (feat_row[f] < 0) rc = -1; /* every feature is a leaf row after shear */
  }
  if (rc == 0) {
    for (int64_t e = 0; e < nnz; ++e) ++sptr[p->sample_idx[e] + 1];
    for (int k = 0; k < n; ++k) sptr[k + 1] += sptr[k];
    int64_t* at = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    if (!at) rc = -1;
    else {
      memcpy(at, sptr, sizeof(int64_t) * (size_t)n);
      for (int f = 0; f < F; ++f) /* ascending features within a sample */
        for (int64_t e = p->feat_ptr[f]; e < p->feat_ptr[f + 1]; ++e) {
          const int s = p->sample_idx[e];
          sfeat[at[s]] = f;
          scnt[at[s]++] = p->counts[e];
        }
      free(at);
    }
  }
  if (threads < 1) threads = 1;
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  sp_build_job* jobs = (sp_build_job*)malloc(sizeof(sp_build_job) * (size_t)threads);
  if (!tids || !jobs) rc = -1;
  out->ptr = NULL, out->row = NULL, out->val = NULL;
  for (int pass = 1; rc == 0 && pass <= 2; ++pass) {
    if (pass == 2) {
      out->ptr = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
      if (!out->ptr) {
        rc = -1;
        break;
      }
      out->ptr[0] = 0;
      for (int k = 0; k < n; ++k) out->ptr[k + 1] = out->ptr[k] + cnt[k];
      out->row = (int32_t*)malloc(sizeof(int32_t) * (size_t)(out->ptr[n] + 1));
      out->val = (double*)malloc(sizeof(double) * (size_t)(out->ptr[n] + 1));
      if (!out->row || !out->val) {
        rc = -1;
        break;
      }
    }
    for (int t = 0; t < threads; ++t) {
      sp_build_job* j = &jobs[t];
      j->p = p, j->weighted = weighted, j->t = t, j->T = threads, j->feat_row = feat_row;
      j->sptr = sptr, j->sfeat = sfeat, j->scnt = scnt, j->cnt = cnt, j->cols = out, j->pass = pass;
      pthread_create(&tids[t], NULL, sp_build, j);
    }
    for (int t = 0; t < threads; ++t) {
      void* r = NULL;
      pthread_join(tids[t], &r);
      if (r) rc = -1;
    }
  }
  free(feat_row), free(sptr), free(sfeat), free(scnt), free(cnt), free(tids), free(jobs);
  return rc;
}

typedef struct sp_job {
  const orc_problem* p;
  const sp_cols* cols;
  int metric, prec, start, s0, s1;
  void *dist, *tot;
} sp_job;

#define DEFINE_SPARSE(NAME, REAL)                                                            \
  static void NAME(const sp_job* j) {                                                        \
    const orc_problem* p = j->p;                                                             \
    const int n = p->n_samples, metric = j->metric;                                          \
    const int64_t* ptr = j->cols->ptr;                                                       \
    const int32_t* row = j->cols->row;                                                       \
    const double* val = j->cols->val;                                                        \
    for (int s = j->s0; s < j->s1; ++s)                                                      \
      for (int k = 0; k < n; ++k) {                                                          \
        int l = k + s + 1;                                                                   \
        if (l >= n) l -= n;                                                                  \
        int64_t a = ptr[k], ae = ptr[k + 1], b = ptr[l], be = ptr[l + 1];                    \
        REAL d = 0, t = 0;                                                                   \
        while (a < ae || b < be) {                                                           \
          const int32_t ra = a < ae ? row[a] : INT32_MAX, rb = b < be ? row[b] : INT32_MAX;   \
          const int32_t r = ra < rb ? ra : rb;                                               \
          const REAL u = ra == r ? (REAL)val[a++] : (REAL)0;                                 \
          const REAL v = rb == r ? (REAL)val[b++] : (REAL)0;                                 \
          const REAL L = (REAL)p->lengths[r];                                                \
          REAL diff = u - v;                                                                 \
          if (diff < (REAL)0) diff = -diff;                                                  \
          d += diff * L;                                                                     \
          if (metric == ORC_UW)                                                              \
            t += (u > v ? u : v) * L;                                                        \
          else if (metric == ORC_WN)                                                         \
            t += (u + v) * L;                                                                \
        }                                                                                    \
        const int64_t o = (int64_t)(s - j->start) * n + k;                                   \
        ((REAL*)j->dist)[o] = d;                                                             \
        if (j->tot) ((REAL*)j->tot)[o] = t;                                                  \
      }                                                                                      \
  }
DEFINE_SPARSE(sparse_f64, double)
DEFINE_SPARSE(sparse_f32, float)

static void* sp_run(void* arg) {
  const sp_job* j = (const sp_job*)arg;
  if (j->prec == 8)
    sparse_f64(j);
  else
    sparse_f32(j);
  return NULL;
}

/* Stripes [start, stop) as orc_compute_stripes (UW, WU, WN), sparse. */
int orc_sparse_stripes(const orc_problem* p, int metric, int prec, int start, int stop, void* dist,
                       void* tot, int finalize, int threads) {
  if (metric != ORC_UW && metric != ORC_WU && metric != ORC_WN) return -1;
  const int n = p->n_samples;
  sp_cols cols;
  if (sp_columns(p, metric != ORC_UW, threads, &cols)) {
    free(cols.ptr), free(cols.row), free(cols.val);
    return -1;
  }
  if (threads < 1) threads = 1;
  if (threads > stop - start) threads = stop - start;
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  sp_job* jobs = (sp_job*)malloc(sizeof(sp_job) * (size_t)threads);
  int rc = (!tids || !jobs) ? -1 : 0;
  const int has_t = metric != ORC_WU;
  for (int w = 0; rc == 0 && w < threads; ++w) {
    sp_job* j = &jobs[w];
    j->p = p, j->cols = &cols, j->metric = metric, j->prec = prec, j->start = start;
    j->s0 = start + (int)((int64_t)(stop - start) * w / threads);
    j->s1 = start + (int)((int64_t)(stop - start) * (w + 1) / threads);
    j->dist = dist, j->tot = has_t ? tot : NULL;
    pthread_create(&tids[w], NULL, sp_run, j);
  }
  if (rc == 0)
    for (int w = 0; w < threads; ++w) pthread_join(tids[w], NULL);
  if (rc == 0 && finalize && has_t) {
    const int64_t slots = (int64_t)(stop - start) * n;
    for (int64_t i = 0; i < slots; ++i) {
      if (prec == 8) {
        const double t = ((double*)tot)[i];
        ((double*)dist)[i] = t == 0.0 ? 0.0 : ((double*)dist)[i] / t;
      } else {
        const float t = ((float*)tot)[i];
        ((float*)dist)[i] = t == 0.0f ? 0.0f : ((float*)dist)[i] / t;
      }
    }
  }
  free(tids), free(jobs), free(cols.ptr), free(cols.row), free(cols.val);
  return rc;
}
