/*
 * nnm_oracle.c -- CPU restatement of the parclust NNM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path (paper_1402_3789_b200/csrc).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path never links, loads or calls anything in oracle/.
 *
 * Parity pinning: the restatement is checked against
 *   - the reference's own known-answer tests (tests/test_oracle_pin.py restates
 *     pkg/tests/test_metrics.py:41-55, test_oracle.py:38-60, test_pairgen.py:199-228,
 *     test_engine.py:50-148), and
 *   - golden fixtures produced by importing the reference here
 *     (tests/golden/make_golden.py -> tests/golden/ fixtures).
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/pkg/src/parclust/).
 *
 * Arithmetic contract (scipy 1.18.1 cdist): per pair, strictly
 * left-to-right FP64 accumulation over coordinates with no FMA contraction.
 * This file MUST be compiled with -ffp-contract=off (see oracle/Makefile).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "nnm_oracle.h"

/* ------------------------------------------------------------------------- */
/* metrics.py:59-73 (internal_pairwise -> scipy cdist kernels)                */
/* ------------------------------------------------------------------------- */

/* internal distance of one pair, scipy accumulation order (metrics.py:67-73) */
double orc_internal_distance(int metric, const double *x, const double *y, int d) {
  double acc = 0.0;
  int k;
  switch (metric) {
    case ORC_EUCLIDEAN:
    case ORC_SQEUCLIDEAN: /* cdist 'sqeuclidean' */
      for (k = 0; k < d; k++) {
        double t = x[k] - y[k];
        acc = acc + t * t;
      }
      return acc;
    case ORC_MANHATTAN: /* cdist 'cityblock' */
      for (k = 0; k < d; k++) acc = acc + fabs(x[k] - y[k]);
      return acc;
    case ORC_CHEBYSHEV: /* cdist 'chebyshev' */
      for (k = 0; k < d; k++) {
        double t = fabs(x[k] - y[k]);
        acc = (t > acc) ? t : acc;
      }
      return acc;
    default:
      return NAN;
  }
}

/* metrics.py:86-90 */
double orc_reported(int metric, double internal) {
  return metric == ORC_EUCLIDEAN ? sqrt(internal) : internal;
}

/* metrics.py:93-103 */
double orc_effective_threshold(int metric, double dmax) {
  return metric == ORC_EUCLIDEAN ? dmax * dmax : dmax;
}

/* ------------------------------------------------------------------------- */
/* pair key (model.py:100-106): (dist, a, b), a < b                           */
/* ------------------------------------------------------------------------- */

typedef struct {
  double d;
  int64_t a, b;
} key_t;

static inline int key_less(const key_t *x, const key_t *y) {
  if (x->d != y->d) return x->d < y->d;
  if (x->a != y->a) return x->a < y->a;
  return x->b < y->b;
}

/* bounded max-heap holding the P smallest keys seen */
typedef struct {
  key_t *v;
  int64_t len, cap;
} heap_t;

static void heap_sift_down(heap_t *h, int64_t i) {
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < h->len && key_less(&h->v[m], &h->v[l])) m = l;
    if (r < h->len && key_less(&h->v[m], &h->v[r])) m = r;
    if (m == i) return;
    key_t t = h->v[i];
    h->v[i] = h->v[m];
    h->v[m] = t;
    i = m;
  }
}

static void heap_offer(heap_t *h, double d, int64_t a, int64_t b) {
  key_t k = {d, a, b};
  if (h->len < h->cap) {
    int64_t i = h->len++;
    h->v[i] = k;
    while (i > 0) {
      int64_t p = (i - 1) / 2;
      if (!key_less(&h->v[p], &h->v[i])) break;
      key_t t = h->v[p];
      h->v[p] = h->v[i];
      h->v[i] = t;
      i = p;
    }
  } else if (key_less(&k, &h->v[0])) {
    h->v[0] = k;
    heap_sift_down(h, 0);
  }
}

static int cmp_key(const void *x, const void *y) {
  const key_t *a = (const key_t *)x, *b = (const key_t *)y;
  if (key_less(a, b)) return -1;
  if (key_less(b, a)) return 1;
  return 0;
}

/* ------------------------------------------------------------------------- */
/* eligibility (pairgen.py:169-210)                                          */
/* ------------------------------------------------------------------------- */

typedef struct {
  const double *X;
  int64_t n;
  int d, metric;
  const int64_t *roots, *sizes;
  int has_thr;
  double thr;
  int64_t kl2, kl3; /* <0: unset */
  const double *XT; /* d x ldt transposed copy (zero padded), built once per call */
  int64_t ldt;
} scan_ctx_t;

/* pairgen.py:169-187: roots differ, dist <= thr, sizes <= kl2, sa+sb <= kl3 */
static inline int pre_eligible(const scan_ctx_t *c, int64_t a, int64_t b) {
  if (c->roots[a] == c->roots[b]) return 0;
  int64_t sa = c->sizes[a], sb = c->sizes[b];
  if (c->kl2 >= 0 && (sa > c->kl2 || sb > c->kl2)) return 0;
  if (c->kl3 >= 0 && sa + sb > c->kl3) return 0;
  return 1;
}

/* ------------------------------------------------------------------------- */
/* top-P selection (pairgen.py:247-324, oracle.py:110-131)                    */
/* ------------------------------------------------------------------------- */

typedef struct {
  const scan_ctx_t *ctx;
  int64_t P;
  int64_t *next_row; /* shared work counter */
  pthread_mutex_t *mu;
  heap_t heap;
} worker_t;

#define ROW_CHUNK 16
#define COL_BLOCK 256
#define RB 4  /* rows per register block */
#define CV 8  /* doubles per vector */

typedef double v8d __attribute__((vector_size(64)));
typedef long long v8l __attribute__((vector_size(64)));

/* Distances of RB rows x[r] to the columns of a transposed block yT[d][COL_BLOCK]
 * (zero padded past cb).  Register-blocked: RB x 2 vectors of accumulators, every
 * yT load is shared by RB rows.  Each pair still accumulates strictly left to right
 * over k with separate IEEE sub / mul / add (SIMD lanes are different pairs; this
 * file is compiled with -ffp-contract=off), so every value stays bit-identical to
 * orc_internal_distance (scipy cdist order). */
__attribute__((target_clones("avx512f", "avx2", "default")))
static void block_dist(int metric, const double *const *x, const double *yT, int64_t ldt, int d,
                       int cb, double (*acc)[COL_BLOCK]) {
  const v8l absmask = {~(1LL << 63), ~(1LL << 63), ~(1LL << 63), ~(1LL << 63),
                       ~(1LL << 63), ~(1LL << 63), ~(1LL << 63), ~(1LL << 63)};
  for (int c0 = 0; c0 < cb; c0 += 2 * CV) {
    v8d a0[RB], a1[RB];
    for (int r = 0; r < RB; r++) {
      a0[r] = (v8d){0, 0, 0, 0, 0, 0, 0, 0};
      a1[r] = a0[r];
    }
    for (int k = 0; k < d; k++) {
      v8d y0, y1;
      memcpy(&y0, yT + (size_t)k * ldt + c0, sizeof(v8d));
      memcpy(&y1, yT + (size_t)k * ldt + c0 + CV, sizeof(v8d));
      for (int r = 0; r < RB; r++) {
        const double xs = x[r][k];
        const v8d xv = {xs, xs, xs, xs, xs, xs, xs, xs};
        v8d t0 = xv - y0, t1 = xv - y1;
        if (metric == ORC_EUCLIDEAN || metric == ORC_SQEUCLIDEAN) {
          v8d s0 = t0 * t0, s1 = t1 * t1;
          a0[r] = a0[r] + s0;
          a1[r] = a1[r] + s1;
        } else {
          t0 = (v8d)((v8l)t0 & absmask);
          t1 = (v8d)((v8l)t1 & absmask);
          if (metric == ORC_MANHATTAN) {
            a0[r] = a0[r] + t0;
            a1[r] = a1[r] + t1;
          } else { /* chebyshev: acc = (t > acc) ? t : acc */
            v8l m0 = t0 > a0[r], m1 = t1 > a1[r];
            a0[r] = (v8d)(((v8l)t0 & m0) | ((v8l)a0[r] & ~m0));
            a1[r] = (v8d)(((v8l)t1 & m1) | ((v8l)a1[r] & ~m1));
          }
        }
      }
    }
    for (int r = 0; r < RB; r++) {
      memcpy(&acc[r][c0], &a0[r], sizeof(v8d));
      memcpy(&acc[r][c0 + CV], &a1[r], sizeof(v8d));
    }
  }
}

static void *topp_worker(void *arg) {
  worker_t *w = (worker_t *)arg;
  const scan_ctx_t *c = w->ctx;
  const int64_t n = c->n;
  const int d = c->d;
  double(*acc)[COL_BLOCK] = (double(*)[COL_BLOCK])malloc(sizeof(double) * RB * COL_BLOCK);
  for (;;) {
    int64_t r0;
    pthread_mutex_lock(w->mu);
    r0 = *w->next_row;
    *w->next_row += ROW_CHUNK;
    pthread_mutex_unlock(w->mu);
    if (r0 >= n) break;
    int64_t r1 = r0 + ROW_CHUNK < n ? r0 + ROW_CHUNK : n;
    for (int64_t b0 = r0 + 1; b0 < n; b0 += COL_BLOCK) {
      const int cb = (int)(n - b0 < COL_BLOCK ? n - b0 : COL_BLOCK);
      const double *yT = c->XT + b0; /* lanes past cb read the zero padding, never used */
      for (int64_t ag = r0; ag < r1; ag += RB) {
        if (ag + 1 >= b0 + cb) continue;
        const double *xr[RB];
        for (int r = 0; r < RB; r++) xr[r] = c->X + (ag + r < r1 ? ag + r : ag) * d;
        block_dist(c->metric, xr, yT, c->ldt, d, cb, acc);
        for (int r = 0; r < RB && ag + r < r1; r++) {
          const int64_t a = ag + r;
          /* a pair whose distance exceeds the threshold (pairgen.py:197-198) or the
           * largest key of a full heap cannot be selected: skip it before the
           * eligibility lookups (the selection itself is unchanged) */
          double lim = c->has_thr ? c->thr : INFINITY;
          if (w->heap.len == w->heap.cap && w->heap.v[0].d < lim) lim = w->heap.v[0].d;
          for (int j = (b0 > a ? 0 : (int)(a + 1 - b0)); j < cb; j++) {
            const double dist = acc[r][j];
            if (dist > lim) continue;
            const int64_t b = b0 + j;
            if (!pre_eligible(c, a, b)) continue;
            heap_offer(&w->heap, dist, a, b);
            if (w->heap.len == w->heap.cap && w->heap.v[0].d < lim) lim = w->heap.v[0].d;
          }
        }
      }
    }
  }
  free(acc);
  return NULL;
}

int64_t orc_top_p(const double *X, int64_t n, int d, int metric, const int64_t *roots,
                  const int64_t *sizes, double thr, int64_t kl2, int64_t kl3, int64_t P,
                  int nthreads, double *out_d, int64_t *out_a, int64_t *out_b) {
  if (P < 1 || n < 1 || d < 1) return -1; /* pairgen.py:256-257 */
  if (nthreads < 1) nthreads = 1;
  const int64_t ldt = n + 2 * COL_BLOCK;
  double *XT = (double *)calloc((size_t)d * ldt, sizeof(double));
  for (int64_t i = 0; i < n; i++)
    for (int k = 0; k < d; k++) XT[(size_t)k * ldt + i] = X[i * d + k];
  scan_ctx_t c = {X, n, d, metric, roots, sizes, !isnan(thr), thr, kl2, kl3, XT, ldt};
  int64_t npairs = n * (n - 1) / 2;
  int64_t cap = P < npairs ? P : npairs;
  if (cap < 1) cap = 1;
  worker_t *ws = (worker_t *)calloc((size_t)nthreads, sizeof(worker_t));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  int64_t next_row = 0;
  for (int t = 0; t < nthreads; t++) {
    ws[t].ctx = &c;
    ws[t].P = P;
    ws[t].next_row = &next_row;
    ws[t].mu = &mu;
    ws[t].heap.cap = cap;
    ws[t].heap.v = (key_t *)malloc((size_t)cap * sizeof(key_t));
  }
  if (nthreads == 1) {
    topp_worker(&ws[0]);
  } else {
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, topp_worker, &ws[t]);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
  }
  /* reduce_topp (pairgen.py:301-316): associative merge of per-thread buffers */
  int64_t total = 0;
  for (int t = 0; t < nthreads; t++) total += ws[t].heap.len;
  key_t *all = (key_t *)malloc((size_t)(total > 0 ? total : 1) * sizeof(key_t));
  int64_t off = 0;
  for (int t = 0; t < nthreads; t++) {
    memcpy(all + off, ws[t].heap.v, (size_t)ws[t].heap.len * sizeof(key_t));
    off += ws[t].heap.len;
    free(ws[t].heap.v);
  }
  qsort(all, (size_t)total, sizeof(key_t), cmp_key); /* lexsort((b,a,dist)) */
  int64_t len = total < P ? total : P;
  for (int64_t i = 0; i < len; i++) {
    out_d[i] = all[i].d;
    out_a[i] = all[i].a;
    out_b[i] = all[i].b;
  }
  free(all);
  free(ws);
  free(th);
  free(XT);
  return len;
}

/* ------------------------------------------------------------------------- */
/* union-find forest (model.py:109-187)                                       */
/* ------------------------------------------------------------------------- */

typedef struct {
  int64_t *parent, *size;
  int64_t count, n;
} forest_t;

static void forest_init(forest_t *f, int64_t n) {
  f->n = n;
  f->count = n;
  f->parent = (int64_t *)malloc((size_t)n * sizeof(int64_t));
  f->size = (int64_t *)malloc((size_t)n * sizeof(int64_t));
  for (int64_t i = 0; i < n; i++) {
    f->parent[i] = i;
    f->size[i] = 1;
  }
}

static void forest_free(forest_t *f) {
  free(f->parent);
  free(f->size);
}

/* model.py:136-146: find with path compression */
static int64_t forest_find(forest_t *f, int64_t i) {
  int64_t r = i;
  while (f->parent[r] != r) r = f->parent[r];
  while (f->parent[i] != r) {
    int64_t nx = f->parent[i];
    f->parent[i] = r;
    i = nx;
  }
  return r;
}

/* model.py:148-160: union keeps the smaller root index */
static int64_t forest_union_roots(forest_t *f, int64_t ri, int64_t rj) {
  int64_t keep = ri < rj ? ri : rj, drop = ri < rj ? rj : ri;
  f->parent[drop] = keep;
  f->size[keep] += f->size[drop];
  f->count--;
  return keep;
}

/* model.py:168-187: full compression, per-point root and size */
static void forest_snapshot(forest_t *f, int64_t *roots, int64_t *sizes) {
  for (int64_t i = 0; i < f->n; i++) roots[i] = forest_find(f, i);
  if (sizes)
    for (int64_t i = 0; i < f->n; i++) sizes[i] = f->size[roots[i]];
}

/* ------------------------------------------------------------------------- */
/* engine.run (engine.py:154-199) with order_batch (:73-87) and                */
/* process_batch (:90-143)                                                    */
/* ------------------------------------------------------------------------- */

static int stop_reason(int64_t count, int64_t kl1) { /* engine.py:146-151 */
  if (count == 1) return ORC_STOP_SINGLE_CLUSTER;
  if (kl1 >= 0 && count <= kl1) return ORC_STOP_KL1;
  return ORC_STOP_NONE;
}

int orc_run(const double *X, int64_t n, int d, int metric, int64_t kl1, int64_t kl2, int64_t kl3,
            int64_t kl4, double dmax, int64_t P, int nthreads, orc_merge_t *out,
            int64_t *out_n_merges, int64_t *out_assign, int64_t *out_rounds, int *out_stop,
            orc_round_t *counters, int64_t counters_cap, int64_t *out_n_counters) {
  if (P < 1 || n < 1 || d < 1) return -1;
  double thr = isnan(dmax) ? NAN : orc_effective_threshold(metric, dmax);
  forest_t f;
  forest_init(&f, n);
  int64_t *roots = (int64_t *)malloc((size_t)n * sizeof(int64_t));
  int64_t *sizes = (int64_t *)malloc((size_t)n * sizeof(int64_t));
  int64_t npairs = n * (n - 1) / 2;
  int64_t cap = P < npairs ? P : (npairs > 0 ? npairs : 1);
  double *bd = (double *)malloc((size_t)cap * sizeof(double));
  int64_t *ba = (int64_t *)malloc((size_t)cap * sizeof(int64_t));
  int64_t *bb = (int64_t *)malloc((size_t)cap * sizeof(int64_t));
  int64_t *order = (int64_t *)malloc((size_t)cap * sizeof(int64_t));
  int64_t nm = 0, rounds = 0, nc = 0;
  int reason;
  for (;;) {
    reason = stop_reason(f.count, kl1);
    if (reason != ORC_STOP_NONE) break;
    forest_snapshot(&f, roots, sizes); /* make_snapshot, pairgen.py:150-166 */
    int64_t len = orc_top_p(X, n, d, metric, roots, sizes, thr, kl2, kl3, cap, nthreads, bd, ba,
                            bb);
    if (len <= 0) {
      reason = ORC_STOP_NO_ELIGIBLE;
      break;
    }
    rounds++;
    /* order_batch: stable partition, priority = min(size_a,size_b) < kl4 at round start */
    int64_t k = 0;
    if (kl4 >= 0) {
      for (int64_t i = 0; i < len; i++) {
        int64_t s = sizes[ba[i]] < sizes[bb[i]] ? sizes[ba[i]] : sizes[bb[i]];
        if (s < kl4) order[k++] = i;
      }
      for (int64_t i = 0; i < len; i++) {
        int64_t s = sizes[ba[i]] < sizes[bb[i]] ? sizes[ba[i]] : sizes[bb[i]];
        if (!(s < kl4)) order[k++] = i;
      }
    } else {
      for (int64_t i = 0; i < len; i++) order[i] = i;
    }
    /* process_batch: live re-checks */
    int64_t same = 0, s2 = 0, s3 = 0, unproc = 0, merged = 0;
    for (int64_t pos = 0; pos < len; pos++) {
      int64_t i = order[pos];
      int64_t a = ba[i], b = bb[i];
      int64_t ra = forest_find(&f, a), rb = forest_find(&f, b);
      if (ra == rb) {
        same++;
        continue;
      }
      int64_t sa = f.size[ra], sb = f.size[rb];
      if (kl2 >= 0 && (sa > kl2 || sb > kl2)) {
        s2++;
        continue;
      }
      if (kl3 >= 0 && sa + sb > kl3) {
        s3++;
        continue;
      }
      int64_t keep = forest_union_roots(&f, ra, rb);
      orc_merge_t *m = &out[nm++];
      m->round = rounds;
      m->root_a = keep;
      m->root_b = keep == ra ? rb : ra;
      m->dist = orc_reported(metric, bd[i]);
      m->new_size = f.size[keep];
      m->point_a = a;
      m->point_b = b;
      merged++;
      if (f.count == 1 || (kl1 >= 0 && f.count <= kl1)) {
        unproc = len - pos - 1;
        break;
      }
    }
    if (counters && nc < counters_cap) {
      orc_round_t *rc = &counters[nc];
      rc->round = rounds;
      rc->selected = len;
      rc->merged = merged;
      rc->same_root = same;
      rc->kl2 = s2;
      rc->kl3 = s3;
      rc->unprocessed = unproc;
    }
    nc++;
  }
  forest_snapshot(&f, out_assign, NULL);
  *out_n_merges = nm;
  *out_rounds = rounds;
  *out_stop = reason;
  if (out_n_counters) *out_n_counters = nc;
  free(roots);
  free(sizes);
  free(bd);
  free(ba);
  free(bb);
  free(order);
  forest_free(&f);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* oracle_single_linkage (oracle.py:59-107): flat Kruskal over all pairs       */
/* ------------------------------------------------------------------------- */

int orc_single_linkage(const double *X, int64_t n, int d, int metric, int64_t kl1, int64_t kl2,
                       int64_t kl3, double dmax, orc_merge_t *out, int64_t *out_n_merges,
                       int64_t *out_assign) {
  if (n < 1 || d < 1) return -1;
  int64_t npairs = n * (n - 1) / 2;
  key_t *all = (key_t *)malloc((size_t)(npairs > 0 ? npairs : 1) * sizeof(key_t));
  if (!all) return -2;
  int64_t p = 0;
  for (int64_t a = 0; a < n; a++)
    for (int64_t b = a + 1; b < n; b++) {
      all[p].d = orc_internal_distance(metric, X + a * d, X + b * d, d);
      all[p].a = a;
      all[p].b = b;
      p++;
    }
  qsort(all, (size_t)npairs, sizeof(key_t), cmp_key); /* oracle.py:48-56 */
  double thr = isnan(dmax) ? NAN : orc_effective_threshold(metric, dmax);
  forest_t f;
  forest_init(&f, n);
  int64_t nm = 0;
  for (int64_t i = 0; i < npairs; i++) {
    if (f.count == 1 || (kl1 >= 0 && f.count <= kl1)) break;
    if (!isnan(thr) && all[i].d > thr) break;
    int64_t rx = forest_find(&f, all[i].a), ry = forest_find(&f, all[i].b);
    if (rx == ry) continue;
    int64_t sx = f.size[rx], sy = f.size[ry];
    if (kl2 >= 0 && (sx > kl2 || sy > kl2)) continue;
    if (kl3 >= 0 && sx + sy > kl3) continue;
    int64_t keep = forest_union_roots(&f, rx, ry);
    orc_merge_t *m = &out[nm++];
    m->round = 0;
    m->root_a = keep;
    m->root_b = keep == rx ? ry : rx;
    m->dist = orc_reported(metric, all[i].d);
    m->new_size = f.size[keep];
    m->point_a = all[i].a;
    m->point_b = all[i].b;
  }
  forest_snapshot(&f, out_assign, NULL);
  *out_n_merges = nm;
  forest_free(&f);
  free(all);
  return 0;
}

/* pairwise tile for metric pinning tests: out[i*ny+j] = internal(x_i, y_j) */
void orc_pairwise(int metric, const double *x, int64_t nx, const double *y, int64_t ny, int d,
                  double *out) {
  for (int64_t i = 0; i < nx; i++)
    for (int64_t j = 0; j < ny; j++)
      out[i * ny + j] = orc_internal_distance(metric, x + i * d, y + j * d, d);
}
