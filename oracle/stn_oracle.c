/*
 * TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference stem executor.
 *
 * This is the parity oracle for the B200 executor: only tests/, the smoke()
 * check of __graft_entry__.py and bench.py's cpu_baseline leg may load it, and
 * only as the checker. The product path (libstn_exec.so) never calls it.
 *
 * It executes a flattened plan (include/stn_exec.h, stn_plan_desc) exactly as
 * the reference `stemtn` runtime does, in the same loop order and with the
 * same IEEE operations, so its results are bitwise identical to the reference
 * (pinned against outputs of the reference itself: tests/golden/, produced by
 * oracle/_ref/ref_tool from /root/reference):
 *   load_leaf     runtime.hpp:367-384  (mixed-radix digits 371-378,
 *                                        restrict_axis tensor.hpp:102-117,
 *                                        from_tensor runtime.hpp:93-100)
 *   permute       runtime.hpp:113-140  (odometer stride walk)
 *   gemm          runtime.hpp:386-418  (D-batched C[d] += A[d] * B[d], loop m,k,n)
 *   run           runtime.hpp:420-453  (live map, cache fetch, peak/mults bookkeeping)
 *   branch cache  runtime.hpp:456-500  (branch steps once, keep consumed outputs)
 *   run_scheme    runtime.hpp:555-605  (ascending-assignment double sum)
 * Complex products are written out as (ar*br - ai*bi, ar*bi + ai*br), which is
 * what GCC emits for std::complex multiplication of finite values; the file is
 * compiled with -ffp-contract=off so no FMA changes the rounding.
 */
#define _POSIX_C_SOURCE 200809L
#include <math.h>
#include <time.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "stn_exec.h"

static __thread char g_err[512];
void stn_set_error_c(const char *msg) {
  strncpy(g_err, msg, sizeof g_err - 1);
  g_err[sizeof g_err - 1] = 0;
}
const char *oracle_last_error(void) { return g_err; }

/* ---- typed tensors ------------------------------------------------------------ */
typedef struct {
  int rank;
  int dims[64];
  size_t n;
  void *data; /* interleaved (re, im) of float or double */
} tt_t;

static size_t elsize(int prec) { return prec == STN_SINGLE ? 8 : 16; }

static int tt_alloc(tt_t *t, int rank, const int *dims, int prec) {
  t->rank = rank;
  t->n = 1;
  for (int i = 0; i < rank; ++i) {
    t->dims[i] = dims[i];
    t->n *= (size_t)dims[i];
  }
  t->data = calloc(t->n ? t->n : 1, elsize(prec));
  return t->data != NULL;
}
static void tt_free(tt_t *t) {
  free(t->data);
  t->data = NULL;
}
static int tt_copy(tt_t *dst, const tt_t *src, int prec) {
  if (!tt_alloc(dst, src->rank, src->dims, prec)) return 0;
  memcpy(dst->data, src->data, src->n * elsize(prec));
  return 1;
}

/* permute: result axis i is input axis perm[i] (runtime.hpp:113-140) */
static int tt_permute(tt_t *out, const tt_t *t, const int32_t *perm, int prec) {
  int r = t->rank;
  int identity = 1;
  for (int i = 0; i < r; ++i) identity &= (perm[i] == i);
  if (r <= 1 || identity) return tt_copy(out, t, prec);
  int od[64];
  for (int i = 0; i < r; ++i) od[i] = t->dims[perm[i]];
  if (!tt_alloc(out, r, od, prec)) return 0;
  size_t in_strides[64], step[64];
  int idx[64];
  in_strides[r - 1] = 1;
  for (int i = r - 2; i >= 0; --i) in_strides[i] = in_strides[i + 1] * (size_t)t->dims[i + 1];
  for (int i = 0; i < r; ++i) {
    step[i] = in_strides[perm[i]];
    idx[i] = 0;
  }
  size_t es = elsize(prec), src = 0;
  char *o = (char *)out->data;
  const char *s = (const char *)t->data;
  for (size_t flat = 0; flat < out->n; ++flat) {
    memcpy(o + flat * es, s + src * es, es);
    for (int ax = r - 1; ax >= 0; --ax) {
      idx[ax]++;
      src += step[ax];
      if (idx[ax] < od[ax]) break;
      src -= (size_t)od[ax] * step[ax];
      idx[ax] = 0;
    }
  }
  return 1;
}

/* ---- plan-side helpers -------------------------------------------------------- */
typedef struct {
  const stn_plan_desc *d;
  int prec;
  int *step_of_node; /* node -> step index or -1 */
  int *leaf_of_node; /* node -> leaf index or -1 */
} plan_t;

static int plan_init(plan_t *p, const stn_plan_desc *d, int prec) {
  p->d = d;
  p->prec = prec;
  p->step_of_node = (int *)malloc(sizeof(int) * (size_t)(d->n_nodes > 0 ? d->n_nodes : 1));
  p->leaf_of_node = (int *)malloc(sizeof(int) * (size_t)(d->n_nodes > 0 ? d->n_nodes : 1));
  if (!p->step_of_node || !p->leaf_of_node) return 0;
  for (int i = 0; i < d->n_nodes; ++i) p->step_of_node[i] = p->leaf_of_node[i] = -1;
  for (int i = 0; i < d->n_steps; ++i) {
    if (d->steps[i].node < 0 || d->steps[i].node >= d->n_nodes) return 0;
    p->step_of_node[d->steps[i].node] = i;
  }
  for (int i = 0; i < d->n_leaves; ++i) {
    if (d->leaves[i].node < 0 || d->leaves[i].node >= d->n_nodes) return 0;
    p->leaf_of_node[d->leaves[i].node] = i;
  }
  return 1;
}
static void plan_free(plan_t *p) {
  free(p->step_of_node);
  free(p->leaf_of_node);
}

/* mixed-radix digits, first sliced edge most significant (runtime.hpp:371-378) */
int oracle_decode_assignment(const stn_plan_desc *d, uint64_t assignment, int32_t *digits) {
  uint64_t rest = assignment;
  for (int i = d->n_sliced; i-- > 0;) {
    uint64_t dim = (uint64_t)d->sliced_dims[i];
    digits[i] = (int32_t)(rest % dim);
    rest /= dim;
  }
  return STN_OK;
}

/* load_leaf (runtime.hpp:367-384): restrict in double, cast to R, permute */
static int load_leaf(const plan_t *p, int node, const int32_t *digits, tt_t *out) {
  const stn_leaf_desc *l = &p->d->leaves[p->leaf_of_node[node]];
  int rank = l->rank, dims[64];
  size_t n = 1;
  for (int i = 0; i < rank; ++i) {
    dims[i] = l->dims[i];
    n *= (size_t)dims[i];
  }
  double *cur = (double *)malloc(16 * (n ? n : 1));
  if (!cur) return 0;
  memcpy(cur, l->values, 16 * n);
  for (int s = 0; s < l->n_sliced; ++s) { /* restrict_axis (tensor.hpp:102-117) */
    int axis = l->sliced_axis[s], index = digits[l->sliced_index[s]];
    size_t outer = 1, inner = 1, ax = (size_t)dims[axis];
    for (int i = 0; i < axis; ++i) outer *= (size_t)dims[i];
    for (int i = axis + 1; i < rank; ++i) inner *= (size_t)dims[i];
    double *nx = (double *)malloc(16 * (outer * inner ? outer * inner : 1));
    if (!nx) {
      free(cur);
      return 0;
    }
    for (size_t o = 0; o < outer; ++o)
      for (size_t in = 0; in < inner; ++in)
        memcpy(nx + 2 * (o * inner + in), cur + 2 * ((o * ax + (size_t)index) * inner + in), 16);
    free(cur);
    cur = nx;
    for (int i = axis; i < rank - 1; ++i) dims[i] = dims[i + 1];
    rank--;
  }
  tt_t typed;
  if (!tt_alloc(&typed, rank, dims, p->prec)) {
    free(cur);
    return 0;
  }
  if (p->prec == STN_SINGLE) {
    float *f = (float *)typed.data;
    for (size_t i = 0; i < 2 * typed.n; ++i) f[i] = (float)cur[i];
  } else {
    memcpy(typed.data, cur, 16 * typed.n);
  }
  free(cur);
  int ok = tt_permute(out, &typed, l->perm, p->prec);
  tt_free(&typed);
  return ok;
}

#define GEMM_LOOP(R)                                                               \
  do {                                                                             \
    const R *pa = (const R *)al.data, *pb = (const R *)bl.data;                    \
    R *pc = (R *)c.data;                                                           \
    for (size_t dd = 0; dd < D; ++dd) {                                            \
      const R *ba = pa + 2 * dd * M * K;                                           \
      const R *bb = pb + 2 * dd * K * N;                                           \
      R *bc = pc + 2 * dd * M * N;                                                 \
      for (size_t m = 0; m < M; ++m)                                               \
        for (size_t k = 0; k < K; ++k) {                                           \
          R ar = ba[2 * (m * K + k)], ai = ba[2 * (m * K + k) + 1];                \
          const R *brow = bb + 2 * k * N;                                          \
          R *crow = bc + 2 * m * N;                                                \
          for (size_t nn = 0; nn < N; ++nn) {                                      \
            R br = brow[2 * nn], bi = brow[2 * nn + 1];                            \
            R re = ar * br - ai * bi;                                              \
            R im = ar * bi + ai * br;                                              \
            crow[2 * nn] += re;                                                    \
            crow[2 * nn + 1] += im;                                                \
          }                                                                        \
        }                                                                          \
    }                                                                              \
  } while (0)

/* gemm (runtime.hpp:386-418) */
static int gemm(const plan_t *p, const stn_step_desc *s, const tt_t *a, const tt_t *b, tt_t *out) {
  tt_t al, bl, c;
  if (!tt_permute(&al, a, s->lperm, p->prec)) return 0;
  if (!tt_permute(&bl, b, s->rperm, p->prec)) {
    tt_free(&al);
    return 0;
  }
  size_t D = (size_t)s->D, M = (size_t)s->M, N = (size_t)s->N, K = (size_t)s->K;
  int produced[64];
  for (int i = 0; i < s->orank; ++i) produced[s->operm[i]] = s->out_dims[i];
  if (!tt_alloc(&c, s->orank, produced, p->prec) || c.n != D * M * N) {
    tt_free(&al);
    tt_free(&bl);
    return 0;
  }
  if (p->prec == STN_SINGLE)
    GEMM_LOOP(float);
  else
    GEMM_LOOP(double);
  tt_free(&al);
  tt_free(&bl);
  int ok = tt_permute(out, &c, s->operm, p->prec);
  tt_free(&c);
  return ok;
}

/* ---- memory-lean gemm (same arithmetic, no materialised transposes) -----------
 * Every element of the reference's product C[d,m,n] is the fold, over k ascending,
 * of crow[n] += amk * brow[n] starting from 0 (runtime.hpp:392, 400-405); its
 * value depends only on that order, not on the loop nest around it. This variant
 * computes each element of the permuted output (runtime.hpp:417) straight from the
 * un-permuted operands through strides (the lperm / rperm / operm bookkeeping of
 * runtime.hpp:387-388, 409-417), so a step holds only a, b and its output: a
 * 2^33-element stem (64 GiB complex64, BASELINE cfg5) needs 128 GiB instead of the
 * reference's 256 GiB (a, al, c and permute(c)). Output elements are independent,
 * so host threads split them without changing a bit. */
typedef struct {
  const stn_step_desc *s;
  const tt_t *a, *b;
  tt_t *out;
  int prec;
  int n_out;
  size_t out_dim[64];
  int64_t out_sa[64], out_sb[64]; /* per canonical output axis, element strides */
  size_t K;
  int64_t *ka, *kb; /* per k (row-major over the K axes), element offsets */
  size_t lo, hi;
} lean_job;

#define LEAN_LOOP(R)                                                                  \
  do {                                                                                \
    const R *pa = (const R *)j->a->data, *pb = (const R *)j->b->data;                 \
    R *po = (R *)j->out->data;                                                        \
    size_t idx[64];                                                                   \
    size_t rem = j->lo;                                                               \
    int64_t ab = 0, bb = 0;                                                           \
    for (int i = j->n_out - 1; i >= 0; --i) {                                         \
      idx[i] = rem % j->out_dim[i];                                                   \
      rem /= j->out_dim[i];                                                           \
      ab += (int64_t)idx[i] * j->out_sa[i];                                           \
      bb += (int64_t)idx[i] * j->out_sb[i];                                           \
    }                                                                                 \
    for (size_t o = j->lo; o < j->hi; ++o) {                                          \
      R cr = 0, ci = 0;                                                               \
      for (size_t k = 0; k < j->K; ++k) {                                             \
        const R *x = pa + 2 * (ab + j->ka[k]), *y = pb + 2 * (bb + j->kb[k]);         \
        R ar = x[0], ai = x[1], br = y[0], bi = y[1];                                 \
        R re = ar * br - ai * bi;                                                     \
        R im = ar * bi + ai * br;                                                     \
        cr += re;                                                                     \
        ci += im;                                                                     \
      }                                                                               \
      po[2 * o] = cr;                                                                 \
      po[2 * o + 1] = ci;                                                             \
      for (int i = j->n_out - 1; i >= 0; --i) { /* odometer over the output axes */  \
        idx[i]++;                                                                     \
        ab += j->out_sa[i];                                                           \
        bb += j->out_sb[i];                                                           \
        if (idx[i] < j->out_dim[i]) break;                                            \
        ab -= (int64_t)j->out_dim[i] * j->out_sa[i];                                  \
        bb -= (int64_t)j->out_dim[i] * j->out_sb[i];                                  \
        idx[i] = 0;                                                                   \
      }                                                                               \
    }                                                                                 \
  } while (0)

static void *lean_worker(void *arg) {
  lean_job *j = (lean_job *)arg;
  if (j->lo >= j->hi) return NULL;
  if (j->prec == STN_SINGLE)
    LEAN_LOOP(float);
  else
    LEAN_LOOP(double);
  return NULL;
}

static int gemm_lean(const plan_t *p, const stn_step_desc *s, const tt_t *a, const tt_t *b,
                     tt_t *out, int threads) {
  const int nd = s->nd, nm = s->nm, nk = s->nk;
  int64_t as[64], bs[64];
  as[a->rank - 1 > 0 ? a->rank - 1 : 0] = 1;
  for (int i = a->rank - 1; i >= 0; --i) as[i] = i == a->rank - 1 ? 1 : as[i + 1] * a->dims[i + 1];
  for (int i = b->rank - 1; i >= 0; --i) bs[i] = i == b->rank - 1 ? 1 : bs[i + 1] * b->dims[i + 1];
  lean_job base;
  memset(&base, 0, sizeof base);
  base.s = s, base.a = a, base.b = b, base.out = out, base.prec = p->prec;
  base.n_out = s->orank;
  /* canonical output axis i = produced [D|M|N] axis operm[i] */
  for (int i = 0; i < s->orank; ++i) {
    int q = s->operm[i];
    base.out_dim[i] = (size_t)s->out_dims[i];
    if (q < nd) {
      base.out_sa[i] = as[s->lperm[q]];
      base.out_sb[i] = bs[s->rperm[q]];
    } else if (q < nd + nm) {
      base.out_sa[i] = as[s->lperm[q]];
      base.out_sb[i] = 0;
    } else {
      base.out_sa[i] = 0;
      base.out_sb[i] = bs[s->rperm[nd + nk + (q - nd - nm)]];
    }
  }
  /* k ascending = row-major over al's K axes (= bl's K axes, same order) */
  size_t K = (size_t)s->K;
  base.K = K;
  base.ka = (int64_t *)malloc(8 * (K ? K : 1));
  base.kb = (int64_t *)malloc(8 * (K ? K : 1));
  if (!base.ka || !base.kb) {
    free(base.ka);
    free(base.kb);
    return 0;
  }
  for (size_t k = 0; k < K; ++k) {
    size_t rem = k;
    int64_t oa = 0, ob = 0;
    for (int q = nk - 1; q >= 0; --q) {
      int la = s->lperm[nd + nm + q], rb = s->rperm[nd + q];
      size_t dim = (size_t)a->dims[la];
      oa += (int64_t)(rem % dim) * as[la];
      ob += (int64_t)(rem % dim) * bs[rb];
      rem /= dim;
    }
    base.ka[k] = oa;
    base.kb[k] = ob;
  }
  if (!tt_alloc(out, s->orank, s->out_dims, p->prec)) {
    free(base.ka);
    free(base.kb);
    return 0;
  }
  size_t n = out->n;
  if (threads < 1) threads = 1;
  if (threads > 1024) threads = 1024;
  if (n < ((size_t)1 << 16)) threads = 1;
  lean_job *jobs = (lean_job *)calloc((size_t)threads, sizeof(lean_job));
  pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
  int ok = jobs && th;
  for (int t = 0; ok && t < threads; ++t) {
    jobs[t] = base;
    jobs[t].lo = n * (size_t)t / (size_t)threads;
    jobs[t].hi = n * (size_t)(t + 1) / (size_t)threads;
  }
  char created[1024] = {0};
  if (threads > 1024) threads = 1024;
  for (int t = 1; ok && t < threads; ++t) {
    if (pthread_create(&th[t], NULL, lean_worker, &jobs[t]) == 0)
      created[t] = 1;
    else
      lean_worker(&jobs[t]);
  }
  if (ok) lean_worker(&jobs[0]);
  for (int t = 1; ok && t < threads; ++t)
    if (created[t]) pthread_join(th[t], NULL);
  free(jobs);
  free(th);
  free(base.ka);
  free(base.kb);
  return ok;
}

/* ---- branch cache --------------------------------------------------------------- */
typedef struct oracle_cache {
  uint64_t identity, mults, elements;
  int prec;
  int n_nodes;
  tt_t *node; /* kept outputs; data == NULL when absent */
} oracle_cache;

void oracle_cache_free(oracle_cache *c) {
  if (!c) return;
  for (int i = 0; i < c->n_nodes; ++i) tt_free(&c->node[i]);
  free(c->node);
  free(c);
}

/* build_cache_typed (runtime.hpp:456-488) */
oracle_cache *oracle_cache_build(const stn_plan_desc *d, int prec) {
  plan_t p;
  if (!plan_init(&p, d, prec)) {
    stn_set_error_c("oracle: malformed plan");
    plan_free(&p);
    return NULL;
  }
  oracle_cache *c = (oracle_cache *)calloc(1, sizeof *c);
  tt_t *all = (tt_t *)calloc((size_t)d->n_nodes, sizeof(tt_t));
  c->node = (tt_t *)calloc((size_t)d->n_nodes, sizeof(tt_t));
  c->n_nodes = d->n_nodes;
  c->prec = prec;
  c->identity = d->identity;
  int32_t zero[4096] = {0};
  int ok = c && all && c->node && d->n_sliced <= 4096;
  for (int i = 0; ok && i < d->n_steps; ++i) {
    const stn_step_desc *s = &d->steps[i];
    if (!s->is_branch) continue;
    tt_t ops[2];
    int ids[2] = {s->lhs, s->rhs};
    for (int k = 0; ok && k < 2; ++k) {
      if (all[ids[k]].data)
        ok = tt_copy(&ops[k], &all[ids[k]], prec);
      else
        ok = p.leaf_of_node[ids[k]] >= 0 && load_leaf(&p, ids[k], zero, &ops[k]);
    }
    if (ok) ok = gemm(&p, s, &ops[0], &ops[1], &all[s->node]);
    tt_free(&ops[0]);
    tt_free(&ops[1]);
    c->mults += s->mults;
  }
  /* keep only outputs consumed by non-branch steps, or the root */
  char *needed = (char *)calloc((size_t)d->n_nodes, 1);
  ok = ok && needed;
  for (int i = 0; ok && i < d->n_steps; ++i)
    if (!d->steps[i].is_branch) needed[d->steps[i].lhs] = needed[d->steps[i].rhs] = 1;
  if (ok) needed[d->root] = 1;
  for (int n = 0; ok && n < d->n_nodes; ++n) {
    if (all[n].data && needed[n]) {
      c->node[n] = all[n];
      c->elements += all[n].n;
      all[n].data = NULL;
    }
    tt_free(&all[n]);
  }
  free(needed);
  free(all);
  plan_free(&p);
  if (!ok) {
    stn_set_error_c("oracle: cache build failed");
    oracle_cache_free(c);
    return NULL;
  }
  return c;
}

int oracle_cache_info(const oracle_cache *c, uint64_t *identity, uint64_t *mults,
                      uint64_t *elements) {
  if (identity) *identity = c->identity;
  if (mults) *mults = c->mults;
  if (elements) *elements = c->elements;
  return STN_OK;
}

/* ---- one subtask (Engine::run, runtime.hpp:420-453) ---------------------------- */
int64_t oracle_out_elements(const stn_plan_desc *d);

/* Per-step wall-clock timing of a (possibly partial) run, for the CPU baseline. */
typedef struct {
  double budget_s; /* stop after the step during which this much time passed (<= 0: all) */
  double *step_ms; /* [cap] per executed per-slice step */
  int32_t cap;
  int32_t done;     /* steps executed */
  int32_t complete; /* 1 if the whole slice ran */
} step_timer;

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static int run_digits_impl(const stn_plan_desc *d, int prec, const int32_t *digits,
                           const oracle_cache *cache, double *out, int64_t out_cap,
                           stn_subtask_info *info, int lean_threads, step_timer *timer) {
  if (cache && cache->identity != d->identity) {
    stn_set_error_c("SubtaskFailure: branch cache belongs to a different plan");
    return STN_ERR_SUBTASK_FAILURE;
  }
  if (cache && cache->prec != prec) {
    stn_set_error_c("SubtaskFailure: branch cache precision mismatch");
    return STN_ERR_SUBTASK_FAILURE;
  }
  plan_t p;
  if (!plan_init(&p, d, prec)) {
    plan_free(&p);
    stn_set_error_c("oracle: malformed plan");
    return STN_ERR_MALFORMED_NETWORK;
  }
  tt_t *live = (tt_t *)calloc((size_t)d->n_nodes, sizeof(tt_t));
  int ok = live != NULL, status = STN_OK;
  int step_count = 0;
  uint64_t mults = 0, peak = 0;
  /* fetch: live (move), cache (copy), leaf */
#define FETCH(nid, dst)                                                               \
  do {                                                                                 \
    if (live[nid].data) {                                                             \
      dst = live[nid];                                                                \
      live[nid].data = NULL;                                                          \
    } else if (cache && cache->node[nid].data) {                                      \
      ok = tt_copy(&dst, &cache->node[nid], prec);                                    \
    } else if (p.leaf_of_node[nid] >= 0) {                                            \
      ok = load_leaf(&p, nid, digits, &dst);                                          \
    } else {                                                                           \
      ok = 0;                                                                          \
      status = STN_ERR_SUBTASK_FAILURE;                                                \
      stn_set_error_c("SubtaskFailure: operand unavailable");                          \
    }                                                                                  \
  } while (0)
  const double t_start = timer ? now_s() : 0.0;
  int stopped = 0;
  for (int i = 0; ok && i < d->n_steps; ++i) {
    const stn_step_desc *s = &d->steps[i];
    if (cache && s->is_branch) continue;
    if (timer && timer->budget_s > 0 && timer->done > 0 && now_s() - t_start > timer->budget_s) {
      stopped = 1;
      break;
    }
    const double t_step = timer ? now_s() : 0.0;
    tt_t a = {0}, b = {0};
    FETCH(s->lhs, a);
    if (ok) FETCH(s->rhs, b);
    if (ok)
      ok = lean_threads > 0 ? gemm_lean(&p, s, &a, &b, &live[s->node], lean_threads)
                            : gemm(&p, s, &a, &b, &live[s->node]);
    tt_free(&a);
    tt_free(&b);
    if (!ok) break;
    step_count++;
    mults += s->mults;
    if (live[s->node].n > peak) peak = live[s->node].n;
    if (timer && timer->done < timer->cap) timer->step_ms[timer->done++] = 1e3 * (now_s() - t_step);
  }
  if (timer) {
    timer->complete = ok && !stopped;
    if (stopped) { /* partial run: no result */
      for (int n = 0; live && n < d->n_nodes; ++n) tt_free(&live[n]);
      free(live);
      plan_free(&p);
      return STN_OK;
    }
  }
  tt_t result = {0};
  if (ok) FETCH(d->root, result);
  if (ok && (int64_t)result.n > out_cap) {
    ok = 0;
    status = STN_ERR_INVALID_ARGUMENT;
    stn_set_error_c("oracle: output buffer too small");
  }
  if (ok) {
    if (prec == STN_SINGLE) {
      const float *f = (const float *)result.data;
      for (size_t j = 0; j < 2 * result.n; ++j) out[j] = (double)f[j];
    } else {
      memcpy(out, result.data, 16 * result.n);
    }
    if (info) {
      info->step_count = step_count;
      info->mults = mults;
      info->peak_elements = peak;
    }
  }
  tt_free(&result);
  for (int n = 0; live && n < d->n_nodes; ++n) tt_free(&live[n]);
  free(live);
  plan_free(&p);
#undef FETCH
  if (!ok && status == STN_OK) {
    status = STN_ERR_OUT_OF_MEMORY;
    stn_set_error_c("oracle: allocation or shape failure");
  }
  return status;
}

int oracle_run_subtask_digits(const stn_plan_desc *d, int prec, const int32_t *digits,
                              const oracle_cache *cache, double *out, int64_t out_cap,
                              stn_subtask_info *info) {
  return run_digits_impl(d, prec, digits, cache, out, out_cap, info, 0, NULL);
}

/* Same result, bit for bit, through gemm_lean on `threads` host threads: the
 * oracle for plans whose stems do not fit the reference's memory pattern. */
int oracle_run_subtask_digits_lean(const stn_plan_desc *d, int prec, const int32_t *digits,
                                   const oracle_cache *cache, double *out, int64_t out_cap,
                                   stn_subtask_info *info, int threads) {
  return run_digits_impl(d, prec, digits, cache, out, out_cap, info, threads < 1 ? 1 : threads,
                         NULL);
}

/* The lean oracle on one slice with per-step wall-clock times, stopping after the
 * step during which `budget_s` elapsed (budget_s <= 0: the whole slice). The CPU
 * baseline of bench.py for plans the reference's own executor cannot hold. */
int oracle_time_slice_lean(const stn_plan_desc *d, int prec, const int32_t *digits,
                           const oracle_cache *cache, int threads, double budget_s,
                           double *step_ms, int32_t cap, int32_t *n_done, int32_t *complete,
                           double *out /* 2*out_elements, or NULL; filled when complete */) {
  step_timer t = {budget_s, step_ms, cap, 0, 0};
  int64_t oe = oracle_out_elements(d);
  double *buf = (double *)calloc(2 * (size_t)(oe > 0 ? oe : 1), 8);
  if (!buf) return STN_ERR_OUT_OF_MEMORY;
  int st = run_digits_impl(d, prec, digits, cache, buf, oe, NULL, threads < 1 ? 1 : threads, &t);
  if (out && st == STN_OK && t.complete) memcpy(out, buf, 16 * (size_t)oe);
  free(buf);
  *n_done = t.done;
  *complete = t.complete;
  return st;
}

int oracle_run_subtask(const stn_plan_desc *d, int prec, uint64_t assignment,
                       const oracle_cache *cache, double *out, int64_t out_cap,
                       stn_subtask_info *info) {
  if (assignment >= d->subtasks) {
    stn_set_error_c("SubtaskFailure: assignment out of range");
    return STN_ERR_SUBTASK_FAILURE;
  }
  int32_t *digits = (int32_t *)calloc((size_t)(d->n_sliced ? d->n_sliced : 1), 4);
  if (!digits) return STN_ERR_OUT_OF_MEMORY;
  oracle_decode_assignment(d, assignment, digits);
  int st = oracle_run_subtask_digits(d, prec, digits, cache, out, out_cap, info);
  if (info) info->assignment = assignment;
  free(digits);
  return st;
}

/* ---- run_scheme: threads over slices, ascending double sum (runtime.hpp:555-605) ---- */
typedef struct {
  const stn_plan_desc *d;
  int prec;
  const oracle_cache *cache;
  uint64_t lo, hi;
  int64_t out_elems;
  double *values; /* [(hi-lo)][2*out_elems] */
  volatile uint64_t next;
  pthread_mutex_t mu;
  int status;
} scheme_job;

static void *scheme_worker(void *arg) {
  scheme_job *j = (scheme_job *)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    uint64_t a = j->next++;
    int failed = j->status != STN_OK;
    pthread_mutex_unlock(&j->mu);
    if (a >= j->hi - j->lo || failed) return NULL;
    int st = oracle_run_subtask(j->d, j->prec, j->lo + a, j->cache,
                                j->values + 2 * (size_t)j->out_elems * a, j->out_elems, NULL);
    if (st != STN_OK) {
      pthread_mutex_lock(&j->mu);
      j->status = st;
      pthread_mutex_unlock(&j->mu);
      return NULL;
    }
  }
}

/* Runs slices [lo, hi) on `threads` host threads with a shared cache. values
 * (optional) receives every per-slice result; sum (optional) the ascending
 * double sum. */
int oracle_run_slices(const stn_plan_desc *d, int prec, const oracle_cache *cache, uint64_t lo,
                      uint64_t hi, int threads, int64_t out_elems, double *values, double *sum) {
  if (hi < lo || threads < 1) return STN_ERR_INVALID_ARGUMENT;
  uint64_t n = hi - lo;
  double *vals = values ? values : (double *)calloc(2 * (size_t)out_elems * (n ? n : 1), 8);
  if (!vals) return STN_ERR_OUT_OF_MEMORY;
  scheme_job j;
  j.d = d, j.prec = prec, j.cache = cache, j.lo = lo, j.hi = hi, j.out_elems = out_elems;
  j.values = vals, j.next = 0, j.status = STN_OK;
  pthread_mutex_init(&j.mu, NULL);
  pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
  int started = 0;
  for (int t = 1; th && t < threads; ++t)
    if (pthread_create(&th[started], NULL, scheme_worker, &j) == 0) started++;
  scheme_worker(&j);
  for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&j.mu);
  if (j.status == STN_OK && sum) {
    for (int64_t i = 0; i < 2 * out_elems; ++i) sum[i] = 0.0;
    for (uint64_t a = 0; a < n; ++a)
      for (int64_t i = 0; i < 2 * out_elems; ++i) sum[i] += vals[2 * (size_t)out_elems * a + i];
  }
  if (!values) free(vals);
  return j.status;
}

/* Root tensor size of a plan (product of the root's canonical dims). */
int64_t oracle_out_elements(const stn_plan_desc *d) {
  for (int i = 0; i < d->n_steps; ++i)
    if (d->steps[i].node == d->root) {
      int64_t n = 1;
      for (int k = 0; k < d->steps[i].orank; ++k) n *= d->steps[i].out_dims[k];
      return n;
    }
  for (int i = 0; i < d->n_leaves; ++i)
    if (d->leaves[i].node == d->root) {
      int64_t n = 1;
      for (int k = 0; k < d->leaves[i].rank; ++k) n *= d->leaves[i].dims[k];
      for (int k = 0; k < d->leaves[i].n_sliced; ++k) n /= d->leaves[i].dims[d->leaves[i].sliced_axis[k]];
      return n;
    }
  return -1;
}
