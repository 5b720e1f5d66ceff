/*
 * Plan files: the serialized stn_plan_desc (include/stn_exec.h).
 *
 * A plan file carries everything the executor reads from the reference's
 * ExecutablePlan (runtime.hpp:60-73): the post-order step list with its
 * permutations and group sizes, the leaf preparations with their vertex
 * tensors, and the sliced-edge dimensions. It is produced by the reference-side
 * adapter (include/stemtn_b200/flatten.hpp) and lets the executor run on a
 * machine that does not have the reference's planner.
 *
 * Layout (little-endian, no padding):
 *   "STNPLAN1"
 *   i32 precision, merge_min_dim, n_nodes, root
 *   u64 identity, subtasks
 *   i32 merged_groups, exec_cw, n_sliced, n_open, n_steps, n_leaves
 *   i32 sliced_dims[n_sliced]
 *   step  x n_steps : i32 node lhs rhs is_branch nd nm nk nn; i64 D M N K; u64 mults;
 *                     i32 lrank rrank orank; i32 lperm[] rperm[] operm[] out_dims[]
 *   leaf  x n_leaves: i32 node vertex rank n_sliced perm_rank; i32 dims[rank];
 *                     i32 sliced_axis[n_sliced] sliced_index[n_sliced] perm[perm_rank];
 *                     f64 values[2*prod(dims)]
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "stn_exec.h"

void stn_set_error_c(const char *msg); /* defined in stn_exec.cpp (or the tool) */

static const char kMagic[8] = {'S', 'T', 'N', 'P', 'L', 'A', 'N', '1'};

static int wr(FILE *f, const void *p, size_t n) { return n == 0 || fwrite(p, 1, n, f) == n; }
static int rd(FILE *f, void *p, size_t n) { return n == 0 || fread(p, 1, n, f) == n; }

int stn_plan_save(const stn_plan_desc *d, const char *path) {
  if (!d || !path) {
    stn_set_error_c("stn_plan_save: NULL argument");
    return STN_ERR_INVALID_ARGUMENT;
  }
  FILE *f = fopen(path, "wb");
  if (!f) {
    stn_set_error_c("stn_plan_save: cannot open output file");
    return STN_ERR_IO;
  }
  int ok = wr(f, kMagic, 8);
  int32_t h1[4] = {d->precision, d->merge_min_dim, d->n_nodes, d->root};
  uint64_t h2[2] = {d->identity, d->subtasks};
  int32_t h3[6] = {d->merged_groups, d->exec_cw, d->n_sliced, d->n_open, d->n_steps, d->n_leaves};
  ok = ok && wr(f, h1, sizeof h1) && wr(f, h2, sizeof h2) && wr(f, h3, sizeof h3);
  ok = ok && wr(f, d->sliced_dims, sizeof(int32_t) * (size_t)d->n_sliced);
  for (int i = 0; ok && i < d->n_steps; ++i) {
    const stn_step_desc *s = &d->steps[i];
    int32_t a[8] = {s->node, s->lhs, s->rhs, s->is_branch, s->nd, s->nm, s->nk, s->nn};
    int64_t g[4] = {s->D, s->M, s->N, s->K};
    int32_t r[3] = {s->lrank, s->rrank, s->orank};
    ok = wr(f, a, sizeof a) && wr(f, g, sizeof g) && wr(f, &s->mults, 8) && wr(f, r, sizeof r) &&
         wr(f, s->lperm, 4 * (size_t)s->lrank) && wr(f, s->rperm, 4 * (size_t)s->rrank) &&
         wr(f, s->operm, 4 * (size_t)s->orank) && wr(f, s->out_dims, 4 * (size_t)s->orank);
  }
  for (int i = 0; ok && i < d->n_leaves; ++i) {
    const stn_leaf_desc *l = &d->leaves[i];
    int32_t a[5] = {l->node, l->vertex, l->rank, l->n_sliced, l->perm_rank};
    size_t n = 1;
    for (int k = 0; k < l->rank; ++k) n *= (size_t)l->dims[k];
    ok = wr(f, a, sizeof a) && wr(f, l->dims, 4 * (size_t)l->rank) &&
         wr(f, l->sliced_axis, 4 * (size_t)l->n_sliced) &&
         wr(f, l->sliced_index, 4 * (size_t)l->n_sliced) &&
         wr(f, l->perm, 4 * (size_t)l->perm_rank) && wr(f, l->values, 16 * n);
  }
  if (fclose(f) != 0) ok = 0;
  if (!ok) {
    stn_set_error_c("stn_plan_save: write failed");
    return STN_ERR_IO;
  }
  return STN_OK;
}

static void *xcalloc(size_t n, size_t sz) { return calloc(n ? n : 1, sz); }

void stn_plan_desc_free(stn_plan_desc *d) {
  if (!d) return;
  for (int i = 0; d->steps && i < d->n_steps; ++i) {
    free((void *)d->steps[i].lperm);
    free((void *)d->steps[i].rperm);
    free((void *)d->steps[i].operm);
    free((void *)d->steps[i].out_dims);
  }
  for (int i = 0; d->leaves && i < d->n_leaves; ++i) {
    free((void *)d->leaves[i].dims);
    free((void *)d->leaves[i].values);
    free((void *)d->leaves[i].sliced_axis);
    free((void *)d->leaves[i].sliced_index);
    free((void *)d->leaves[i].perm);
  }
  free((void *)d->steps);
  free((void *)d->leaves);
  free((void *)d->sliced_dims);
  free(d);
}

#define RANK_CAP 4096

int stn_plan_load(const char *path, stn_plan_desc **out) {
  if (!path || !out) {
    stn_set_error_c("stn_plan_load: NULL argument");
    return STN_ERR_INVALID_ARGUMENT;
  }
  *out = NULL;
  FILE *f = fopen(path, "rb");
  if (!f) {
    stn_set_error_c("stn_plan_load: cannot open plan file");
    return STN_ERR_IO;
  }
  stn_plan_desc *d = (stn_plan_desc *)xcalloc(1, sizeof *d);
  char magic[8];
  int32_t h1[4], h3[6];
  uint64_t h2[2];
  int ok = d && rd(f, magic, 8) && memcmp(magic, kMagic, 8) == 0 && rd(f, h1, sizeof h1) &&
           rd(f, h2, sizeof h2) && rd(f, h3, sizeof h3);
  if (ok) {
    d->precision = h1[0];
    d->merge_min_dim = h1[1];
    d->n_nodes = h1[2];
    d->root = h1[3];
    d->identity = h2[0];
    d->subtasks = h2[1];
    d->merged_groups = h3[0];
    d->exec_cw = h3[1];
    d->n_sliced = h3[2];
    d->n_open = h3[3];
    d->n_steps = h3[4];
    d->n_leaves = h3[5];
    ok = d->n_sliced >= 0 && d->n_steps >= 0 && d->n_leaves >= 0 && d->n_sliced < (1 << 20) &&
         d->n_steps < (1 << 26) && d->n_leaves < (1 << 26);
  }
  if (ok) {
    int32_t *sd = (int32_t *)xcalloc((size_t)d->n_sliced, 4);
    d->sliced_dims = sd;
    ok = sd && rd(f, sd, 4 * (size_t)d->n_sliced);
  }
  if (ok) {
    stn_step_desc *steps = (stn_step_desc *)xcalloc((size_t)d->n_steps, sizeof *steps);
    d->steps = steps;
    ok = steps != NULL;
    for (int i = 0; ok && i < d->n_steps; ++i) {
      stn_step_desc *s = &steps[i];
      int32_t a[8], r[3];
      int64_t g[4];
      ok = rd(f, a, sizeof a) && rd(f, g, sizeof g) && rd(f, &s->mults, 8) && rd(f, r, sizeof r);
      if (!ok) break;
      s->node = a[0], s->lhs = a[1], s->rhs = a[2], s->is_branch = a[3];
      s->nd = a[4], s->nm = a[5], s->nk = a[6], s->nn = a[7];
      s->D = g[0], s->M = g[1], s->N = g[2], s->K = g[3];
      s->lrank = r[0], s->rrank = r[1], s->orank = r[2];
      ok = r[0] >= 0 && r[1] >= 0 && r[2] >= 0 && r[0] < RANK_CAP && r[1] < RANK_CAP &&
           r[2] < RANK_CAP;
      if (!ok) break;
      int32_t *lp = (int32_t *)xcalloc((size_t)s->lrank, 4);
      int32_t *rp = (int32_t *)xcalloc((size_t)s->rrank, 4);
      int32_t *op = (int32_t *)xcalloc((size_t)s->orank, 4);
      int32_t *od = (int32_t *)xcalloc((size_t)s->orank, 4);
      s->lperm = lp, s->rperm = rp, s->operm = op, s->out_dims = od;
      ok = lp && rp && op && od && rd(f, lp, 4 * (size_t)s->lrank) &&
           rd(f, rp, 4 * (size_t)s->rrank) && rd(f, op, 4 * (size_t)s->orank) &&
           rd(f, od, 4 * (size_t)s->orank);
    }
  }
  if (ok) {
    stn_leaf_desc *leaves = (stn_leaf_desc *)xcalloc((size_t)d->n_leaves, sizeof *leaves);
    d->leaves = leaves;
    ok = leaves != NULL;
    for (int i = 0; ok && i < d->n_leaves; ++i) {
      stn_leaf_desc *l = &leaves[i];
      int32_t a[5];
      ok = rd(f, a, sizeof a);
      if (!ok) break;
      l->node = a[0], l->vertex = a[1], l->rank = a[2], l->n_sliced = a[3], l->perm_rank = a[4];
      ok = l->rank >= 0 && l->rank < RANK_CAP && l->n_sliced >= 0 && l->n_sliced <= l->rank &&
           l->perm_rank >= 0 && l->perm_rank < RANK_CAP;
      if (!ok) break;
      int32_t *dims = (int32_t *)xcalloc((size_t)l->rank, 4);
      int32_t *sa = (int32_t *)xcalloc((size_t)l->n_sliced, 4);
      int32_t *si = (int32_t *)xcalloc((size_t)l->n_sliced, 4);
      int32_t *pm = (int32_t *)xcalloc((size_t)l->perm_rank, 4);
      l->dims = dims, l->sliced_axis = sa, l->sliced_index = si, l->perm = pm;
      ok = dims && sa && si && pm && rd(f, dims, 4 * (size_t)l->rank) &&
           rd(f, sa, 4 * (size_t)l->n_sliced) && rd(f, si, 4 * (size_t)l->n_sliced) &&
           rd(f, pm, 4 * (size_t)l->perm_rank);
      if (!ok) break;
      size_t n = 1;
      for (int k = 0; k < l->rank; ++k) {
        if (dims[k] <= 0 || n > ((size_t)1 << 32)) ok = 0;
        n *= (size_t)(dims[k] > 0 ? dims[k] : 1);
      }
      if (!ok) break;
      double *v = (double *)xcalloc(2 * n, 8);
      l->values = v;
      ok = v && rd(f, v, 16 * n);
    }
  }
  if (ok) {
    char extra;
    ok = fread(&extra, 1, 1, f) == 0; /* no trailing bytes */
  }
  fclose(f);
  if (!ok) {
    stn_plan_desc_free(d);
    stn_set_error_c("stn_plan_load: malformed or truncated plan file");
    return STN_ERR_SCHEMA_ERROR;
  }
  *out = d;
  return STN_OK;
}
