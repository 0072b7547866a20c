/*
 * stc_oracle.c -- CPU restatement of the reference's contraction path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg use it, and only as the checker or as the
 * timed CPU baseline ("kind": "port").
 *
 * It restates, in plain C with fp contraction disabled, the algorithm of the
 * reference package strassen_tc (Python + numba; /root/reference/pkg/src):
 *
 *   bundle scatter vectors        scatter.py:105-112   (first bundle label fastest)
 *   block-scatter vectors         scatter.py:26-40     (constant positive stride, else 0)
 *   make_view / pad / split       scatter.py:115-165
 *   quadrant_views                strassen.py:101-127  (row-major ids, top level most significant)
 *   strassen_terms                strassen.py:56-94    (substitution, outer level first)
 *   pack_a_block / pack_b_block   _jit.py:27-131       (zero, then sum views in order)
 *   microtile                     _jit.py:134-143      (p outermost rank-1 updates)
 *   store_tile / macro_kernel     _jit.py:158-220
 *   accum_dense / unpack_sum      _jit.py:223-309
 *   run_fused (5 loops)           driver.py:76-126     (jc -> pc -> pack B -> ic -> pack A -> macro)
 *   run_gemm_dense                driver.py:139-152
 *   contract ABC / AB / NAIVE     strassen.py:141-207
 *   contract_reference            oracle.py:62-92      (j, i, p loops, P innermost)
 *   _seq_sum_sq                   oracle.py:102-107
 *
 * Every accumulation happens in the same order as the reference, so results
 * are bitwise identical to it (pinned by tests/test_oracle_golden.py against
 * fixtures generated from the reference itself, tests/golden/make_golden.py).
 * The only liberty taken: the jr-chunk thread pool (driver.py:93-117) is an
 * OpenMP loop over the same chunks, which the reference proves bitwise neutral
 * (pkg/tests/test_driver.py:165-171).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORA_PAD INT64_MIN
#define ORA_MAXLAB 16

typedef struct {
  int32_t nlab;
  int32_t _pad;
  int64_t ext[ORA_MAXLAB];
  int64_t str[ORA_MAXLAB];
} ora_bundle;

typedef struct {
  ora_bundle a_row, a_col; /* A matricised as I x P */
  ora_bundle b_row, b_col; /* B matricised as P x J */
  ora_bundle c_row, c_col; /* C matricised as I x J */
  int64_t a_base, b_base, c_base;
} ora_problem;

typedef struct {
  int64_t mc, nc, kc, mr, nr, kr;
} ora_blocking;

typedef struct {
  double total_flops;
  int64_t fast_blocks, slow_blocks, fast_updates, slow_updates, leaf_multiplies;
} ora_stats;

/* ------------------------------------------------------------------ views */

typedef struct {
  const double *data; /* parent storage (read) */
  double *wdata;      /* parent storage (write) or NULL */
  int64_t m, n, rb, cb;
  int64_t *rscat, *cscat, *rbs, *cbs;
  int64_t row_unit, col_unit;
} view_t;

static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

int64_t ora_bundle_len(const ora_bundle *b) {
  int64_t n = 1;
  for (int d = 0; d < b->nlab; ++d) n *= b->ext[d];
  return n;
}

/* scatter.py:105-112 -- offsets of the bundle's linear index, first label fastest. */
void ora_bundle_scatter(const ora_bundle *b, int64_t base, int64_t *out) {
  int64_t len = 1;
  out[0] = base;
  for (int d = 0; d < b->nlab; ++d) {
    int64_t e = b->ext[d], s = b->str[d];
    /* new[idx + len*x] = old[idx] + x*s  (the old index stays fastest) */
    for (int64_t x = e - 1; x >= 0; --x)
      for (int64_t i = 0; i < len; ++i) out[x * len + i] = out[i] + x * s;
    len *= e;
  }
}

/* scatter.py:26-40 */
void ora_block_vector(const int64_t *scat, int64_t len, int64_t blk, int64_t unit, int64_t *out) {
  int64_t nb = cdiv(len, blk);
  for (int64_t b = 0; b < nb; ++b) {
    int64_t lo = b * blk, hi = lo + blk < len ? lo + blk : len;
    int has_pad = 0;
    for (int64_t i = lo; i < hi; ++i)
      if (scat[i] == ORA_PAD) has_pad = 1;
    out[b] = 0;
    if (has_pad) continue;
    if (hi - lo == 1) {
      out[b] = unit > 0 ? unit : 0;
      continue;
    }
    int64_t d = scat[lo + 1] - scat[lo];
    if (d <= 0) continue;
    int ok = 1;
    for (int64_t i = lo + 1; i < hi; ++i)
      if (scat[i] - scat[i - 1] != d) { ok = 0; break; }
    if (ok) out[b] = d;
  }
}

static view_t *view_new(const double *data, double *wdata, const int64_t *rscat, int64_t m,
                        const int64_t *cscat, int64_t n, int64_t rb, int64_t cb, int64_t ru, int64_t cu) {
  view_t *v = (view_t *)calloc(1, sizeof(view_t));
  v->data = data; v->wdata = wdata; v->m = m; v->n = n; v->rb = rb; v->cb = cb;
  v->row_unit = ru; v->col_unit = cu;
  v->rscat = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
  v->cscat = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  memcpy(v->rscat, rscat, sizeof(int64_t) * (size_t)m);
  memcpy(v->cscat, cscat, sizeof(int64_t) * (size_t)n);
  v->rbs = (int64_t *)malloc(sizeof(int64_t) * (size_t)cdiv(m, rb));
  v->cbs = (int64_t *)malloc(sizeof(int64_t) * (size_t)cdiv(n, cb));
  ora_block_vector(v->rscat, m, rb, ru, v->rbs);
  ora_block_vector(v->cscat, n, cb, cu, v->cbs);
  return v;
}

static void view_free(view_t *v) {
  if (!v) return;
  free(v->rscat); free(v->cscat); free(v->rbs); free(v->cbs); free(v);
}

/* scatter.py:115-131 (base folded into the column scatter). */
static view_t *make_view(const double *data, double *wdata, const ora_bundle *rows, const ora_bundle *cols,
                         int64_t base, int64_t rb, int64_t cb) {
  int64_t m = ora_bundle_len(rows), n = ora_bundle_len(cols);
  int64_t *rs = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
  int64_t *cs = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  ora_bundle_scatter(rows, 0, rs);
  ora_bundle_scatter(cols, base, cs);
  int64_t ru = rows->nlab ? rows->str[0] : 1, cu = cols->nlab ? cols->str[0] : 1;
  view_t *v = view_new(data, wdata, rs, m, cs, n, rb, cb, ru, cu);
  free(rs); free(cs);
  return v;
}

/* scatter.py:143-152 */
static view_t *split_view(const view_t *v, int64_t r0, int64_t r1, int64_t c0, int64_t c1) {
  return view_new(v->data, v->wdata, v->rscat + r0, r1 - r0, v->cscat + c0, c1 - c0, v->rb, v->cb,
                  v->row_unit, v->col_unit);
}

/* scatter.py:155-165 */
static view_t *pad_view(const view_t *v, int64_t mt, int64_t nt) {
  int64_t *rs = (int64_t *)malloc(sizeof(int64_t) * (size_t)mt);
  int64_t *cs = (int64_t *)malloc(sizeof(int64_t) * (size_t)nt);
  for (int64_t i = 0; i < mt; ++i) rs[i] = i < v->m ? v->rscat[i] : ORA_PAD;
  for (int64_t j = 0; j < nt; ++j) cs[j] = j < v->n ? v->cscat[j] : ORA_PAD;
  view_t *p = view_new(v->data, v->wdata, rs, mt, cs, nt, v->rb, v->cb, v->row_unit, v->col_unit);
  free(rs); free(cs);
  return p;
}

static void quad_rec(const view_t *v, int lev, view_t **out, int *pos) {
  if (lev == 0) {
    out[(*pos)++] = split_view(v, 0, v->m, 0, v->n);
    return;
  }
  int64_t h = v->m / 2, w = v->n / 2;
  const int64_t rr[4][2] = {{0, h}, {0, h}, {h, 2 * h}, {h, 2 * h}};
  const int64_t cc[4][2] = {{0, w}, {w, 2 * w}, {0, w}, {w, 2 * w}};
  for (int q = 0; q < 4; ++q) {
    view_t *s = split_view(v, rr[q][0], rr[q][1], cc[q][0], cc[q][1]);
    quad_rec(s, lev - 1, out, pos);
    view_free(s);
  }
}

/* strassen.py:101-127: pad to a multiple of 2^L, split recursively. */
static void quadrant_views(const view_t *v, int level, view_t **out) {
  int64_t step = (int64_t)1 << level;
  view_t *p = pad_view(v, cdiv(v->m, step) * step, cdiv(v->n, step) * step);
  int pos = 0;
  quad_rec(p, level, out, &pos);
  view_free(p);
}

/* ------------------------------------------------------------------ terms */

/* strassen.py:56-65 -- the seven-product table: {quadrant, sign} per operand. */
static const int L1_A[7][2][2] = {{{0, 1}, {3, 1}}, {{2, 1}, {3, 1}}, {{0, 1}, {0, 0}}, {{3, 1}, {0, 0}},
                                  {{0, 1}, {1, 1}}, {{2, 1}, {0, -1}}, {{1, 1}, {3, -1}}};
static const int L1_NA[7] = {2, 2, 1, 1, 2, 2, 2};
static const int L1_B[7][2][2] = {{{0, 1}, {3, 1}}, {{0, 1}, {0, 0}}, {{1, 1}, {3, -1}}, {{2, 1}, {0, -1}},
                                  {{3, 1}, {0, 0}}, {{0, 1}, {1, 1}}, {{2, 1}, {3, 1}}};
static const int L1_NB[7] = {2, 1, 2, 2, 1, 2, 2};
static const int L1_C[7][2][2] = {{{0, 1}, {3, 1}}, {{2, 1}, {3, -1}}, {{1, 1}, {3, 1}}, {{0, 1}, {2, 1}},
                                  {{1, 1}, {0, -1}}, {{3, 1}, {0, 0}}, {{0, 1}, {0, 0}}};
static const int L1_NC[7] = {2, 2, 2, 2, 2, 1, 1};

/* One operand list: n (q, sign) pairs, stored flat. */
typedef struct {
  int n;
  int *q;
  int *s;
} ops_t;

typedef struct {
  ops_t a, b, c;
} term_t;

static ops_t expand_ops(const int outer[][2], int nouter, const ops_t *inner, int mult) {
  ops_t r;
  r.n = nouter * inner->n;
  r.q = (int *)malloc(sizeof(int) * (size_t)r.n);
  r.s = (int *)malloc(sizeof(int) * (size_t)r.n);
  int k = 0;
  for (int o = 0; o < nouter; ++o)
    for (int i = 0; i < inner->n; ++i) {
      r.q[k] = outer[o][0] * mult + inner->q[i];
      r.s[k] = outer[o][1] * inner->s[i];
      ++k;
    }
  return r;
}

static void free_terms(term_t *t, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    free(t[i].a.q); free(t[i].a.s); free(t[i].b.q); free(t[i].b.s); free(t[i].c.q); free(t[i].c.s);
  }
  free(t);
}

/* strassen.py:70-94: level-(l) table = level-1 outer x level-(l-1) inner. */
static term_t *make_terms(int level, int64_t *count) {
  int64_t n = 1;
  term_t *t = (term_t *)calloc(1, sizeof(term_t));
  for (int k = 0; k < 3; ++k) {
    ops_t *o = k == 0 ? &t[0].a : k == 1 ? &t[0].b : &t[0].c;
    o->n = 1; o->q = (int *)malloc(sizeof(int)); o->s = (int *)malloc(sizeof(int));
    o->q[0] = 0; o->s[0] = 1;
  }
  for (int lev = 1; lev <= level; ++lev) {
    int mult = 1;
    for (int i = 1; i < lev; ++i) mult *= 4;
    term_t *nt = (term_t *)calloc((size_t)(7 * n), sizeof(term_t));
    for (int o = 0; o < 7; ++o)
      for (int64_t i = 0; i < n; ++i) {
        term_t *d = &nt[o * n + i];
        d->a = expand_ops(L1_A[o], L1_NA[o], &t[i].a, mult);
        d->b = expand_ops(L1_B[o], L1_NB[o], &t[i].b, mult);
        d->c = expand_ops(L1_C[o], L1_NC[o], &t[i].c, mult);
      }
    free_terms(t, n);
    t = nt;
    n *= 7;
  }
  *count = n;
  return t;
}

/* Flat export of the term table for tests: per term, na nb nc then (q,s) pairs. */
int64_t ora_strassen_terms(int level, int *buf, int64_t cap) {
  int64_t n;
  term_t *t = make_terms(level, &n);
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i) {
    const ops_t *o3[3] = {&t[i].a, &t[i].b, &t[i].c};
    if (k + 3 <= cap) { buf[k] = t[i].a.n; buf[k + 1] = t[i].b.n; buf[k + 2] = t[i].c.n; }
    k += 3;
    for (int s = 0; s < 3; ++s)
      for (int j = 0; j < o3[s]->n; ++j) {
        if (k + 2 <= cap) { buf[k] = o3[s]->q[j]; buf[k + 1] = o3[s]->s[j]; }
        k += 2;
      }
  }
  free_terms(t, n);
  return k;
}

/* ------------------------------------------------------------ kernels */

typedef struct {
  int n;
  view_t **v;
  double *coeff;
} side_t;

/* _jit.py:27-79 */
static void pack_a_block(double *out, int64_t depth, const side_t *sd, int64_t r0, int64_t rcount, int64_t k0,
                         int64_t kcount, int64_t mr, int64_t kr, int force_slow, int64_t *fast, int64_t *slow) {
  int64_t nsl = cdiv(rcount, mr), nch = cdiv(kcount, kr);
  for (int64_t s = 0; s < nsl; ++s) {
    int64_t i0 = s * mr, ilim = rcount - i0 < mr ? rcount - i0 : mr;
    double *o = out + s * depth * mr;
    for (int64_t p = 0; p < kcount; ++p)
      for (int64_t i = 0; i < mr; ++i) o[p * mr + i] = 0.0;
    for (int64_t c = 0; c < nch; ++c) {
      int64_t p0 = c * kr, plim = kcount - p0 < kr ? kcount - p0 : kr;
      int regular = !force_slow;
      for (int t = 0; regular && t < sd->n; ++t)
        if (sd->v[t]->rbs[(r0 + i0) / mr] == 0 || sd->v[t]->cbs[(k0 + p0) / kr] == 0) regular = 0;
      if (regular) {
        ++*fast;
        for (int t = 0; t < sd->n; ++t) {
          const view_t *v = sd->v[t];
          double co = sd->coeff[t];
          int64_t rbase = v->rscat[r0 + i0], cbase = v->cscat[k0 + p0];
          int64_t rstep = v->rbs[(r0 + i0) / mr], cstep = v->cbs[(k0 + p0) / kr];
          for (int64_t p = 0; p < plim; ++p) {
            int64_t off = cbase + p * cstep;
            for (int64_t i = 0; i < ilim; ++i) o[(p0 + p) * mr + i] += co * v->data[rbase + i * rstep + off];
          }
        }
      } else {
        ++*slow;
        for (int t = 0; t < sd->n; ++t) {
          const view_t *v = sd->v[t];
          double co = sd->coeff[t];
          for (int64_t p = 0; p < plim; ++p) {
            int64_t cc = v->cscat[k0 + p0 + p];
            if (cc == ORA_PAD) continue;
            for (int64_t i = 0; i < ilim; ++i) {
              int64_t rr = v->rscat[r0 + i0 + i];
              if (rr == ORA_PAD) continue;
              o[(p0 + p) * mr + i] += co * v->data[rr + cc];
            }
          }
        }
      }
    }
  }
}

/* _jit.py:82-131 */
static void pack_b_block(double *out, int64_t depth, const side_t *sd, int64_t k0, int64_t kcount, int64_t c0,
                         int64_t ccount, int64_t kr, int64_t nr, int force_slow, int64_t *fast, int64_t *slow) {
  int64_t nsl = cdiv(ccount, nr), nch = cdiv(kcount, kr);
  for (int64_t s = 0; s < nsl; ++s) {
    int64_t j0 = s * nr, jlim = ccount - j0 < nr ? ccount - j0 : nr;
    double *o = out + s * depth * nr;
    for (int64_t p = 0; p < kcount; ++p)
      for (int64_t j = 0; j < nr; ++j) o[p * nr + j] = 0.0;
    for (int64_t c = 0; c < nch; ++c) {
      int64_t p0 = c * kr, plim = kcount - p0 < kr ? kcount - p0 : kr;
      int regular = !force_slow;
      for (int t = 0; regular && t < sd->n; ++t)
        if (sd->v[t]->rbs[(k0 + p0) / kr] == 0 || sd->v[t]->cbs[(c0 + j0) / nr] == 0) regular = 0;
      if (regular) {
        ++*fast;
        for (int t = 0; t < sd->n; ++t) {
          const view_t *v = sd->v[t];
          double co = sd->coeff[t];
          int64_t rbase = v->rscat[k0 + p0], cbase = v->cscat[c0 + j0];
          int64_t rstep = v->rbs[(k0 + p0) / kr], cstep = v->cbs[(c0 + j0) / nr];
          for (int64_t p = 0; p < plim; ++p) {
            int64_t off = rbase + p * rstep;
            for (int64_t j = 0; j < jlim; ++j) o[(p0 + p) * nr + j] += co * v->data[off + cbase + j * cstep];
          }
        }
      } else {
        ++*slow;
        for (int t = 0; t < sd->n; ++t) {
          const view_t *v = sd->v[t];
          double co = sd->coeff[t];
          for (int64_t p = 0; p < plim; ++p) {
            int64_t rr = v->rscat[k0 + p0 + p];
            if (rr == ORA_PAD) continue;
            for (int64_t j = 0; j < jlim; ++j) {
              int64_t cc = v->cscat[c0 + j0 + j];
              if (cc == ORA_PAD) continue;
              o[(p0 + p) * nr + j] += co * v->data[rr + cc];
            }
          }
        }
      }
    }
  }
}

/* _jit.py:158-186 */
static int store_tile(const double *acc, const view_t *v, double coeff, int64_t i0, int64_t ilim, int64_t j0,
                      int64_t jlim, int64_t mr, int64_t nr, int force_slow) {
  int64_t bi = i0 / mr, bj = j0 / nr;
  double *cd = v->wdata;
  if (!force_slow && v->rbs[bi] != 0 && v->cbs[bj] != 0) {
    int64_t rbase = v->rscat[i0], cbase = v->cscat[j0], rstep = v->rbs[bi], cstep = v->cbs[bj];
    for (int64_t i = 0; i < ilim; ++i) {
      int64_t off = rbase + i * rstep + cbase;
      for (int64_t j = 0; j < jlim; ++j) cd[off + j * cstep] += coeff * acc[i * nr + j];
    }
    return 1;
  }
  for (int64_t i = 0; i < ilim; ++i) {
    int64_t rr = v->rscat[i0 + i];
    if (rr == ORA_PAD) continue;
    for (int64_t j = 0; j < jlim; ++j) {
      int64_t cc = v->cscat[j0 + j];
      if (cc == ORA_PAD) continue;
      cd[rr + cc] += coeff * acc[i * nr + j];
    }
  }
  return 0;
}

/* _jit.py:189-220 with microtile (_jit.py:134-143) inlined. */
static void macro_kernel(const double *abuf, int64_t adepth, const double *bbuf, int64_t bdepth, int64_t kcount,
                         const side_t *cs, int64_t ic, int64_t mcount, int64_t jc, int64_t jr0, int64_t jr1,
                         int64_t mr, int64_t nr, int force_slow, int64_t *fast, int64_t *slow, int64_t *tiles) {
  double acc[64 * 64];
  for (int64_t jr = jr0; jr < jr1; jr += nr) {
    int64_t jlim = jr1 - jr < nr ? jr1 - jr : nr, sb = jr / nr;
    for (int64_t ir = 0; ir < mcount; ir += mr) {
      int64_t ilim = mcount - ir < mr ? mcount - ir : mr, sa = ir / mr;
      for (int64_t x = 0; x < mr * nr; ++x) acc[x] = 0.0;
      const double *a = abuf + sa * adepth * mr, *b = bbuf + sb * bdepth * nr;
      for (int64_t p = 0; p < kcount; ++p)
        for (int64_t i = 0; i < mr; ++i) {
          double av = a[p * mr + i];
          for (int64_t j = 0; j < nr; ++j) acc[i * nr + j] += av * b[p * nr + j];
        }
      ++*tiles;
      for (int t = 0; t < cs->n; ++t) {
        if (store_tile(acc, cs->v[t], cs->coeff[t], ic + ir, ilim, jc + jr, jlim, mr, nr, force_slow))
          ++*fast;
        else
          ++*slow;
      }
    }
  }
}

/* driver.py:64-73 */
static int jr_chunks(int64_t ncount, int64_t nr, int threads, int64_t *lo, int64_t *hi) {
  int64_t sl = cdiv(ncount, nr);
  int64_t nch = threads < sl ? threads : sl;
  int64_t per = sl / nch, extra = sl % nch, start = 0;
  for (int64_t t = 0; t < nch; ++t) {
    int64_t take = per + (t < extra ? 1 : 0);
    lo[t] = start * nr;
    hi[t] = (start + take) * nr < ncount ? (start + take) * nr : ncount;
    start += take;
  }
  return (int)nch;
}

/* driver.py:76-126 */
static void run_fused(const side_t *as, const side_t *bs, const side_t *cs, const ora_blocking *bp, double *abuf,
                      int64_t adepth, double *bbuf, int64_t bdepth, int threads, int force_slow, ora_stats *st) {
  int64_t m = as->v[0]->m, k = as->v[0]->n, n = bs->v[0]->n;
  int64_t *lo = (int64_t *)malloc(sizeof(int64_t) * (size_t)(threads + 1));
  int64_t *hi = (int64_t *)malloc(sizeof(int64_t) * (size_t)(threads + 1));
  for (int64_t jc = 0; jc < n; jc += bp->nc) {
    int64_t ncount = n - jc < bp->nc ? n - jc : bp->nc;
    for (int64_t pc = 0; pc < k; pc += bp->kc) {
      int64_t kcount = k - pc < bp->kc ? k - pc : bp->kc;
      pack_b_block(bbuf, bdepth, bs, pc, kcount, jc, ncount, bp->kr, bp->nr, force_slow, &st->fast_blocks,
                   &st->slow_blocks);
      for (int64_t ic = 0; ic < m; ic += bp->mc) {
        int64_t mcount = m - ic < bp->mc ? m - ic : bp->mc;
        pack_a_block(abuf, adepth, as, ic, mcount, pc, kcount, bp->mr, bp->kr, force_slow, &st->fast_blocks,
                     &st->slow_blocks);
        int nch = jr_chunks(ncount, bp->nr, threads > 1 ? threads : 1, lo, hi);
        int64_t f = 0, s = 0, tl = 0;
#pragma omp parallel for num_threads(nch) reduction(+ : f, s, tl) schedule(static, 1) if (nch > 1)
        for (int c = 0; c < nch; ++c)
          macro_kernel(abuf, adepth, bbuf, bdepth, kcount, cs, ic, mcount, jc, lo[c], hi[c], bp->mr, bp->nr,
                       force_slow, &f, &s, &tl);
        st->fast_updates += f;
        st->slow_updates += s;
        st->total_flops += 2.0 * (double)bp->mr * (double)bp->nr * (double)kcount * (double)tl;
      }
    }
  }
  st->leaf_multiplies += 1;
  free(lo); free(hi);
}

/* _jit.py:223-256 ; mat is column-major (ld = m). */
static void accum_dense(const double *mat, int64_t m, int64_t n, const view_t *v, double coeff, int force_slow,
                        ora_stats *st) {
  int64_t rb = v->rb, cb = v->cb;
  double *cd = v->wdata;
  for (int64_t bj = 0; bj < cdiv(n, cb); ++bj) {
    int64_t j0 = bj * cb, jlim = n - j0 < cb ? n - j0 : cb;
    for (int64_t bi = 0; bi < cdiv(m, rb); ++bi) {
      int64_t i0 = bi * rb, ilim = m - i0 < rb ? m - i0 : rb;
      if (!force_slow && v->rbs[bi] != 0 && v->cbs[bj] != 0) {
        ++st->fast_updates;
        int64_t rbase = v->rscat[i0], cbase = v->cscat[j0], rstep = v->rbs[bi], cstep = v->cbs[bj];
        for (int64_t i = 0; i < ilim; ++i) {
          int64_t off = rbase + i * rstep + cbase;
          for (int64_t j = 0; j < jlim; ++j) cd[off + j * cstep] += coeff * mat[(i0 + i) + (j0 + j) * m];
        }
      } else {
        ++st->slow_updates;
        for (int64_t i = 0; i < ilim; ++i) {
          int64_t rr = v->rscat[i0 + i];
          if (rr == ORA_PAD) continue;
          for (int64_t j = 0; j < jlim; ++j) {
            int64_t cc = v->cscat[j0 + j];
            if (cc == ORA_PAD) continue;
            cd[rr + cc] += coeff * mat[(i0 + i) + (j0 + j) * m];
          }
        }
      }
    }
  }
}

/* _jit.py:259-309 ; out is column-major m x n. */
static void unpack_sum(double *out, const side_t *sd, int force_slow, ora_stats *st) {
  const view_t *v0 = sd->v[0];
  int64_t m = v0->m, n = v0->n, rb = v0->rb, cb = v0->cb;
  for (int64_t x = 0; x < m * n; ++x) out[x] = 0.0;
  for (int64_t bj = 0; bj < cdiv(n, cb); ++bj) {
    int64_t j0 = bj * cb, jlim = n - j0 < cb ? n - j0 : cb;
    for (int64_t bi = 0; bi < cdiv(m, rb); ++bi) {
      int64_t i0 = bi * rb, ilim = m - i0 < rb ? m - i0 : rb;
      int regular = !force_slow;
      for (int t = 0; regular && t < sd->n; ++t)
        if (sd->v[t]->rbs[bi] == 0 || sd->v[t]->cbs[bj] == 0) regular = 0;
      if (regular) {
        ++st->fast_blocks;
        for (int t = 0; t < sd->n; ++t) {
          const view_t *v = sd->v[t];
          double co = sd->coeff[t];
          int64_t rbase = v->rscat[i0], cbase = v->cscat[j0], rstep = v->rbs[bi], cstep = v->cbs[bj];
          for (int64_t i = 0; i < ilim; ++i) {
            int64_t off = rbase + i * rstep + cbase;
            for (int64_t j = 0; j < jlim; ++j) out[(i0 + i) + (j0 + j) * m] += co * v->data[off + j * cstep];
          }
        }
      } else {
        ++st->slow_blocks;
        for (int t = 0; t < sd->n; ++t) {
          const view_t *v = sd->v[t];
          double co = sd->coeff[t];
          for (int64_t i = 0; i < ilim; ++i) {
            int64_t rr = v->rscat[i0 + i];
            if (rr == ORA_PAD) continue;
            for (int64_t j = 0; j < jlim; ++j) {
              int64_t cc = v->cscat[j0 + j];
              if (cc == ORA_PAD) continue;
              out[(i0 + i) + (j0 + j) * m] += co * v->data[rr + cc];
            }
          }
        }
      }
    }
  }
}

/* --------------------------------------------------------------- contract */

static side_t make_side(view_t **quads, const ops_t *ops) {
  side_t s;
  s.n = ops->n;
  s.v = (view_t **)malloc(sizeof(view_t *) * (size_t)ops->n);
  s.coeff = (double *)malloc(sizeof(double) * (size_t)ops->n);
  for (int i = 0; i < ops->n; ++i) { s.v[i] = quads[ops->q[i]]; s.coeff[i] = (double)ops->s[i]; }
  return s;
}

static void free_side(side_t *s) { free(s->v); free(s->coeff); }

/* strassen.py:141-207.  variant: 0 = ABC, 1 = AB, 2 = NAIVE. Returns 0 on success. */
int ora_contract(const ora_problem *pr, const double *A, const double *B, double *C, int level, int variant,
                 const ora_blocking *bp, int threads, int force_slow, ora_stats *st) {
  if (level < 0 || variant < 0 || variant > 2) return 1;
  if (bp->mr * bp->nr > 64 * 64) return 2;
  memset(st, 0, sizeof(*st));
  int64_t nterms;
  term_t *terms = make_terms(level, &nterms);
  view_t *va = make_view(A, NULL, &pr->a_row, &pr->a_col, pr->a_base, bp->mr, bp->kr);
  view_t *vb = make_view(B, NULL, &pr->b_row, &pr->b_col, pr->b_base, bp->kr, bp->nr);
  view_t *vc = make_view(C, C, &pr->c_row, &pr->c_col, pr->c_base, bp->mr, bp->nr);
  int64_t nq = (int64_t)1 << (2 * level);
  view_t **qa = (view_t **)calloc((size_t)nq, sizeof(view_t *));
  view_t **qb = (view_t **)calloc((size_t)nq, sizeof(view_t *));
  view_t **qc = (view_t **)calloc((size_t)nq, sizeof(view_t *));
  if (level == 0) {
    qa[0] = va; qb[0] = vb; qc[0] = vc;
  } else {
    quadrant_views(va, level, qa);
    quadrant_views(vb, level, qb);
    quadrant_views(vc, level, qc);
  }
  int64_t mq = qa[0]->m, kq = qa[0]->n, nqq = qb[0]->n;
  /* PackedBuffer.a_panel / b_panel (kernels.py:87-99) */
  int64_t arows = bp->mc < mq ? bp->mc : mq, adepth = bp->kc < kq ? bp->kc : kq;
  int64_t bcols = bp->nc < nqq ? bp->nc : nqq, bdepth = adepth;
  double *abuf = (double *)calloc((size_t)(cdiv(arows, bp->mr) * adepth * bp->mr), sizeof(double));
  double *bbuf = (double *)calloc((size_t)(cdiv(bcols, bp->nr) * bdepth * bp->nr), sizeof(double));

  if (variant == 0) {
    for (int64_t t = 0; t < nterms; ++t) {
      side_t as = make_side(qa, &terms[t].a), bs = make_side(qb, &terms[t].b), cs = make_side(qc, &terms[t].c);
      run_fused(&as, &bs, &cs, bp, abuf, adepth, bbuf, bdepth, threads, force_slow, st);
      free_side(&as); free_side(&bs); free_side(&cs);
    }
  } else {
    double *M = (double *)calloc((size_t)(mq * nqq), sizeof(double));
    ora_bundle mr_b = {1, 0, {mq}, {1}}, mc_b = {1, 0, {nqq}, {mq}};
    view_t *mv = make_view(M, M, &mr_b, &mc_b, 0, bp->mr, bp->nr);
    double one = 1.0;
    side_t mside = {1, &mv, &one};
    double *ad = NULL, *bd = NULL;
    view_t *adv = NULL, *bdv = NULL;
    if (variant == 2) {
      ad = (double *)calloc((size_t)(mq * kq), sizeof(double));
      bd = (double *)calloc((size_t)(kq * nqq), sizeof(double));
      ora_bundle ar = {1, 0, {mq}, {1}}, ac = {1, 0, {kq}, {mq}};
      ora_bundle br = {1, 0, {kq}, {1}}, bc = {1, 0, {nqq}, {kq}};
      adv = make_view(ad, NULL, &ar, &ac, 0, bp->mr, bp->kr);
      bdv = make_view(bd, NULL, &br, &bc, 0, bp->kr, bp->nr);
    }
    for (int64_t t = 0; t < nterms; ++t) {
      side_t as = make_side(qa, &terms[t].a), bs = make_side(qb, &terms[t].b);
      memset(M, 0, sizeof(double) * (size_t)(mq * nqq));
      if (variant == 1) {
        run_fused(&as, &bs, &mside, bp, abuf, adepth, bbuf, bdepth, threads, force_slow, st);
      } else {
        unpack_sum(ad, &as, force_slow, st);
        unpack_sum(bd, &bs, force_slow, st);
        side_t sa = {1, &adv, &one}, sb = {1, &bdv, &one};
        run_fused(&sa, &sb, &mside, bp, abuf, adepth, bbuf, bdepth, threads, force_slow, st);
      }
      for (int j = 0; j < terms[t].c.n; ++j)
        accum_dense(M, mq, nqq, qc[terms[t].c.q[j]], (double)terms[t].c.s[j], force_slow, st);
      free_side(&as); free_side(&bs);
    }
    view_free(mv); view_free(adv); view_free(bdv);
    free(M); free(ad); free(bd);
  }

  free(abuf); free(bbuf);
  if (level > 0) {
    for (int64_t q = 0; q < nq; ++q) { view_free(qa[q]); view_free(qb[q]); view_free(qc[q]); }
  }
  view_free(va); view_free(vb); view_free(vc);
  free(qa); free(qb); free(qc);
  free_terms(terms, nterms);
  return 0;
}

/* oracle.py:62-92: C[ci+cj] += sum_p A[ai+ap] * B[bp+bj]; loops j, i, p (P innermost). */
int ora_contract_reference(const ora_problem *pr, const double *A, const double *B, double *C, int threads) {
  int64_t m = ora_bundle_len(&pr->a_row), k = ora_bundle_len(&pr->a_col), n = ora_bundle_len(&pr->b_col);
  int64_t *c_ri = (int64_t *)malloc(sizeof(int64_t) * (size_t)m), *c_cj = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  int64_t *a_ri = (int64_t *)malloc(sizeof(int64_t) * (size_t)m), *a_cp = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
  int64_t *b_rp = (int64_t *)malloc(sizeof(int64_t) * (size_t)k), *b_cj = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  ora_bundle_scatter(&pr->c_row, pr->c_base, c_ri);
  ora_bundle_scatter(&pr->c_col, 0, c_cj);
  ora_bundle_scatter(&pr->a_row, pr->a_base, a_ri);
  ora_bundle_scatter(&pr->a_col, 0, a_cp);
  ora_bundle_scatter(&pr->b_row, pr->b_base, b_rp);
  ora_bundle_scatter(&pr->b_col, 0, b_cj);
#pragma omp parallel for num_threads(threads > 0 ? threads : 1) schedule(dynamic, 1) if (threads > 1)
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int64_t p = 0; p < k; ++p) acc += A[a_ri[i] + a_cp[p]] * B[b_rp[p] + b_cj[j]];
      C[c_ri[i] + c_cj[j]] += acc;
    }
  free(c_ri); free(c_cj); free(a_ri); free(a_cp); free(b_rp); free(b_cj);
  return 0;
}

/* oracle.py:102-107 */
/* Component calls on raw scatter vectors (tests of the device pack_a / pack_b / microkernel):
 * kernels.py:166-201 through pack_a_block / pack_b_block above.  Views are given by
 * their scatter vectors (rows[t] of length m, cols[t] of length n) and unit strides;
 * the block vectors are rebuilt at (rb, cb) as BlockScatterView.from_scatter does. */
int ora_pack_panel(int which, const double *data, int nviews, const int64_t *const *rows, int64_t m,
                   const int64_t *const *cols, int64_t n, int64_t rb, int64_t cb, int64_t row_unit,
                   int64_t col_unit, const double *coeffs, int64_t x0, int64_t xcount, int64_t k0, int64_t kcount,
                   int force_slow, double *out, int64_t depth, int64_t *fast, int64_t *slow) {
  side_t sd;
  sd.n = nviews;
  sd.v = (view_t **)malloc(sizeof(view_t *) * (size_t)nviews);
  sd.coeff = (double *)malloc(sizeof(double) * (size_t)nviews);
  for (int t = 0; t < nviews; ++t) {
    sd.v[t] = view_new(data, NULL, rows[t], m, cols[t], n, rb, cb, row_unit, col_unit);
    sd.coeff[t] = coeffs[t];
  }
  *fast = *slow = 0;
  if (which == 0)
    pack_a_block(out, depth, &sd, x0, xcount, k0, kcount, rb, cb, force_slow, fast, slow);
  else
    pack_b_block(out, depth, &sd, k0, kcount, x0, xcount, rb, cb, force_slow, fast, slow);
  for (int t = 0; t < nviews; ++t) view_free(sd.v[t]);
  free(sd.v); free(sd.coeff);
  return 0;
}

/* kernels.py:204-233: microtile_mats (_jit.py:145-155) on (mr, >= k) x (>= k, nr) row-major
 * slivers, then store_tile into every target (view t: rows[t] of length tm[t], cols[t] of
 * length tn[t], block vectors at (mr, nr)), clipped to the view. */
int ora_microtile(const double *a, int64_t lda, const double *b, int64_t ldb, int64_t k, int64_t mr, int64_t nr,
                  double *cdata, int ntargets, const int64_t *const *rows, const int64_t *tm,
                  const int64_t *const *cols, const int64_t *tn, const int64_t *row_unit, const int64_t *col_unit,
                  const double *coeffs, const int64_t *i0, const int64_t *j0, int force_slow, int64_t *fast,
                  int64_t *slow) {
  *fast = *slow = 0;
  if (k == 0) return 0;
  double *acc = (double *)calloc((size_t)(mr * nr), sizeof(double));
  for (int64_t p = 0; p < k; ++p)
    for (int64_t i = 0; i < mr; ++i) {
      double av = a[i * lda + p];
      for (int64_t j = 0; j < nr; ++j) acc[i * nr + j] += av * b[p * ldb + j];
    }
  for (int t = 0; t < ntargets; ++t) {
    view_t *v = view_new(cdata, cdata, rows[t], tm[t], cols[t], tn[t], mr, nr, row_unit[t], col_unit[t]);
    int64_t ilim = v->m - i0[t] < mr ? v->m - i0[t] : mr, jlim = v->n - j0[t] < nr ? v->n - j0[t] : nr;
    if (store_tile(acc, v, coeffs[t], i0[t], ilim, j0[t], jlim, mr, nr, force_slow)) ++*fast; else ++*slow;
    view_free(v);
  }
  free(acc);
  return 0;
}

double ora_seq_sum_sq(const double *x, int64_t n) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += x[i] * x[i];
  return acc;
}

/* Debug/parity helpers: the reference's view vectors for one view, and its quadrants. */
int ora_view_vectors(const ora_bundle *rows, const ora_bundle *cols, int64_t base, int64_t rb, int64_t cb,
                     int level, int quadrant, int64_t *rscat, int64_t *cscat, int64_t *rbs, int64_t *cbs,
                     int64_t *mn) {
  view_t *v = make_view(NULL, NULL, rows, cols, base, rb, cb);
  view_t *q = v;
  view_t **qs = NULL;
  int64_t nq = (int64_t)1 << (2 * level);
  if (level > 0) {
    qs = (view_t **)calloc((size_t)nq, sizeof(view_t *));
    quadrant_views(v, level, qs);
    q = qs[quadrant];
  }
  mn[0] = q->m; mn[1] = q->n;
  if (rscat) memcpy(rscat, q->rscat, sizeof(int64_t) * (size_t)q->m);
  if (cscat) memcpy(cscat, q->cscat, sizeof(int64_t) * (size_t)q->n);
  if (rbs) memcpy(rbs, q->rbs, sizeof(int64_t) * (size_t)cdiv(q->m, rb));
  if (cbs) memcpy(cbs, q->cbs, sizeof(int64_t) * (size_t)cdiv(q->n, cb));
  if (qs) {
    for (int64_t i = 0; i < nq; ++i) view_free(qs[i]);
    free(qs);
  }
  view_free(v);
  return 0;
}

int ora_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
