/*
 * yo_oracle.c — CPU restatement of the reference's Newton-step hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load this library, and only as the checker
 * or the reported CPU baseline.  The product path (paper_2605_23088_b200)
 * never links or calls it.
 *
 * It exports the C-ABI of include/yasps_b200.h with the prefix `yo_` and
 * restates, function by function, the algorithm of the reference relsim
 * (/root/reference/proj), deliberately NOT the GPU algorithm:
 *   - local g / H of each energy in the UNCOMPRESSED width (the reference's
 *     symbolic derivatives, diff.cpp:528-708) via second-order forward-mode
 *     jets over the energy formulas of energies.cpp:20-174;
 *   - local_compress (assembly.cpp:266-282), symmetrisation and psd_project
 *     (assembly.cpp:8-17) with a dense cyclic-Jacobi EVD of the m x m block;
 *     ReducedProject route (assembly.cpp:299-320);
 *   - placement walk (index_gen.cpp:77-122), make_pattern (assembly.cpp:201-219),
 *     build_global_structure + BlockSparseHessian::build (223-246, 22-61) with a
 *     comparison sort on (rows, cols, row, col), value_offset binary search
 *     (63-81), serial instance-order scatter (346-372), DiagAccumulator (158-180);
 *   - spmv_add (solver.cpp:10-82, serial), BlockJacobiPreconditioner
 *     (93-146), pcg (151-200) verbatim, Engine::minimize_step (engine.cpp:75-101);
 *   - refresh_dynamic_pairs (sim.cpp:456-484) all-pairs loop.
 * Parity pinning: the reference itself is built here from its unmodified
 * sources against eigen-lite (oracle/ref_build.sh -> oracle/_ref: relsim, its
 * ten doctest suites — all passing — and oracle/ref_driver.cpp).  The goldens
 * of tests/golden are the reference's own step records; tests/test_golden.py
 * and tests/test_reference.py check this restatement against them (bit-exact
 * structure and pairs, equal PCG iteration counts, values <= 1e-9), and
 * tests/test_oracle.py against the reference's known-answer tests.
 */
#include <math.h>
#include <pthread.h>
#include <setjmp.h>
#include <stdatomic.h>
#include <unistd.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/yasps_b200.h"

#define MAXW 24
#define MAXK 4

enum { K_SNH = 0, K_BENDING, K_INERTIA, K_ORTHO, K_PP, K_REPULSIVE, K_PT, K_EE, K_PE };

typedef struct {
  int64_t n;
  int rc;
  int64_t start;
  double* init;
} Target;

typedef struct {
  int kind;
  int64_t n;
  int ta, tb;
  int64_t* v2b;
  double* rest;
} Domain;

typedef struct {
  int nchild;
  int* child;
  int kappa_u, width;
} Union;

typedef struct {
  int uni, dynamic;
  int arity; /* points per instance: 2 pairs, 3 point-edge, 4 point-triangle / edge-edge */
  int64_t n;
  int64_t* pairs;
  /* contact candidates (yo_set_stencil_primitives): kind 1 PT, 2 EE (self), 3 PE */
  int pkind, aa, ab;
  int64_t na, nb;
  int64_t *pa, *pb;
} PairSet;

typedef struct {
  int64_t index; /* 1-based, 0 = pad */
  int len, col;
} Slot;

typedef struct {
  int64_t gstart;
  int len, comp_col;
} UBlock;

typedef struct {
  int ua, ub;
  int64_t value_offset;
} Dest;

typedef struct {
  int nu, m, nd;
  UBlock ub[MAXK];
  int slot2ub[MAXK];
  Dest d[MAXK * (MAXK + 1) / 2];
} Plan;

typedef struct {
  int kind, dynamic, mode;
  int64_t n;
  int kappa, width;
  double prm[6];
  int target, domain, pairset;
  int64_t* conn;
  double* cdata;
  double* anchor;
  Slot* slots;
  Plan* plans;
  int64_t nplans;
} Energy;

typedef struct {
  int rows, cols;
  int64_t row, col;
} Coord;

typedef struct {
  int64_t rows, cols, coord_start, count, value_start;
} Group;

typedef struct {
  int64_t s;
  int ng;
  Group* groups;
  int64_t nb;
  int64_t* row;
  int64_t* col;
  int64_t* voff;
  int64_t nv;
  double* values;
} Bsr;

typedef struct yo_context yo_context;

struct yo_context {
  char err[1024];
  int err_cls;
  jmp_buf jb;
  Target* t;
  int nt;
  Domain* d;
  int nd;
  Union* u;
  int nu;
  PairSet* ps;
  int nps;
  Energy* e;
  int ne;
  int finalized;
  uint64_t epoch, seen_epoch;
  int64_t s;
  double *X, *X0, *G, *DX;
  int64_t nblk;
  int64_t* bstart;
  int* brc;
  int64_t* bvoff;
  int64_t diag_vals;
  double* diag;
  double* minv;
  int32_t regularized;
  Bsr H[2];
  double* hist;
  int64_t hist_n;
  /* free-standing systems */
  Bsr* sys;
  int nsys;
  /* row-partitioned solve (restatement of ys_dist.cu) */
  int dist_on, dist_rank, dist_n;
  ys_allgather_fn dist_fn;
  void* dist_user;
  int64_t dist_bounds[65], dist_exp_off[65];
};

/* ------------------------------------------------------------------------
 * Errors.  Inside the parallel local-evaluation phase (the reference's
 * parallel_for over instances, assembly.cpp:334-336) a failing instance
 * records its error and unwinds to its own thread-local jump buffer; the
 * serial phase then reports the failure of the lowest instance index, as the
 * serial loop would. */
static _Thread_local jmp_buf* TL_JB;
static _Thread_local int TL_CLS;
static _Thread_local char TL_MSG[256];

static void fail(yo_context* c, int cls, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  if (TL_JB) {
    vsnprintf(TL_MSG, sizeof(TL_MSG), fmt, ap);
    va_end(ap);
    TL_CLS = cls;
    longjmp(*TL_JB, 1);
  }
  vsnprintf(c->err, sizeof(c->err), fmt, ap);
  va_end(ap);
  c->err_cls = cls;
  longjmp(c->jb, cls);
}

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz);
  if (!p) abort();
  return p;
}

#define GROW(arr, cnt) (arr = realloc(arr, sizeof(*(arr)) * (size_t)((cnt) + 1)))

/* ------------------------------------------------------------------------
 * Second-order forward-mode jets: value, gradient and Hessian w.r.t. the n
 * uncompressed local parameters (the reference's symbolic J and H,
 * diff.cpp:374-442 + 631-705).
 * ------------------------------------------------------------------------ */
typedef struct {
  double v;
  double g[MAXW];
  double h[MAXW * MAXW];
} Jet;

static _Thread_local int JN;          /* active dimension */
static _Thread_local yo_context* JC;  /* for errors */

static void j_const(Jet* o, double v) {
  o->v = v;
  memset(o->g, 0, sizeof(double) * JN);
  memset(o->h, 0, sizeof(double) * JN * JN);
}
static void j_var(Jet* o, double v, int i) {
  j_const(o, v);
  o->g[i] = 1.0;
}
static void j_lin(Jet* o, const Jet* a, double sa, const Jet* b, double sb) { /* sa*a + sb*b */
  Jet t;
  t.v = sa * a->v + sb * b->v;
  for (int i = 0; i < JN; ++i) t.g[i] = sa * a->g[i] + sb * b->g[i];
  for (int i = 0; i < JN * JN; ++i) t.h[i] = sa * a->h[i] + sb * b->h[i];
  *o = t;
}
static void j_add(Jet* o, const Jet* a, const Jet* b) { j_lin(o, a, 1.0, b, 1.0); }
static void j_sub(Jet* o, const Jet* a, const Jet* b) { j_lin(o, a, 1.0, b, -1.0); }
static void j_scale(Jet* o, const Jet* a, double s) {
  Jet t;
  t.v = s * a->v;
  for (int i = 0; i < JN; ++i) t.g[i] = s * a->g[i];
  for (int i = 0; i < JN * JN; ++i) t.h[i] = s * a->h[i];
  *o = t;
}
static void j_addc(Jet* o, const Jet* a, double c) {
  *o = *a;
  o->v += c;
}
static void j_mul(Jet* o, const Jet* a, const Jet* b) {
  Jet t;
  t.v = a->v * b->v;
  for (int i = 0; i < JN; ++i) t.g[i] = a->g[i] * b->v + a->v * b->g[i];
  for (int i = 0; i < JN; ++i)
    for (int k = 0; k < JN; ++k)
      t.h[i * JN + k] = a->h[i * JN + k] * b->v + a->v * b->h[i * JN + k] + a->g[i] * b->g[k] + b->g[i] * a->g[k];
  *o = t;
}
/* f(a) with derivatives f1, f2 */
static void j_unary(Jet* o, const Jet* a, double f, double f1, double f2) {
  Jet t;
  t.v = f;
  for (int i = 0; i < JN; ++i) t.g[i] = f1 * a->g[i];
  for (int i = 0; i < JN; ++i)
    for (int k = 0; k < JN; ++k) t.h[i * JN + k] = f1 * a->h[i * JN + k] + f2 * a->g[i] * a->g[k];
  *o = t;
}
static void j_div(Jet* o, const Jet* a, const Jet* b) {
  if (b->v == 0.0) fail(JC, YS_ERR_NUMERICAL, "division by zero");
  Jet inv;
  j_unary(&inv, b, 1.0 / b->v, -1.0 / (b->v * b->v), 2.0 / (b->v * b->v * b->v));
  j_mul(o, a, &inv);
}
static void j_log(Jet* o, const Jet* a) {
  if (a->v <= 0.0) fail(JC, YS_ERR_NUMERICAL, "log of non-positive value");
  j_unary(o, a, log(a->v), 1.0 / a->v, -1.0 / (a->v * a->v));
}
/* Euclidean norm of k jets: sqrt(sum a_i^2); its derivative divides by the
 * norm (diff.cpp:259-262), undefined at zero. */
static void j_norm(Jet* o, const Jet* a, int k) {
  Jet s, q;
  j_const(&s, 0.0);
  for (int i = 0; i < k; ++i) {
    j_mul(&q, &a[i], &a[i]);
    j_add(&s, &s, &q);
  }
  const double r = sqrt(s.v);
  if (JN > 0 && r == 0.0) fail(JC, YS_ERR_NUMERICAL, "division by zero");
  if (JN == 0) {
    o->v = r;
    return;
  }
  j_unary(o, &s, r, 0.5 / r, -0.25 / (r * s.v));
}
static void j_cross(Jet* o, const Jet* a, const Jet* b) {
  Jet t1, t2, r[3];
  for (int k = 0; k < 3; ++k) {
    const int i1 = (k + 1) % 3, i2 = (k + 2) % 3;
    j_mul(&t1, &a[i1], &b[i2]);
    j_mul(&t2, &a[i2], &b[i1]);
    j_sub(&r[k], &t1, &t2);
  }
  o[0] = r[0];
  o[1] = r[1];
  o[2] = r[2];
}

/* ------------------------------------------------------------------------
 * Symmetric EVD (cyclic Jacobi) and psd_project (assembly.cpp:8-17)
 * ------------------------------------------------------------------------ */
static void psd_project(double* a, int n) {
  double v[MAXW * MAXW];
  double s[MAXW * MAXW];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) s[i * n + j] = 0.5 * (a[i * n + j] + a[j * n + i]);
  for (int i = 0; i < n * n; ++i) v[i] = 0.0;
  for (int i = 0; i < n; ++i) v[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += s[p * n + q] * s[p * n + q];
    if (off == 0.0) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = s[p * n + q], app = s[p * n + p], aqq = s[q * n + q];
        const double g = 100.0 * fabs(apq);
        if (fabs(app) + g == fabs(app) && fabs(aqq) + g == fabs(aqq)) {
          s[p * n + q] = s[q * n + p] = 0.0;
          continue;
        }
        const double theta = 0.5 * (aqq - app) / apq;
        double t = 1.0 / (fabs(theta) + sqrt(theta * theta + 1.0));
        if (theta < 0.0) t = -t;
        const double cc = 1.0 / sqrt(t * t + 1.0), sn = t * cc, tau = sn / (1.0 + cc);
        s[p * n + p] = app - t * apq;
        s[q * n + q] = aqq + t * apq;
        s[p * n + q] = s[q * n + p] = 0.0;
        for (int k = 0; k < n; ++k) {
          if (k == p || k == q) continue;
          const double akp = s[k * n + p], akq = s[k * n + q];
          s[k * n + p] = s[p * n + k] = akp - sn * (akq + tau * akp);
          s[k * n + q] = s[q * n + k] = akq + sn * (akp - tau * akq);
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = v[k * n + p], vkq = v[k * n + q];
          v[k * n + p] = vkp - sn * (vkq + tau * vkp);
          v[k * n + q] = vkq + sn * (vkp - tau * vkq);
        }
      }
  }
  double lam[MAXW];
  for (int k = 0; k < n; ++k) lam[k] = s[k * n + k] < 0.0 ? 0.0 : s[k * n + k];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc += v[i * n + k] * lam[k] * v[j * n + k];
      a[i * n + j] = acc;
    }
}

/* ------------------------------------------------------------------------
 * Layout and placement (index_gen.cpp:22-38, 77-122)
 * ------------------------------------------------------------------------ */
static int dom_kappa(const Domain* d) { return d->kind == YS_POINTS_FREE ? 1 : d->kind == YS_POINTS_AFFINE ? 2 : 0; }
static int dom_width(const Domain* d) { return d->kind == YS_POINTS_FREE ? 3 : d->kind == YS_POINTS_AFFINE ? 12 : 0; }

/* DataSlot for free points; Seq[JoinRep(v2b, A), JoinRep(v2b, t)] for affine. */
static int point_slots(yo_context* c, const Domain* d, int64_t i, int col, Slot* out) {
  if (d->kind == YS_POINTS_FREE) {
    out[0].index = c->t[d->ta].start + 3 * i + 1;
    out[0].len = 3;
    out[0].col = col;
    return 1;
  }
  if (d->kind == YS_POINTS_AFFINE) {
    const int64_t b = d->v2b[i];
    out[0].index = c->t[d->ta].start + 9 * b + 1;
    out[0].len = 9;
    out[0].col = col;
    out[1].index = c->t[d->tb].start + 3 * b + 1;
    out[1].len = 3;
    out[1].col = col + 9;
    return 2;
  }
  return 0;
}

/* PrimitiveUnion::decode (scene.cpp:227-237) */
static int union_decode(yo_context* c, const Union* u, int64_t g, int64_t* local) {
  int64_t off = 0, total = 0;
  for (int k = 0; k < u->nchild; ++k) total += c->d[u->child[k]].n;
  if (g < 0 || g >= total) fail(c, YS_ERR_VALIDATION, "union decode: index %lld out of range [0, %lld)", (long long)g, (long long)total);
  int br = 0;
  int64_t broff = 0;
  for (int k = 0; k < u->nchild; ++k) {
    if (off <= g) {
      br = k;
      broff = off;
    }
    off += c->d[u->child[k]].n;
  }
  /* upper_bound - 1 then skip empty children */
  while (c->d[u->child[br]].n == 0) ++br;
  *local = g - broff;
  return br;
}

static void energy_slots(yo_context* c, const Energy* e, int64_t i, Slot* s) {
  for (int k = 0; k < e->kappa; ++k) {
    s[k].index = 0;
    s[k].len = 0;
    s[k].col = 0;
  }
  switch (e->kind) {
    case K_SNH:
    case K_BENDING:
      for (int l = 0; l < 4; ++l) {
        s[l].index = c->t[e->target].start + 3 * e->conn[4 * i + l] + 1;
        s[l].len = 3;
        s[l].col = 3 * l;
      }
      break;
    case K_ORTHO:
      s[0].index = c->t[e->target].start + 9 * i + 1;
      s[0].len = 9;
      s[0].col = 0;
      break;
    case K_INERTIA:
      point_slots(c, &c->d[e->domain], i, 0, s);
      break;
    default: { /* JoinRep(stencil2v, UnionSel): pairs (arity 2) and contact stencils */
      const PairSet* p = &c->ps[e->pairset];
      const Union* u = &c->u[p->uni];
      for (int l = 0; l < p->arity; ++l) {
        int64_t local;
        const int br = union_decode(c, u, p->pairs[p->arity * i + l], &local);
        point_slots(c, &c->d[u->child[br]], local, l * u->width, s + l * u->kappa_u);
      }
    }
  }
}

/* make_pattern (assembly.cpp:201-219) */
static void make_pattern(const Slot* s, int kappa, Plan* p) {
  p->nu = 0;
  p->m = 0;
  for (int k = 0; k < kappa; ++k) {
    p->slot2ub[k] = -1;
    if (s[k].index == 0) continue;
    const int64_t gs = s[k].index - 1;
    int found = -1;
    for (int u = 0; u < p->nu; ++u)
      if (p->ub[u].gstart == gs) found = u;
    if (found < 0) {
      found = p->nu++;
      p->ub[found].gstart = gs;
      p->ub[found].len = s[k].len;
      p->ub[found].comp_col = p->m;
      p->m += s[k].len;
    }
    p->slot2ub[k] = found;
  }
}

/* ------------------------------------------------------------------------
 * BlockSparseHessian::build (assembly.cpp:22-61) and value_offset (63-81)
 * ------------------------------------------------------------------------ */
static int coord_cmp(const void* a, const void* b) {
  const Coord* x = (const Coord*)a;
  const Coord* y = (const Coord*)b;
  if (x->rows != y->rows) return x->rows < y->rows ? -1 : 1;
  if (x->cols != y->cols) return x->cols < y->cols ? -1 : 1;
  if (x->row != y->row) return x->row < y->row ? -1 : 1;
  if (x->col != y->col) return x->col < y->col ? -1 : 1;
  return 0;
}

static void bsr_free(Bsr* h) {
  free(h->groups);
  free(h->row);
  free(h->col);
  free(h->voff);
  free(h->values);
  memset(h, 0, sizeof(*h));
}

static void bsr_build(yo_context* c, Bsr* h, Coord* coords, int64_t n, int64_t total) {
  for (int64_t k = 0; k < n; ++k) {
    const Coord* q = &coords[k];
    if (q->row < 0 || q->col < 0 || q->row + q->rows > total || q->col + q->cols > total)
      fail(c, YS_ERR_VALIDATION, "block coordinate outside the global system");
    if (q->row > q->col) fail(c, YS_ERR_INTERNAL, "block coordinate not upper-triangular");
  }
  qsort(coords, (size_t)n, sizeof(Coord), coord_cmp);
  int64_t m = 0;
  for (int64_t k = 0; k < n; ++k)
    if (k == 0 || coord_cmp(&coords[k], &coords[m - 1]) != 0) coords[m++] = coords[k];
  bsr_free(h);
  h->s = total;
  h->nb = m;
  h->row = xcalloc((size_t)m, sizeof(int64_t));
  h->col = xcalloc((size_t)m, sizeof(int64_t));
  h->voff = xcalloc((size_t)m, sizeof(int64_t));
  h->groups = xcalloc((size_t)(m + 1), sizeof(Group));
  int64_t acc = 0;
  for (int64_t i = 0; i < m;) {
    int64_t j = i;
    Group g;
    g.rows = coords[i].rows;
    g.cols = coords[i].cols;
    g.coord_start = i;
    g.value_start = acc;
    while (j < m && coords[j].rows == g.rows && coords[j].cols == g.cols) ++j;
    g.count = j - i;
    acc += g.count * g.rows * g.cols;
    h->groups[h->ng++] = g;
    i = j;
  }
  for (int gi = 0; gi < h->ng; ++gi) {
    const Group* g = &h->groups[gi];
    for (int64_t k = 0; k < g->count; ++k) {
      const Coord* q = &coords[g->coord_start + k];
      h->row[g->coord_start + k] = q->row;
      h->col[g->coord_start + k] = q->col;
      h->voff[g->coord_start + k] = g->value_start + k * g->rows * g->cols;
    }
  }
  h->nv = acc;
  h->values = xcalloc((size_t)acc, sizeof(double));
}

static int64_t value_offset(yo_context* c, const Bsr* h, int rows, int cols, int64_t row, int64_t col) {
  for (int gi = 0; gi < h->ng; ++gi) {
    const Group* g = &h->groups[gi];
    if (g->rows != rows || g->cols != cols) continue;
    int64_t lo = g->coord_start, hi = g->coord_start + g->count;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (h->row[mid] < row || (h->row[mid] == row && h->col[mid] < col)) lo = mid + 1;
      else hi = mid;
    }
    if (lo < g->coord_start + g->count && h->row[lo] == row && h->col[lo] == col) return h->voff[lo];
    break;
  }
  fail(c, YS_ERR_INTERNAL, "block (%lld,%lld) of shape %dx%d not present in the global structure", (long long)row,
       (long long)col, rows, cols);
  return -1;
}

static uint64_t structure_checksum(const Bsr* h) {
  uint64_t x = 1469598103934665603ull;
#define MIX(v)               \
  do {                       \
    x ^= (uint64_t)(v);      \
    x *= 1099511628211ull;   \
  } while (0)
  MIX(h->s);
  for (int g = 0; g < h->ng; ++g) {
    MIX(h->groups[g].rows);
    MIX(h->groups[g].cols);
    MIX(h->groups[g].count);
  }
  for (int64_t i = 0; i < h->nb; ++i) {
    MIX(h->row[i]);
    MIX(h->col[i]);
  }
#undef MIX
  return x;
}

/* ------------------------------------------------------------------------
 * Group structure (engine.cpp:34-39)
 * ------------------------------------------------------------------------ */
static int64_t energy_count(yo_context* c, const Energy* e) { return e->pairset >= 0 ? c->ps[e->pairset].n : e->n; }

static void build_group(yo_context* c, int which) {
  int64_t ncoord = 0, cap = 0;
  Coord* coords = NULL;
  for (int ei = 0; ei < c->ne; ++ei) {
    Energy* e = &c->e[ei];
    if (e->dynamic != which) continue;
    e->n = energy_count(c, e);
    free(e->slots);
    free(e->plans);
    e->slots = xcalloc((size_t)(e->n * (e->kappa ? e->kappa : 1)), sizeof(Slot));
    e->plans = xcalloc((size_t)e->n, sizeof(Plan));
    e->nplans = e->n;
    if (e->kappa == 0) continue;
    for (int64_t i = 0; i < e->n; ++i) {
      Slot* s = e->slots + i * e->kappa;
      energy_slots(c, e, i, s);
      Plan* p = &e->plans[i];
      make_pattern(s, e->kappa, p);
      for (int a = 0; a < p->nu; ++a)
        for (int b = a; b < p->nu; ++b) {
          const UBlock* ua = &p->ub[a];
          const UBlock* ub = &p->ub[b];
          const UBlock* lo = ua->gstart <= ub->gstart ? ua : ub;
          const UBlock* hi = ua->gstart <= ub->gstart ? ub : ua;
          if (ncoord == cap) {
            cap = cap ? 2 * cap : 1024;
            coords = realloc(coords, sizeof(Coord) * (size_t)cap);
          }
          coords[ncoord].rows = lo->len;
          coords[ncoord].cols = hi->len;
          coords[ncoord].row = lo->gstart;
          coords[ncoord].col = hi->gstart;
          ++ncoord;
        }
    }
  }
  bsr_build(c, &c->H[which], coords, ncoord, c->s);
  free(coords);
  /* build_instance_plans (assembly.cpp:248-264) */
  for (int ei = 0; ei < c->ne; ++ei) {
    Energy* e = &c->e[ei];
    if (e->dynamic != which || e->kappa == 0) continue;
    for (int64_t i = 0; i < e->n; ++i) {
      Plan* p = &e->plans[i];
      p->nd = 0;
      for (int a = 0; a < p->nu; ++a)
        for (int b = a; b < p->nu; ++b) {
          Dest* d = &p->d[p->nd++];
          const int sw = p->ub[a].gstart > p->ub[b].gstart;
          d->ua = sw ? b : a;
          d->ub = sw ? a : b;
          d->value_offset = value_offset(c, &c->H[which], p->ub[d->ua].len, p->ub[d->ub].len, p->ub[d->ua].gstart,
                                         p->ub[d->ub].gstart);
        }
    }
  }
}

/* ------------------------------------------------------------------------
 * Energy formulas in jets (energies.cpp)
 * ------------------------------------------------------------------------ */
/* Point position of domain d, point i, whose parameters sit at columns
 * [col, col + width) of the local vector (or are constants for fixed). */
static void point_jets(yo_context* c, const Domain* d, int64_t i, int col, const double* X, Jet* p) {
  if (d->kind == YS_POINTS_FREE) {
    const double* q = X + c->t[d->ta].start + 3 * i;
    for (int k = 0; k < 3; ++k) j_var(&p[k], q[k], col + k);
  } else if (d->kind == YS_POINTS_AFFINE) {
    const int64_t b = d->v2b[i];
    const double* A = X + c->t[d->ta].start + 9 * b;
    const double* t = X + c->t[d->tb].start + 3 * b;
    const double* r = d->rest + 3 * i;
    for (int k = 0; k < 3; ++k) {
      /* position = affine.matmul(rest) + trans (sim.cpp:247) */
      Jet acc, a, q;
      j_const(&acc, 0.0);
      for (int j = 0; j < 3; ++j) {
        j_var(&a, A[3 * k + j], col + 3 * k + j);
        j_scale(&q, &a, r[j]);
        j_add(&acc, &acc, &q);
      }
      j_var(&a, t[k], col + 9 + k);
      j_add(&p[k], &acc, &a);
    }
  } else {
    for (int k = 0; k < 3; ++k) j_const(&p[k], d->rest[3 * i + k]);
  }
}

static void point_value(yo_context* c, const Domain* d, int64_t i, const double* X, double* p) {
  if (d->kind == YS_POINTS_FREE) {
    const double* q = X + c->t[d->ta].start + 3 * i;
    p[0] = q[0]; p[1] = q[1]; p[2] = q[2];
  } else if (d->kind == YS_POINTS_AFFINE) {
    const int64_t b = d->v2b[i];
    const double* A = X + c->t[d->ta].start + 9 * b;
    const double* t = X + c->t[d->tb].start + 3 * b;
    const double* r = d->rest + 3 * i;
    for (int k = 0; k < 3; ++k) p[k] = ((A[3 * k] * r[0] + A[3 * k + 1] * r[1]) + A[3 * k + 2] * r[2]) + t[k];
  } else {
    p[0] = d->rest[3 * i]; p[1] = d->rest[3 * i + 1]; p[2] = d->rest[3 * i + 2];
  }
}

/* Stable Neo-Hookean psi(F) with F the row-major 3x3 of Jets (energies.cpp:78-113) */
static void snh_psi(const Energy* e, int64_t t, Jet F[9], Jet* psi) {
  const double* binv = e->cdata + 10 * t;
  const double vol = binv[9];
  const double mu = e->prm[0], lambda = e->prm[1], alpha = e->prm[2], w = e->prm[3];
  Jet fi[9], q, acc;
  /* fi = F^T Binv */
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      j_const(&acc, 0.0);
      for (int k = 0; k < 3; ++k) {
        j_scale(&q, &F[3 * k + i], binv[3 * k + j]);
        j_add(&acc, &acc, &q);
      }
      fi[3 * i + j] = acc;
    }
  /* ic = tr(fi^T fi) */
  Jet ic;
  j_const(&ic, 0.0);
  for (int k = 0; k < 9; ++k) {
    j_mul(&q, &fi[k], &fi[k]);
    j_add(&ic, &ic, &q);
  }
  /* J = det fi (cofactor expansion on the first row) */
  Jet m1, m2, c0, c1, c2, J;
  j_mul(&m1, &fi[4], &fi[8]);
  j_mul(&m2, &fi[5], &fi[7]);
  j_sub(&c0, &m1, &m2);
  j_mul(&m1, &fi[3], &fi[8]);
  j_mul(&m2, &fi[5], &fi[6]);
  j_sub(&c1, &m1, &m2);
  j_mul(&m1, &fi[3], &fi[7]);
  j_mul(&m2, &fi[4], &fi[6]);
  j_sub(&c2, &m1, &m2);
  j_mul(&J, &fi[0], &c0);
  j_mul(&q, &fi[1], &c1);
  j_sub(&J, &J, &q);
  j_mul(&q, &fi[2], &c2);
  j_add(&J, &J, &q);
  /* psi = V w [mu/2 (ic-3) - mu/2 log(ic+1) + lambda/2 (J-alpha)^2] */
  Jet a1, a2, a3, lg, js;
  j_addc(&a1, &ic, -3.0);
  j_scale(&a1, &a1, mu / 2.0);
  j_addc(&lg, &ic, 1.0);
  j_log(&lg, &lg);
  j_scale(&a2, &lg, mu / 2.0);
  j_addc(&js, &J, -alpha);
  j_mul(&a3, &js, &js);
  j_scale(&a3, &a3, lambda / 2.0);
  j_sub(&acc, &a1, &a2);
  j_add(&acc, &acc, &a3);
  j_scale(psi, &acc, vol * w);
}

/* Local energy / gradient / Hessian in the uncompressed width; vars = JN. */
/* ------------------------------------------------------------------------
 * Point-triangle / edge-edge / point-edge barriers — NOT IN THE REFERENCE
 * (its contact is point-point only, proj/README.md:110-111), so this is the
 * specification the B200 kernels are checked against (with finite
 * differences and PSD checks): the point-point barrier of energies.cpp:30-47
 * on the squared distance d between the stencil's primitives, IPC's distance
 * types chosen on the current positions (Ericson, Real-Time Collision
 * Detection 5.1.5 / 5.1.9), FullProject.
 * ------------------------------------------------------------------------ */
enum { CT_PP = 0, CT_PE = 1, CT_PT = 2, CT_EE = 3 };
typedef struct {
  int type, a, b, c, e;
} ContactSel;

static double c_dot(const double* x, const double* y) { return x[0] * y[0] + x[1] * y[1] + x[2] * y[2]; }
static void c_sub(const double* x, const double* y, double* o) {
  o[0] = x[0] - y[0];
  o[1] = x[1] - y[1];
  o[2] = x[2] - y[2];
}
static ContactSel csel(int t, int a, int b, int c, int e) {
  ContactSel r = {t, a, b, c, e};
  return r;
}

static ContactSel classify_pt(double x[4][3]) {
  double ab[3], ac[3], ap[3], bp[3], cp[3];
  c_sub(x[2], x[1], ab);
  c_sub(x[3], x[1], ac);
  c_sub(x[0], x[1], ap);
  const double d1 = c_dot(ab, ap), d2 = c_dot(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) return csel(CT_PP, 0, 1, 0, 0);
  c_sub(x[0], x[2], bp);
  const double d3 = c_dot(ab, bp), d4 = c_dot(ac, bp);
  if (d3 >= 0.0 && d4 <= d3) return csel(CT_PP, 0, 2, 0, 0);
  const double vc = d1 * d4 - d3 * d2;
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) return csel(CT_PE, 0, 1, 2, 0);
  c_sub(x[0], x[3], cp);
  const double d5 = c_dot(ab, cp), d6 = c_dot(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) return csel(CT_PP, 0, 3, 0, 0);
  const double vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) return csel(CT_PE, 0, 1, 3, 0);
  const double va = d3 * d6 - d5 * d4;
  if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) return csel(CT_PE, 0, 2, 3, 0);
  return csel(CT_PT, 0, 1, 2, 3);
}

static ContactSel classify_pe(double x[4][3]) {
  double ed[3], ap[3];
  c_sub(x[2], x[1], ed);
  c_sub(x[0], x[1], ap);
  const double t = c_dot(ap, ed), ee = c_dot(ed, ed);
  if (t <= 0.0) return csel(CT_PP, 0, 1, 0, 0);
  if (t >= ee) return csel(CT_PP, 0, 2, 0, 0);
  return csel(CT_PE, 0, 1, 2, 0);
}

static ContactSel classify_ee(double x[4][3]) {
  double d1[3], d2[3], r[3];
  c_sub(x[1], x[0], d1);
  c_sub(x[3], x[2], d2);
  c_sub(x[0], x[2], r);
  const double a = c_dot(d1, d1), e = c_dot(d2, d2), f = c_dot(d2, r);
  const double cc = c_dot(d1, r), b = c_dot(d1, d2);
  const double denom = a * e - b * b;
  double s;
  int s_clamped;
  if (denom > 1e-20 * (a * e)) {
    s = (b * f - cc * e) / denom;
    s_clamped = s <= 0.0 || s >= 1.0;
    s = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);
  } else {
    s = 0.0;
    s_clamped = 1;
  }
  const double tn = b * s + f;
  if (tn <= 0.0) {
    const double sn = -cc;
    s_clamped = sn <= 0.0 || sn >= a;
    s = sn <= 0.0 ? 0.0 : (sn >= a ? 1.0 : sn / a);
    if (s_clamped) return csel(CT_PP, s == 0.0 ? 0 : 1, 2, 0, 0);
    return csel(CT_PE, 2, 0, 1, 0);
  }
  if (tn >= e) {
    const double sn = b - cc;
    s_clamped = sn <= 0.0 || sn >= a;
    s = sn <= 0.0 ? 0.0 : (sn >= a ? 1.0 : sn / a);
    if (s_clamped) return csel(CT_PP, s == 0.0 ? 0 : 1, 3, 0, 0);
    return csel(CT_PE, 3, 0, 1, 0);
  }
  if (s_clamped) return csel(CT_PE, s == 0.0 ? 0 : 1, 2, 3, 0);
  return csel(CT_EE, 0, 1, 2, 3);
}

/* value-only squared distance of the selected type: the same operations in
 * the same order as the B200 candidate test (ys_contact4.cuh contact_dist2_value) */
static void c_cross(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}
static double contact_dist2_value(ContactSel s, double x[4][3]) {
  double u[3], v[3], w[3], n[3];
  if (s.type == CT_PP) {
    c_sub(x[s.b], x[s.a], u);
    return c_dot(u, u);
  }
  if (s.type == CT_PE) {
    c_sub(x[s.b], x[s.a], u);
    c_sub(x[s.c], x[s.a], v);
    c_sub(x[s.c], x[s.b], w);
    c_cross(u, v, n);
    return c_dot(n, n) / c_dot(w, w);
  }
  if (s.type == CT_PT) {
    c_sub(x[s.a], x[s.b], u);
    c_sub(x[s.c], x[s.b], v);
    c_sub(x[s.e], x[s.b], w);
    c_cross(v, w, n);
    const double sp = c_dot(u, n);
    return (sp * sp) / c_dot(n, n);
  }
  c_sub(x[s.b], x[s.a], u);
  c_sub(x[s.e], x[s.c], v);
  c_sub(x[s.c], x[s.a], w);
  c_cross(u, v, n);
  const double sp = c_dot(w, n);
  return (sp * sp) / c_dot(n, n);
}

static void j_dot3(Jet* o, const Jet* a, const Jet* b) {
  Jet q;
  j_mul(o, &a[0], &b[0]);
  j_mul(&q, &a[1], &b[1]);
  j_add(o, o, &q);
  j_mul(&q, &a[2], &b[2]);
  j_add(o, o, &q);
}

/* squared distance of the selected type over the stencil's point jets P */
static void contact_dist2(ContactSel s, Jet (*P)[3], Jet* d) {
  Jet u[3], v[3], w[3], n[3], sp, num, den;
  int k;
  if (s.type == CT_PP) {
    for (k = 0; k < 3; ++k) j_sub(&u[k], &P[s.b][k], &P[s.a][k]);
    j_dot3(d, u, u);
  } else if (s.type == CT_PE) {
    for (k = 0; k < 3; ++k) {
      j_sub(&u[k], &P[s.b][k], &P[s.a][k]);
      j_sub(&v[k], &P[s.c][k], &P[s.a][k]);
      j_sub(&w[k], &P[s.c][k], &P[s.b][k]);
    }
    j_cross(n, u, v);
    j_dot3(&num, n, n);
    j_dot3(&den, w, w);
    j_div(d, &num, &den);
  } else if (s.type == CT_PT) {
    for (k = 0; k < 3; ++k) {
      j_sub(&u[k], &P[s.a][k], &P[s.b][k]);
      j_sub(&v[k], &P[s.c][k], &P[s.b][k]);
      j_sub(&w[k], &P[s.e][k], &P[s.b][k]);
    }
    j_cross(n, v, w);
    j_dot3(&sp, u, n);
    j_mul(&num, &sp, &sp);
    j_dot3(&den, n, n);
    j_div(d, &num, &den);
  } else {
    for (k = 0; k < 3; ++k) {
      j_sub(&u[k], &P[s.b][k], &P[s.a][k]);
      j_sub(&v[k], &P[s.e][k], &P[s.c][k]);
      j_sub(&w[k], &P[s.c][k], &P[s.a][k]);
    }
    j_cross(n, u, v);
    j_dot3(&sp, w, n);
    j_mul(&num, &sp, &sp);
    j_dot3(&den, n, n);
    j_div(d, &num, &den);
  }
}

/* w kappa (d - dhat)^2 log(d / dhat)^2 on a jet d (energies.cpp:30-39) */
static void pp_barrier(const Energy* e, const Jet* d, Jet* E) {
  Jet i5, len, lg, acc;
  j_scale(&i5, d, 1.0 / e->prm[0]);
  i5.v = d->v / e->prm[0];
  j_addc(&len, d, -e->prm[0]);
  j_log(&lg, &i5);
  j_mul(&acc, &len, &len);
  j_scale(&acc, &acc, e->prm[1]);
  j_mul(&acc, &acc, &lg);
  j_mul(&acc, &acc, &lg);
  j_scale(E, &acc, e->prm[2]);
}

static void local_eval(yo_context* c, const Energy* e, int64_t i, const double* X, Jet* E) {
  switch (e->kind) {
    case K_SNH: {
      Jet x[12], F[9];
      for (int l = 0; l < 4; ++l) {
        const double* q = X + c->t[e->target].start + 3 * e->conn[4 * i + l];
        for (int k = 0; k < 3; ++k) j_var(&x[3 * l + k], q[k], 3 * l + k);
      }
      for (int r = 0; r < 3; ++r)
        for (int cc = 0; cc < 3; ++cc) j_sub(&F[3 * r + cc], &x[3 * (cc + 1) + r], &x[r]);
      snh_psi(e, i, F, E);
      break;
    }
    case K_BENDING: {
      Jet x[12], e0[3], e1[3], e2[3], n1[3], n2[3], N1, N2, u[3], U;
      for (int l = 0; l < 4; ++l) {
        const double* q = X + c->t[e->target].start + 3 * e->conn[4 * i + l];
        for (int k = 0; k < 3; ++k) j_var(&x[3 * l + k], q[k], 3 * l + k);
      }
      for (int k = 0; k < 3; ++k) {
        j_sub(&e0[k], &x[3 + k], &x[k]);
        j_sub(&e1[k], &x[6 + k], &x[k]);
        j_sub(&e2[k], &x[9 + k], &x[k]);
      }
      j_cross(n1, e0, e1); /* (x1-x0) x (x2-x0) */
      j_cross(n2, e2, e0); /* (x3-x0) x (x1-x0) */
      j_norm(&N1, n1, 3);
      j_norm(&N2, n2, 3);
      for (int k = 0; k < 3; ++k) {
        Jet h1, h2;
        j_div(&h1, &n1[k], &N1);
        j_div(&h2, &n2[k], &N2);
        j_sub(&u[k], &h1, &h2);
      }
      j_norm(&U, u, 3);
      j_scale(E, &U, e->cdata[i]);
      break;
    }
    case K_ORTHO: {
      Jet A[9], M[9], q, acc, tr;
      const double* a = X + c->t[e->target].start + 9 * i;
      for (int k = 0; k < 9; ++k) j_var(&A[k], a[k], k);
      for (int r = 0; r < 3; ++r)
        for (int cc = 0; cc < 3; ++cc) {
          j_const(&acc, 0.0);
          for (int k = 0; k < 3; ++k) {
            j_mul(&q, &A[3 * k + r], &A[3 * k + cc]);
            j_add(&acc, &acc, &q);
          }
          j_addc(&M[3 * r + cc], &acc, r == cc ? -1.0 : 0.0);
        }
      j_const(&tr, 0.0);
      for (int k = 0; k < 9; ++k) {
        j_mul(&q, &M[k], &M[k]);
        j_add(&tr, &tr, &q);
      }
      j_scale(E, &tr, 0.5 * e->prm[0]);
      break;
    }
    case K_INERTIA: {
      const Domain* d = &c->d[e->domain];
      Jet p[3], dv[3], q, acc;
      point_jets(c, d, i, 0, X, p);
      j_const(&acc, 0.0);
      for (int k = 0; k < 3; ++k) {
        j_addc(&dv[k], &p[k], -e->anchor[3 * i + k]);
        j_mul(&q, &dv[k], &dv[k]);
        j_add(&acc, &acc, &q);
      }
      j_scale(E, &acc, 0.5 * e->cdata[i]);
      break;
    }
    case K_PT:
    case K_EE:
    case K_PE: {
      const PairSet* ps = &c->ps[e->pairset];
      const Union* u = &c->u[ps->uni];
      Jet P[4][3], d;
      double xv[4][3];
      for (int l = 0; l < ps->arity; ++l) {
        int64_t loc;
        const int br = union_decode(c, u, ps->pairs[ps->arity * i + l], &loc);
        point_jets(c, &c->d[u->child[br]], loc, l * u->width, X, P[l]);
        point_value(c, &c->d[u->child[br]], loc, X, xv[l]);
      }
      const ContactSel sel = e->kind == K_PT ? classify_pt(xv) : e->kind == K_EE ? classify_ee(xv) : classify_pe(xv);
      contact_dist2(sel, P, &d);
      pp_barrier(e, &d, E);
      break;
    }
    default: {
      const PairSet* ps = &c->ps[e->pairset];
      const Union* u = &c->u[ps->uni];
      Jet p0[3], p1[3], dv[3], q, d;
      int64_t l0, l1;
      const int b0 = union_decode(c, u, ps->pairs[2 * i], &l0);
      const int b1 = union_decode(c, u, ps->pairs[2 * i + 1], &l1);
      point_jets(c, &c->d[u->child[b0]], l0, 0, X, p0);
      point_jets(c, &c->d[u->child[b1]], l1, u->width, X, p1);
      if (e->kind == K_REPULSIVE) {
        /* weight / (p0 - p1).norm() (energies.cpp:22-24) */
        Jet nrm, w;
        for (int k = 0; k < 3; ++k) j_sub(&dv[k], &p0[k], &p1[k]);
        j_norm(&nrm, dv, 3);
        j_const(&w, e->prm[2]);
        j_div(E, &w, &nrm);
        break;
      }
      /* dvec = p1 - p0; d = dvec.dvec; kappa (d - dhat)^2 log(d/dhat)^2 (energies.cpp:30-39) */
      j_const(&d, 0.0);
      for (int k = 0; k < 3; ++k) {
        j_sub(&dv[k], &p1[k], &p0[k]);
        j_mul(&q, &dv[k], &dv[k]);
        j_add(&d, &d, &q);
      }
      Jet i5, len, lg, acc;
      j_scale(&i5, &d, 1.0 / e->prm[0]);
      i5.v = d.v / e->prm[0];
      j_addc(&len, &d, -e->prm[0]);
      j_log(&lg, &i5);
      j_mul(&acc, &len, &len);
      j_scale(&acc, &acc, e->prm[1]);
      j_mul(&acc, &acc, &lg);
      j_mul(&acc, &acc, &lg);
      j_scale(E, &acc, e->prm[2]);
    }
  }
}

/* Energy only (JN = 0): same formulas, no derivatives. */
static double local_energy(yo_context* c, const Energy* e, int64_t i, const double* X) {
  Jet E;
  const int save = JN;
  JN = 0;
  local_eval(c, e, i, X, &E);
  JN = save;
  return E.v;
}

/* ------------------------------------------------------------------------
 * assemble_local + assemble_group (assembly.cpp:284-374)
 * ------------------------------------------------------------------------ */
static void diag_add(yo_context* c, int64_t gstart, const double* b, int len) {
  /* DiagAccumulator::add (assembly.cpp:176-180): binary search on starts */
  int64_t lo = 0, hi = c->nblk;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (c->bstart[mid] < gstart) lo = mid + 1;
    else hi = mid;
  }
  if (lo == c->nblk || c->bstart[lo] != gstart) fail(c, YS_ERR_INTERNAL, "diagonal block start not aligned");
  double* d = c->diag + c->bvoff[lo];
  for (int k = 0; k < len * len; ++k) d[k] += b[k];
}

/* One instance's local gradient (width) and compressed, symmetrised,
 * projected Hessian (m x m): assemble_local (assembly.cpp:284-321). */
static void local_assemble(yo_context* c, const Energy* e, int64_t i, int project, int with_h, Jet* E, double* g,
                           double* hc) {
  const Slot* s = e->slots + i * e->kappa;
  const Plan* p = &e->plans[i];
  const int m = p->m;
  const int reduced = e->mode == YS_PROJECT_REDUCED && e->kind == K_SNH;
  if (!reduced) {
    JN = e->width;
    JC = c;
    local_eval(c, e, i, c->X, E);
    for (int k = 0; k < e->width; ++k) g[k] = E->g[k];
    if (!with_h) return;
    /* local_compress (assembly.cpp:266-282) */
    for (int k = 0; k < m * m; ++k) hc[k] = 0.0;
    for (int a = 0; a < e->kappa; ++a) {
      const int us = p->slot2ub[a];
      if (us < 0) continue;
      for (int b = 0; b < e->kappa; ++b) {
        const int ut = p->slot2ub[b];
        if (ut < 0) continue;
        for (int r = 0; r < s[a].len; ++r)
          for (int q = 0; q < s[b].len; ++q)
            hc[(p->ub[us].comp_col + r) * m + p->ub[ut].comp_col + q] += E->h[(s[a].col + r) * e->width + s[b].col + q];
      }
    }
    /* 0.5 (H + H^T), then psd_project */
    double sym[MAXW * MAXW];
    for (int r = 0; r < m; ++r)
      for (int q = 0; q < m; ++q) sym[r * m + q] = 0.5 * (hc[r * m + q] + hc[q * m + r]);
    memcpy(hc, sym, sizeof(double) * m * m);
    if (project && m > 0) psd_project(hc, m);
    return;
  }
  /* ReducedProject: inner variable vec_rm(F) (9), J = dF/dx (9 x 12) */
  JN = 9;
  JC = c;
  Jet F[9];
  double x[12];
  for (int l = 0; l < 4; ++l)
    for (int k = 0; k < 3; ++k) x[3 * l + k] = c->X[c->t[e->target].start + 3 * e->conn[4 * i + l] + k];
  for (int r = 0; r < 3; ++r)
    for (int cc = 0; cc < 3; ++cc) j_var(&F[3 * r + cc], x[3 * (cc + 1) + r] - x[r], 3 * r + cc);
  snh_psi(e, i, F, E);
  double J[9 * 12];
  memset(J, 0, sizeof(J));
  for (int r = 0; r < 3; ++r)
    for (int cc = 0; cc < 3; ++cc) {
      J[(3 * r + cc) * 12 + 3 * (cc + 1) + r] = 1.0;
      J[(3 * r + cc) * 12 + r] = -1.0;
    }
  for (int k = 0; k < 12; ++k) {
    double acc = 0.0;
    for (int q = 0; q < 9; ++q) acc += E->g[q] * J[q * 12 + k];
    g[k] = acc;
  }
  if (!with_h) return;
  double hin[81];
  for (int r = 0; r < 9; ++r)
    for (int q = 0; q < 9; ++q) hin[r * 9 + q] = 0.5 * (E->h[r * 9 + q] + E->h[q * 9 + r]);
  if (project) psd_project(hin, 9);
  double jc[9 * MAXW];
  memset(jc, 0, sizeof(jc));
  for (int a = 0; a < e->kappa; ++a) {
    const int us = p->slot2ub[a];
    if (us < 0) continue;
    for (int q = 0; q < 9; ++q)
      for (int r = 0; r < s[a].len; ++r) jc[q * m + p->ub[us].comp_col + r] += J[q * 12 + s[a].col + r];
  }
  for (int r = 0; r < m; ++r)
    for (int q = 0; q < m; ++q) {
      double acc = 0.0;
      for (int a = 0; a < 9; ++a)
        for (int b = 0; b < 9; ++b) acc += jc[a * m + r] * hin[a * 9 + b] * jc[b * m + q];
      hc[r * m + q] = acc;
    }
}

/* Instance loop of assemble_group (assembly.cpp:323-374): local results of a
 * chunk of instances in parallel (host threads, dynamic blocks of 64; each
 * instance is independent, so the results are those of the serial loop bit
 * for bit), then the scatter serially in instance order.  YO_THREADS caps the
 * thread count (default: all online CPUs). */
#define CHUNK 32768
typedef struct {
  yo_context* c;
  const Energy* e;
  int64_t i0, n;
  int project, with_h;
  atomic_llong next;
  double *gbuf, *hbuf;
  int* ebuf;
  char (*mbuf)[256];
} LocalJob;

static void* local_worker(void* arg) {
  LocalJob* j = (LocalJob*)arg;
  static _Thread_local Jet E;
  for (;;) {
    const int64_t k0 = atomic_fetch_add(&j->next, 64);
    if (k0 >= j->n) break;
    const int64_t k1 = k0 + 64 < j->n ? k0 + 64 : j->n;
    for (int64_t k = k0; k < k1; ++k) {
      jmp_buf jb;
      j->ebuf[k] = 0;
      if (setjmp(jb)) {
        TL_JB = NULL;
        j->ebuf[k] = TL_CLS;
        memcpy(j->mbuf[k], TL_MSG, 256);
        continue;
      }
      TL_JB = &jb;
      local_assemble(j->c, j->e, j->i0 + k, j->project, j->with_h, &E, j->gbuf + k * MAXW,
                     j->hbuf + k * MAXW * MAXW);
      TL_JB = NULL;
    }
  }
  return NULL;
}

static int host_threads(void) {
  const char* v = getenv("YO_THREADS");
  long n = v ? atol(v) : sysconf(_SC_NPROCESSORS_ONLN);
  return n < 1 ? 1 : n > 256 ? 256 : (int)n;
}

static void assemble_group(yo_context* c, int which, int project, int with_h) {
  double* gbuf = (double*)xcalloc((size_t)CHUNK * MAXW, sizeof(double));
  double* hbuf = (double*)xcalloc((size_t)CHUNK * MAXW * MAXW, sizeof(double));
  int* ebuf = (int*)xcalloc(CHUNK, sizeof(int));
  char(*mbuf)[256] = calloc(CHUNK, 256);
  const int nt = host_threads();
  pthread_t th[256];
  for (int ei = 0; ei < c->ne; ++ei) {
    Energy* e = &c->e[ei];
    if (e->dynamic != which || e->n == 0 || e->kappa == 0) continue;
    if (e->nplans != energy_count(c, e)) {
      free(gbuf), free(hbuf), free(ebuf), free(mbuf);
      fail(c, YS_ERR_VALIDATION, "energy '%d': instance plans are stale; rebuild the dynamic structures", ei);
    }
    for (int64_t i0 = 0; i0 < e->n; i0 += CHUNK) {
      const int64_t n = e->n - i0 < CHUNK ? e->n - i0 : CHUNK;
      LocalJob job = {c, e, i0, n, project, with_h, 0, gbuf, hbuf, ebuf, mbuf};
      atomic_init(&job.next, 0);
      const int use = (int)(n / 256 + 1) < nt ? (int)(n / 256 + 1) : nt;
      for (int t = 1; t < use; ++t) pthread_create(&th[t], NULL, local_worker, &job);
      local_worker(&job);
      for (int t = 1; t < use; ++t) pthread_join(th[t], NULL);
      for (int64_t k = 0; k < n; ++k)
        if (ebuf[k]) {
          int cls = ebuf[k];
          char msg[256];
          memcpy(msg, mbuf[k], 256);
          free(gbuf), free(hbuf), free(ebuf), free(mbuf);
          fail(c, cls, "%s", msg);
        }
      /* scatter in instance order (assembly.cpp:346-372) */
      for (int64_t k = 0; k < n; ++k) {
        const int64_t i = i0 + k;
        const Slot* s = e->slots + i * e->kappa;
        const Plan* p = &e->plans[i];
        const int m = p->m;
        const double* g = gbuf + k * MAXW;
        const double* hc = hbuf + k * MAXW * MAXW;
        for (int a = 0; a < e->kappa; ++a) {
          if (s[a].index == 0) continue;
          for (int r = 0; r < s[a].len; ++r) c->G[s[a].index - 1 + r] += g[s[a].col + r];
        }
        if (!with_h) continue;
        for (int d = 0; d < p->nd; ++d) {
          const UBlock* lo = &p->ub[p->d[d].ua];
          const UBlock* hi = &p->ub[p->d[d].ub];
          double* dst = c->H[which].values + p->d[d].value_offset;
          for (int r = 0; r < lo->len; ++r)
            for (int q = 0; q < hi->len; ++q) dst[r * hi->len + q] += hc[(lo->comp_col + r) * m + hi->comp_col + q];
        }
        for (int u = 0; u < p->nu; ++u) {
          double b[81];
          const UBlock* ub = &p->ub[u];
          for (int r = 0; r < ub->len; ++r)
            for (int q = 0; q < ub->len; ++q) b[r * ub->len + q] = hc[(ub->comp_col + r) * m + ub->comp_col + q];
          diag_add(c, ub->gstart, b, ub->len);
        }
      }
    }
  }
  free(gbuf), free(hbuf), free(ebuf), free(mbuf);
}

static void assemble(yo_context* c, int project, int with_h) {
  if (c->seen_epoch != c->epoch)
    fail(c, YS_ERR_VALIDATION, "dynamic structures are stale after resize_dynamic; call refresh_dynamic()");
  memset(c->G, 0, sizeof(double) * (size_t)c->s);
  memset(c->diag, 0, sizeof(double) * (size_t)c->diag_vals);
  for (int w = 0; w < 2; ++w) memset(c->H[w].values, 0, sizeof(double) * (size_t)c->H[w].nv);
  assemble_group(c, 0, project, with_h);
  assemble_group(c, 1, project, with_h);
}

/* ------------------------------------------------------------------------
 * Solver (solver.cpp)
 * ------------------------------------------------------------------------ */
static void spmv_range(const Bsr* h, const Group* g, int64_t k0, int64_t k1, const double* x, double* y) {
  const int R = (int)g->rows, Cc = (int)g->cols;
  for (int64_t k = k0; k < k1; ++k) {
    const int64_t bi = g->coord_start + k;
    const double* b = h->values + h->voff[bi];
    const int64_t r = h->row[bi], cc = h->col[bi];
    for (int i = 0; i < R; ++i) {
      double acc = 0.0;
      for (int j = 0; j < Cc; ++j) acc += b[i * Cc + j] * x[cc + j];
      y[r + i] += acc;
    }
    if (r != cc)
      for (int j = 0; j < Cc; ++j) {
        double acc = 0.0;
        for (int i = 0; i < R; ++i) acc += b[i * Cc + j] * x[r + i];
        y[cc + j] += acc;
      }
  }
}

typedef struct {
  const Bsr* h;
  const Group* g;
  int64_t k0, k1;
  const double* x;
  double* y;
} SpmvShard;

static void* spmv_shard(void* a) {
  SpmvShard* s = (SpmvShard*)a;
  spmv_range(s->h, s->g, s->k0, s->k1, s->x, s->y);
  return NULL;
}

/* spmv_add (solver.cpp:59-82).  YO_SPMV_THREADS > 1 (the reference's
 * "threads" > 1) with >= 1024 blocks: per group, block shards into per-thread
 * partial vectors, reduced in shard order — the reference's threaded rounding.
 * Default 1: the serial, deterministic order (the parity checker's mode). */
static void spmv_add(const Bsr* h, const double* x, double* y) {
  const char* v = getenv("YO_SPMV_THREADS");
  int nt = v ? atoi(v) : 1;
  if (nt > 64) nt = 64;
  if (nt <= 1 || h->nb < 1024) {
    for (int gi = 0; gi < h->ng; ++gi) spmv_range(h, &h->groups[gi], 0, h->groups[gi].count, x, y);
    return;
  }
  const int64_t n = h->s;
  double* part = (double*)xcalloc((size_t)nt * (size_t)n, sizeof(double));
  pthread_t th[64];
  SpmvShard sh[64];
  for (int gi = 0; gi < h->ng; ++gi) {
    const Group* g = &h->groups[gi];
    const int64_t per = (g->count + nt - 1) / nt;
    int used = 0;
    for (int t = 0; t < nt; ++t) {
      const int64_t b = t * per, e = b + per < g->count ? b + per : g->count;
      if (b >= e) break;
      sh[t] = (SpmvShard){h, g, b, e, x, part + (size_t)t * (size_t)n};
      pthread_create(&th[t], NULL, spmv_shard, &sh[t]);
      ++used;
    }
    for (int t = 0; t < used; ++t) pthread_join(th[t], NULL);
  }
  for (int t = 0; t < nt; ++t)
    for (int64_t i = 0; i < n; ++i) y[i] += part[(size_t)t * (size_t)n + (size_t)i];
  free(part);
}

/* Eigen dynamic inverse() = PartialPivLU (solver.cpp:107) */
static void lu_inverse(const double* B, int n, double* inv) {
  double a[144];
  int piv[12];
  memcpy(a, B, sizeof(double) * n * n);
  for (int k = 0; k < n; ++k) piv[k] = k;
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = fabs(a[k * n + k]);
    for (int r = k + 1; r < n; ++r)
      if (fabs(a[r * n + k]) > best) {
        best = fabs(a[r * n + k]);
        p = r;
      }
    if (p != k) {
      for (int cc = 0; cc < n; ++cc) {
        const double t = a[k * n + cc];
        a[k * n + cc] = a[p * n + cc];
        a[p * n + cc] = t;
      }
      const int t = piv[k];
      piv[k] = piv[p];
      piv[p] = t;
    }
    for (int r = k + 1; r < n; ++r) {
      const double f = a[r * n + k] / a[k * n + k];
      a[r * n + k] = f;
      for (int cc = k + 1; cc < n; ++cc) a[r * n + cc] -= f * a[k * n + cc];
    }
  }
  for (int col = 0; col < n; ++col) {
    double y[12];
    for (int r = 0; r < n; ++r) {
      double v = piv[r] == col ? 1.0 : 0.0;
      for (int cc = 0; cc < r; ++cc) v -= a[r * n + cc] * y[cc];
      y[r] = v;
    }
    for (int r = n - 1; r >= 0; --r) {
      double v = y[r];
      for (int cc = r + 1; cc < n; ++cc) v -= a[r * n + cc] * y[cc];
      y[r] = v / a[r * n + r];
    }
    for (int r = 0; r < n; ++r) inv[r * n + col] = y[r];
  }
}

static double inv_residual(const double* B, const double* I, int n, int* finite) {
  double r = 0.0;
  *finite = 1;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc += B[i * n + k] * I[k * n + j];
      acc -= i == j ? 1.0 : 0.0;
      r += acc * acc;
      if (!isfinite(I[i * n + j])) *finite = 0;
    }
  return sqrt(r);
}

/* BlockJacobiPreconditioner::build (solver.cpp:93-122) */
static void build_precond(yo_context* c) {
  c->regularized = 0;
  for (int64_t b = 0; b < c->nblk; ++b) {
    const int m = c->brc[b];
    const double* B = c->diag + c->bvoff[b];
    double* inv = c->minv + c->bvoff[b];
    int zero = 1;
    double nb = 0.0, tr = 0.0;
    for (int k = 0; k < m * m; ++k) {
      if (!(fabs(B[k]) <= 0.0)) zero = 0;
      nb += B[k] * B[k];
    }
    for (int k = 0; k < m; ++k) tr += B[k * m + k];
    if (zero) {
      for (int k = 0; k < m * m; ++k) inv[k] = k % (m + 1) == 0 ? 1.0 : 0.0;
      ++c->regularized;
      continue;
    }
    int fin;
    lu_inverse(B, m, inv);
    double res = inv_residual(B, inv, m, &fin);
    if (!fin || res > 1e-6 * (1.0 + sqrt(nb))) {
      double eps = 1e-12 * tr / m;
      if (eps <= 0.0) eps = 1e-12;
      double reg[144];
      double nr = 0.0;
      for (int k = 0; k < m * m; ++k) {
        reg[k] = B[k] + (k % (m + 1) == 0 ? eps : 0.0);
        nr += reg[k] * reg[k];
      }
      lu_inverse(reg, m, inv);
      ++c->regularized;
      res = inv_residual(reg, inv, m, &fin);
      if (!fin || res > 1e-3 * (1.0 + sqrt(nr)))
        fail(c, YS_ERR_NUMERICAL, "diagonal block at DoF range [%lld, %lld) is singular", (long long)c->bstart[b],
             (long long)(c->bstart[b] + m));
    }
  }
}

static void precond_apply(yo_context* c, const double* r, double* z) {
  for (int64_t b = 0; b < c->nblk; ++b) {
    const int m = c->brc[b];
    const double* M = c->minv + c->bvoff[b];
    const int64_t s0 = c->bstart[b];
    for (int i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int k = 0; k < m; ++k) acc += M[i * m + k] * r[s0 + k];
      z[s0 + i] = acc;
    }
  }
}

static double dot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* pcg (solver.cpp:151-200) */
static void pcg(yo_context* c, Bsr* h0, Bsr* h1, const double* g, double tol, int64_t max_iter, double* x,
                int64_t* iters, double* relres, int* converged) {
  const int64_t n = c->s;
  memset(x, 0, sizeof(double) * (size_t)n);
  free(c->hist);
  c->hist = xcalloc((size_t)(max_iter + 2), sizeof(double));
  c->hist_n = 0;
  *iters = 0;
  *relres = 0.0;
  *converged = 0;
  const double gnorm = sqrt(dot(g, g, n));
  if (gnorm == 0.0) {
    *converged = 1;
    return;
  }
  double* r = xcalloc((size_t)n, sizeof(double));
  double* z = xcalloc((size_t)n, sizeof(double));
  double* p = xcalloc((size_t)n, sizeof(double));
  double* hp = xcalloc((size_t)n, sizeof(double));
  memcpy(r, g, sizeof(double) * (size_t)n);
  precond_apply(c, r, z);
  memcpy(p, z, sizeof(double) * (size_t)n);
  double rz = dot(r, z, n);
  c->hist[c->hist_n++] = 1.0;
  for (int64_t it = 0; it < max_iter; ++it) {
    memset(hp, 0, sizeof(double) * (size_t)n);
    spmv_add(h0, p, hp);
    if (h1) spmv_add(h1, p, hp);
    const double php = dot(p, hp, n);
    if (!isfinite(php) || php <= 0.0) {
      if (php == 0.0) break;
      free(r); free(z); free(p); free(hp);
      fail(c, YS_ERR_NUMERICAL, "PCG diverged at iteration %lld (non-finite or negative curvature)", (long long)it);
    }
    const double alpha = rz / php;
    for (int64_t i = 0; i < n; ++i) x[i] += alpha * p[i];
    for (int64_t i = 0; i < n; ++i) r[i] -= alpha * hp[i];
    *iters = it + 1;
    const double rel = sqrt(dot(r, r, n)) / gnorm;
    c->hist[c->hist_n++] = rel;
    if (!isfinite(rel)) {
      free(r); free(z); free(p); free(hp);
      fail(c, YS_ERR_NUMERICAL, "PCG diverged at iteration %lld (non-finite residual)", (long long)it);
    }
    precond_apply(c, r, z);
    const double rz_new = dot(r, z, n);
    if (rel <= tol) {
      *converged = 1;
      break;
    }
    const double beta = rz_new / rz;
    rz = rz_new;
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  *relres = c->hist[c->hist_n - 1];
  free(r); free(z); free(p); free(hp);
}

/* ------------------------------------------------------------------------
 * Row-partitioned PCG over nranks processes (the algorithm of
 * ys_dist.cu restated serially per rank).  Partition: W(R) = entries of block
 * rows < R (each upper block once at its row, off-diagonal blocks once more
 * at their column row, both stores) + R; bounds[k] = first R with
 * W(R) >= k W(NB) / n.  Halo: a block (R, C) with owner(R) != owner(C)
 * exports rows R and C.  Dot products: the rank's partial over its rows in
 * row order, then the allgathered partials summed in rank order.
 * ------------------------------------------------------------------------ */
static int owner_of(const int64_t* bounds, int n, int64_t v) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (bounds[mid] <= v) lo = mid;
    else hi = mid;
  }
  return lo;
}

static void dist_gather(yo_context* c, const double* send, double* recv, int64_t count) {
  if (c->dist_fn(c->dist_user, send, recv, count) != 0)
    fail(c, YS_ERR_CUDA, "distributed solve: the host allgather callback failed");
}

static void dist_spmv_rows(const Bsr* h, int64_t a, int64_t b, const double* x, double* y) {
  for (int64_t bi = 0; bi < h->nb; ++bi) {
    const double* B = h->values + h->voff[bi];
    const int64_t r = h->row[bi], cc = h->col[bi];
    if (r / 3 >= a && r / 3 < b)
      for (int i = 0; i < 3; ++i) y[r + i] += B[3 * i] * x[cc] + B[3 * i + 1] * x[cc + 1] + B[3 * i + 2] * x[cc + 2];
    if (r != cc && cc / 3 >= a && cc / 3 < b)
      for (int j = 0; j < 3; ++j) y[cc + j] += B[j] * x[r] + B[3 + j] * x[r + 1] + B[6 + j] * x[r + 2];
  }
}

static void dist_pcg(yo_context* c, double tol, int64_t max_iter, double* x, int64_t* iters, double* relres,
                     int* converged) {
  const int n = c->dist_n, me = c->dist_rank;
  const int64_t NB = c->nblk, s = c->s;
  for (int64_t b = 0; b < NB; ++b)
    if (c->brc[b] != 3) fail(c, YS_ERR_VALIDATION, "distributed PCG supports uniform 3x3 block systems only");
  /* partition: the static structure's entries (fixed across Newton
   * iterations, so the device knows each rank's instances before evaluating) */
  int64_t* W = xcalloc((size_t)NB + 1, sizeof(int64_t));
  for (int w = 0; w < 1; ++w)
    for (int64_t bi = 0; bi < c->H[w].nb; ++bi) {
      W[c->H[w].row[bi] / 3 + 1] += 1;
      if (c->H[w].row[bi] != c->H[w].col[bi]) W[c->H[w].col[bi] / 3 + 1] += 1;
    }
  for (int64_t R = 0; R < NB; ++R) W[R + 1] += W[R] + 1;
  int64_t* bounds = c->dist_bounds;
  bounds[0] = 0;
  bounds[n] = NB;
  for (int k = 1; k < n; ++k) {
    const int64_t target = W[NB] * k / n;
    int64_t lo = 0, hi = NB;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (W[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    bounds[k] = lo;
  }
  free(W);
  /* halo */
  unsigned char* need = xcalloc((size_t)NB, 1);
  for (int w = 0; w < 2; ++w)
    for (int64_t bi = 0; bi < c->H[w].nb; ++bi) {
      const int64_t R = c->H[w].row[bi] / 3, C = c->H[w].col[bi] / 3;
      if (R != C && owner_of(bounds, n, R) != owner_of(bounds, n, C)) need[R] = need[C] = 1;
    }
  int64_t nexp = 0;
  int64_t* exp = xcalloc((size_t)NB + 1, sizeof(int64_t));
  for (int64_t R = 0; R < NB; ++R)
    if (need[R]) exp[nexp++] = R;
  free(need);
  int64_t* off = c->dist_exp_off;
  for (int k = 0; k <= n; ++k) {
    int64_t lo = 0, hi = nexp;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (exp[mid] < bounds[k]) lo = mid + 1;
      else hi = mid;
    }
    off[k] = lo;
  }
  int64_t maxe = 0, maxr = 0;
  for (int k = 0; k < n; ++k) {
    if (off[k + 1] - off[k] > maxe) maxe = off[k + 1] - off[k];
    if (bounds[k + 1] - bounds[k] > maxr) maxr = bounds[k + 1] - bounds[k];
  }
  const int64_t a = bounds[me], b = bounds[me + 1];
  const int64_t big = 3 * (maxe > maxr ? maxe : maxr) + 2;
  double* send = xcalloc((size_t)big, sizeof(double));
  double* recv = xcalloc((size_t)big * (size_t)n, sizeof(double));
  double* r = xcalloc((size_t)s, sizeof(double));
  double* z = xcalloc((size_t)s, sizeof(double));
  double* p = xcalloc((size_t)s, sizeof(double));
  double* hp = xcalloc((size_t)s, sizeof(double));
  double part[2], all[128];
  memset(x, 0, sizeof(double) * (size_t)s);
  free(c->hist);
  c->hist = xcalloc((size_t)(max_iter + 2), sizeof(double));
  c->hist_n = 0;
  *iters = 0;
  *relres = 0.0;
  *converged = 0;
  /* r = g, z = M^-1 r, p = z on owned rows */
  part[0] = part[1] = 0.0;
  for (int64_t R = a; R < b; ++R) {
    const double* M = c->minv + c->bvoff[R];
    for (int i = 0; i < 3; ++i) r[3 * R + i] = c->G[3 * R + i];
    for (int i = 0; i < 3; ++i) {
      z[3 * R + i] = M[3 * i] * r[3 * R] + M[3 * i + 1] * r[3 * R + 1] + M[3 * i + 2] * r[3 * R + 2];
      p[3 * R + i] = z[3 * R + i];
      part[0] += r[3 * R + i] * r[3 * R + i];
      part[1] += r[3 * R + i] * z[3 * R + i];
    }
  }
  dist_gather(c, part, all, 2);
  double gg = 0.0, rz = 0.0;
  for (int k = 0; k < n; ++k) {
    gg += all[2 * k];
    rz += all[2 * k + 1];
  }
  const double gnorm = sqrt(gg);
  int status = gnorm == 0.0 ? 1 : (max_iter > 0 ? 0 : 5);
  if (gnorm != 0.0) c->hist[c->hist_n++] = 1.0;
  else *converged = 1;
  int64_t it = 0;
  while (status == 0) {
    if (maxe > 0) { /* halo of p */
      const int64_t mine = off[me + 1] - off[me];
      for (int64_t i = 0; i < mine; ++i)
        for (int d = 0; d < 3; ++d) send[3 * i + d] = p[3 * exp[off[me] + i] + d];
      dist_gather(c, send, recv, 3 * maxe);
      for (int k = 0; k < n; ++k) {
        if (k == me) continue;
        for (int64_t e = off[k]; e < off[k + 1]; ++e)
          for (int d = 0; d < 3; ++d) p[3 * exp[e] + d] = recv[(k * maxe + (e - off[k])) * 3 + d];
      }
    }
    memset(hp, 0, sizeof(double) * (size_t)s);
    dist_spmv_rows(&c->H[0], a, b, p, hp);
    dist_spmv_rows(&c->H[1], a, b, p, hp);
    part[0] = 0.0;
    for (int64_t i = 3 * a; i < 3 * b; ++i) part[0] += p[i] * hp[i];
    dist_gather(c, part, all, 1);
    double php = 0.0;
    for (int k = 0; k < n; ++k) php += all[k];
    if (!isfinite(php) || php <= 0.0) {
      if (php == 0.0) break;
      fail(c, YS_ERR_NUMERICAL, "PCG diverged at iteration %lld (non-finite or negative curvature)", (long long)it);
    }
    const double alpha = rz / php;
    part[0] = part[1] = 0.0;
    for (int64_t R = a; R < b; ++R) {
      const double* M = c->minv + c->bvoff[R];
      for (int i = 0; i < 3; ++i) {
        x[3 * R + i] += alpha * p[3 * R + i];
        r[3 * R + i] -= alpha * hp[3 * R + i];
      }
      for (int i = 0; i < 3; ++i) {
        z[3 * R + i] = M[3 * i] * r[3 * R] + M[3 * i + 1] * r[3 * R + 1] + M[3 * i + 2] * r[3 * R + 2];
        part[0] += r[3 * R + i] * r[3 * R + i];
        part[1] += r[3 * R + i] * z[3 * R + i];
      }
    }
    dist_gather(c, part, all, 2);
    double rr = 0.0, rzn = 0.0;
    for (int k = 0; k < n; ++k) {
      rr += all[2 * k];
      rzn += all[2 * k + 1];
    }
    const double rel = sqrt(rr) / gnorm;
    *iters = ++it;
    c->hist[c->hist_n++] = rel;
    if (!isfinite(rel))
      fail(c, YS_ERR_NUMERICAL, "PCG diverged at iteration %lld (non-finite residual)", (long long)(it - 1));
    if (rel <= tol) {
      *converged = 1;
      break;
    }
    if (it >= max_iter) break;
    const double beta = rzn / rz;
    rz = rzn;
    for (int64_t i = 3 * a; i < 3 * b; ++i) p[i] = z[i] + beta * p[i];
  }
  if (c->hist_n) *relres = c->hist[c->hist_n - 1];
  if (n > 1) { /* every rank returns the full step */
    for (int64_t i = 0; i < 3 * (b - a); ++i) send[i] = x[3 * a + i];
    dist_gather(c, send, recv, 3 * maxr);
    for (int64_t R = 0; R < NB; ++R) {
      const int k = owner_of(bounds, n, R);
      for (int d = 0; d < 3; ++d) x[3 * R + d] = recv[(k * maxr + (R - bounds[k])) * 3 + d];
    }
  }
  free(exp); free(send); free(recv); free(r); free(z); free(p); free(hp);
}

/* ------------------------------------------------------------------------
 * Engine construction (engine.cpp:7-20)
 * ------------------------------------------------------------------------ */
static void finalize(yo_context* c) {
  if (c->finalized) fail(c, YS_ERR_DECL, "ys_finalize: the engine is already built (ys_finalize)");
  if (c->nt == 0) fail(c, YS_ERR_DECL, "no minimize targets registered");
  int64_t acc = 0, nb = 0, dv = 0;
  for (int t = 0; t < c->nt; ++t) {
    c->t[t].start = acc;
    acc += c->t[t].n * c->t[t].rc;
    nb += c->t[t].n;
    dv += c->t[t].n * c->t[t].rc * c->t[t].rc;
  }
  c->s = acc;
  c->nblk = nb;
  c->diag_vals = dv;
  c->bstart = xcalloc((size_t)nb, sizeof(int64_t));
  c->brc = xcalloc((size_t)nb, sizeof(int));
  c->bvoff = xcalloc((size_t)nb, sizeof(int64_t));
  int64_t b = 0, vo = 0;
  for (int t = 0; t < c->nt; ++t)
    for (int64_t i = 0; i < c->t[t].n; ++i, ++b) {
      c->bstart[b] = c->t[t].start + i * c->t[t].rc;
      c->brc[b] = c->t[t].rc;
      c->bvoff[b] = vo;
      vo += (int64_t)c->t[t].rc * c->t[t].rc;
    }
  c->X = xcalloc((size_t)acc, sizeof(double));
  c->X0 = xcalloc((size_t)acc, sizeof(double));
  c->G = xcalloc((size_t)acc, sizeof(double));
  c->DX = xcalloc((size_t)acc, sizeof(double));
  c->diag = xcalloc((size_t)dv, sizeof(double));
  c->minv = xcalloc((size_t)dv, sizeof(double));
  for (int t = 0; t < c->nt; ++t)
    if (c->t[t].init) memcpy(c->X + c->t[t].start, c->t[t].init, sizeof(double) * c->t[t].n * c->t[t].rc);
  c->finalized = 1;
  build_group(c, 0);
  build_group(c, 1);
  c->seen_epoch = c->epoch;
}

/* ======================================================================== */
/* extern C API                                                             */

#define API_BEGIN(c)                      \
  if (!(c)) return YS_ERR_VALIDATION;      \
  {                                        \
    int st_ = setjmp((c)->jb);             \
    if (st_) return st_;                   \
  }
#define API_END return YS_OK;

static void require_fin(yo_context* c) {
  if (!c->finalized) fail(c, YS_ERR_VALIDATION, "engine not built: call ys_finalize first");
}
static void require_not_fin(yo_context* c, const char* what) {
  if (c->finalized) fail(c, YS_ERR_DECL, "%s: the engine is already built (ys_finalize)", what);
}
static void check_target(yo_context* c, int t, int rc, const char* what) {
  if (t < 0 || t >= c->nt) fail(c, YS_ERR_DECL, "%s: unknown target", what);
  if (rc > 0 && c->t[t].rc != rc) fail(c, YS_ERR_DECL, "%s: target must have %d values per instance", what, rc);
}

int yo_create(yo_context** out, int32_t device) {
  (void)device;
  *out = xcalloc(1, sizeof(yo_context));
  return YS_OK;
}

void yo_destroy(yo_context* c) {
  if (!c) return;
  for (int t = 0; t < c->nt; ++t) free(c->t[t].init);
  free(c->t);
  for (int k = 0; k < c->nd; ++k) {
    free(c->d[k].v2b);
    free(c->d[k].rest);
  }
  free(c->d);
  for (int k = 0; k < c->nu; ++k) free(c->u[k].child);
  free(c->u);
  for (int k = 0; k < c->nps; ++k) free(c->ps[k].pairs);
  free(c->ps);
  for (int k = 0; k < c->ne; ++k) {
    free(c->e[k].conn);
    free(c->e[k].cdata);
    free(c->e[k].anchor);
    free(c->e[k].slots);
    free(c->e[k].plans);
  }
  free(c->e);
  free(c->X); free(c->X0); free(c->G); free(c->DX);
  free(c->bstart); free(c->brc); free(c->bvoff); free(c->diag); free(c->minv);
  bsr_free(&c->H[0]);
  bsr_free(&c->H[1]);
  for (int k = 0; k < c->nsys; ++k) bsr_free(&c->sys[k]);
  free(c->sys);
  free(c->hist);
  free(c);
}

const char* yo_last_error(const yo_context* c) { return c ? c->err : "null context"; }
int yo_last_error_class(const yo_context* c) { return c ? c->err_cls : YS_ERR_VALIDATION; }
const char* yo_version(void) { return "yasps oracle (CPU restatement of relsim)"; }

int yo_add_target(yo_context* c, int64_t n, int32_t rc, int32_t* id) {
  API_BEGIN(c);
  require_not_fin(c, "ys_add_target");
  if (n < 0) fail(c, YS_ERR_DECL, "negative instance count");
  GROW(c->t, c->nt);
  memset(&c->t[c->nt], 0, sizeof(Target));
  c->t[c->nt].n = n;
  c->t[c->nt].rc = rc;
  if (id) *id = c->nt;
  c->nt++;
  API_END;
}

int yo_set_target_values(yo_context* c, int32_t t, const double* v) {
  API_BEGIN(c);
  check_target(c, t, 0, "ys_set_target_values");
  const int64_t n = c->t[t].n * c->t[t].rc;
  if (!c->finalized) {
    free(c->t[t].init);
    c->t[t].init = xcalloc((size_t)n, sizeof(double));
    memcpy(c->t[t].init, v, sizeof(double) * (size_t)n);
  } else {
    memcpy(c->X + c->t[t].start, v, sizeof(double) * (size_t)n);
  }
  API_END;
}

int yo_get_target_values(yo_context* c, int32_t t, double* v) {
  API_BEGIN(c);
  check_target(c, t, 0, "ys_get_target_values");
  const int64_t n = c->t[t].n * c->t[t].rc;
  if (!c->finalized) {
    if (c->t[t].init) memcpy(v, c->t[t].init, sizeof(double) * (size_t)n);
    else memset(v, 0, sizeof(double) * (size_t)n);
  } else {
    memcpy(v, c->X + c->t[t].start, sizeof(double) * (size_t)n);
  }
  API_END;
}

int yo_total_dofs(yo_context* c, int64_t* s) {
  API_BEGIN(c);
  int64_t acc = 0;
  for (int t = 0; t < c->nt; ++t) acc += c->t[t].n * c->t[t].rc;
  *s = acc;
  API_END;
}

int yo_add_points(yo_context* c, int32_t kind, int64_t n, int32_t ta, int32_t tb, const int64_t* v2b,
                  const double* rest, int32_t* id) {
  API_BEGIN(c);
  require_not_fin(c, "ys_add_points");
  Domain d;
  memset(&d, 0, sizeof(d));
  d.kind = kind;
  d.n = n;
  d.ta = -1;
  d.tb = -1;
  if (kind == YS_POINTS_FREE) {
    check_target(c, ta, 3, "free points");
    if (c->t[ta].n != n) fail(c, YS_ERR_DECL, "free points: count differs from the position target");
    d.ta = ta;
  } else if (kind == YS_POINTS_AFFINE) {
    check_target(c, ta, 9, "affine points (affine matrix)");
    check_target(c, tb, 3, "affine points (translation)");
    d.ta = ta;
    d.tb = tb;
    d.v2b = xcalloc((size_t)n, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
      if (v2b[i] < 0 || v2b[i] >= c->t[ta].n)
        fail(c, YS_ERR_VALIDATION, "connectivity 'v2b': index %lld at position %lld out of range [0, %lld)",
             (long long)v2b[i], (long long)i, (long long)c->t[ta].n);
      d.v2b[i] = v2b[i];
    }
    d.rest = xcalloc((size_t)(3 * n), sizeof(double));
    memcpy(d.rest, rest, sizeof(double) * (size_t)(3 * n));
  } else if (kind == YS_POINTS_FIXED) {
    d.rest = xcalloc((size_t)(3 * n), sizeof(double));
    memcpy(d.rest, rest, sizeof(double) * (size_t)(3 * n));
  } else {
    fail(c, YS_ERR_DECL, "unknown point-domain kind");
  }
  GROW(c->d, c->nd);
  c->d[c->nd] = d;
  *id = c->nd++;
  API_END;
}

int yo_get_points(yo_context* c, int32_t dom, double* out) {
  API_BEGIN(c);
  require_fin(c);
  if (dom < 0 || dom >= c->nd) fail(c, YS_ERR_DECL, "unknown point domain");
  for (int64_t i = 0; i < c->d[dom].n; ++i) point_value(c, &c->d[dom], i, c->X, out + 3 * i);
  API_END;
}

int yo_add_point_union(yo_context* c, int32_t n, const int32_t* doms, int32_t* id) {
  API_BEGIN(c);
  require_not_fin(c, "ys_add_point_union");
  if (n < 1) fail(c, YS_ERR_DECL, "primitive union needs at least one child");
  Union u;
  u.nchild = n;
  u.child = xcalloc((size_t)n, sizeof(int));
  u.kappa_u = 0;
  u.width = 0;
  for (int k = 0; k < n; ++k) {
    if (doms[k] < 0 || doms[k] >= c->nd) fail(c, YS_ERR_DECL, "unknown point domain");
    u.child[k] = doms[k];
    if (dom_kappa(&c->d[doms[k]]) > u.kappa_u) u.kappa_u = dom_kappa(&c->d[doms[k]]);
    if (dom_width(&c->d[doms[k]]) > u.width) u.width = dom_width(&c->d[doms[k]]);
  }
  GROW(c->u, c->nu);
  c->u[c->nu] = u;
  *id = c->nu++;
  API_END;
}

int yo_add_stencil_set(yo_context* c, int32_t uni, int32_t arity, int32_t dynamic, int32_t* id) {
  API_BEGIN(c);
  require_not_fin(c, "ys_add_stencil_set");
  if (uni < 0 || uni >= c->nu) fail(c, YS_ERR_DECL, "unknown primitive union");
  if (arity < 2 || arity > 4) fail(c, YS_ERR_DECL, "stencil arity must be 2, 3 or 4");
  GROW(c->ps, c->nps);
  memset(&c->ps[c->nps], 0, sizeof(PairSet));
  c->ps[c->nps].uni = uni;
  c->ps[c->nps].arity = arity;
  c->ps[c->nps].dynamic = dynamic != 0;
  *id = c->nps++;
  API_END;
}

/* Contact candidates of the PT / EE / PE barriers (not in the reference; its
 * candidates are point-point only, sim.cpp:456-484): the all-pairs loop that
 * specifies the B200 grid search (ys_stencil.cu).  Every (a, b) (EE: b > a)
 * sharing no point, not all points fixed, with the squared distance of its
 * distance type strictly below dhat, in (a, b) order. */
int yo_set_stencil_primitives(yo_context* c, int32_t set, int32_t kind, int64_t n_a, const int64_t* prims_a,
                              int64_t n_b, const int64_t* prims_b) {
  API_BEGIN(c);
  if (set < 0 || set >= c->nps) fail(c, YS_ERR_DECL, "unknown stencil set");
  PairSet* p = &c->ps[set];
  if (kind < 1 || kind > 3) fail(c, YS_ERR_VALIDATION, "stencil kind must be 1 (PT), 2 (EE) or 3 (PE)");
  const int aa = kind == 2 ? 2 : 1, ab = kind == 1 ? 3 : 2;
  if (aa + ab != p->arity) fail(c, YS_ERR_DECL, "stencil kind does not match the set's arity");
  if (kind == 2) n_b = 0;
  free(p->pa);
  free(p->pb);
  p->pa = xcalloc((size_t)(n_a * aa), sizeof(int64_t));
  p->pb = xcalloc((size_t)(n_b * ab), sizeof(int64_t));
  memcpy(p->pa, prims_a, sizeof(int64_t) * (size_t)(n_a * aa));
  if (n_b) memcpy(p->pb, prims_b, sizeof(int64_t) * (size_t)(n_b * ab));
  p->pkind = kind;
  p->aa = aa;
  p->ab = ab;
  p->na = n_a;
  p->nb = n_b;
  API_END;
}

int yo_refresh_stencils(yo_context* c, int32_t set, double dhat, int64_t* out_n) {
  API_BEGIN(c);
  require_fin(c);
  if (set < 0 || set >= c->nps) fail(c, YS_ERR_DECL, "unknown stencil set");
  PairSet* p = &c->ps[set];
  if (!p->pkind) fail(c, YS_ERR_VALIDATION, "stencil set has no primitives (ys_set_stencil_primitives)");
  const Union* u = &c->u[p->uni];
  int64_t total = 0;
  for (int k = 0; k < u->nchild; ++k) total += c->d[u->child[k]].n;
  double* pts = xcalloc((size_t)(3 * total), sizeof(double));
  char* fixed = xcalloc((size_t)total, 1);
  int64_t acc = 0;
  for (int k = 0; k < u->nchild; ++k) {
    const Domain* d = &c->d[u->child[k]];
    for (int64_t i = 0; i < d->n; ++i) {
      point_value(c, d, i, c->X, pts + 3 * (acc + i));
      fixed[acc + i] = d->kind == YS_POINTS_FIXED;
    }
    acc += d->n;
  }
  const int self = p->pkind == 2, ar = p->aa + p->ab;
  const int kind = p->pkind == 1 ? K_PT : p->pkind == 2 ? K_EE : K_PE;
  const int64_t* B = self ? p->pa : p->pb;
  const int64_t nb = self ? p->na : p->nb;
  const int abb = self ? p->aa : p->ab;
  int64_t cnt = 0, cap = 256;
  int64_t* idx = xcalloc((size_t)(ar * cap), sizeof(int64_t));
  for (int64_t a = 0; a < p->na; ++a)
    for (int64_t b = self ? a + 1 : 0; b < nb; ++b) {
      int64_t st[4];
      int shared = 0, allfixed = 1;
      for (int i = 0; i < p->aa; ++i) st[i] = p->pa[p->aa * a + i];
      for (int j = 0; j < abb; ++j) st[p->aa + j] = B[abb * b + j];
      for (int i = 0; i < p->aa; ++i)
        for (int j = 0; j < abb; ++j) shared |= st[i] == st[p->aa + j];
      if (shared) continue;
      for (int l = 0; l < ar; ++l) allfixed &= fixed[st[l]];
      if (allfixed) continue;
      double x[4][3];
      for (int l = 0; l < ar; ++l)
        for (int k = 0; k < 3; ++k) x[l][k] = pts[3 * st[l] + k];
      const ContactSel sel = kind == K_PT ? classify_pt(x) : kind == K_EE ? classify_ee(x) : classify_pe(x);
      if (!(contact_dist2_value(sel, x) < dhat)) continue;
      if (cnt == cap) {
        cap *= 2;
        idx = realloc(idx, sizeof(int64_t) * (size_t)(ar * cap));
      }
      for (int l = 0; l < ar; ++l) idx[ar * cnt + l] = st[l];
      ++cnt;
    }
  free(p->pairs);
  p->pairs = idx;
  p->n = cnt;
  c->epoch++;
  free(pts);
  free(fixed);
  if (out_n) *out_n = cnt;
  API_END;
}

int yo_add_pair_set(yo_context* c, int32_t uni, int32_t dynamic, int32_t* id) {
  return yo_add_stencil_set(c, uni, 2, dynamic, id);
}

int yo_set_pairs(yo_context* c, int32_t ps, int64_t n, const int64_t* pairs) {
  API_BEGIN(c);
  if (ps < 0 || ps >= c->nps) fail(c, YS_ERR_DECL, "unknown pair set");
  PairSet* p = &c->ps[ps];
  if (!p->dynamic && c->finalized) fail(c, YS_ERR_VALIDATION, "resize_dynamic on static primitive contact.pp");
  if (n < 0) fail(c, YS_ERR_VALIDATION, "negative instance count");
  int64_t total = 0;
  for (int k = 0; k < c->u[p->uni].nchild; ++k) total += c->d[c->u[p->uni].child[k]].n;
  for (int64_t k = 0; k < p->arity * n; ++k)
    if (pairs[k] < 0 || pairs[k] >= total)
      fail(c, YS_ERR_VALIDATION, "connectivity 'pp2v': index %lld at position %lld out of range [0, %lld)",
           (long long)pairs[k], (long long)k, (long long)total);
  free(p->pairs);
  p->pairs = xcalloc((size_t)(p->arity * n), sizeof(int64_t));
  memcpy(p->pairs, pairs, sizeof(int64_t) * (size_t)(p->arity * n));
  p->n = n;
  c->epoch++;
  API_END;
}

int yo_pair_count(yo_context* c, int32_t ps, int64_t* n) {
  API_BEGIN(c);
  if (ps < 0 || ps >= c->nps) fail(c, YS_ERR_DECL, "unknown pair set");
  *n = c->ps[ps].n;
  API_END;
}

int yo_get_pairs(yo_context* c, int32_t ps, int64_t* out) {
  API_BEGIN(c);
  if (ps < 0 || ps >= c->nps) fail(c, YS_ERR_DECL, "unknown pair set");
  memcpy(out, c->ps[ps].pairs, sizeof(int64_t) * (size_t)(c->ps[ps].arity * c->ps[ps].n));
  API_END;
}

/* Simulation::refresh_dynamic_pairs (sim.cpp:456-484) */
int yo_refresh_pairs(yo_context* c, int32_t ps, double dhat, const int32_t* child_fixed, int64_t* out_n) {
  API_BEGIN(c);
  require_fin(c);
  if (ps < 0 || ps >= c->nps) fail(c, YS_ERR_DECL, "unknown pair set");
  PairSet* p = &c->ps[ps];
  if (p->arity != 2) fail(c, YS_ERR_DECL, "ys_refresh_pairs: point-point pair sets only");
  const Union* u = &c->u[p->uni];
  int64_t total = 0;
  for (int k = 0; k < u->nchild; ++k) total += c->d[u->child[k]].n;
  double* pts = xcalloc((size_t)(3 * total), sizeof(double));
  int64_t* base = xcalloc((size_t)u->nchild, sizeof(int64_t));
  int64_t acc = 0;
  for (int k = 0; k < u->nchild; ++k) {
    base[k] = acc;
    for (int64_t i = 0; i < c->d[u->child[k]].n; ++i) point_value(c, &c->d[u->child[k]], i, c->X, pts + 3 * (acc + i));
    acc += c->d[u->child[k]].n;
  }
  int64_t cnt = 0, cap = 1024;
  int64_t* idx = xcalloc((size_t)(2 * cap), sizeof(int64_t));
  for (int ca = 0; ca < u->nchild; ++ca)
    for (int cb = ca + 1; cb < u->nchild; ++cb) {
      const int fa = child_fixed ? child_fixed[ca] != 0 : c->d[u->child[ca]].kind == YS_POINTS_FIXED;
      const int fb = child_fixed ? child_fixed[cb] != 0 : c->d[u->child[cb]].kind == YS_POINTS_FIXED;
      if (fa && fb) continue;
      for (int64_t i = 0; i < c->d[u->child[ca]].n; ++i)
        for (int64_t j = 0; j < c->d[u->child[cb]].n; ++j) {
          const double* a = pts + 3 * (base[ca] + i);
          const double* b = pts + 3 * (base[cb] + j);
          const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
          const double d2 = (dx * dx + dy * dy) + dz * dz;
          if (d2 < dhat) {
            if (cnt == cap) {
              cap *= 2;
              idx = realloc(idx, sizeof(int64_t) * (size_t)(2 * cap));
            }
            idx[2 * cnt] = base[ca] + i;
            idx[2 * cnt + 1] = base[cb] + j;
            ++cnt;
          }
        }
    }
  free(p->pairs);
  p->pairs = idx;
  p->n = cnt;
  c->epoch++;
  free(pts);
  free(base);
  if (out_n) *out_n = cnt;
  API_END;
}

static int add_energy(yo_context* c, Energy* e) {
  GROW(c->e, c->ne);
  c->e[c->ne] = *e;
  return c->ne++;
}

int yo_add_stable_neo_hookean(yo_context* c, int32_t pos, int64_t nt, const int64_t* t2v, const double* rest,
                              double E, double nu, double weight, int32_t via_f, int32_t* id) {
  API_BEGIN(c);
  require_not_fin(c, "add_stable_neo_hookean");
  check_target(c, pos, 3, "stable Neo-Hookean positions");
  Energy e;
  memset(&e, 0, sizeof(e));
  e.kind = K_SNH;
  e.n = nt;
  e.kappa = 4;
  e.width = 12;
  e.target = pos;
  e.domain = e.pairset = -1;
  e.mode = via_f ? YS_PROJECT_REDUCED : YS_PROJECT_FULL;
  const double mu = E / (2.0 * (1.0 + nu));
  const double lambda = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  e.prm[0] = mu;
  e.prm[1] = lambda;
  e.prm[2] = 1.0 + 3.0 * mu / (4.0 * lambda);
  e.prm[3] = weight;
  e.conn = xcalloc((size_t)(4 * nt), sizeof(int64_t));
  e.cdata = xcalloc((size_t)(10 * nt), sizeof(double));
  for (int64_t t = 0; t < nt; ++t) {
    for (int l = 0; l < 4; ++l) {
      if (t2v[4 * t + l] < 0 || t2v[4 * t + l] >= c->t[pos].n)
        fail(c, YS_ERR_VALIDATION, "connectivity 'tet2v': index %lld at position %lld out of range [0, %lld)",
             (long long)t2v[4 * t + l], (long long)(4 * t + l), (long long)c->t[pos].n);
      e.conn[4 * t + l] = t2v[4 * t + l];
    }
    double fr[9];
    const int64_t i0 = t2v[4 * t];
    for (int col = 0; col < 3; ++col) {
      const int64_t ic = t2v[4 * t + col + 1];
      for (int r = 0; r < 3; ++r) fr[3 * r + col] = rest[ic * 3 + r] - rest[i0 * 3 + r];
    }
    const double det = fr[0] * (fr[4] * fr[8] - fr[5] * fr[7]) - fr[1] * (fr[3] * fr[8] - fr[5] * fr[6]) +
                       fr[2] * (fr[3] * fr[7] - fr[4] * fr[6]);
    if (fabs(det) < 1e-14) fail(c, YS_ERR_VALIDATION, "degenerate rest tetrahedron %lld", (long long)t);
    /* Binv = (fr^T)^-1 via the adjugate */
    double b[9], inv[9];
    for (int r = 0; r < 3; ++r)
      for (int col = 0; col < 3; ++col) b[3 * r + col] = fr[3 * col + r];
    lu_inverse(b, 3, inv);
    for (int k = 0; k < 9; ++k) e.cdata[10 * t + k] = inv[k];
    e.cdata[10 * t + 9] = fabs(det) / 6.0;
  }
  *id = add_energy(c, &e);
  API_END;
}

int yo_add_bending(yo_context* c, int32_t pos, int64_t nh, const int64_t* h2v, const double* rest, double k,
                   double weight, int32_t* id) {
  API_BEGIN(c);
  require_not_fin(c, "add_bending");
  check_target(c, pos, 3, "bending positions");
  Energy e;
  memset(&e, 0, sizeof(e));
  e.kind = K_BENDING;
  e.n = nh;
  e.kappa = 4;
  e.width = 12;
  e.target = pos;
  e.domain = e.pairset = -1;
  e.conn = xcalloc((size_t)(4 * nh), sizeof(int64_t));
  e.cdata = xcalloc((size_t)nh, sizeof(double));
  for (int64_t h = 0; h < nh; ++h) {
    for (int l = 0; l < 4; ++l) e.conn[4 * h + l] = h2v[4 * h + l];
    const int64_t a = h2v[4 * h], bb = h2v[4 * h + 1];
    double acc = 0.0;
    for (int d = 0; d < 3; ++d) {
      const double diff = rest[a * 3 + d] - rest[bb * 3 + d];
      acc += diff * diff;
    }
    e.cdata[h] = (k * weight) * sqrt(acc);
  }
  *id = add_energy(c, &e);
  API_END;
}

int yo_add_inertia(yo_context* c, int32_t dom, const double* mass, const double* xt, int32_t* id) {
  API_BEGIN(c);
  require_not_fin(c, "add_inertia");
  if (dom < 0 || dom >= c->nd) fail(c, YS_ERR_DECL, "unknown point domain");
  Energy e;
  memset(&e, 0, sizeof(e));
  e.kind = K_INERTIA;
  e.n = c->d[dom].n;
  e.kappa = dom_kappa(&c->d[dom]);
  e.width = dom_width(&c->d[dom]);
  e.domain = dom;
  e.target = e.pairset = -1;
  e.cdata = xcalloc((size_t)e.n, sizeof(double));
  e.anchor = xcalloc((size_t)(3 * e.n), sizeof(double));
  memcpy(e.cdata, mass, sizeof(double) * (size_t)e.n);
  memcpy(e.anchor, xt, sizeof(double) * (size_t)(3 * e.n));
  *id = add_energy(c, &e);
  API_END;
}

int yo_set_inertia_anchor(yo_context* c, int32_t id, const double* xt) {
  API_BEGIN(c);
  if (id < 0 || id >= c->ne || c->e[id].kind != K_INERTIA) fail(c, YS_ERR_DECL, "ys_set_inertia_anchor: not an inertia energy");
  memcpy(c->e[id].anchor, xt, sizeof(double) * (size_t)(3 * c->e[id].n));
  API_END;
}

int yo_add_affine_orthogonality(yo_context* c, int32_t amat, double k, double weight, int32_t* id) {
  API_BEGIN(c);
  require_not_fin(c, "add_affine_orthogonality");
  check_target(c, amat, 9, "affine orthogonality");
  Energy e;
  memset(&e, 0, sizeof(e));
  e.kind = K_ORTHO;
  e.n = c->t[amat].n;
  e.kappa = 1;
  e.width = 9;
  e.target = amat;
  e.domain = e.pairset = -1;
  e.prm[0] = k * weight;
  *id = add_energy(c, &e);
  API_END;
}

static int add_pair(yo_context* c, int kind, int32_t ps, double dhat, double kappa, double weight, int32_t mode,
                    int32_t* id) {
  API_BEGIN(c);
  require_not_fin(c, kind == K_PP ? "add_point_point_barrier" : "add_repulsive_energy");
  if (ps < 0 || ps >= c->nps) fail(c, YS_ERR_DECL, "unknown pair set");
  const Union* u = &c->u[c->ps[ps].uni];
  Energy e;
  memset(&e, 0, sizeof(e));
  e.kind = kind;
  e.dynamic = c->ps[ps].dynamic;
  e.mode = mode;
  e.pairset = ps;
  e.target = e.domain = -1;
  e.n = c->ps[ps].n;
  e.kappa = 2 * u->kappa_u;
  e.width = 2 * u->width;
  e.prm[0] = dhat;
  e.prm[1] = kappa;
  e.prm[2] = weight;
  *id = add_energy(c, &e);
  API_END;
}

static int add_contact(yo_context* c, int kind, int32_t ps, double dhat, double kappa, double weight, int32_t* id) {
  API_BEGIN(c);
  require_not_fin(c, kind == K_PT ? "point_triangle" : kind == K_EE ? "edge_edge" : "point_edge");
  if (ps < 0 || ps >= c->nps) fail(c, YS_ERR_DECL, "unknown stencil set");
  const int want = kind == K_PE ? 3 : 4;
  const char* nm = kind == K_PT ? "point_triangle" : kind == K_EE ? "edge_edge" : "point_edge";
  if (c->ps[ps].arity != want) fail(c, YS_ERR_DECL, "%s needs a stencil set of arity %d", nm, want);
  const Union* u = &c->u[c->ps[ps].uni];
  if (u->kappa_u != 1) fail(c, YS_ERR_DECL, "%s: unions of free and fixed points only", nm);
  if (!(dhat > 0.0)) fail(c, YS_ERR_VALIDATION, "dhat must be positive");
  Energy e;
  memset(&e, 0, sizeof(e));
  e.kind = kind;
  e.dynamic = c->ps[ps].dynamic;
  e.mode = YS_PROJECT_FULL;
  e.pairset = ps;
  e.target = e.domain = -1;
  e.n = c->ps[ps].n;
  e.kappa = want;
  e.width = 3 * want;
  e.prm[0] = dhat;
  e.prm[1] = kappa;
  e.prm[2] = weight;
  *id = add_energy(c, &e);
  API_END;
}

int yo_add_point_triangle_barrier(yo_context* c, int32_t ps, double dhat, double kappa, double weight, int32_t* id) {
  return add_contact(c, K_PT, ps, dhat, kappa, weight, id);
}
int yo_add_edge_edge_barrier(yo_context* c, int32_t ps, double dhat, double kappa, double weight, int32_t* id) {
  return add_contact(c, K_EE, ps, dhat, kappa, weight, id);
}
int yo_add_point_edge_barrier(yo_context* c, int32_t ps, double dhat, double kappa, double weight, int32_t* id) {
  return add_contact(c, K_PE, ps, dhat, kappa, weight, id);
}

int yo_add_point_point_barrier(yo_context* c, int32_t ps, double dhat, double kappa, double weight, int32_t mode,
                               int32_t* id) {
  return add_pair(c, K_PP, ps, dhat, kappa, weight, mode, id);
}
int yo_add_repulsive(yo_context* c, int32_t ps, double weight, int32_t mode, int32_t* id) {
  return add_pair(c, K_REPULSIVE, ps, 0.0, 0.0, weight, mode, id);
}

int yo_finalize(yo_context* c) {
  API_BEGIN(c);
  finalize(c);
  API_END;
}

int yo_refresh_dynamic(yo_context* c) {
  API_BEGIN(c);
  require_fin(c);
  if (c->seen_epoch != c->epoch) {
    build_group(c, 1);
    c->seen_epoch = c->epoch;
  }
  API_END;
}

int yo_dynamic_stale(yo_context* c, int32_t* st) {
  API_BEGIN(c);
  *st = c->seen_epoch != c->epoch;
  API_END;
}

int yo_assemble(yo_context* c, int32_t project, int32_t with_h) {
  API_BEGIN(c);
  require_fin(c);
  assemble(c, project, with_h);
  API_END;
}

int yo_get_gradient(yo_context* c, double* g) {
  API_BEGIN(c);
  require_fin(c);
  memcpy(g, c->G, sizeof(double) * (size_t)c->s);
  API_END;
}

/* Engine::total_energy (engine.cpp:64-68): serial per energy, then across */
static double total_energy(yo_context* c, double* per) {
  double sum = 0.0;
  JC = c;
  for (int ei = 0; ei < c->ne; ++ei) {
    const Energy* e = &c->e[ei];
    const int64_t n = energy_count(c, e);
    double t = 0.0;
    for (int64_t i = 0; i < n; ++i) t += local_energy(c, e, i, c->X);
    if (per) per[ei] = t;
    sum += t;
  }
  return sum;
}

int yo_total_energy(yo_context* c, double* e) {
  API_BEGIN(c);
  require_fin(c);
  *e = total_energy(c, NULL);
  API_END;
}

int yo_energy_totals(yo_context* c, double* t) {
  API_BEGIN(c);
  require_fin(c);
  total_energy(c, t);
  API_END;
}

int yo_apply_hessian(yo_context* c, const double* x, double* y) {
  API_BEGIN(c);
  require_fin(c);
  spmv_add(&c->H[0], x, y);
  spmv_add(&c->H[1], x, y);
  API_END;
}

int yo_minimize_step(yo_context* c, double tol, int64_t max_iter, double* dx, ys_step_stats* stats) {
  API_BEGIN(c);
  require_fin(c);
  if (c->seen_epoch != c->epoch) {
    build_group(c, 1);
    c->seen_epoch = c->epoch;
  }
  assemble(c, 1, 1);
  build_precond(c);
  if (max_iter < 0) max_iter = 2 * c->s > 64 ? 2 * c->s : 64;
  int64_t it;
  double rel;
  int conv;
  if (c->dist_on) dist_pcg(c, tol, max_iter, c->DX, &it, &rel, &conv);
  else pcg(c, &c->H[0], &c->H[1], c->G, tol, max_iter, c->DX, &it, &rel, &conv);
  memcpy(c->X0, c->X, sizeof(double) * (size_t)c->s);
  if (dx) memcpy(dx, c->DX, sizeof(double) * (size_t)c->s);
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    stats->pcg_iterations = it;
    stats->pcg_residual = rel;
    stats->pcg_converged = conv;
    stats->regularized_blocks = c->regularized;
  }
  API_END;
}

int yo_pcg_history(yo_context* c, int64_t cap, double* h, int64_t* count) {
  API_BEGIN(c);
  const int64_t n = cap < c->hist_n ? cap : c->hist_n;
  if (n > 0) memcpy(h, c->hist, sizeof(double) * (size_t)n);
  *count = c->hist_n;
  API_END;
}

int yo_gather_targets(yo_context* c, double* x) {
  API_BEGIN(c);
  require_fin(c);
  memcpy(x, c->X, sizeof(double) * (size_t)c->s);
  API_END;
}

int yo_scatter_targets(yo_context* c, const double* x) {
  API_BEGIN(c);
  require_fin(c);
  memcpy(c->X, x, sizeof(double) * (size_t)c->s);
  API_END;
}

int yo_step_targets(yo_context* c, double alpha, double* max_abs) {
  API_BEGIN(c);
  require_fin(c);
  double m = 0.0;
  for (int64_t i = 0; i < c->s; ++i) {
    const double ad = alpha * c->DX[i];
    c->X[i] = c->X0[i] - ad;
    if (fabs(ad) > m) m = fabs(ad);
  }
  if (max_abs) *max_abs = m;
  API_END;
}

static Bsr* which_h(yo_context* c, int32_t w) { return &c->H[w ? 1 : 0]; }

int yo_hessian_info(yo_context* c, int32_t w, int64_t* ng, int64_t* nb, int64_t* nv, uint64_t* cs) {
  API_BEGIN(c);
  require_fin(c);
  Bsr* h = which_h(c, w);
  if (ng) *ng = h->ng;
  if (nb) *nb = h->nb;
  if (nv) *nv = h->nv;
  if (cs) *cs = structure_checksum(h);
  API_END;
}

int yo_hessian_groups(yo_context* c, int32_t w, int64_t* g) {
  API_BEGIN(c);
  Bsr* h = which_h(c, w);
  for (int k = 0; k < h->ng; ++k) {
    g[5 * k] = h->groups[k].rows;
    g[5 * k + 1] = h->groups[k].cols;
    g[5 * k + 2] = h->groups[k].coord_start;
    g[5 * k + 3] = h->groups[k].count;
    g[5 * k + 4] = h->groups[k].value_start;
  }
  API_END;
}

int yo_hessian_coords(yo_context* c, int32_t w, int64_t* row, int64_t* col) {
  API_BEGIN(c);
  Bsr* h = which_h(c, w);
  memcpy(row, h->row, sizeof(int64_t) * (size_t)h->nb);
  memcpy(col, h->col, sizeof(int64_t) * (size_t)h->nb);
  API_END;
}

int yo_hessian_values(yo_context* c, int32_t w, double* v) {
  API_BEGIN(c);
  Bsr* h = which_h(c, w);
  memcpy(v, h->values, sizeof(double) * (size_t)h->nv);
  API_END;
}

int yo_energy_info(yo_context* c, int32_t id, int64_t* n, int32_t* kappa, int32_t* width, int32_t* dyn) {
  API_BEGIN(c);
  if (id < 0 || id >= c->ne) fail(c, YS_ERR_DECL, "unknown energy");
  if (n) *n = energy_count(c, &c->e[id]);
  if (kappa) *kappa = c->e[id].kappa;
  if (width) *width = c->e[id].width;
  if (dyn) *dyn = c->e[id].dynamic;
  API_END;
}

int yo_energy_slots(yo_context* c, int32_t id, int64_t* index, int32_t* len, int32_t* col) {
  API_BEGIN(c);
  require_fin(c);
  if (id < 0 || id >= c->ne) fail(c, YS_ERR_DECL, "unknown energy");
  const Energy* e = &c->e[id];
  for (int64_t k = 0; k < e->nplans * e->kappa; ++k) {
    index[k] = e->slots[k].index;
    len[k] = e->slots[k].len;
    col[k] = e->slots[k].col;
  }
  API_END;
}

int yo_energy_compressed_sizes(yo_context* c, int32_t id, int32_t* m) {
  API_BEGIN(c);
  require_fin(c);
  if (id < 0 || id >= c->ne) fail(c, YS_ERR_DECL, "unknown energy");
  for (int64_t i = 0; i < c->e[id].nplans; ++i) m[i] = c->e[id].plans[i].m;
  API_END;
}

int yo_diag_blocks(yo_context* c, double* out) {
  API_BEGIN(c);
  require_fin(c);
  memcpy(out, c->diag, sizeof(double) * (size_t)c->diag_vals);
  API_END;
}

int yo_bump_dynamic_epoch(yo_context* c) {
  API_BEGIN(c);
  c->epoch++;
  API_END;
}

int yo_stream(yo_context* c, void** stream) {
  API_BEGIN(c);
  *stream = NULL;
  API_END;
}

/* Execution options (ys_set_option): the oracle is sequential, "overlap" has no effect. */
int yo_set_option(yo_context* c, const char* name, int64_t value) {
  API_BEGIN(c);
  (void)value;
  if (!name || strcmp(name, "overlap") != 0) fail(c, YS_ERR_VALIDATION, "unknown option '%s'", name ? name : "");
  API_END;
}

/* --- free-standing BSR ---------------------------------------------------- */
int yo_bsr_build(yo_context* c, int64_t s, int64_t n, const int64_t* coords, int32_t* id) {
  API_BEGIN(c);
  Coord* q = xcalloc((size_t)n, sizeof(Coord));
  for (int64_t k = 0; k < n; ++k) {
    q[k].rows = (int)coords[4 * k];
    q[k].cols = (int)coords[4 * k + 1];
    q[k].row = coords[4 * k + 2];
    q[k].col = coords[4 * k + 3];
  }
  GROW(c->sys, c->nsys);
  memset(&c->sys[c->nsys], 0, sizeof(Bsr));
  bsr_build(c, &c->sys[c->nsys], q, n, s);
  free(q);
  *id = c->nsys++;
  API_END;
}

static Bsr* sys_of(yo_context* c, int32_t id) {
  if (id < 0 || id >= c->nsys) fail(c, YS_ERR_DECL, "unknown BSR system");
  return &c->sys[id];
}

int yo_bsr_info(yo_context* c, int32_t id, int64_t* ng, int64_t* nb, int64_t* nv, uint64_t* cs) {
  API_BEGIN(c);
  Bsr* h = sys_of(c, id);
  if (ng) *ng = h->ng;
  if (nb) *nb = h->nb;
  if (nv) *nv = h->nv;
  if (cs) *cs = structure_checksum(h);
  API_END;
}

int yo_bsr_groups(yo_context* c, int32_t id, int64_t* g) {
  API_BEGIN(c);
  Bsr* h = sys_of(c, id);
  for (int k = 0; k < h->ng; ++k) {
    g[5 * k] = h->groups[k].rows;
    g[5 * k + 1] = h->groups[k].cols;
    g[5 * k + 2] = h->groups[k].coord_start;
    g[5 * k + 3] = h->groups[k].count;
    g[5 * k + 4] = h->groups[k].value_start;
  }
  API_END;
}

int yo_bsr_coords(yo_context* c, int32_t id, int64_t* row, int64_t* col) {
  API_BEGIN(c);
  Bsr* h = sys_of(c, id);
  memcpy(row, h->row, sizeof(int64_t) * (size_t)h->nb);
  memcpy(col, h->col, sizeof(int64_t) * (size_t)h->nb);
  API_END;
}

int yo_bsr_set_values(yo_context* c, int32_t id, const double* v) {
  API_BEGIN(c);
  Bsr* h = sys_of(c, id);
  memcpy(h->values, v, sizeof(double) * (size_t)h->nv);
  API_END;
}

int yo_bsr_spmv(yo_context* c, int32_t id, const double* x, double* y) {
  API_BEGIN(c);
  spmv_add(sys_of(c, id), x, y);
  API_END;
}

int yo_bsr_pcg(yo_context* c, int32_t id, int32_t bs, const double* g, double tol, int64_t max_iter, double* x,
               int64_t* iters, double* rel, int32_t* conv) {
  API_BEGIN(c);
  Bsr* h = sys_of(c, id);
  /* block layout of the system: uniform square blocks of the first group */
  const int b = h->ng ? (int)h->groups[0].rows : 3;
  const int m = bs ? bs : b;
  yo_context* sc = xcalloc(1, sizeof(yo_context));
  sc->s = h->s;
  sc->nblk = h->s / m;
  sc->bstart = xcalloc((size_t)sc->nblk, sizeof(int64_t));
  sc->brc = xcalloc((size_t)sc->nblk, sizeof(int));
  sc->bvoff = xcalloc((size_t)sc->nblk, sizeof(int64_t));
  sc->diag_vals = sc->nblk * m * m;
  sc->diag = xcalloc((size_t)sc->diag_vals, sizeof(double));
  sc->minv = xcalloc((size_t)sc->diag_vals, sizeof(double));
  for (int64_t k = 0; k < sc->nblk; ++k) {
    sc->bstart[k] = k * m;
    sc->brc[k] = m;
    sc->bvoff[k] = k * m * m;
  }
  int st = setjmp(sc->jb);
  if (st) {
    snprintf(c->err, sizeof(c->err), "%s", sc->err);
    c->err_cls = st;
    return st;
  }
  if (bs == 0) {
    for (int64_t k = 0; k < sc->nblk; ++k)
      for (int q = 0; q < m * m; ++q) sc->minv[k * m * m + q] = q % (m + 1) == 0 ? 1.0 : 0.0;
  } else {
    /* diagonal blocks of the system itself */
    for (int gi = 0; gi < h->ng; ++gi)
      for (int64_t k = 0; k < h->groups[gi].count; ++k) {
        const int64_t bi = h->groups[gi].coord_start + k;
        if (h->row[bi] != h->col[bi]) continue;
        double* d = sc->diag + (h->row[bi] / m) * m * m;
        for (int q = 0; q < m * m; ++q) d[q] += h->values[h->voff[bi] + q];
      }
    build_precond(sc);
  }
  int64_t it;
  double rr;
  int cv;
  pcg(sc, h, NULL, g, tol, max_iter, x, &it, &rr, &cv);
  free(sc->bstart); free(sc->brc); free(sc->bvoff); free(sc->diag); free(sc->minv); free(sc->hist);
  free(sc);
  if (iters) *iters = it;
  if (rel) *rel = rr;
  if (conv) *conv = cv;
  API_END;
}

/* multi-rank solve entry points (ys_dist_init_host / finalize / info) */
int yo_dist_init_host(yo_context* c, int32_t rank, int32_t nranks, ys_allgather_fn fn, void* user) {
  API_BEGIN(c);
  if (nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks)
    fail(c, YS_ERR_VALIDATION, "distributed solve: rank %d of %d is out of range (1..64 ranks)", rank, nranks);
  if (!fn) fail(c, YS_ERR_VALIDATION, "distributed solve: null allgather callback");
  c->dist_on = 1;
  c->dist_rank = rank;
  c->dist_n = nranks;
  c->dist_fn = fn;
  c->dist_user = user;
  c->dist_bounds[0] = 0;
  c->dist_bounds[1] = c->nblk;
  memset(c->dist_exp_off, 0, sizeof(c->dist_exp_off));
  API_END;
}

int yo_dist_finalize(yo_context* c) {
  API_BEGIN(c);
  c->dist_on = 0;
  API_END;
}

/* The oracle evaluates every instance on every rank (the device evaluates
 * only the instances touching its rows; the solve is the same). */
int yo_dist_eval_counts(yo_context* c, int64_t* evaluated, int64_t* total) {
  API_BEGIN(c);
  int64_t all = 0;
  for (int ei = 0; ei < c->ne; ++ei)
    if (!c->e[ei].dynamic && (c->e[ei].kind == K_SNH || c->e[ei].kind == K_BENDING)) all += c->e[ei].n;
  if (evaluated) *evaluated = all;
  if (total) *total = all;
  API_END;
}

int yo_dist_info(yo_context* c, int32_t* rank, int32_t* nranks, int64_t* bounds, int64_t* halo_rows,
                 int64_t* export_rows) {
  API_BEGIN(c);
  const int n = c->dist_on ? c->dist_n : 1;
  if (rank) *rank = c->dist_on ? c->dist_rank : 0;
  if (nranks) *nranks = n;
  if (bounds) {
    if (c->dist_on) memcpy(bounds, c->dist_bounds, sizeof(int64_t) * (size_t)(n + 1));
    else {
      bounds[0] = 0;
      bounds[1] = c->nblk;
    }
  }
  const int64_t mine = c->dist_on ? c->dist_exp_off[c->dist_rank + 1] - c->dist_exp_off[c->dist_rank] : 0;
  if (halo_rows) *halo_rows = c->dist_on ? c->dist_exp_off[n] - mine : 0;
  if (export_rows) *export_rows = mine;
  API_END;
}
