/* oracle.c — plain, slow, sequential CPU oracle for the hpar hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2309_01906_b200/); it includes only libc headers.
 *
 * What it computes:
 *   1. Results by their plain definition, sequential over ascending i
 *      ("directive-erased sequential execution"):
 *        sum int32 -> int64 (two's complement wrap), sum fp32 -> fp64,
 *        min / max, 256-bin histogram of bytes, row sums, segment sums.
 *   2. The partition of the iteration space by a nest, step by step:
 *      a child task's local list is the subset of its parent's local list
 *      chosen by own(schedule, n, T, child)
 *      applied level by level, outermost first, each level refining only
 *      the loop it is bound to                   (PAPER P:211-225 bind_ancestor).
 *      dynamic(c) is modelled as round-robin static(c) ("claimed ...
 *      in trace-deterministic round-robin order").
 *   3. Per-level partials: leaf partial = fold over its owned iterations in
 *      execution order; parent partial = fold of its children's partials in
 *      ascending child id, starting from the identity  (S:377 ordered fold;
 *      PAPER P:83-85 "on each level, one of the tasks collects the results
 *      from all sibling tasks").
 *   4. Coverage fingerprints (verify protocol).
 *   5. The owner of one iteration of a flat nest (own() followed for one
 *      position), for fingerprints at full size (2^32-2^34 iterations).
 *
 * Build: gcc -O2 -std=c99 -fPIC -shared (no -ffast-math, no threads).
 * Nothing here is tuned; clarity over speed.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- schedule codes (the oracle's own numbering) ------------------------ */
enum { OR_STATIC = 0, OR_STATIC_CHUNK = 1, OR_DYNAMIC = 2, OR_NONE = 3 };
/* ---- ops ---------------------------------------------------------------- */
/* OR_AFFINE: element x (int64) is the affine map y -> a*y + b (mod 2^64)
 * with a = 2x + 1, b = x*x (b = x would be conjugate to a product); the fold composes the maps in ascending order
 * (apply the left operand first): associative, NOT commutative — the
 * user-defined non-commutative reduction of P:86 / S:377. */
enum { OR_SUM = 0, OR_MIN = 1, OR_MAX = 2, OR_HIST256 = 3, OR_AFFINE = 4 };
/* ---- element types ------------------------------------------------------ */
enum { OR_I32 = 0, OR_I64 = 1, OR_F32 = 2, OR_F64 = 3, OR_U8 = 4 };
/* ---- error codes -------------------------------------------------------- */
enum { OR_OK = 0, OR_E_SCHEDULE = -1, OR_E_INVALID = -2, OR_E_NOMEM = -3 };

typedef struct {
  int32_t sched;  /* OR_STATIC ... OR_NONE                          */
  int32_t loop;   /* 0 or 1: which loop this level workshares        */
  int64_t chunk;  /* chunk size for static(c)/dynamic(c)             */
  int64_t T;      /* number of sibling tasks (fan-out per parent)    */
} or_level;

/* ========================================================================
 * 1. own(): which positions of a parent list of length n child t of T owns.
 *    SPEC S:337:
 *      static (no chunk): contiguous blocks, sizes differing by <= 1,
 *                         earlier tasks get the larger blocks;
 *      static(c):         chunks of c round-robin, position p -> task
 *                         floor(p/c) mod T;
 *      dynamic(c):        modelled as static(c) (see header);
 *      none:              task t owns position t if t < n, nothing else;
 *                         n > T is an error (PAPER P:251, S:338 diagnose UB).
 *    Writes the owned positions in ascending order to out (if non-NULL) and
 *    returns their count, or a negative error code.
 * ======================================================================== */
int64_t or_own(int32_t sched, int64_t chunk, int64_t n, int64_t T, int64_t t, int64_t* out) {
  if (T < 1 || t < 0 || t >= T || n < 0) return OR_E_INVALID;
  int64_t cnt = 0;
  if (sched == OR_STATIC) {
    int64_t q = n / T, r = n % T;
    int64_t begin = t * q + (t < r ? t : r);
    int64_t size = q + (t < r ? 1 : 0);
    for (int64_t p = begin; p < begin + size; ++p) {
      if (out) out[cnt] = p;
      ++cnt;
    }
    return cnt;
  }
  if (sched == OR_STATIC_CHUNK || sched == OR_DYNAMIC) {
    if (chunk < 1) return OR_E_INVALID;
    for (int64_t p = 0; p < n; ++p) {
      if ((p / chunk) % T == t) {
        if (out) out[cnt] = p;
        ++cnt;
      }
    }
    return cnt;
  }
  if (sched == OR_NONE) {
    if (n > T) return OR_E_SCHEDULE;
    if (t < n) {
      if (out) out[0] = t;
      return 1;
    }
    return 0;
  }
  return OR_E_INVALID;
}

/* ========================================================================
 * 2./3. The nest walk.  A task at nest level a holds one local list per loop
 * (loop 0, loop 1).  Its children at level a+1 refine the list of the loop
 * level a+1 is bound to and inherit the other list unchanged.  The loop-1
 * list is kept as the chain of (level, id) refinements and materialised per
 * row, because for CSR nests its length depends on the row (offsets).
 * ======================================================================== */

typedef struct {
  /* the nest */
  const or_level* lv;
  int nlev;
  int nloops;
  /* the iteration space */
  int64_t n0, n1;          /* loop extents (n1: dense inner extent)       */
  const int64_t* offsets;  /* CSR row offsets [n0+1] or NULL              */
  /* the data (may be NULL when only the partition is wanted) */
  int32_t dtype;
  const void* x;           /* flat / CSR values / dense rows              */
  int64_t ld;              /* dense row stride in elements                */
  int32_t op;
  /* outputs (each may be NULL) */
  int64_t* owner;          /* per iteration: mixed-radix leaf id          */
  uint32_t* count;         /* per iteration: number of visits             */
  void** partials;         /* per nest level: partials array or NULL      */
  int32_t keyed;           /* 0: one total; 1: per loop-0 iteration       */
  int keyed_first_inner;   /* first nest level bound to loop 1 (keyed)    */
  /* work state */
  int64_t ids[16];         /* current task id at every nest level         */
  int64_t* list0[17];      /* loop-0 list storage at depth a              */
  const int64_t* l0p[17];  /* loop-0 local list at depth a (may alias)    */
  int64_t len0[17];
  int64_t* tmp1[17];       /* scratch for the loop-1 refinement chain     */
  int64_t cap1;
  int err;
} or_walk;

/* ---- accumulator: a tagged value (sum/min/max) or 256 bins ------------- */
typedef struct {
  int64_t i;
  double f;
  uint64_t aa, ab;  /* OR_AFFINE: the map y -> aa*y + ab */
  uint64_t bins[256];
} or_acc;

static int is_float(int32_t dt) { return dt == OR_F32 || dt == OR_F64; }

static void acc_identity(const or_walk* w, or_acc* a) {
  a->i = 0;
  a->f = 0.0;
  if (w->op == OR_MIN) { a->i = INT64_MAX; a->f = 1.0 / 0.0; }
  if (w->op == OR_MAX) { a->i = INT64_MIN; a->f = -1.0 / 0.0; }
  if (w->op == OR_HIST256) memset(a->bins, 0, sizeof(a->bins));
  a->aa = 1;  /* identity map */
  a->ab = 0;
}

/* fold b into a (a := a (+) b); ordered: a is the left operand */
static void acc_fold(const or_walk* w, or_acc* a, const or_acc* b) {
  if (w->op == OR_AFFINE) {  /* a := b o a  (a applied first) */
    const uint64_t na = b->aa * a->aa;
    const uint64_t nb = b->aa * a->ab + b->ab;
    a->aa = na;
    a->ab = nb;
    return;
  }
  if (w->op == OR_HIST256) {
    for (int k = 0; k < 256; ++k) a->bins[k] += b->bins[k];
    return;
  }
  if (is_float(w->dtype)) {
    if (w->op == OR_SUM) a->f = a->f + b->f;
    if (w->op == OR_MIN) a->f = (b->f < a->f) ? b->f : a->f;
    if (w->op == OR_MAX) a->f = (b->f > a->f) ? b->f : a->f;
  } else {
    if (w->op == OR_SUM) a->i = (int64_t)((uint64_t)a->i + (uint64_t)b->i);
    if (w->op == OR_MIN) a->i = (b->i < a->i) ? b->i : a->i;
    if (w->op == OR_MAX) a->i = (b->i > a->i) ? b->i : a->i;
  }
}

/* fold element number idx of the input into a */
static void acc_element(const or_walk* w, or_acc* a, int64_t idx) {
  or_acc e;
  if (w->op == OR_HIST256) {
    const uint8_t v = ((const uint8_t*)w->x)[idx];
    a->bins[v] += 1;
    return;
  }
  if (w->op == OR_AFFINE) {
    const uint64_t v = (uint64_t)((const int64_t*)w->x)[idx];
    e.aa = 2 * v + 1;
    e.ab = v * v;
    acc_fold(w, a, &e);
    return;
  }
  switch (w->dtype) {
    case OR_I32: e.i = ((const int32_t*)w->x)[idx]; break;
    case OR_I64: e.i = ((const int64_t*)w->x)[idx]; break;
    case OR_F32: e.f = (double)((const float*)w->x)[idx]; break;
    case OR_F64: e.f = ((const double*)w->x)[idx]; break;
    default: e.i = ((const uint8_t*)w->x)[idx]; break;
  }
  acc_fold(w, a, &e);
}

static void acc_store(const or_walk* w, void* arr, int64_t slot, const or_acc* a) {
  if (w->op == OR_AFFINE) {
    ((uint64_t*)arr)[2 * slot] = a->aa;
    ((uint64_t*)arr)[2 * slot + 1] = a->ab;
  } else if (w->op == OR_HIST256) {
    memcpy((uint64_t*)arr + slot * 256, a->bins, sizeof(a->bins));
  } else if (is_float(w->dtype)) {
    ((double*)arr)[slot] = a->f;
  } else {
    ((int64_t*)arr)[slot] = a->i;
  }
}

/* Materialise the loop-1 list of the current task for a row of length n:
 * apply every level < upto that is bound to loop 1, in nest order. */
static int64_t loop1_list(or_walk* w, int upto, int64_t n, int64_t** result) {
  int64_t len = n;
  int64_t* cur = w->tmp1[0];
  for (int64_t p = 0; p < n; ++p) cur[p] = p;
  int slot = 0;
  for (int a = 0; a < upto; ++a) {
    if (w->lv[a].loop != 1) continue;
    int64_t* nxt = w->tmp1[(slot + 1) % 2 + 1];
    int64_t* pos = w->tmp1[3];
    int64_t c = or_own(w->lv[a].sched, w->lv[a].chunk, len, w->lv[a].T, w->ids[a], pos);
    if (c < 0) { w->err = (int)c; return 0; }
    for (int64_t q = 0; q < c; ++q) nxt[q] = cur[pos[q]];
    cur = nxt;
    len = c;
    slot = (slot + 1) % 2;
  }
  *result = cur;
  return len;
}

static int64_t row_len(const or_walk* w, int64_t i) {
  if (w->nloops == 1) return 1;
  if (w->offsets) return w->offsets[i + 1] - w->offsets[i];
  return w->n1;
}
static int64_t elem_index(const or_walk* w, int64_t i, int64_t j) {
  if (w->nloops == 1) return i;
  if (w->offsets) return w->offsets[i] + j;
  return i * w->ld + j;
}
static int64_t iter_index(const or_walk* w, int64_t i, int64_t j) {
  if (w->nloops == 1) return i;
  if (w->offsets) return w->offsets[i] + j;
  return i * w->n1 + j;
}

/* global id of the current task at level a (mixed radix over levels 0..a) */
static int64_t task_gid(const or_walk* w, int a) {
  int64_t g = 0;
  for (int b = 0; b <= a; ++b) g = g * w->lv[b].T + w->ids[b];
  return g;
}
/* id of the current task at level a local to the keyed row owner */
static int64_t task_lid(const or_walk* w, int a) {
  int64_t g = 0;
  for (int b = w->keyed_first_inner; b <= a; ++b) g = g * w->lv[b].T + w->ids[b];
  return g;
}
static int64_t tasks_below_owner(const or_walk* w, int a) {
  int64_t g = 1;
  for (int b = w->keyed_first_inner; b <= a; ++b) g *= w->lv[b].T;
  return g;
}

/* ---- TOTAL mode: depth-first walk, returns the partial of the task ------ */
static void walk_total(or_walk* w, int a, or_acc* out) {
  acc_identity(w, out);
  if (w->err) return;
  if (a == w->nlev) {
    /* leaf: execute the owned iterations in order (loop 0 outer, loop 1 inner) */
    const int64_t leaf = task_gid(w, w->nlev - 1);
    int64_t* l1 = NULL;
    int64_t l1_len = -1, l1_for = -1;
    for (int64_t q = 0; q < w->len0[a]; ++q) {
      const int64_t i = w->l0p[a][q];
      const int64_t n = row_len(w, i);
      if (w->nloops == 1) {
        l1_len = 1;
      } else if (n != l1_for) {
        l1_len = loop1_list(w, w->nlev, n, &l1);
        l1_for = n;
        if (w->err) return;
      }
      for (int64_t r = 0; r < l1_len; ++r) {
        const int64_t j = (w->nloops == 1) ? 0 : l1[r];
        const int64_t it = iter_index(w, i, j);
        if (w->owner) w->owner[it] = leaf;
        if (w->count) w->count[it] += 1;
        if (w->x) acc_element(w, out, elem_index(w, i, j));
      }
    }
    return;
  }
  const or_level* L = &w->lv[a];
  or_acc* child = (or_acc*)malloc(sizeof(or_acc));
  if (!child) { w->err = OR_E_NOMEM; return; }
  for (int64_t t = 0; t < L->T; ++t) {
    w->ids[a] = t;
    if (L->loop == 0) {
      int64_t* pos = w->list0[a + 1];
      int64_t c = or_own(L->sched, L->chunk, w->len0[a], L->T, t, pos);
      if (c < 0) { w->err = (int)c; break; }
      for (int64_t q = 0; q < c; ++q) pos[q] = w->l0p[a][pos[q]];
      w->l0p[a + 1] = pos;
      w->len0[a + 1] = c;
    } else {
      /* loop-1 refinement is applied lazily at the leaf (per row length);
       * loop-0 list passes through unchanged */
      w->l0p[a + 1] = w->l0p[a];
      w->len0[a + 1] = w->len0[a];
      if (w->nloops == 1) { w->err = OR_E_INVALID; break; }
    }
    walk_total(w, a + 1, child);
    if (w->err) break;
    if (w->partials && w->partials[a]) acc_store(w, w->partials[a], task_gid(w, a), child);
    acc_fold(w, out, child);  /* ascending child id */
  }
  free(child);
}

/* ---- KEYED mode: loop-0 levels are a prefix [0, k); for every row i of a
 * row owner, walk the inner (loop-1) levels and fold per inner task. ------ */
static void walk_inner(or_walk* w, int a, int64_t i, or_acc* out) {
  acc_identity(w, out);
  if (w->err) return;
  if (a == w->nlev) {
    const int64_t leaf = task_gid(w, w->nlev - 1);
    int64_t* l1 = NULL;
    const int64_t l1_len = loop1_list(w, w->nlev, row_len(w, i), &l1);
    if (w->err) return;
    for (int64_t r = 0; r < l1_len; ++r) {
      const int64_t it = iter_index(w, i, l1[r]);
      if (w->owner) w->owner[it] = leaf;
      if (w->count) w->count[it] += 1;
      if (w->x) acc_element(w, out, elem_index(w, i, l1[r]));
    }
    return;
  }
  or_acc* child = (or_acc*)malloc(sizeof(or_acc));
  if (!child) { w->err = OR_E_NOMEM; return; }
  for (int64_t t = 0; t < w->lv[a].T; ++t) {
    w->ids[a] = t;
    walk_inner(w, a + 1, i, child);
    if (w->err) break;
    if (w->partials && w->partials[a]) {
      const int64_t slot = i * tasks_below_owner(w, a) + task_lid(w, a);
      acc_store(w, w->partials[a], slot, child);
    }
    acc_fold(w, out, child);
  }
  free(child);
}

static void walk_keyed(or_walk* w, int a, void* out_rows) {
  if (w->err) return;
  if (a == w->keyed_first_inner) {
    /* a row owner: every row of its loop-0 list */
    or_acc* row = (or_acc*)malloc(sizeof(or_acc));
    if (!row) { w->err = OR_E_NOMEM; return; }
    for (int64_t q = 0; q < w->len0[a]; ++q) {
      const int64_t i = w->l0p[a][q];
      walk_inner(w, a, i, row);
      if (w->err) break;
      if (out_rows) acc_store(w, out_rows, i, row);
    }
    free(row);
    return;
  }
  const or_level* L = &w->lv[a];
  for (int64_t t = 0; t < L->T; ++t) {
    w->ids[a] = t;
    int64_t* pos = w->list0[a + 1];
    int64_t c = or_own(L->sched, L->chunk, w->len0[a], L->T, t, pos);
    if (c < 0) { w->err = (int)c; return; }
    for (int64_t q = 0; q < c; ++q) pos[q] = w->l0p[a][pos[q]];
    w->l0p[a + 1] = pos;
    w->len0[a + 1] = c;
    walk_keyed(w, a + 1, out_rows);
  }
}

/* ========================================================================
 * or_nest_run: the nest semantics.
 *   lv/nlev        the nest (outermost first; nlev <= 16)
 *   nloops         1 (flat, n0 iterations) or 2 (n0 x n1 dense, or CSR)
 *   offsets        CSR offsets [n0+1] (nloops == 2) or NULL for dense
 *   dtype/x/ld/op  input data (x may be NULL: partition only)
 *   keyed          0: one total (TOTAL mode); 1: one result per loop-0
 *                  iteration (requires loop-0 levels to be a prefix)
 *   result         TOTAL: one accumulator value (int64 / double / 256 u64)
 *                  KEYED: per-row values [n0]
 *   owner/count    per-iteration coverage (iteration index: i, i*n1+j, or
 *                  offsets[i]+j), may be NULL; count must be zeroed by caller
 *   partials       per nest level array or NULL (TOTAL: indexed by the
 *                  task's global mixed-radix id; KEYED: inner levels only,
 *                  indexed row * tasks_per_owner + local id)
 * Returns OR_OK or a negative error.
 * ======================================================================== */
int or_nest_run(const or_level* lv, int nlev, int nloops, int64_t n0, int64_t n1,
                const int64_t* offsets, int32_t dtype, const void* x, int64_t ld, int32_t op,
                int32_t keyed, void* result, int64_t* owner, uint32_t* count, void** partials) {
  if (nlev < 1 || nlev > 16 || (nloops != 1 && nloops != 2) || n0 < 0) return OR_E_INVALID;
  or_walk w;
  memset(&w, 0, sizeof(w));
  w.lv = lv; w.nlev = nlev; w.nloops = nloops; w.n0 = n0; w.n1 = n1;
  w.offsets = offsets; w.dtype = dtype; w.x = x; w.ld = ld; w.op = op;
  w.owner = owner; w.count = count; w.partials = partials; w.keyed = keyed;
  for (int a = 0; a < nlev; ++a) {
    if (lv[a].loop < 0 || lv[a].loop >= nloops || lv[a].T < 1) return OR_E_INVALID;
  }
  if (keyed) {
    if (nloops != 2) return OR_E_INVALID;
    int k = 0;
    while (k < nlev && lv[k].loop == 0) ++k;
    for (int a = k; a < nlev; ++a)
      if (lv[a].loop != 1) return OR_E_INVALID;  /* loop-0 levels must be a prefix */
    w.keyed_first_inner = k;
  }
  /* buffers */
  int64_t maxrow = 1;
  if (nloops == 2) {
    if (offsets) {
      for (int64_t i = 0; i < n0; ++i)
        if (offsets[i + 1] - offsets[i] > maxrow) maxrow = offsets[i + 1] - offsets[i];
    } else {
      maxrow = n1 > 1 ? n1 : 1;
    }
  }
  w.cap1 = maxrow;
  int ok = 1;
  for (int a = 0; a <= nlev; ++a) {
    w.list0[a] = (int64_t*)malloc((size_t)(n0 > 0 ? n0 : 1) * sizeof(int64_t));
    if (!w.list0[a]) ok = 0;
  }
  for (int s = 0; s < 4; ++s) {
    w.tmp1[s] = (int64_t*)malloc((size_t)maxrow * sizeof(int64_t));
    if (!w.tmp1[s]) ok = 0;
  }
  if (ok) {
    for (int64_t i = 0; i < n0; ++i) w.list0[0][i] = i;
    w.l0p[0] = w.list0[0];
    w.len0[0] = n0;
    if (!keyed) {
      or_acc* total = (or_acc*)malloc(sizeof(or_acc));
      if (!total) {
        w.err = OR_E_NOMEM;
      } else {
        walk_total(&w, 0, total);
        if (!w.err && result) acc_store(&w, result, 0, total);
        free(total);
      }
    } else {
      walk_keyed(&w, 0, result);
    }
  } else {
    w.err = OR_E_NOMEM;
  }
  for (int a = 0; a <= nlev; ++a) free(w.list0[a]);
  for (int s = 0; s < 4; ++s) free(w.tmp1[s]);
  return w.err;
}

/* ========================================================================
 * 1. Results by their plain definitions.
 * ======================================================================== */
int64_t or_sum_i32(const int32_t* x, int64_t n) {
  uint64_t s = 0;  /* two's complement wrap == exact int64 sum below 2^63 */
  for (int64_t i = 0; i < n; ++i) s += (uint64_t)(int64_t)x[i];
  return (int64_t)s;
}
double or_sum_f32(const float* x, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += (double)x[i];
  return s;
}
double or_min_f32(const float* x, int64_t n) {
  double m = 1.0 / 0.0;
  for (int64_t i = 0; i < n; ++i) if ((double)x[i] < m) m = (double)x[i];
  return m;
}
double or_max_f32(const float* x, int64_t n) {
  double m = -1.0 / 0.0;
  for (int64_t i = 0; i < n; ++i) if ((double)x[i] > m) m = (double)x[i];
  return m;
}
int64_t or_min_i32(const int32_t* x, int64_t n) {
  int64_t m = INT64_MAX;
  for (int64_t i = 0; i < n; ++i) if (x[i] < m) m = x[i];
  return m;
}
int64_t or_max_i32(const int32_t* x, int64_t n) {
  int64_t m = INT64_MIN;
  for (int64_t i = 0; i < n; ++i) if (x[i] > m) m = x[i];
  return m;
}
void or_hist256(const uint8_t* x, int64_t n, uint64_t* bins) {
  for (int k = 0; k < 256; ++k) bins[k] = 0;
  for (int64_t i = 0; i < n; ++i) bins[x[i]] += 1;
}
void or_rowsum_f32(const float* a, int64_t rows, int64_t cols, int64_t ld, double* out) {
  for (int64_t r = 0; r < rows; ++r) {
    double s = 0.0;
    for (int64_t c = 0; c < cols; ++c) s += (double)a[r * ld + c];
    out[r] = s;
  }
}
void or_segsum_f32(const float* v, const int64_t* offsets, int64_t rows, double* out) {
  for (int64_t r = 0; r < rows; ++r) {
    double s = 0.0;
    for (int64_t e = offsets[r]; e < offsets[r + 1]; ++e) s += (double)v[e];
    out[r] = s;
  }
}
/* exact closed form for inputs k * 2^-24: the integer numerator sum */
uint64_t or_sum_u64(const uint64_t* k, int64_t n) {
  uint64_t s = 0;
  for (int64_t i = 0; i < n; ++i) s += k[i];
  return s;
}

/* ========================================================================
 * 4. Coverage fingerprints (verify protocol).
 *    fp_mix(i)      = fmix64(i * 0x9E3779B97F4A7C15 + 0x632BE59BD9B4E019)
 *    fp_mix2(i, o)  = fmix64(fp_mix(i) ^ (o * 0xD6E8FEB86659FD93))
 *    F_once  = sum_i fp_mix(i)            mod 2^64
 *    F_owner = sum_i fp_mix2(i, owner(i)) mod 2^64
 * ======================================================================== */
static uint64_t fmix64(uint64_t z) {
  z ^= z >> 33;
  z *= 0xFF51AFD7ED558CCDull;
  z ^= z >> 33;
  z *= 0xC4CEB9FE1A85EC53ull;
  z ^= z >> 33;
  return z;
}
uint64_t or_fp_mix(uint64_t i) { return fmix64(i * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull); }
uint64_t or_fp_mix2(uint64_t i, uint64_t o) { return fmix64(or_fp_mix(i) ^ (o * 0xD6E8FEB86659FD93ull)); }
uint64_t or_fp_once(uint64_t begin, int64_t n) {
  uint64_t s = 0;
  for (int64_t e = 0; e < n; ++e) s += or_fp_mix(begin + (uint64_t)e);
  return s;
}
uint64_t or_fp_owner(const int64_t* owner, uint64_t begin, int64_t n) {
  uint64_t s = 0;
  for (int64_t e = 0; e < n; ++e) s += or_fp_mix2(begin + (uint64_t)e, (uint64_t)owner[e]);
  return s;
}

/* ========================================================================
 * 5. Owner of ONE iteration of a flat nest, without materialising lists
 *    (needed at 2^32-2^34 iterations, where or_nest_run's per-level lists do
 *    not fit in host memory).  Same semantics as the nest walk: own() applied
 *    level by level, outermost first, but followed for one
 *    position p of the parent's list instead of for all of them:
 *      static:    the task t whose block [t*q + min(t,r), (t+1)*q + min(t+1,r))
 *                 holds p; p's position in t's list is p - block start;
 *      static(c) / dynamic(c) (modelled as static(c)):
 *                 chunk k = p / c belongs to task k mod T; it is that task's
 *                 (k / T)-th chunk, so p's position is (k / T) * c + p mod c;
 *      none:      task p (error if n > T), position 0.
 *    The child's list length is own()'s count for t, in closed form
 *    (or_own_count); tests pin both against or_own / or_nest_run / brute.py.
 *    Every level must be bound to loop 0.  Returns the mixed-radix leaf id
 *    (the same packing as task_gid), or a negative error code.
 * ======================================================================== */
int64_t or_own_count(int32_t sched, int64_t chunk, int64_t n, int64_t T, int64_t t) {
  if (T < 1 || t < 0 || t >= T || n < 0) return OR_E_INVALID;
  if (sched == OR_STATIC) return n / T + (t < n % T ? 1 : 0);
  if (sched == OR_STATIC_CHUNK || sched == OR_DYNAMIC) {
    if (chunk < 1) return OR_E_INVALID;
    const int64_t full = n / chunk, rest = n % chunk;        /* whole chunks, ragged tail */
    int64_t cnt = (full / T + (t < full % T ? 1 : 0)) * chunk;  /* whole chunks of task t   */
    if (rest > 0 && full % T == t) cnt += rest;               /* the tail chunk is number full */
    return cnt;
  }
  if (sched == OR_NONE) {
    if (n > T) return OR_E_SCHEDULE;
    return t < n ? 1 : 0;
  }
  return OR_E_INVALID;
}

int64_t or_owner_flat(const or_level* lv, int nlev, int64_t n, int64_t i) {
  if (nlev < 1 || nlev > 16 || i < 0 || i >= n) return OR_E_INVALID;
  int64_t p = i, len = n, leaf = 0;
  for (int a = 0; a < nlev; ++a) {
    const or_level* L = &lv[a];
    if (L->loop != 0 || L->T < 1) return OR_E_INVALID;
    int64_t t = 0, pos = 0;
    if (L->sched == OR_STATIC) {
      const int64_t q = len / L->T, r = len % L->T;
      /* blocks 0..r-1 have q+1 positions, the rest q */
      if (p < r * (q + 1)) {
        t = p / (q + 1);
        pos = p - t * (q + 1);
      } else {
        t = r + (p - r * (q + 1)) / q;
        pos = p - (t * q + r);
      }
    } else if (L->sched == OR_STATIC_CHUNK || L->sched == OR_DYNAMIC) {
      if (L->chunk < 1) return OR_E_INVALID;
      const int64_t k = p / L->chunk;
      t = k % L->T;
      pos = (k / L->T) * L->chunk + p % L->chunk;
    } else if (L->sched == OR_NONE) {
      if (len > L->T) return OR_E_SCHEDULE;
      t = p;
      pos = 0;
    } else {
      return OR_E_INVALID;
    }
    len = or_own_count(L->sched, L->chunk, len, L->T, t);
    if (len < 0) return len;
    p = pos;
    leaf = leaf * L->T + t;
  }
  return leaf;
}

/* Fingerprints of the iterations [begin, begin + count) of a flat nest over
 * n iterations, computed one iteration at a time from or_owner_flat:
 *   out[0] += sum fp_mix(g0 + i),  out[1] += sum fp_mix2(g0 + i, owner(i))
 * (mod 2^64), g0 = the global index of iteration 0 (the rank's first).  The
 * sums are exact in Z/2^64, so disjoint ranges may be fingerprinted
 * separately and added.  Returns OR_OK or a negative error. */
int or_fp_flat_range(const or_level* lv, int nlev, int64_t n, int64_t begin, int64_t count, uint64_t g0,
                     uint64_t* out) {
  if (begin < 0 || count < 0 || begin + count > n) return OR_E_INVALID;
  uint64_t f_once = 0, f_owner = 0;
  for (int64_t i = begin; i < begin + count; ++i) {
    const int64_t o = or_owner_flat(lv, nlev, n, i);
    if (o < 0) return (int)o;
    f_once += or_fp_mix(g0 + (uint64_t)i);
    f_owner += or_fp_mix2(g0 + (uint64_t)i, (uint64_t)o);
  }
  out[0] += f_once;
  out[1] += f_owner;
  return OR_OK;
}

/* The recurrence the affine fold computes, run directly: y <- a_i*y + b_i for
 * i ascending, from y0 (a different algorithm than composing maps). */
uint64_t or_affine_run(const int64_t* x, int64_t n, uint64_t y0) {
  uint64_t y = y0;
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t v = (uint64_t)x[i];
    y = (2 * v + 1) * y + v * v;
  }
  return y;
}
