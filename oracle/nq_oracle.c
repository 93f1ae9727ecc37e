/*
 * nq_oracle.c — TEST INFRASTRUCTURE ONLY (see nq_oracle.h).
 *
 * A plain-C restatement of the reference counting path. Each function cites the
 * reference lines it follows (paths relative to /root/reference/proj/include/nqueens/).
 * The code is written for clarity, not speed: it is the checker, never the product.
 */
#include "nq_oracle.h"

#include <pthread.h>
#include <stdarg.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* nqo_last_error(void) { return g_err; }

/* checked_add / checked_mul — errors.hpp:23-35 */
static int add_ok(uint64_t a, uint64_t b, uint64_t* r) { return !__builtin_add_overflow(a, b, r); }
static int mul_ok(uint64_t a, uint64_t b, uint64_t* r) { return !__builtin_mul_overflow(a, b, r); }

/* board_mask — bitboard.hpp:15-17 */
uint32_t nqo_board_mask(int n) { return n >= 32 ? 0xffffffffu : ((1u << n) - 1u); }

/* valid_positions — bitboard.hpp:21-23 */
uint32_t nqo_valid_positions(uint32_t cur, uint32_t left, uint32_t right, int n) {
  return nqo_board_mask(n) & ~(cur | left | right);
}

/* apply_placement — bitboard.hpp:38-45 (left shift truncates at bit 31) */
static void place(uint32_t* cur, uint32_t* left, uint32_t* right, uint32_t p) {
  *cur |= p;
  *left = (uint32_t)((*left | p) << 1);
  *right = (*right | p) >> 1;
}

/* detail::check_board — solver.hpp:45-48 */
static int check_board(int n) {
  if (n < 1 || n > 32) return fail(NQO_ECONFIG, "board size must be in [1, 32], got %d", n);
  return NQO_OK;
}

/* count_recursive_impl — solver.hpp:50-63 */
static int rec(int n, uint32_t cur, uint32_t left, uint32_t right, uint64_t* out) {
  if (cur == nqo_board_mask(n)) { *out = 1; return NQO_OK; }
  uint64_t sum = 0;
  uint32_t v = nqo_valid_positions(cur, left, right, n);
  while (v) {
    const uint32_t p = v & (~v + 1u);
    v -= p;
    uint32_t c = cur, l = left, r = right;
    place(&c, &l, &r, p);
    uint64_t sub;
    int rc = rec(n, c, l, r, &sub);
    if (rc) return rc;
    if (!add_ok(sum, sub, &sum)) return fail(NQO_EOVERFLOW, "solution count overflows 64 bits");
  }
  *out = sum;
  return NQO_OK;
}

int nqo_count_recursive(int n, uint32_t cur, uint32_t left, uint32_t right, uint64_t* count) {
  int rc = check_board(n);
  if (rc) return rc;
  return rec(n, cur, left, right, count);
}

/* require_feasible — stack_config.hpp:43-45 (required_depth), :59-71. The message
 * names the reference's built-in table (stack_config.hpp:29-35). */
static int feasible(int stack_depth, int n, int placed, int last_row) {
  static const struct { const char* name; int depth; } cfgs[] = {
      {"config1", 24}, {"config2", 19}, {"config3", 16}, {"config4", 12}, {"config5", 6}};
  const int need = n - placed - (last_row ? 1 : 0);
  if (need <= stack_depth) return NQO_OK;
  const char* fit = NULL;
  int fit_depth = 1 << 30;
  for (size_t i = 0; i < sizeof cfgs / sizeof cfgs[0]; ++i)
    if (cfgs[i].depth >= need && cfgs[i].depth < fit_depth) { fit = cfgs[i].name; fit_depth = cfgs[i].depth; }
  if (fit)
    return fail(NQO_ECONFIG, "stack supports depth %d but n=%d, pre_rows=%d needs %d; "
                "smallest sufficient config is '%s'", stack_depth, n, placed, need, fit);
  return fail(NQO_ECONFIG, "stack supports depth %d but n=%d, pre_rows=%d needs %d; "
              "no built-in config is deep enough", stack_depth, n, placed, need);
}

/* count_iterative — solver.hpp:79-130 */
int nqo_count_iterative(int n, const nqo_sub* sub, int stack_depth, uint64_t* count,
                        int* high_water) {
  int rc = check_board(n);
  if (rc) return rc;
  const int placed = (int)(sub->row & 0xff);
  rc = feasible(stack_depth, n, placed, 0);
  if (rc) return rc;
  const uint32_t last = nqo_board_mask(n);
  uint32_t cur = sub->cols, left = sub->diag, right = sub->antidiag;
  *high_water = 0;
  if (cur == last) { *count = 1; return NQO_OK; }
  uint32_t v = nqo_valid_positions(cur, left, right, n);
  if (v == 0) { *count = 0; return NQO_OK; }
  uint32_t st[4 * 33];
  int top = 4, high = 0;
  uint64_t sum = 0;
  st[0] = cur; st[1] = left; st[2] = right; st[3] = v;
  while (top) {
    cur = st[top - 4]; left = st[top - 3]; right = st[top - 2]; v = st[top - 1];
    const int h = __builtin_popcount(cur) - placed + 1;
    if (h > high) high = h;
    const uint32_t p = v & (~v + 1u);
    v -= p;
    st[top - 1] = v;
    top -= v == 0 ? 4 : 0;
    cur |= p;
    if (cur == last) {
      if (!add_ok(sum, 1, &sum)) return fail(NQO_EOVERFLOW, "solution count overflows 64 bits");
      continue;
    }
    left = (uint32_t)((left | p) << 1);
    right = (right | p) >> 1;
    v = nqo_valid_positions(cur, left, right, n);
    if (!v) continue;
    st[top] = cur; st[top + 1] = left; st[top + 2] = right; st[top + 3] = v;
    top += 4;
  }
  *count = sum;
  *high_water = high;
  return NQO_OK;
}

/* count_iterative_lastrow — solver.hpp:138-191. nodes counts loop iterations. */
int nqo_count_lastrow(int n, const nqo_sub* sub, int stack_depth, uint64_t* count,
                      int* high_water, uint64_t* nodes) {
  int rc = check_board(n);
  if (rc) return rc;
  const int placed = (int)(sub->row & 0xff);
  rc = feasible(stack_depth, n, placed, 1);
  if (rc) return rc;
  const uint32_t last = nqo_board_mask(n);
  uint32_t cur = sub->cols, left = sub->diag, right = sub->antidiag;
  *high_water = 0;
  if (nodes) *nodes = 0;
  if (placed >= n) { *count = cur == last ? 1u : 0u; return NQO_OK; }
  uint32_t v = nqo_valid_positions(cur, left, right, n);
  if (placed == n - 1) { *count = (uint64_t)__builtin_popcount(v); return NQO_OK; }
  if (v == 0) { *count = 0; return NQO_OK; }
  uint32_t st[4 * 33];
  int top = 4, high = 0;
  uint64_t sum = 0, it = 0;
  st[0] = cur; st[1] = left; st[2] = right; st[3] = v;
  while (top) {
    cur = st[top - 4]; left = st[top - 3]; right = st[top - 2]; v = st[top - 1];
    ++it;
    const int h = __builtin_popcount(cur) - placed + 1;
    if (h > high) high = h;
    const uint32_t p = v & (~v + 1u);
    v -= p;
    st[top - 1] = v;
    top -= v == 0 ? 4 : 0;
    cur |= p;
    left = (uint32_t)((left | p) << 1);
    right = (right | p) >> 1;
    v = nqo_valid_positions(cur, left, right, n);
    if (v == 0 || __builtin_popcount(cur) == n - 1) {
      if (!add_ok(sum, (uint64_t)__builtin_popcount(v), &sum))
        return fail(NQO_EOVERFLOW, "solution count overflows 64 bits");
      continue;
    }
    st[top] = cur; st[top + 1] = left; st[top + 2] = right; st[top + 3] = v;
    top += 4;
  }
  *count = sum;
  *high_water = high;
  if (nodes) *nodes = it;
  return NQO_OK;
}

/* ---- frontier: subproblems.hpp ------------------------------------------------ */

typedef struct {
  nqo_sub* out;
  uint64_t cap, len;
  FILE* text;
} sink_t;

static void emit(sink_t* s, uint32_t cur, uint32_t left, uint32_t right, int placed, int mult) {
  if (s->text)
    fprintf(s->text, "%llu %x %x %x %d %d\n", (unsigned long long)s->len, cur, left, right,
            placed, mult); /* write_batch — subproblems.hpp:169-178 */
  if (s->out && s->len < s->cap) {
    nqo_sub* r = &s->out[s->len];
    r->cols = cur; r->diag = left; r->antidiag = right;
    r->row = (uint32_t)placed | ((uint32_t)mult << 8);
  }
  s->len++;
}

/* detail::expand_rows — subproblems.hpp:41-55 */
static void expand(int n, uint32_t cur, uint32_t left, uint32_t right, int row, int target,
                   int mult, sink_t* s) {
  if (row == target) { emit(s, cur, left, right, target, mult); return; }
  uint32_t v = nqo_valid_positions(cur, left, right, n);
  while (v) {
    const uint32_t p = v & (~v + 1u);
    v -= p;
    uint32_t c = cur, l = left, r = right;
    place(&c, &l, &r, p);
    expand(n, c, l, r, row + 1, target, mult, s);
  }
}

/* detail::check_plan — subproblems.hpp:32-39 */
static int check_plan(int n, int R) {
  int rc = check_board(n);
  if (rc) return rc;
  if (R < 1 || R >= n) return fail(NQO_ECONFIG, "pre_rows must satisfy 1 <= R < n (n=%d, R=%d)", n, R);
  if (R > 8) return fail(NQO_ECONFIG, "pre_rows above 8 is not supported");
  return NQO_OK;
}

/* for_each_subproblem — subproblems.hpp:80-108 */
static int walk(int n, int R, sink_t* s) {
  int rc = check_plan(n, R);
  if (rc) return rc;
  for (int c = 0; c < n / 2; ++c) {
    uint32_t cur = 0, l = 0, r = 0;
    place(&cur, &l, &r, 1u << c);
    expand(n, cur, l, r, 1, R, 2, s);
  }
  if (n % 2 == 1) {
    const int c = (n - 1) / 2;
    uint32_t cur = 0, l = 0, r = 0;
    place(&cur, &l, &r, 1u << c);
    if (R == 1) {
      emit(s, cur, l, r, 1, 1);
    } else {
      const uint32_t left_half = c >= 1 ? (1u << (c - 1)) - 1u : 0u;
      uint32_t v = nqo_valid_positions(cur, l, r, n) & left_half;
      while (v) {
        const uint32_t p = v & (~v + 1u);
        v -= p;
        uint32_t c2 = cur, l2 = l, r2 = r;
        place(&c2, &l2, &r2, p);
        expand(n, c2, l2, r2, 2, R, 2, s);
      }
    }
  }
  return NQO_OK;
}

int nqo_generate(int n, int pre_rows, nqo_sub* out, uint64_t cap, uint64_t* total) {
  sink_t s = {out, cap, 0, NULL};
  int rc = walk(n, pre_rows, &s);
  if (rc) return rc;
  *total = s.len;
  return NQO_OK;
}

int nqo_write_batch(int n, int pre_rows, FILE* out, uint64_t* lines) {
  sink_t s = {NULL, 0, 0, out};
  int rc = walk(n, pre_rows, &s);
  if (rc) return rc;
  *lines = s.len;
  return NQO_OK;
}

/* detail::count_rows — subproblems.hpp:58-71 */
static uint64_t count_rows(int n, uint32_t cur, uint32_t left, uint32_t right, int row,
                           int target) {
  if (row == target) return 1;
  uint32_t v = nqo_valid_positions(cur, left, right, n);
  if (row == target - 1) return (uint64_t)__builtin_popcount(v);
  uint64_t sum = 0;
  while (v) {
    const uint32_t p = v & (~v + 1u);
    v -= p;
    uint32_t c = cur, l = left, r = right;
    place(&c, &l, &r, p);
    sum += count_rows(n, c, l, r, row + 1, target);
  }
  return sum;
}

/* count_subproblems — subproblems.hpp:118-145 */
int nqo_count_subproblems(int n, int pre_rows, uint64_t* total) {
  int rc = check_plan(n, pre_rows);
  if (rc) return rc;
  uint64_t t = 0;
  for (int c = 0; c < n / 2; ++c) {
    uint32_t cur = 0, l = 0, r = 0;
    place(&cur, &l, &r, 1u << c);
    t += count_rows(n, cur, l, r, 1, pre_rows);
  }
  if (n % 2 == 1) {
    const int c = (n - 1) / 2;
    uint32_t cur = 0, l = 0, r = 0;
    place(&cur, &l, &r, 1u << c);
    if (pre_rows == 1) {
      t += 1;
    } else {
      const uint32_t left_half = c >= 1 ? (1u << (c - 1)) - 1u : 0u;
      uint32_t v = nqo_valid_positions(cur, l, r, n) & left_half;
      while (v) {
        const uint32_t p = v & (~v + 1u);
        v -= p;
        uint32_t c2 = cur, l2 = l, r2 = r;
        place(&c2, &l2, &r2, p);
        t += count_rows(n, c2, l2, r2, 2, pre_rows);
      }
    }
  }
  *total = t;
  return NQO_OK;
}

/* aggregate — subproblems.hpp:149-165: same 64-bit state key, sequential order so
 * the first error surfaced matches the reference. Open-addressing set. */
int nqo_aggregate(const nqo_sub* subs, const uint64_t* counts, uint64_t len, uint64_t* total) {
  uint64_t cap = 16;
  while (cap < 2 * len + 16) cap <<= 1;
  uint64_t* keys = (uint64_t*)calloc(cap, sizeof(uint64_t));
  unsigned char* used = (unsigned char*)calloc(cap, 1);
  if (!keys || !used) { free(keys); free(used); return fail(NQO_ECONFIG, "out of memory"); }
  uint64_t t = 0;
  int rc = NQO_OK;
  for (uint64_t i = 0; i < len && rc == NQO_OK; ++i) {
    const nqo_sub* s = &subs[i];
    uint64_t key = s->cols;
    key = key * 0x9e3779b97f4a7c15ull ^ s->diag;
    key = key * 0x9e3779b97f4a7c15ull ^ s->antidiag;
    key = key * 0x9e3779b97f4a7c15ull ^ (uint64_t)(s->row & 0xff);
    uint64_t h = (key ^ (key >> 29)) & (cap - 1);
    int dup = 0;
    while (used[h]) {
      if (keys[h] == key) { dup = 1; break; }
      h = (h + 1) & (cap - 1);
    }
    if (dup) { rc = fail(NQO_ECONFIG, "duplicate subproblem in aggregation input"); break; }
    used[h] = 1;
    keys[h] = key;
    uint64_t w;
    if (!mul_ok((uint64_t)(s->row >> 8), counts[i], &w) || !add_ok(t, w, &t))
      rc = fail(NQO_EOVERFLOW, "solution count overflows 64 bits");
  }
  free(keys);
  free(used);
  if (rc == NQO_OK) *total = t;
  return rc;
}

/* partition_uniform — scheduler.hpp:61-73 */
int nqo_partition_uniform(uint64_t task_count, int workers, uint64_t* ranges) {
  if (workers < 1) return fail(NQO_ECONFIG, "worker_count must be >= 1");
  const uint64_t base = task_count / (uint64_t)workers, rem = task_count % (uint64_t)workers;
  uint64_t next = 0;
  for (int i = 0; i < workers; ++i) {
    const uint64_t size = base + ((uint64_t)i < rem ? 1 : 0);
    ranges[2 * i] = next;
    ranges[2 * i + 1] = next + size;
    next += size;
  }
  return NQO_OK;
}

/* partition_weighted — scheduler.hpp:76-102 */
int nqo_partition_weighted(uint64_t task_count, const double* weights, int workers,
                           uint64_t* ranges) {
  if (workers < 1) return fail(NQO_ECONFIG, "weighted partition needs at least one weight");
  double sum = 0;
  for (int i = 0; i < workers; ++i) {
    if (!(weights[i] > 0)) return fail(NQO_ECONFIG, "partition weights must be positive");
    sum += weights[i];
  }
  uint64_t assigned = 0;
  for (int i = 0; i < workers; ++i) {
    const double share = (double)task_count * (weights[i] / sum);
    ranges[2 * i + 1] = (uint64_t)share; /* floor for non-negative values */
    assigned += ranges[2 * i + 1];
  }
  for (int i = 0; assigned < task_count; i = (i + 1) % workers) {
    ranges[2 * i + 1]++;
    assigned++;
  }
  uint64_t next = 0;
  for (int i = 0; i < workers; ++i) {
    const uint64_t size = ranges[2 * i + 1];
    ranges[2 * i] = next;
    ranges[2 * i + 1] = next + size;
    next += size;
  }
  return NQO_OK;
}

/* ---- threaded batch solve: execute_batch stealing branch, scheduler.hpp:266-389 ---- */

typedef struct {
  int n;
  const nqo_sub* subs;
  uint64_t len, chunk;
  uint64_t* cursor;
  uint64_t* per_sub;
  uint64_t sum, nodes;
  int rc;
  char err[256];
} worker_t;

static void* worker_main(void* arg) {
  worker_t* w = (worker_t*)arg;
  for (;;) {
    const uint64_t first = __atomic_fetch_add(w->cursor, w->chunk, __ATOMIC_RELAXED);
    if (first >= w->len) break;
    const uint64_t last = first + w->chunk < w->len ? first + w->chunk : w->len;
    for (uint64_t i = first; i < last; ++i) {
      uint64_t c = 0, nd = 0, wsum;
      int high;
      int rc = nqo_count_lastrow(w->n, &w->subs[i], 32, &c, &high, &nd);
      if (rc == NQO_OK && (!mul_ok((uint64_t)(w->subs[i].row >> 8), c, &wsum) ||
                           !add_ok(w->sum, wsum, &w->sum)))
        rc = fail(NQO_EOVERFLOW, "solution count overflows 64 bits");
      if (rc) {
        w->rc = rc;
        snprintf(w->err, sizeof w->err, "failed on subproblem %llu: %s",
                 (unsigned long long)i, nqo_last_error());
        return NULL;
      }
      w->nodes += nd;
      if (w->per_sub) w->per_sub[i] = c;
    }
  }
  return NULL;
}

int nqo_solve_batch(int n, const nqo_sub* subs, uint64_t len, int threads, uint64_t chunk,
                    uint64_t* total, uint64_t* nodes, uint64_t* per_sub_counts) {
  if (threads < 1) return fail(NQO_ECONFIG, "worker_count must be >= 1");
  if (chunk == 0) return fail(NQO_ECONFIG, "chunk_size must be >= 1");
  uint64_t cursor = 0;
  worker_t* ws = (worker_t*)calloc((size_t)threads, sizeof(worker_t));
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int i = 0; i < threads; ++i) {
    ws[i].n = n; ws[i].subs = subs; ws[i].len = len; ws[i].chunk = chunk;
    ws[i].cursor = &cursor; ws[i].per_sub = per_sub_counts;
    pthread_create(&tid[i], NULL, worker_main, &ws[i]);
  }
  for (int i = 0; i < threads; ++i) pthread_join(tid[i], NULL);
  int rc = NQO_OK;
  uint64_t t = 0, nd = 0;
  for (int i = 0; i < threads && rc == NQO_OK; ++i) {
    if (ws[i].rc) { rc = fail(ws[i].rc, "worker %d %s", i, ws[i].err); break; }
    if (!add_ok(t, ws[i].sum, &t)) rc = fail(NQO_EOVERFLOW, "solution count overflows 64 bits");
    nd += ws[i].nodes;
  }
  free(ws);
  free(tid);
  if (rc == NQO_OK) { *total = t; if (nodes) *nodes = nd; }
  return rc;
}
