/* TEST INFRASTRUCTURE ONLY — see mssz_oracle.h.
 *
 * Type-independent parts: grid topology (grid.cpp), label pointer jumping
 * (mss.cpp:51-97), error plumbing (errors.hpp).  The per-type body lives in
 * mssz_oracle_body.inc, included once for float and once for double.
 */
#include "mssz_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

enum { ERR_USAGE = 2, ERR_IO = 3, ERR_BOUND = 4, ERR_NONCONV = 5, ERR_CORRUPT = 6, ERR_INTERNAL = 7 };
enum { K_FPMAX = 0, K_FPMIN = 1, K_FNMAX = 2, K_FNMIN = 3 };
enum { RULE_SELF = 0, RULE_G_ASC = 1, RULE_F_DESC = 2 };

static _Thread_local char g_err[512];

static int fail(int kind, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return kind;
}

const char* mssz_oracle_last_error(void) { return g_err; }
void mssz_oracle_free(void* p) { free(p); }

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ---- grid topology: grid.cpp:8-16 (stencils), :23-37 (neighbors), :39-55 (build) ---- */

typedef struct {
  int ndims;
  uint64_t dims[3];
  uint64_t n;
} topo_t;

static const int kOff2[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {1, 1, 0}, {-1, -1, 0}};
static const int kOff3[14][3] = {{1, 0, 0},  {-1, 0, 0},  {0, 1, 0},  {0, -1, 0}, {0, 0, 1},
                                 {0, 0, -1}, {1, 1, 0},   {-1, -1, 0}, {0, 1, 1},  {0, -1, -1},
                                 {1, 0, 1},  {-1, 0, -1}, {1, 1, 1},  {-1, -1, -1}};

static int topo_build(int ndims, const uint64_t* dims, topo_t* t) {
  const uint64_t cap = (uint64_t)1 << 40; /* grid.cpp:19 */
  if (ndims != 2 && ndims != 3) return fail(ERR_USAGE, "dims must have 2 or 3 extents");
  t->ndims = ndims;
  t->dims[0] = t->dims[1] = t->dims[2] = 1;
  uint64_t count = 1;
  for (int a = 0; a < ndims; ++a) {
    if (dims[a] < 2) return fail(ERR_USAGE, "every grid extent must be >= 2");
    if (dims[a] > cap / count) return fail(ERR_USAGE, "grid exceeds the address-space cap");
    t->dims[a] = dims[a];
    count *= dims[a];
  }
  t->n = count;
  return 0;
}

/* Writes neighbours in stencil order; unsigned wraparound rejects -1. */
static int topo_neighbors(const topo_t* t, uint64_t v, uint64_t out[14]) {
  const uint64_t c0 = v % t->dims[0];
  const uint64_t c1 = (v / t->dims[0]) % t->dims[1];
  const uint64_t c2 = v / (t->dims[0] * t->dims[1]);
  const int (*off)[3] = t->ndims == 2 ? kOff2 : kOff3;
  const int stencil = t->ndims == 2 ? 6 : 14;
  int n = 0;
  for (int k = 0; k < stencil; ++k) {
    uint64_t x = c0 + (uint64_t)(int64_t)off[k][0];
    uint64_t y = c1 + (uint64_t)(int64_t)off[k][1];
    uint64_t z = c2 + (uint64_t)(int64_t)off[k][2];
    if (x >= t->dims[0] || y >= t->dims[1] || z >= t->dims[2]) continue;
    out[n++] = x + t->dims[0] * (y + t->dims[1] * z);
  }
  return n;
}

int mssz_oracle_build_topology(int ndims, const uint64_t* dims, uint64_t* vertex_count) {
  topo_t t;
  int rc = topo_build(ndims, dims, &t);
  if (rc) return rc;
  *vertex_count = t.n;
  return 0;
}

int mssz_oracle_neighbors(int ndims, const uint64_t* dims, uint64_t v, uint64_t* out, int* n) {
  topo_t t;
  int rc = topo_build(ndims, dims, &t);
  if (rc) return rc;
  if (v >= t.n) return fail(ERR_USAGE, "vertex out of range");
  *n = topo_neighbors(&t, v, out);
  return 0;
}

/* ---- labels: mss.cpp:51-97 (round-synchronous doubling, cap bit_width(n-1)+2) ---- */

static int bit_width_u64(uint64_t x) {
  int w = 0;
  while (x) {
    ++w;
    x >>= 1;
  }
  return w;
}

static int jump_to_fixpoint(uint64_t n, const uint64_t* parent, uint64_t* cur, uint64_t* next) {
  memcpy(cur, parent, sizeof(uint64_t) * n);
  const int cap = bit_width_u64(n - 1) + 2;
  uint64_t* src = cur;
  uint64_t* dst = next;
  for (int round = 0; round < cap; ++round) {
    int changed = 0;
    /* round-synchronous (reads src, writes dst): thread-count invariant */
#pragma omp parallel for schedule(static) reduction(| : changed)
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t hop = src[src[i]];
      dst[i] = hop;
      if (hop != src[i]) changed = 1;
    }
    uint64_t* tmp = src;
    src = dst;
    dst = tmp;
    if (!changed) {
      if (src != cur) memcpy(cur, src, sizeof(uint64_t) * n);
      return 0;
    }
  }
  return fail(ERR_INTERNAL, "path compression exceeded its round cap (corrupt direction field)");
}

static int labels_into(uint64_t n, const uint64_t* asc, const uint64_t* desc, uint64_t* M,
                       uint64_t* m, uint64_t* scratch) {
  int rc = jump_to_fixpoint(n, asc, M, scratch);
  if (rc) return rc;
  return jump_to_fixpoint(n, desc, m, scratch);
}

int mssz_oracle_compute_labels(int ndims, const uint64_t* dims, const uint64_t* asc,
                               const uint64_t* desc, uint64_t* max_label, uint64_t* min_label) {
  topo_t t;
  int rc = topo_build(ndims, dims, &t);
  if (rc) return rc;
  for (uint64_t i = 0; i < t.n; ++i)
    if (asc[i] >= t.n || desc[i] >= t.n) return fail(ERR_INTERNAL, "direction out of range");
  uint64_t* scratch = (uint64_t*)malloc(sizeof(uint64_t) * t.n);
  rc = labels_into(t.n, asc, desc, max_label, min_label, scratch);
  free(scratch);
  return rc;
}

/* ---- per-type body ---- */

#define T float
#define SUF f32
#define NEXTAFTER nextafterf
#include "mssz_oracle_body.inc"
#undef T
#undef SUF
#undef NEXTAFTER

#define T double
#define SUF f64
#define NEXTAFTER nextafter
#include "mssz_oracle_body.inc"
#undef T
#undef SUF
#undef NEXTAFTER
