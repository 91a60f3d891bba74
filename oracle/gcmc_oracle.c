/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference per-move
 * energy path (see gcmc_oracle.h). Citations are to
 * /root/reference/proj/include/gcmc/<file>:<line>. Compiled with
 * -ffp-contract=off so every a*b+c rounds twice, like the reference's
 * x86-64 build without -march (proj/CMakeLists.txt:1-18). */
#include "gcmc_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];
const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------ mt19937_64
 * The engine of RngStream (rng.hpp:84) is std::mt19937_64; its algorithm
 * is fixed by the C++ standard ([rand.eng.mers], [rand.predef]). */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x000000007FFFFFFFULL

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (uint64_t i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + i;
  r->idx = MT_N;
  r->draws = 0;
}

static void mt_twist(uint64_t* x) {
  int k;
  for (k = 0; k < MT_N - MT_M; ++k) {
    const uint64_t y = (x[k] & MT_UM) | (x[k + 1] & MT_LM);
    x[k] = x[k + MT_M] ^ (y >> 1) ^ ((y & 1) ? MT_A : 0);
  }
  for (; k < MT_N - 1; ++k) {
    const uint64_t y = (x[k] & MT_UM) | (x[k + 1] & MT_LM);
    x[k] = x[k + MT_M - MT_N] ^ (y >> 1) ^ ((y & 1) ? MT_A : 0);
  }
  const uint64_t y = (x[MT_N - 1] & MT_UM) | (x[0] & MT_LM);
  x[MT_N - 1] = x[MT_M - 1] ^ (y >> 1) ^ ((y & 1) ? MT_A : 0);
}

uint64_t orc_rng_next(orc_rng* r) {
  if (r->idx >= MT_N) {
    mt_twist(r->mt);
    r->idx = 0;
  }
  uint64_t z = r->mt[r->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

/* rng.hpp:28-31: top 53 bits / 2^53 */
double orc_uniform(orc_rng* r) {
  ++r->draws;
  return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53;
}

/* rng.hpp:38-41 */
uint64_t orc_index_from(double u, uint64_t n) {
  const uint64_t i = (uint64_t)(u * (double)n);
  return i < n ? i : n - 1;
}

/* ------------------------------------------------------------ box.hpp */
/* box.hpp:24-31 */
double orc_wrap_axis(double v, double l) {
  double r = fmod(v, l);
  if (r < 0.0) r += l;
  if (r >= l) r = 0.0;
  return r;
}

/* box.hpp:37-41 */
int orc_wrap_position(const double* p, double l, double* out) {
  if (!isfinite(p[0]) || !isfinite(p[1]) || !isfinite(p[2])) return -1;
  out[0] = orc_wrap_axis(p[0], l);
  out[1] = orc_wrap_axis(p[1], l);
  out[2] = orc_wrap_axis(p[2], l);
  return 0;
}

/* box.hpp:45-55 */
double orc_min_image_dist2(const double* a, const double* b, double l) {
  const double inv_l = 1.0 / l;
  double dx = a[0] - b[0];
  double dy = a[1] - b[1];
  double dz = a[2] - b[2];
  dx -= l * nearbyint(dx * inv_l);
  dy -= l * nearbyint(dy * inv_l);
  dz -= l * nearbyint(dz * inv_l);
  return dx * dx + dy * dy + dz * dz;
}

/* ------------------------------------------------------------ potential.hpp */
orc_lj orc_lj_make(double eps, double sigma, double rc) {
  orc_lj p = {eps, sigma, rc, sigma * sigma, rc * rc}; /* potential.hpp:25-26 */
  return p;
}

/* potential.hpp:39-46 */
int orc_lj_pair(double r2, const orc_lj* p, double* u, double* w) {
  if (!(r2 > 0.0)) return -1;
  if (r2 > p->r_cut2) {
    *u = 0.0;
    *w = 0.0;
    return 0;
  }
  const double s2 = p->sigma2 / r2;
  const double s6 = s2 * s2 * s2;
  const double s12 = s6 * s6;
  *u = 4.0 * p->epsilon * (s12 - s6);
  *w = 24.0 * p->epsilon * (2.0 * s12 - s6);
  return 0;
}

/* potential.hpp:51-54 (floor 1e-12 sigma^2, energy 1e30: :30,34) */
void orc_lj_pair_clamped(double r2, const orc_lj* p, double* u, double* w) {
  if (r2 < 1e-12 * p->sigma2) {
    *u = 1e30;
    *w = 1e30;
    return;
  }
  orc_lj_pair(r2, p, u, w);
}

/* potential.hpp:63-72 */
void orc_tail_corrections(double rho, double eps, double sigma, double rc, double* u, double* pr) {
  const double sr3 = (sigma / rc) * (sigma / rc) * (sigma / rc);
  const double sr9 = sr3 * sr3 * sr3;
  const double s3 = sigma * sigma * sigma;
  const double pi = 3.141592653589793238462643383279502884;
  *u = (8.0 / 3.0) * pi * rho * eps * s3 * (sr9 / 3.0 - sr3);
  *pr = (16.0 / 3.0) * pi * rho * rho * eps * s3 * (2.0 / 3.0 * sr9 - sr3);
}

/* ------------------------------------------------------------ engine.hpp:28-59 */
static double metropolis(double ratio) { return ratio < 1.0 ? ratio : 1.0; }
double orc_displacement_acceptance(double du, double beta) { return metropolis(exp(-beta * du)); }
double orc_insertion_acceptance(double du, uint64_t n, double v, double beta, double mu,
                                double lam) {
  const double l3 = lam * lam * lam;
  return metropolis(v / (l3 * (double)(n + 1)) * exp(beta * (mu - du)));
}
double orc_deletion_acceptance(double du, uint64_t n, double v, double beta, double mu,
                               double lam) {
  const double l3 = lam * lam * lam;
  return metropolis(l3 * (double)n / v * exp(-beta * (mu + du)));
}

/* ------------------------------------------------------------ grid geometry */
/* cell_grid.hpp:27-33 */
void orc_compute_cell_dims(double l, double rc, int32_t* dims, double* size) {
  int t = (int)(l / rc);
  while ((double)(t + 1) * rc <= l) ++t;
  while (t > 1 && (double)t * rc > l) --t;
  if (t < 3) t = 3;
  *dims = t;
  *size = l / t;
}
/* cell_grid.hpp:36-38 */
int32_t orc_default_cell_capacity(double rc, double sigma) { return rc <= 4.0 * sigma ? 48 : 96; }

/* microcell_grid.hpp:29-35 */
void orc_microcell_dims(double l, double sigma, int32_t* dims, double* last_w) {
  const double cells = l / sigma;
  const double whole = floor(cells);
  const double frac = cells - whole;
  if (frac < 1e-9) {
    *dims = (int32_t)llround(whole);
    *last_w = 1.0;
    return;
  }
  *dims = (int32_t)whole + 1;
  *last_w = frac;
}
/* microcell_grid.hpp:39-41 */
int32_t orc_microcell_extent(double rc, double sigma) { return (int32_t)ceil(rc / sigma); }

static int window_side(int j, int base, double deficit, double rc) {
  int k = base;
  while ((double)k - ((j >= 1 && j <= k) ? deficit : 0.0) < rc) ++k;
  return k;
}

/* microcell_grid.hpp:54-73 */
void orc_microcell_axis_window(int32_t center, double rc_abs, double sigma, int32_t dims,
                               double last_w, int32_t* lo, int32_t* count) {
  const double rc = rc_abs / sigma;
  const double deficit = 1.0 - last_w;
  const int base = orc_microcell_extent(rc_abs, sigma);
  int to_right = (dims - 1 - center) % dims;
  if (to_right < 0) to_right += dims;
  const int to_left = (center + 1) % dims;
  const int right = window_side(to_right, base, deficit, rc);
  const int left = window_side(to_left, base, deficit, rc);
  *lo = -left;
  *count = (left + right + 1 >= dims) ? dims : left + right + 1;
}

static long long arc_global_cell(double t, double l, double inv_sigma, int dims) {
  const double w = orc_wrap_axis(t, l);
  const long long k = llround((t - w) / l);
  int c = (int)(w * inv_sigma);
  if (c >= dims) c = dims - 1;
  return k * dims + c;
}

/* microcell_grid.hpp:85-103 */
void orc_microcell_axis_arc(double x, double rc, double sigma, double l, int32_t dims,
                            int32_t* first, int32_t* count) {
  const double pad = 1e-9 * sigma;
  const double inv_sigma = 1.0 / sigma;
  const long long lo = arc_global_cell(x - rc - pad, l, inv_sigma, dims);
  const long long span = arc_global_cell(x + rc + pad, l, inv_sigma, dims) - lo + 1;
  *first = (int32_t)(((lo % dims) + dims) % dims);
  *count = span >= dims ? dims : (int32_t)span;
}

/* grid_common.hpp:11-21 */
static void sort_ids(int32_t* ids, int n) {
  for (int i = 1; i < n; ++i) {
    const int32_t v = ids[i];
    int j = i - 1;
    while (j >= 0 && ids[j] > v) {
      ids[j + 1] = ids[j];
      --j;
    }
    ids[j + 1] = v;
  }
}

/* grid_common.hpp:27-47: returns count, fills out (<= 343 for h=3; caller sized) */
static int cube_axis(int c, int h, int dims, int* out) {
  const int count = (2 * h + 1) < dims ? (2 * h + 1) : dims;
  int v = (c - h) % dims;
  if (v < 0) v += dims;
  for (int i = 0; i < count; ++i) {
    out[i] = v;
    if (++v == dims) v = 0;
  }
  return count;
}

/* ------------------------------------------------------------ strategies */
typedef struct {
  double sum, c;
} kahan; /* kahan.hpp:8-20 */
static void kadd(kahan* k, double v) {
  const double y = v - k->c;
  const double t = k->sum + y;
  k->c = (t - k->sum) - y;
  k->sum = t;
}

struct orc_grid {
  int kind;
  double l;
  orc_lj lj;
  double* pos; /* AoS xyz */
  uint64_t n, capn;
  /* grid */
  int dims;
  double inv_cell;  /* cell list: 1/S; microcell: 1/sigma */
  double last_w;    /* microcell boundary cell width */
  int cap, peak;
  uint64_t ncells;
  int32_t* occ;
  int32_t* slots;
  int32_t* table; /* cell list: 27 per cell */
};

static const double* P(const orc_grid* g, uint64_t i) { return g->pos + 3 * i; }

static int coord(const orc_grid* g, double v) {
  const int c = (int)(v * g->inv_cell);
  return c < g->dims ? c : g->dims - 1;
}
int32_t orc_grid_cell_of(const orc_grid* g, const double* p) {
  return coord(g, p[0]) + g->dims * (coord(g, p[1]) + g->dims * coord(g, p[2]));
}

static uint64_t slot_index(const orc_grid* g, int cell, int k) {
  /* microcell slot-major k*ncells+c (microcell_grid.hpp:480);
   * cell list cell-major c*cap+k (cell_grid.hpp:245) */
  return g->kind == ORC_MICROCELL ? (uint64_t)k * g->ncells + (uint64_t)cell
                                  : (uint64_t)cell * g->cap + (uint64_t)k;
}

/* microcell_grid.hpp:472-483, cell_grid.hpp:237-248 */
static int insert_id(orc_grid* g, int cell, int32_t id) {
  int32_t* occ = &g->occ[cell];
  if (*occ >= g->cap) {
    snprintf(g_err, sizeof g_err,
             "%s: cell %d exceeds capacity %d (occupancy %d); rerun with a larger %s",
             g->kind == ORC_MICROCELL ? "microcell" : "cell_list", cell, g->cap, *occ,
             g->kind == ORC_MICROCELL ? "microcell_capacity" : "cell_capacity");
    return ORC_CELL_OVERFLOW;
  }
  g->slots[slot_index(g, cell, *occ)] = id;
  ++*occ;
  if (*occ > g->peak) g->peak = *occ;
  return ORC_OK;
}

/* microcell_grid.hpp:485-499, cell_grid.hpp:250-262 */
static int remove_id(orc_grid* g, int cell, int32_t id) {
  int32_t* occ = &g->occ[cell];
  for (int k = 0; k < *occ; ++k) {
    if (g->slots[slot_index(g, cell, k)] == id) {
      g->slots[slot_index(g, cell, k)] = g->slots[slot_index(g, cell, *occ - 1)];
      --*occ;
      return ORC_OK;
    }
  }
  snprintf(g_err, sizeof g_err, "particle %d not found in cell %d", id, cell);
  return ORC_NOT_FOUND;
}

/* microcell_grid.hpp:501-513, cell_grid.hpp:264-275 */
static int relabel_id(orc_grid* g, int cell, int32_t from, int32_t to) {
  for (int k = 0; k < g->occ[cell]; ++k) {
    if (g->slots[slot_index(g, cell, k)] == from) {
      g->slots[slot_index(g, cell, k)] = to;
      return ORC_OK;
    }
  }
  snprintf(g_err, sizeof g_err, "particle %d not found in cell %d", from, cell);
  return ORC_NOT_FOUND;
}

int32_t orc_grid_build(orc_grid* g) {
  if (g->kind == ORC_ALL_PAIRS) return ORC_OK;
  memset(g->occ, 0, g->ncells * sizeof(int32_t));
  for (uint64_t i = 0; i < g->n; ++i) {
    const int rc = insert_id(g, orc_grid_cell_of(g, P(g, i)), (int32_t)i);
    if (rc) return rc;
  }
  return ORC_OK;
}

orc_grid* orc_grid_create(int32_t kind, const double* xyz, uint64_t n, uint64_t capacity_n,
                          double l, double eps, double sigma, double rc, int32_t cell_cap,
                          int32_t* status) {
  orc_grid* g = (orc_grid*)calloc(1, sizeof *g);
  g->kind = kind;
  g->l = l;
  g->lj = orc_lj_make(eps, sigma, rc);
  g->capn = capacity_n > n ? capacity_n : n + 1;
  g->pos = (double*)malloc(3 * g->capn * sizeof(double));
  memcpy(g->pos, xyz, 3 * n * sizeof(double));
  g->n = n;
  if (kind == ORC_MICROCELL) {
    orc_microcell_dims(l, sigma, &g->dims, &g->last_w);
    g->inv_cell = 1.0 / sigma;
    g->cap = cell_cap > 0 ? cell_cap : 5; /* microcell_grid.hpp:149 */
  } else if (kind == ORC_CELL_LIST) {
    double size;
    orc_compute_cell_dims(l, rc, &g->dims, &size);
    g->inv_cell = 1.0 / size;
    g->cap = cell_cap > 0 ? cell_cap : orc_default_cell_capacity(rc, sigma);
  }
  if (kind != ORC_ALL_PAIRS) {
    const int d = g->dims;
    g->ncells = (uint64_t)d * d * d;
    g->occ = (int32_t*)calloc(g->ncells, sizeof(int32_t));
    g->slots = (int32_t*)malloc(g->ncells * g->cap * sizeof(int32_t));
    for (uint64_t i = 0; i < g->ncells * g->cap; ++i) g->slots[i] = -1;
    if (kind == ORC_CELL_LIST) { /* cell_grid.hpp:59-65 */
      g->table = (int32_t*)malloc(g->ncells * 27 * sizeof(int32_t));
      int xs[3], ys[3], zs[3];
      uint64_t t = 0;
      for (int z = 0; z < d; ++z)
        for (int y = 0; y < d; ++y)
          for (int x = 0; x < d; ++x) {
            cube_axis(x, 1, d, xs);
            cube_axis(y, 1, d, ys);
            cube_axis(z, 1, d, zs);
            for (int a = 0; a < 3; ++a)
              for (int b = 0; b < 3; ++b)
                for (int c = 0; c < 3; ++c) g->table[t++] = xs[c] + d * (ys[b] + d * zs[a]);
          }
    }
  }
  *status = orc_grid_build(g);
  return g;
}

void orc_grid_destroy(orc_grid* g) {
  if (!g) return;
  free(g->pos);
  free(g->occ);
  free(g->slots);
  free(g->table);
  free(g);
}
uint64_t orc_grid_size(const orc_grid* g) { return g->n; }
const double* orc_grid_positions(const orc_grid* g) { return g->pos; }
void orc_grid_info(const orc_grid* g, int32_t* dims, int32_t* cap, uint64_t* ncells) {
  *dims = g->dims;
  *cap = g->cap;
  *ncells = g->ncells;
}
const int32_t* orc_grid_occ(const orc_grid* g) { return g->occ; }
const int32_t* orc_grid_slots(const orc_grid* g) { return g->slots; }
int32_t orc_grid_peak(const orc_grid* g) { return g->peak; }

/* Visits occupants of one cell in ascending id order
 * (microcell_grid.hpp:341-356, cell_grid.hpp:208-221). */
typedef struct {
  const orc_grid* g;
  const double* a; /* first endpoint */
  const double* b; /* second endpoint or NULL */
  uint64_t exclude;
  kahan u, w, ub, wb;
} acc_ctx;

static void visit_pair(acc_ctx* x, uint64_t j) {
  if (j == x->exclude) return;
  const orc_grid* g = x->g;
  const double rc2 = g->lj.r_cut2;
  double u, w;
  const double r2 = orc_min_image_dist2(x->a, P(g, j), g->l);
  if (r2 <= rc2) {
    orc_lj_pair_clamped(r2, &g->lj, &u, &w);
    kadd(&x->u, u);
    kadd(&x->w, w);
  }
  if (x->b) {
    const double r2o = orc_min_image_dist2(x->b, P(g, j), g->l);
    if (r2o <= rc2) {
      orc_lj_pair_clamped(r2o, &g->lj, &u, &w);
      kadd(&x->ub, u);
      kadd(&x->wb, w);
    }
  }
}

static void visit_cell(acc_ctx* x, int c) {
  const orc_grid* g = x->g;
  const int occ = g->occ[c];
  if (occ == 0) return;
  int32_t ids[128];
  for (int k = 0; k < occ; ++k) ids[k] = g->slots[slot_index(g, c, k)];
  sort_ids(ids, occ);
  for (int k = 0; k < occ; ++k) visit_pair(x, (uint64_t)ids[k]);
}

/* Cells x-fastest over axis lists (microcell_grid.hpp:392-409, 435-456). */
static void visit_box(acc_ctx* x, const int* xs, int nx, const int* ys, int ny, const int* zs,
                      int nz) {
  const int d = x->g->dims;
  for (int iz = 0; iz < nz; ++iz)
    for (int iy = 0; iy < ny; ++iy)
      for (int ix = 0; ix < nx; ++ix) visit_cell(x, xs[ix] + d * (ys[iy] + d * zs[iz]));
}

static int fill_run(int first, int count, int dims, int* out) {
  int v = first;
  for (int i = 0; i < count; ++i) {
    out[i] = v;
    if (++v == dims) v = 0;
  }
  return count;
}

/* Per-position arc window (microcell_grid.hpp:393-409) */
static void micro_arc_box(const orc_grid* g, const double* p, int* xs, int* nx, int* ys, int* ny,
                          int* zs, int* nz) {
  int32_t f, c;
  orc_microcell_axis_arc(p[0], g->lj.r_cut, g->lj.sigma, g->l, g->dims, &f, &c);
  *nx = fill_run(f, c, g->dims, xs);
  orc_microcell_axis_arc(p[1], g->lj.r_cut, g->lj.sigma, g->l, g->dims, &f, &c);
  *ny = fill_run(f, c, g->dims, ys);
  orc_microcell_axis_arc(p[2], g->lj.r_cut, g->lj.sigma, g->l, g->dims, &f, &c);
  *nz = fill_run(f, c, g->dims, zs);
}

/* Same-cell window (microcell_grid.hpp:301-311, 435-456) */
static int micro_window_axis(const orc_grid* g, int center, int* out) {
  int32_t lo, count;
  orc_microcell_axis_window(center, g->lj.r_cut, g->lj.sigma, g->dims, g->last_w, &lo, &count);
  int v = (center + lo) % g->dims;
  if (v < 0) v += g->dims;
  return fill_run(v, count, g->dims, out);
}

/* sum over the window around p (strategy-specific), excluding `exclude`;
 * b != NULL evaluates a second endpoint over the same window. */
static void sum_window(acc_ctx* x, int mode_cell, int cell) {
  const orc_grid* g = x->g;
  if (g->kind == ORC_ALL_PAIRS) { /* strategy.hpp:64-116 */
    for (uint64_t j = 0; j < g->n; ++j) visit_pair(x, j);
    return;
  }
  if (g->kind == ORC_CELL_LIST) { /* cell_grid.hpp:208-221 */
    const int32_t* t = &g->table[(uint64_t)cell * 27];
    for (int i = 0; i < 27; ++i) visit_cell(x, t[i]);
    return;
  }
  int xs[512], ys[512], zs[512], nx, ny, nz;
  if (mode_cell) {
    const int d = g->dims;
    nx = micro_window_axis(g, cell % d, xs);
    ny = micro_window_axis(g, (cell / d) % d, ys);
    nz = micro_window_axis(g, cell / (d * d), zs);
  } else {
    micro_arc_box(g, x->a, xs, &nx, ys, &ny, zs, &nz);
  }
  visit_box(x, xs, nx, ys, ny, zs, nz);
}

static void sum_around(const orc_grid* g, const double* p, uint64_t exclude, double* u,
                       double* w) {
  acc_ctx x;
  memset(&x, 0, sizeof x);
  x.g = g;
  x.a = p;
  x.exclude = exclude;
  sum_window(&x, 0, g->kind == ORC_CELL_LIST ? orc_grid_cell_of(g, p) : 0);
  *u = x.u.sum;
  *w = x.w.sum;
}

static int require_valid(const orc_grid* g, uint64_t pid) {
  if (pid >= g->n) {
    snprintf(g_err, sizeof g_err, "%s: invalid particle id",
             g->kind == ORC_ALL_PAIRS ? "all_pairs"
                                      : (g->kind == ORC_CELL_LIST ? "cell_list" : "microcell"));
    return ORC_INVALID_PID;
  }
  return ORC_OK;
}

/* strategy.hpp:64-87, cell_grid.hpp:97-126, microcell_grid.hpp:200-231 */
int32_t orc_delta_displace(const orc_grid* g, uint64_t pid, const double* p, double* du,
                           double* dw) {
  if (require_valid(g, pid)) return ORC_INVALID_PID;
  double old[3] = {P(g, pid)[0], P(g, pid)[1], P(g, pid)[2]};
  const int both = g->kind == ORC_ALL_PAIRS ||
                   orc_grid_cell_of(g, old) == orc_grid_cell_of(g, p);
  if (both) {
    acc_ctx x;
    memset(&x, 0, sizeof x);
    x.g = g;
    x.a = p;
    x.b = old;
    x.exclude = pid;
    sum_window(&x, 1, g->kind == ORC_ALL_PAIRS ? 0 : orc_grid_cell_of(g, p));
    *du = x.u.sum - x.ub.sum;
    *dw = x.w.sum - x.wb.sum;
    return ORC_OK;
  }
  double nu, nw, ou, ow;
  sum_around(g, p, pid, &nu, &nw);
  sum_around(g, old, pid, &ou, &ow);
  *du = nu - ou;
  *dw = nw - ow;
  return ORC_OK;
}

int32_t orc_delta_insert(const orc_grid* g, const double* p, double* du, double* dw) {
  sum_around(g, p, g->n, du, dw);
  return ORC_OK;
}

int32_t orc_delta_delete(const orc_grid* g, uint64_t pid, double* du, double* dw) {
  if (require_valid(g, pid)) return ORC_INVALID_PID;
  double u, w;
  sum_around(g, P(g, pid), pid, &u, &w);
  *du = -u;
  *dw = -w;
  return ORC_OK;
}

static int grow(orc_grid* g) {
  if (g->n < g->capn) return 0;
  g->capn *= 2;
  g->pos = (double*)realloc(g->pos, 3 * g->capn * sizeof(double));
  return 0;
}

/* microcell_grid.hpp:243-251 */
int32_t orc_commit_displace(orc_grid* g, uint64_t pid, const double* p) {
  if (require_valid(g, pid)) return ORC_INVALID_PID;
  double* q = g->pos + 3 * pid;
  if (g->kind == ORC_ALL_PAIRS) {
    memcpy(q, p, 3 * sizeof(double));
    return ORC_OK;
  }
  const int oc = orc_grid_cell_of(g, q), nc = orc_grid_cell_of(g, p);
  memcpy(q, p, 3 * sizeof(double));
  if (oc == nc) return ORC_OK;
  int rc = remove_id(g, oc, (int32_t)pid);
  if (rc) return rc;
  return insert_id(g, nc, (int32_t)pid);
}

/* microcell_grid.hpp:253-257 */
int32_t orc_commit_insert(orc_grid* g, const double* p, uint64_t* pid) {
  grow(g);
  memcpy(g->pos + 3 * g->n, p, 3 * sizeof(double));
  *pid = g->n++;
  if (g->kind == ORC_ALL_PAIRS) return ORC_OK;
  return insert_id(g, orc_grid_cell_of(g, p), (int32_t)*pid);
}

/* microcell_grid.hpp:259-268 + particles.hpp:35-41 */
int32_t orc_commit_delete(orc_grid* g, uint64_t pid) {
  if (require_valid(g, pid)) return ORC_INVALID_PID;
  const uint64_t last = g->n - 1;
  if (g->kind != ORC_ALL_PAIRS) {
    int rc = remove_id(g, orc_grid_cell_of(g, P(g, pid)), (int32_t)pid);
    if (rc) return rc;
    if (pid != last) {
      rc = relabel_id(g, orc_grid_cell_of(g, P(g, last)), (int32_t)last, (int32_t)pid);
      if (rc) return rc;
    }
  }
  if (pid != last) memcpy(g->pos + 3 * pid, g->pos + 3 * last, 3 * sizeof(double));
  g->n--;
  return ORC_OK;
}

static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* microcell_grid.hpp:270-292 / cell_grid.hpp:168-191: per-cell sorted
 * occupant sets equal a fresh binning. */
int32_t orc_rebuild_check(const orc_grid* g) {
  if (g->kind == ORC_ALL_PAIRS) return 1;
  int32_t* occ = (int32_t*)calloc(g->ncells, sizeof(int32_t));
  int32_t* fresh = (int32_t*)malloc(g->ncells * g->cap * sizeof(int32_t));
  int clean = 1;
  for (uint64_t i = 0; i < g->n && clean; ++i) {
    const int c = orc_grid_cell_of(g, P(g, i));
    if (occ[c] >= g->cap) {
      snprintf(g_err, sizeof g_err, "rebin overflow in cell %d", c);
      clean = 0;
      break;
    }
    fresh[(uint64_t)c * g->cap + occ[c]++] = (int32_t)i;
  }
  for (uint64_t c = 0; c < g->ncells && clean; ++c) {
    if (occ[c] != g->occ[c]) {
      snprintf(g_err, sizeof g_err, "cell %llu: occupancy %d, rebinned %d",
               (unsigned long long)c, g->occ[c], occ[c]);
      clean = 0;
      break;
    }
    int32_t a[128];
    for (int k = 0; k < occ[c]; ++k) a[k] = g->slots[slot_index(g, (int)c, k)];
    qsort(a, (size_t)occ[c], sizeof(int32_t), cmp_i32);
    qsort(fresh + c * g->cap, (size_t)occ[c], sizeof(int32_t), cmp_i32);
    if (memcmp(a, fresh + c * g->cap, (size_t)occ[c] * sizeof(int32_t)) != 0) {
      snprintf(g_err, sizeof g_err, "cell %llu: occupant sets differ from fresh binning",
               (unsigned long long)c);
      clean = 0;
    }
  }
  free(occ);
  free(fresh);
  return clean;
}

/* engine.hpp:74-94 */
int32_t orc_total_energy(const double* xyz, uint64_t n, double l, double eps, double sigma,
                         double rc, double* u, double* w) {
  const orc_lj lj = orc_lj_make(eps, sigma, rc);
  kahan ku = {0, 0}, kw = {0, 0};
  const double floor2 = 1e-12 * lj.sigma2;
  for (uint64_t i = 0; i + 1 < n; ++i) {
    for (uint64_t j = i + 1; j < n; ++j) {
      const double r2 = orc_min_image_dist2(xyz + 3 * i, xyz + 3 * j, l);
      if (r2 > lj.r_cut2) continue;
      if (r2 < floor2) {
        snprintf(g_err, sizeof g_err, "total_energy: particles %llu and %llu overlap",
                 (unsigned long long)i, (unsigned long long)j);
        return ORC_OVERLAP;
      }
      double pu, pw;
      orc_lj_pair(r2, &lj, &pu, &pw);
      kadd(&ku, pu);
      kadd(&kw, pw);
    }
  }
  *u = ku.sum;
  *w = kw.sum;
  return ORC_OK;
}

/* init_config.hpp:19-64 (coarse grid with per-cell linked lists; the clash
 * test's outcome does not depend on visit order). */
int32_t orc_random_initial_configuration(uint64_t n, double l, double min_sep, orc_rng* r,
                                         double* out) {
  int dims = (int)(l / min_sep);
  if (dims < 1) dims = 1;
  const double inv_width = dims / l;
  const uint64_t ncells = (uint64_t)dims * dims * dims;
  int64_t* head = (int64_t*)malloc(ncells * sizeof(int64_t));
  int64_t* next = (int64_t*)malloc((n ? n : 1) * sizeof(int64_t));
  for (uint64_t c = 0; c < ncells; ++c) head[c] = -1;
  const double min_sep2 = min_sep * min_sep;
  uint64_t count = 0, rejects = 0;
#define CRD(v) ((int)((v) * inv_width) < dims ? (int)((v) * inv_width) : dims - 1)
  while (count < n) {
    double raw[3];
    raw[0] = orc_uniform(r) * l;
    raw[1] = orc_uniform(r) * l;
    raw[2] = orc_uniform(r) * l;
    double c3[3];
    orc_wrap_position(raw, l, c3);
    int xs[3], ys[3], zs[3];
    const int nx = cube_axis(CRD(c3[0]), 1, dims, xs);
    const int ny = cube_axis(CRD(c3[1]), 1, dims, ys);
    const int nz = cube_axis(CRD(c3[2]), 1, dims, zs);
    int clash = 0;
    for (int a = 0; a < nz && !clash; ++a)
      for (int b = 0; b < ny && !clash; ++b)
        for (int c = 0; c < nx && !clash; ++c)
          for (int64_t j = head[xs[c] + dims * (ys[b] + dims * zs[a])]; j >= 0; j = next[j])
            if (orc_min_image_dist2(c3, out + 3 * j, l) < min_sep2) {
              clash = 1;
              break;
            }
    if (clash) {
      if (++rejects >= 1000000) {
        snprintf(g_err, sizeof g_err, "initial configuration: too many consecutive rejections");
        free(head);
        free(next);
        return ORC_ARG;
      }
      continue;
    }
    rejects = 0;
    memcpy(out + 3 * count, c3, sizeof c3);
    const uint64_t cell = CRD(c3[0]) + dims * (CRD(c3[1]) + dims * (uint64_t)CRD(c3[2]));
    next[count] = head[cell];
    head[cell] = (int64_t)count;
    ++count;
  }
#undef CRD
  free(head);
  free(next);
  return ORC_OK;
}

/* ------------------------------------------------------------ Simulation */
struct orc_sim {
  orc_params p;
  orc_grid* g;
  orc_rng rng;
  orc_state st;
  double volume, beta;
};

orc_sim* orc_sim_create(const orc_params* p, const double* xyz, uint64_t n, const orc_rng* rng,
                        uint64_t step, double energy, double virial, int32_t* status) {
  orc_sim* s = (orc_sim*)calloc(1, sizeof *s);
  s->p = *p;
  const double l = p->box_length;
  const double vol = l * l * l;
  const uint64_t capn = (uint64_t)(vol * 1.5) + n + 64;
  const int cap = p->strategy == ORC_MICROCELL ? p->microcell_capacity : p->cell_capacity;
  s->g = orc_grid_create(p->strategy, xyz, n, capn, l, p->epsilon, p->sigma, p->r_cut, cap, status);
  s->rng = *rng;
  s->st.step = step;
  s->st.energy = energy;
  s->st.virial = virial;
  s->volume = vol;
  s->beta = 1.0 / p->temperature; /* config.hpp:66 */
  return s;
}

void orc_sim_destroy(orc_sim* s) {
  if (!s) return;
  orc_grid_destroy(s->g);
  free(s);
}

static double sim_density(const orc_sim* s) { return (double)s->g->n / s->volume; }

/* engine.hpp:277-291 */
static double sim_pressure(const orc_sim* s) {
  double pr = sim_density(s) * s->p.temperature + s->st.virial / (3.0 * s->volume);
  if (s->p.tail_corrections) {
    double tu, tp;
    orc_tail_corrections(sim_density(s), s->p.epsilon, s->p.sigma, s->p.r_cut, &tu, &tp);
    pr += tp;
  }
  return pr;
}
static double sim_reported_energy(const orc_sim* s) {
  double u = s->st.energy;
  if (s->p.tail_corrections) {
    double tu, tp;
    orc_tail_corrections(sim_density(s), s->p.epsilon, s->p.sigma, s->p.r_cut, &tu, &tp);
    u += (double)s->g->n * tu;
  }
  return u;
}

/* engine.hpp:345-348 */
static void point_from(const orc_sim* s, double u1, double u2, double u3, double* out) {
  const double l = s->p.box_length;
  const double raw[3] = {u1 * l, u2 * l, u3 * l};
  orc_wrap_position(raw, l, out);
}

/* engine.hpp:293-308, 350-426 */
int32_t orc_sim_run(orc_sim* s, uint64_t nsteps, orc_outcome* trace) {
  for (uint64_t it = 0; it < nsteps; ++it) {
    orc_outcome o = {0, 0, 0.0, 0.0, 0.0, 0};
    int rc = ORC_OK;
    const double selector = orc_uniform(&s->rng);
    if (selector < s->p.displace_percent) {
      o.kind = 0;
      ++s->st.attempted[0];
      const double pick = orc_uniform(&s->rng);
      const double u1 = orc_uniform(&s->rng), u2 = orc_uniform(&s->rng), u3 = orc_uniform(&s->rng);
      const double acc = orc_uniform(&s->rng);
      if (s->g->n > 0) {
        const uint64_t pid = orc_index_from(pick, s->g->n);
        double np[3];
        if (s->p.max_displacement > 0.0) {
          const double cap = s->p.max_displacement;
          const double* q = P(s->g, pid);
          const double raw[3] = {q[0] + (2.0 * u1 - 1.0) * cap, q[1] + (2.0 * u2 - 1.0) * cap,
                                 q[2] + (2.0 * u3 - 1.0) * cap};
          orc_wrap_position(raw, s->p.box_length, np);
        } else {
          point_from(s, u1, u2, u3, np);
        }
        orc_delta_displace(s->g, pid, np, &o.delta_u, &o.delta_w);
        o.acceptance_prob = orc_displacement_acceptance(o.delta_u, s->beta);
        if (acc < o.acceptance_prob) {
          rc = orc_commit_displace(s->g, pid, np);
          o.accepted = 1;
        }
      }
    } else if (orc_uniform(&s->rng) < 0.5) {
      o.kind = 2;
      ++s->st.attempted[2];
      const double pick = orc_uniform(&s->rng);
      const double acc = orc_uniform(&s->rng);
      if (s->g->n > 0) {
        const uint64_t pid = orc_index_from(pick, s->g->n);
        orc_delta_delete(s->g, pid, &o.delta_u, &o.delta_w);
        o.acceptance_prob = orc_deletion_acceptance(o.delta_u, s->g->n, s->volume, s->beta,
                                                    s->p.chemical_potential, s->p.lambda);
        if (acc < o.acceptance_prob) {
          rc = orc_commit_delete(s->g, pid);
          o.accepted = 1;
        }
      }
    } else {
      o.kind = 1;
      ++s->st.attempted[1];
      const double u1 = orc_uniform(&s->rng), u2 = orc_uniform(&s->rng), u3 = orc_uniform(&s->rng);
      const double acc = orc_uniform(&s->rng);
      double np[3];
      point_from(s, u1, u2, u3, np);
      orc_delta_insert(s->g, np, &o.delta_u, &o.delta_w);
      o.acceptance_prob = orc_insertion_acceptance(o.delta_u, s->g->n, s->volume, s->beta,
                                                   s->p.chemical_potential, s->p.lambda);
      if (acc < o.acceptance_prob) {
        uint64_t pid;
        rc = orc_commit_insert(s->g, np, &pid);
        o.accepted = 1;
      }
    }
    if (rc) return rc;
    if (o.accepted) { /* engine.hpp:413-417 */
      s->st.energy += o.delta_u;
      s->st.virial += o.delta_w;
      ++s->st.accepted[o.kind];
    }
    ++s->st.step;
    if (s->st.step > s->p.equilibration_steps &&
        (s->st.step - s->p.equilibration_steps) % s->p.sampling_interval == 0) {
      ++s->st.samples; /* engine.hpp:419-426 */
      const double n = (double)s->g->n;
      s->st.sum_n += n;
      s->st.sum_n2 += n * n;
      s->st.sum_u += sim_reported_energy(s);
      s->st.sum_p += sim_pressure(s);
    }
    o.n_after = s->g->n;
    if (trace) trace[it] = o;
  }
  return ORC_OK;
}

void orc_sim_state(const orc_sim* s, orc_state* out) { *out = s->st; }
const orc_grid* orc_sim_grid(const orc_sim* s) { return s->g; }
const orc_rng* orc_sim_rng(const orc_sim* s) { return &s->rng; }
