/*
 * TEST INFRASTRUCTURE ONLY — see taskmd_oracle.h. Plain-C restatement of the
 * reference taskmd LJ path (single subnode: n_sub = 1), with compensated sums.
 * Reference citations are relative to /root/reference/proj/include/taskmd/.
 */
#include "taskmd_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---- LJ (potentials.hpp:41-75) ------------------------------------------ */

void tmo_lj_prepare(double eps, double sigma, double rc, int shifted, tmo_lj* q) {
  /* lj_prepare, potentials.hpp:49-61 */
  q->sigma2 = sigma * sigma;
  q->rc2 = rc * rc;
  q->eps4 = 4.0 * eps;
  q->eps24 = 24.0 * eps;
  q->shift = 0.0;
  if (shifted) {
    const double s2 = q->sigma2 / q->rc2;
    const double s6 = s2 * s2 * s2;
    q->shift = q->eps4 * (s6 * s6 - s6);
  }
}

void tmo_lj_eval(double r2, const tmo_lj* p, double* energy, double* ff) {
  /* lj_eval, potentials.hpp:65-75: exactly zero at and beyond the cutoff */
  if (r2 >= p->rc2) {
    *energy = 0.0;
    *ff = 0.0;
    return;
  }
  const double inv = p->sigma2 / r2;
  const double i6 = inv * inv * inv;
  *energy = p->eps4 * (i6 * i6 - i6) - p->shift;
  *ff = p->eps24 * (2.0 * i6 * i6 - i6) / r2;
}

/* ---- box / grid (box.hpp:47-51, cell_grid.hpp:36-78) -------------------- */

double tmo_wrap1(double p, double length) {
  double r = p - length * floor(p / length);
  if (r >= length) r -= length;
  return r;
}

int tmo_cell_grid(const double box[3], double r_cut, double r_skin, int dims[3],
                  double cell_len[3]) {
  /* build_cell_grid, cell_grid.hpp:54-78 */
  if (!(r_cut > 0.0) || !isfinite(r_cut)) return 1;
  if (!(r_skin >= 0.0) || !isfinite(r_skin)) return 1;
  const double rv = r_cut + r_skin;
  for (int k = 0; k < 3; ++k) {
    if (!isfinite(box[k]) || box[k] <= 0.0) return 1;
    if (box[k] < rv) return 1;
    const int d = (int)floor(box[k] / rv);
    dims[k] = d < 1 ? 1 : d;
  }
  for (int k = 0; k < 3; ++k) cell_len[k] = box[k] / dims[k];
  return 0;
}

static int coord1(double p, double len, int dims) {
  /* cell_coords, cell_grid.hpp:36-46 */
  int v = (int)floor(p / len);
  if (v < 0) v = 0;
  if (v >= dims) v = dims - 1;
  return v;
}

int tmo_cell_of(const double p[3], const int dims[3], const double cell_len[3]) {
  const int cx = coord1(p[0], cell_len[0], dims[0]);
  const int cy = coord1(p[1], cell_len[1], dims[1]);
  const int cz = coord1(p[2], cell_len[2], dims[2]);
  return cx + dims[0] * (cy + dims[1] * cz); /* linear, cell_grid.hpp:26-28 */
}

/* ---- counter RNG (random.hpp:23-81) -------------------------------------- */

static uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static uint64_t chash(uint64_t seed, uint64_t ctx, uint64_t step, uint64_t id,
                      uint64_t lane) {
  uint64_t h = mix64(seed ^ 0x243f6a8885a308d3ull);
  h = mix64(h ^ ctx);
  h = mix64(h ^ step);
  h = mix64(h ^ id);
  return mix64(h ^ lane);
}

static double u_co(uint64_t b) { return (double)(b >> 11) * 0x1.0p-53; }
static double u_oc(uint64_t b) { return (double)((b >> 11) + 1) * 0x1.0p-53; }

void tmo_counter_uniform3(uint64_t seed, uint64_t ctx, uint64_t step, uint64_t id,
                          double out[3]) {
  for (int l = 0; l < 3; ++l) out[l] = u_co(chash(seed, ctx, step, id, (uint64_t)l));
}

void tmo_counter_normal3(uint64_t seed, uint64_t ctx, uint64_t step, uint64_t id,
                         double out[3]) {
  const double a0 = u_oc(chash(seed, ctx, step, id, 0));
  const double a1 = u_co(chash(seed, ctx, step, id, 1));
  const double a2 = u_oc(chash(seed, ctx, step, id, 2));
  const double a3 = u_co(chash(seed, ctx, step, id, 3));
  const double two_pi = 6.283185307179586476925286766559;
  const double r0 = sqrt(-2.0 * log(a0));
  const double r1 = sqrt(-2.0 * log(a2));
  out[0] = r0 * cos(two_pi * a1);
  out[1] = r0 * sin(two_pi * a1);
  out[2] = r1 * cos(two_pi * a3);
}

void tmo_thermal_velocities(int64_t n, const int64_t* id, const double* mass,
                            double temperature, uint64_t seed, double* vel) {
  /* thermal_velocities + zero_net_momentum, generators.hpp:19-39 */
  double p[3] = {0.0, 0.0, 0.0}, mt = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    const double m = mass ? mass[k] : 1.0;
    const double sc = sqrt(temperature / m);
    double g[3];
    tmo_counter_normal3(seed, 2 /* kVelocityInit */, 0, (uint64_t)id[k], g);
    for (int a = 0; a < 3; ++a) vel[3 * k + a] = sc * g[a];
  }
  for (int64_t k = 0; k < n; ++k) {
    const double m = mass ? mass[k] : 1.0;
    for (int a = 0; a < 3; ++a) p[a] += m * vel[3 * k + a];
    mt += m;
  }
  if (mt == 0.0) return;
  const double inv = 1.0 / mt;
  double drift[3];
  for (int a = 0; a < 3; ++a) drift[a] = inv * p[a];
  for (int64_t k = 0; k < n; ++k)
    for (int a = 0; a < 3; ++a) vel[3 * k + a] -= drift[a];
}

int tmo_gen_fcc(int cells, double rho, double offset, int64_t* id, double* pos,
                double box[3]) {
  /* FCC lattice of SURVEY §8(d) (absent from generators.hpp) */
  static const double b[4][3] = {{0, 0, 0}, {0.5, 0.5, 0}, {0.5, 0, 0.5}, {0, 0.5, 0.5}};
  if (cells < 1 || !(rho > 0.0)) return 1;
  const int64_t n = 4LL * cells * cells * cells;
  const double L = cbrt((double)n / rho);
  const double a = L / cells;
  int64_t k = 0;
  for (int z = 0; z < cells; ++z)
    for (int y = 0; y < cells; ++y)
      for (int x = 0; x < cells; ++x)
        for (int q = 0; q < 4; ++q, ++k) {
          id[k] = k;
          pos[3 * k] = (x + b[q][0] + offset) * a;
          pos[3 * k + 1] = (y + b[q][1] + offset) * a;
          pos[3 * k + 2] = (z + b[q][2] + offset) * a;
        }
  box[0] = box[1] = box[2] = L;
  return 0;
}

/* ---- compensated accumulation ------------------------------------------- */

typedef struct {
  long double s, c;
} nsum;

static void nadd(nsum* a, long double x) { /* Neumaier */
  const long double t = a->s + x;
  if (fabsl(a->s) >= fabsl(x)) a->c += (a->s - t) + x;
  else a->c += (x - t) + a->s;
  a->s = t;
}
static long double nval(const nsum* a) { return a->s + a->c; }

/* ---- system --------------------------------------------------------------- */

typedef struct {
  int32_t a, b;
  uint8_t code[3]; /* image of b: 0 none, 1 +L, 2 -L (ghost shift, subnode.hpp:84-90) */
} hpair;

struct tmo_system {
  int64_t n;
  int64_t *id;
  double *mass, *pos, *vel, *snap;
  nsum* f;          /* per-particle compensated forces */
  double* fd;       /* rounded forces (what the integrator uses) */
  double box[3];
  int dims[3];
  double cell_len[3];
  int ncells;
  double rv2, thr, dt;
  tmo_lj lj;
  int32_t *cell, *start, *items; /* CSR cell lists, ascending id inside a cell */
  hpair* pairs;
  int64_t npairs, cap;
  int64_t step;
  uint64_t rebuilds;
  long double pe, w;
  char err[256];
};


static int64_t* g_sort_ids; /* qsort has no context argument in C11 */
static int by_id(const void* x, const void* y) {
  const int64_t a = g_sort_ids[*(const int32_t*)x], b = g_sort_ids[*(const int32_t*)y];
  return (a > b) - (a < b);
}

/* distribute_records (domain.hpp:54-65): wrap every position, bin by cell. */
static int resort(tmo_system* s) {
  for (int64_t k = 0; k < s->n; ++k) {
    double* p = s->pos + 3 * k;
    if (!isfinite(p[0]) || !isfinite(p[1]) || !isfinite(p[2])) {
      snprintf(s->err, sizeof s->err, "non-finite position for particle id %lld",
               (long long)s->id[k]);
      return 2;
    }
    for (int a = 0; a < 3; ++a) p[a] = tmo_wrap1(p[a], s->box[a]);
    s->cell[k] = tmo_cell_of(p, s->dims, s->cell_len);
  }
  memset(s->start, 0, sizeof(int32_t) * (size_t)(s->ncells + 1));
  for (int64_t k = 0; k < s->n; ++k) s->start[s->cell[k] + 1]++;
  for (int c = 0; c < s->ncells; ++c) s->start[c + 1] += s->start[c];
  int32_t* fill = calloc((size_t)s->ncells, sizeof(int32_t));
  for (int64_t k = 0; k < s->n; ++k) {
    const int c = s->cell[k];
    s->items[s->start[c] + fill[c]++] = (int32_t)k;
  }
  free(fill);
  g_sort_ids = s->id;
  for (int c = 0; c < s->ncells; ++c) {
    qsort(s->items + s->start[c], (size_t)(s->start[c + 1] - s->start[c]),
          sizeof(int32_t), by_id);
  }
  return 0;
}

static double image(double x, uint8_t code, double L) {
  /* ghost copy position: source + shift (decomp.hpp:191-193) */
  return code == 0 ? x : (code == 1 ? x + L : x + (-L));
}

/* build_sorted_list (neighbor_list.hpp:51-111) as a pair set: same-cell
 * b after a, then the 13 half-stencil offsets (neighbor_list.hpp:35-44) with
 * periodic ghost images; own image skipped when the stencil wraps onto the
 * source cell (91-93); keep r2 <= rv2 (inclusive, 83/95). */
static void build_pairs(tmo_system* s) {
  static const int st[13][3] = {{1, -1, -1}, {1, 0, -1}, {1, 1, -1}, {1, -1, 0},
                                {1, 0, 0},   {1, 1, 0},  {1, -1, 1}, {1, 0, 1},
                                {1, 1, 1},   {0, 1, -1}, {0, 1, 0},  {0, 1, 1},
                                {0, 0, 1}};
  s->npairs = 0;
  for (int c = 0; c < s->ncells; ++c) {
    const int cc[3] = {c % s->dims[0], (c / s->dims[0]) % s->dims[1],
                       c / (s->dims[0] * s->dims[1])};
    for (int32_t ia = s->start[c]; ia < s->start[c + 1]; ++ia) {
      const int32_t a = s->items[ia];
      const double* pa = s->pos + 3 * a;
      for (int32_t ib = ia + 1; ib < s->start[c + 1]; ++ib) {
        const int32_t b = s->items[ib];
        const double* pb = s->pos + 3 * b;
        const double dx = pa[0] - pb[0], dy = pa[1] - pb[1], dz = pa[2] - pb[2];
        if (dx * dx + dy * dy + dz * dz <= s->rv2) {
          if (s->npairs == s->cap) {
            s->cap = s->cap * 2 + 1024;
            s->pairs = realloc(s->pairs, sizeof(hpair) * (size_t)s->cap);
          }
          hpair h = {a, b, {0, 0, 0}};
          s->pairs[s->npairs++] = h;
        }
      }
      for (int o = 0; o < 13; ++o) {
        int t[3];
        uint8_t code[3];
        for (int k = 0; k < 3; ++k) {
          t[k] = cc[k] + st[o][k];
          code[k] = 0;
          if (t[k] < 0) { t[k] += s->dims[k]; code[k] = 2; }
          else if (t[k] >= s->dims[k]) { t[k] -= s->dims[k]; code[k] = 1; }
        }
        const int tc = t[0] + s->dims[0] * (t[1] + s->dims[1] * t[2]);
        for (int32_t ib = s->start[tc]; ib < s->start[tc + 1]; ++ib) {
          const int32_t b = s->items[ib];
          if (tc == c && s->id[b] == s->id[a]) continue;
          const double* pb = s->pos + 3 * b;
          const double dx = pa[0] - image(pb[0], code[0], s->box[0]);
          const double dy = pa[1] - image(pb[1], code[1], s->box[1]);
          const double dz = pa[2] - image(pb[2], code[2], s->box[2]);
          if (dx * dx + dy * dy + dz * dz <= s->rv2) {
            if (s->npairs == s->cap) {
              s->cap = s->cap * 2 + 1024;
              s->pairs = realloc(s->pairs, sizeof(hpair) * (size_t)s->cap);
            }
            hpair h = {a, b, {code[0], code[1], code[2]}};
            s->pairs[s->npairs++] = h;
          }
        }
      }
    }
  }
  memcpy(s->snap, s->pos, sizeof(double) * 3 * (size_t)s->n);
}

/* compute_pair_forces (neighbor_list.hpp:150-187) over the pair set, with
 * compensated per-particle force, PE and virial sums. */
static int forces(tmo_system* s) {
  for (int64_t k = 0; k < s->n; ++k) {
    for (int a = 0; a < 3; ++a) s->f[3 * k + a].s = s->f[3 * k + a].c = 0.0L;
  }
  nsum pe = {0, 0}, w = {0, 0};
  for (int64_t q = 0; q < s->npairs; ++q) {
    const hpair* h = s->pairs + q;
    const double* pa = s->pos + 3 * h->a;
    const double* pb = s->pos + 3 * h->b;
    const double d[3] = {pa[0] - image(pb[0], h->code[0], s->box[0]),
                         pa[1] - image(pb[1], h->code[1], s->box[1]),
                         pa[2] - image(pb[2], h->code[2], s->box[2])};
    const double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
    if (r2 >= s->lj.rc2) continue;
    if (r2 == 0.0) {
      snprintf(s->err, sizeof s->err, "overlapping particles: ids %lld and %lld coincide",
               (long long)s->id[h->a], (long long)s->id[h->b]);
      return 2;
    }
    double e, ff;
    tmo_lj_eval(r2, &s->lj, &e, &ff);
    nadd(&pe, e);
    nadd(&w, (long double)ff * r2);
    for (int a = 0; a < 3; ++a) {
      const long double fa = (long double)ff * d[a];
      nadd(&s->f[3 * h->a + a], fa);
      nadd(&s->f[3 * h->b + a], -fa);
    }
  }
  s->pe = nval(&pe);
  s->w = nval(&w);
  for (int64_t k = 0; k < 3 * s->n; ++k) s->fd[k] = (double)nval(&s->f[k]);
  return 0;
}

tmo_system* tmo_create(int64_t n, const int64_t* id, const double* mass,
                       const double* pos, const double* vel, const double box[3],
                       double eps, double sigma, double r_cut, int shifted,
                       double r_skin, double dt, int* status) {
  tmo_system* s = calloc(1, sizeof *s);
  *status = 0;
  if (n < 1 || tmo_cell_grid(box, r_cut, r_skin, s->dims, s->cell_len) != 0) {
    *status = 1;
    snprintf(s->err, sizeof s->err, "invalid configuration");
    return s;
  }
  s->n = n;
  memcpy(s->box, box, sizeof s->box);
  s->ncells = s->dims[0] * s->dims[1] * s->dims[2];
  const double rv = r_cut + r_skin;
  s->rv2 = rv * rv;
  s->thr = 0.25 * r_skin * r_skin;
  s->dt = dt;
  tmo_lj_prepare(eps, sigma, r_cut, shifted, &s->lj);
  s->id = malloc(sizeof(int64_t) * (size_t)n);
  s->mass = malloc(sizeof(double) * (size_t)n);
  s->pos = malloc(sizeof(double) * 3 * (size_t)n);
  s->vel = calloc(3 * (size_t)n, sizeof(double));
  s->snap = malloc(sizeof(double) * 3 * (size_t)n);
  s->f = calloc(3 * (size_t)n, sizeof(nsum));
  s->fd = calloc(3 * (size_t)n, sizeof(double));
  s->cell = malloc(sizeof(int32_t) * (size_t)n);
  s->items = malloc(sizeof(int32_t) * (size_t)n);
  s->start = malloc(sizeof(int32_t) * (size_t)(s->ncells + 1));
  memcpy(s->id, id, sizeof(int64_t) * (size_t)n);
  memcpy(s->pos, pos, sizeof(double) * 3 * (size_t)n);
  if (vel) memcpy(s->vel, vel, sizeof(double) * 3 * (size_t)n);
  for (int64_t k = 0; k < n; ++k) s->mass[k] = mass ? mass[k] : 1.0;
  if ((*status = resort(s)) != 0) return s;
  build_pairs(s);
  *status = forces(s);
  return s;
}

/* Engine::step (engine.hpp:80-126) without thermostat, one subnode. */
int tmo_step(tmo_system* s, int64_t nsteps) {
  const double hdt = 0.5 * s->dt;
  for (int64_t st = 0; st < nsteps; ++st) {
    s->step += 1;
    double best = 0.0;
    for (int64_t k = 0; k < s->n; ++k) { /* half_kick_and_drift 174-189 */
      const double inv_m = 1.0 / s->mass[k];
      for (int a = 0; a < 3; ++a) {
        s->vel[3 * k + a] += s->fd[3 * k + a] * inv_m * hdt;
        s->pos[3 * k + a] += s->vel[3 * k + a] * s->dt;
      }
      const double dx = s->pos[3 * k] - s->snap[3 * k];
      const double dy = s->pos[3 * k + 1] - s->snap[3 * k + 1];
      const double dz = s->pos[3 * k + 2] - s->snap[3 * k + 2];
      const double d2 = dx * dx + dy * dy + dz * dz; /* max_displacement2 114-136 */
      if (d2 > best) best = d2;
    }
    if (best > s->thr) { /* needs_rebuild 141-144 */
      int rc = resort(s);
      if (rc) return rc;
      build_pairs(s);
      s->rebuilds += 1;
    }
    int rc = forces(s);
    if (rc) {
      char tail[64];
      snprintf(tail, sizeof tail, " (at step %lld)", (long long)s->step);
      strncat(s->err, tail, sizeof s->err - strlen(s->err) - 1);
      return rc;
    }
    for (int64_t k = 0; k < s->n; ++k) { /* thermostat_and_half_kick 209-239 */
      const double inv_m = 1.0 / s->mass[k];
      for (int a = 0; a < 3; ++a) s->vel[3 * k + a] += s->fd[3 * k + a] * inv_m * hdt;
      for (int a = 0; a < 3; ++a) {
        if (!isfinite(s->vel[3 * k + a]) || !isfinite(s->fd[3 * k + a])) {
          snprintf(s->err, sizeof s->err,
                   "non-finite velocity or force on particle id %lld (at step %lld)",
                   (long long)s->id[k], (long long)s->step);
          return 2;
        }
      }
    }
  }
  return 0;
}

void tmo_observe(const tmo_system* s, double out[5]) {
  nsum ke = {0, 0};
  for (int64_t k = 0; k < s->n; ++k) {
    const double* v = s->vel + 3 * k;
    nadd(&ke, 0.5 * s->mass[k] * (v[0] * v[0] + v[1] * v[1] + v[2] * v[2]));
  }
  const double kin = (double)nval(&ke);
  out[0] = (double)s->step;
  out[1] = kin;
  out[2] = (double)s->pe;
  out[3] = (double)s->w;
  out[4] = 2.0 * kin / (3.0 * (double)s->n); /* soa_store.hpp:200-204 */
}

static int cmp_pair(const void* x, const void* y) {
  const int64_t* a = x;
  const int64_t* b = y;
  if (a[0] != b[0]) return (a[0] > b[0]) - (a[0] < b[0]);
  return (a[1] > b[1]) - (a[1] < b[1]);
}

int64_t tmo_pairs(const tmo_system* s, int64_t* out, int64_t cap) {
  if (!out || cap < s->npairs) return s->npairs;
  for (int64_t q = 0; q < s->npairs; ++q) {
    const int64_t a = s->id[s->pairs[q].a], b = s->id[s->pairs[q].b];
    out[2 * q] = a < b ? a : b;
    out[2 * q + 1] = a < b ? b : a;
  }
  qsort(out, (size_t)s->npairs, 2 * sizeof(int64_t), cmp_pair);
  return s->npairs;
}

static int32_t* order_by_id(const tmo_system* s) {
  int32_t* o = malloc(sizeof(int32_t) * (size_t)s->n);
  for (int64_t k = 0; k < s->n; ++k) o[k] = (int32_t)k;
  g_sort_ids = s->id;
  qsort(o, (size_t)s->n, sizeof(int32_t), by_id);
  return o;
}

void tmo_cell_of_all(const tmo_system* s, int64_t* id, int32_t* cell) {
  int32_t* o = order_by_id(s);
  for (int64_t r = 0; r < s->n; ++r) {
    id[r] = s->id[o[r]];
    cell[r] = s->cell[o[r]];
  }
  free(o);
}

void tmo_forces(const tmo_system* s, int64_t* id, double* f) {
  int32_t* o = order_by_id(s);
  for (int64_t r = 0; r < s->n; ++r) {
    id[r] = s->id[o[r]];
    for (int a = 0; a < 3; ++a) f[3 * r + a] = s->fd[3 * o[r] + a];
  }
  free(o);
}

void tmo_flatten(const tmo_system* s, int64_t* id, double* pos, double* vel) {
  int32_t* o = order_by_id(s);
  for (int64_t r = 0; r < s->n; ++r) {
    id[r] = s->id[o[r]];
    for (int a = 0; a < 3; ++a) {
      if (pos) pos[3 * r + a] = tmo_wrap1(s->pos[3 * o[r] + a], s->box[a]);
      if (vel) vel[3 * r + a] = s->vel[3 * o[r] + a];
    }
  }
  free(o);
}

uint64_t tmo_rebuild_count(const tmo_system* s) { return s->rebuilds; }
int64_t tmo_size(const tmo_system* s) { return s->n; }
const char* tmo_error(const tmo_system* s) { return s->err; }

void tmo_destroy(tmo_system* s) {
  if (!s) return;
  free(s->id); free(s->mass); free(s->pos); free(s->vel); free(s->snap);
  free(s->f); free(s->fd); free(s->cell); free(s->items); free(s->start);
  free(s->pairs);
  free(s);
}
