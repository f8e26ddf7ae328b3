/* oracle/hfmm_oracle.c — CPU restatement (plain C11, FP64) of the reference's FMM matvec path.
 *
 * TEST INFRASTRUCTURE ONLY — see hfmm_oracle.h.  Parity status: PINNED against the compiled
 * reference (oracle/_ref) and its committed fixtures (tests/golden).
 *
 * Each function names the reference file:line whose behaviour it restates.  The code is an
 * independent re-expression: iterative tree build, flat pair lists, sorted shift de-duplication,
 * OpenMP over target groups.  "ref:" paths are relative to /root/reference/proj/core.
 */
#include "hfmm_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex zc;
#define HO_PI 3.14159265358979323846264338327950288
#define HO_MAXLEVEL 21 /* ref: include/hfmm/octree.hpp:26 */

static inline int nm(int n, int m) { return n * (n + 1) + m; } /* ref: special.hpp:29 */
static inline int nmdim(int p) { return (p + 1) * (p + 1); }    /* ref: special.hpp:30 */
static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* ------------------------------------------------------------------------------------------
 * special functions
 * ---------------------------------------------------------------------------------------- */

/* ref: src/special.cpp:16-54 — ascending series below 0.5, Miller downward recurrence
 * (start nmax+16+floor(z), rescale at 1e250, normalise by j0 = sin z / z) otherwise. */
void ho_sph_jn(int nmax, double z, double* out) {
  if (fabs(z) < 0.5) {
    const double h = 0.5 * z * z;
    double zpow = 1.0, dfact = 1.0;
    for (int n = 0; n <= nmax; ++n) {
      double term = 1.0, sum = 1.0;
      for (int j = 1; j < 40; ++j) {
        term *= -h / ((double)j * (2 * n + 2 * j + 1));
        sum += term;
        if (fabs(term) < 1e-18 * fabs(sum)) break;
      }
      out[n] = zpow / dfact * sum;
      zpow *= z;
      dfact *= (double)(2 * n + 3);
    }
    return;
  }
  const int start = nmax + 16 + (int)fabs(z);
  double above = 0.0, cur = 1e-30;
  double* keep = (double*)calloc((size_t)nmax + 1, sizeof(double));
  for (int n = start; n >= 0; --n) {
    const double below = (2.0 * n + 3.0) / z * cur - above;
    above = cur;
    cur = below;
    if (n <= nmax) keep[n] = cur;
    if (fabs(cur) > 1e250) {
      cur *= 1e-250;
      above *= 1e-250;
      for (int i = n < nmax ? n : nmax; i <= nmax; ++i) keep[i] *= 1e-250;
    }
  }
  const double j0 = fabs(z) < 1e-6 ? 1.0 - z * z / 6.0 : sin(z) / z;
  const double scale = j0 / cur;
  for (int n = 0; n <= nmax; ++n) out[n] = keep[n] * scale;
  free(keep);
}

/* the same for a complex argument (the reference's sph_jn takes cplx z: special.cpp:7-54) */
static zc sph_j0_z(zc z) {
  if (cabs(z) < 1e-6) {
    const zc z2 = z * z;
    return 1.0 - z2 / 6.0 + z2 * z2 / 120.0;
  }
  return csin(z) / z;
}
static void sph_jn_z(int nmax, zc z, zc* out) {
  const double az = cabs(z);
  if (az < 0.5) {
    const zc h = 0.5 * z * z;
    zc zpow = 1.0;
    double dfact = 1.0;
    for (int n = 0; n <= nmax; ++n) {
      zc term = 1.0, sum = 1.0;
      for (int j = 1; j < 40; ++j) {
        term *= -h / (double)(j * (2 * n + 2 * j + 1));
        sum += term;
        if (cabs(term) < 1e-18 * cabs(sum)) break;
      }
      out[n] = zpow / dfact * sum;
      zpow *= z;
      dfact *= (double)(2 * n + 3);
    }
    return;
  }
  const int start = nmax + 16 + (int)az;
  zc above = 0.0, cur = 1e-30;
  zc* keep = (zc*)calloc((size_t)nmax + 1, sizeof(zc));
  for (int n = start; n >= 0; --n) {
    const zc below = (2.0 * n + 3.0) / z * cur - above;
    above = cur;
    cur = below;
    if (n <= nmax) keep[n] = cur;
    if (cabs(cur) > 1e250) {
      cur *= 1e-250;
      above *= 1e-250;
      for (int i = n < nmax ? n : nmax; i <= nmax; ++i) keep[i] *= 1e-250;
    }
  }
  const zc scale = sph_j0_z(z) / cur;
  for (int n = 0; n <= nmax; ++n) out[n] = keep[n] * scale;
  free(keep);
}

/* j_n for a real or complex argument (a real argument keeps the real-arithmetic path) */
static void radial_j(int nmax, zc z, zc* out) {
  if (cimag(z) == 0.0) {
    double* jr = (double*)malloc(sizeof(double) * ((size_t)nmax + 1));
    ho_sph_jn(nmax, creal(z), jr);
    for (int n = 0; n <= nmax; ++n) out[n] = jr[n];
    free(jr);
  } else {
    sph_jn_z(nmax, z, out);
  }
}

/* ref: src/special.cpp:56-65 — h0 = -i e^{iz}/z, h1 = -e^{iz}(z+i)/z^2, upward recurrence */
static void sph_hn_c(int nmax, zc z, zc* out) {
  const zc e = cexp(I * z);
  out[0] = -I * e / z;
  if (nmax == 0) return;
  out[1] = -e * (z + I) / (z * z);
  for (int n = 1; n < nmax; ++n) out[n + 1] = (2.0 * n + 1.0) / z * out[n] - out[n - 1];
}
void ho_sph_hn(int nmax, double z, double* o) { sph_hn_c(nmax, z, (zc*)o); }

/* ref: src/special.cpp:80-124 — orthonormal Y_n^m with Condon-Shortley phase from the
 * fully-normalised Legendre recurrences; zero vector keeps only the monopole. */
static void ynm_c(int nmax, const double d[3], zc* out) {
  const int dim = nmdim(nmax);
  const double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  if (r == 0.0) {
    for (int i = 0; i < dim; ++i) out[i] = 0;
    out[0] = sqrt(1.0 / (4.0 * HO_PI));
    return;
  }
  double ct = d[2] / r;
  if (ct > 1) ct = 1;
  if (ct < -1) ct = -1;
  const double theta = acos(ct), phi = atan2(d[1], d[0]);
  const double x = cos(theta), s = sin(theta);
  double* pb = (double*)malloc(sizeof(double) * (size_t)(nmax + 1) * (nmax + 2) / 2);
#define PB(n, m) pb[(n) * ((n) + 1) / 2 + (m)]
  PB(0, 0) = sqrt(1.0 / (4.0 * HO_PI));
  for (int m = 1; m <= nmax; ++m) PB(m, m) = -sqrt((2.0 * m + 1.0) / (2.0 * m)) * s * PB(m - 1, m - 1);
  for (int m = 0; m < nmax; ++m) PB(m + 1, m) = sqrt(2.0 * m + 3.0) * x * PB(m, m);
  for (int m = 0; m <= nmax; ++m)
    for (int n = m + 2; n <= nmax; ++n) {
      const double den = (double)n * n - (double)m * m;
      const double a = sqrt((4.0 * n * n - 1.0) / den);
      const double b = sqrt(((2.0 * n + 1.0) * (n - 1.0 + m) * (n - 1.0 - m)) / ((2.0 * n - 3.0) * den));
      PB(n, m) = a * x * PB(n - 1, m) - b * PB(n - 2, m);
    }
  for (int n = 0; n <= nmax; ++n) {
    out[nm(n, 0)] = PB(n, 0);
    for (int m = 1; m <= n; ++m) {
      const zc v = PB(n, m) * (cos(m * phi) + I * sin(m * phi));
      out[nm(n, m)] = v;
      out[nm(n, -m)] = (m & 1 ? -1.0 : 1.0) * conj(v);
    }
  }
#undef PB
  free(pb);
}
void ho_ynm(int nmax, const double dir[3], double* o) { ynm_c(nmax, dir, (zc*)o); }

/* ref: src/special.cpp:126-155 — Racah sum over log-factorials in long double */
static long double lfact(int n) {
  static long double tab[512];
  static int ready = 0;
  if (!ready) {
#pragma omp critical(ho_lfact)
    if (!ready) {
      tab[0] = 0;
      for (int i = 1; i < 512; ++i) tab[i] = tab[i - 1] + logl((long double)i);
      ready = 1;
    }
  }
  return tab[n];
}
double ho_wigner3j(int j1, int j2, int j3, int m1, int m2, int m3) {
  if (m1 + m2 + m3 != 0) return 0;
  if (j3 < abs(j1 - j2) || j3 > j1 + j2) return 0;
  if (abs(m1) > j1 || abs(m2) > j2 || abs(m3) > j3) return 0;
  const long double pre =
      0.5L * (lfact(j1 + j2 - j3) + lfact(j1 - j2 + j3) + lfact(-j1 + j2 + j3) -
              lfact(j1 + j2 + j3 + 1) + lfact(j1 + m1) + lfact(j1 - m1) + lfact(j2 + m2) +
              lfact(j2 - m2) + lfact(j3 + m3) + lfact(j3 - m3));
  int lo = 0, hi = j1 + j2 - j3;
  if (j2 - j3 - m1 > lo) lo = j2 - j3 - m1;
  if (j1 - j3 + m2 > lo) lo = j1 - j3 + m2;
  if (j1 - m1 < hi) hi = j1 - m1;
  if (j2 + m2 < hi) hi = j2 + m2;
  long double sum = 0;
  for (int t = lo; t <= hi; ++t) {
    const long double den = lfact(t) + lfact(j1 + j2 - j3 - t) + lfact(j1 - m1 - t) +
                            lfact(j2 + m2 - t) + lfact(j3 - j2 + m1 + t) + lfact(j3 - j1 - m2 + t);
    const long double term = expl(pre - den);
    sum += (t & 1) ? -term : term;
  }
  const int ph = j1 - j2 - m3;
  return (double)((((ph % 2) + 2) % 2) ? -sum : sum);
}

/* ------------------------------------------------------------------------------------------
 * translation operators
 * ---------------------------------------------------------------------------------------- */

/* ref: src/expansion.cpp:47-84 — coupling table: for (nu,mu | n,m) the (lambda, coeff) terms with
 * coeff = 4pi (-1)^m sqrt((2nu+1)(2lam+1)(2n+1)/4pi) (nu lam n;000) (nu lam n;-mu,mu-m,m),
 * lambda from max(|n-nu|,|m-mu|) (parity-adjusted) to n+nu step 2; zero terms dropped. */
typedef struct {
  int order;
  uint32_t* off; /* dim*dim+1 */
  int* lam;
  double* coef;
} gaunt_t;

static gaunt_t* gaunt_build(int order) {
  const int dim = nmdim(order);
  gaunt_t* g = (gaunt_t*)calloc(1, sizeof(gaunt_t));
  g->order = order;
  g->off = (uint32_t*)calloc((size_t)dim * dim + 1, sizeof(uint32_t));
  size_t cap = 1024, cnt = 0;
  g->lam = (int*)malloc(cap * sizeof(int));
  g->coef = (double*)malloc(cap * sizeof(double));
  for (int nu = 0; nu <= order; ++nu)
    for (int mu = -nu; mu <= nu; ++mu)
      for (int n = 0; n <= order; ++n)
        for (int m = -n; m <= n; ++m) {
          g->off[(size_t)nm(nu, mu) * dim + nm(n, m)] = (uint32_t)cnt;
          int lo = abs(n - nu) > abs(m - mu) ? abs(n - nu) : abs(m - mu);
          if ((lo ^ (n + nu)) & 1) ++lo;
          for (int l = lo; l <= n + nu; l += 2) {
            const double w0 = sqrt((2 * nu + 1) * (2 * l + 1) * (2 * n + 1) / (4 * HO_PI)) *
                              ho_wigner3j(nu, l, n, 0, 0, 0);
            const double wm = ho_wigner3j(nu, l, n, -mu, mu - m, m);
            const double c = 4 * HO_PI * (m % 2 ? -1.0 : 1.0) * w0 * wm;
            if (c == 0) continue;
            if (cnt == cap) {
              cap *= 2;
              g->lam = (int*)realloc(g->lam, cap * sizeof(int));
              g->coef = (double*)realloc(g->coef, cap * sizeof(double));
            }
            g->lam[cnt] = l;
            g->coef[cnt] = c;
            ++cnt;
          }
        }
  g->off[(size_t)dim * dim] = (uint32_t)cnt;
  return g;
}

/* ref: src/expansion.cpp:86-93 — one shared table per order */
static gaunt_t* gaunt_get(int order) {
  static gaunt_t* cache[64];
  gaunt_t* g;
#pragma omp critical(ho_gaunt)
  {
    if (!cache[order]) cache[order] = gaunt_build(order);
    g = cache[order];
  }
  return g;
}

static const zc kIpow[4] = {1, I, -1, -I};

/* ref: src/expansion.cpp:95-124 — T[(nu,mu),(n,m)] = sum_lam i^(nu+lam-n) G z_lam(k|t|)
 * Y_lam^(m-mu)(t^), z = j (regular) or h (singular); row-major dim x dim. */
static void translation_matrix_c(zc k, const double t[3], int order, int singular, zc* T) {
  const gaunt_t* g = gaunt_get(order);
  const int dim = nmdim(order), lmax = 2 * order;
  const zc z = k * sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
  zc* rad = (zc*)malloc(sizeof(zc) * (lmax + 1));
  if (singular)
    sph_hn_c(lmax, z, rad);
  else
    radial_j(lmax, z, rad);
  zc* harm = (zc*)malloc(sizeof(zc) * nmdim(lmax));
  ynm_c(lmax, t, harm);
  for (int nu = 0; nu <= order; ++nu)
    for (int mu = -nu; mu <= nu; ++mu)
      for (int n = 0; n <= order; ++n)
        for (int m = -n; m <= n; ++m) {
          const size_t slot = (size_t)nm(nu, mu) * dim + nm(n, m);
          zc s = 0;
          for (uint32_t e = g->off[slot]; e < g->off[slot + 1]; ++e) {
            const int l = g->lam[e];
            s += kIpow[(((nu + l - n) % 4) + 4) % 4] * g->coef[e] * rad[l] * harm[nm(l, m - mu)];
          }
          T[slot] = s;
        }
  free(rad);
  free(harm);
}
void ho_translation_matrix(double k, const double t[3], int order, int singular, double* out) {
  translation_matrix_c(k, t, order, singular, (zc*)out);
}
void ho_translation_matrix_complex_k(double kr, double ki, const double t[3], int order, int singular,
                                     double* out) {
  translation_matrix_c(kr + I * ki, t, order, singular, (zc*)out);
}

/* ref: src/expansion.cpp:126-139 — out += T * in */
static void apply_dense(const zc* T, int dim, const zc* in, zc* out) {
  for (int o = 0; o < dim; ++o) {
    zc s = 0;
    const zc* row = T + (size_t)o * dim;
    for (int i = 0; i < dim; ++i) s += row[i] * in[i];
    out[o] += s;
  }
}

/* ref: src/expansion.cpp:157-175 — M_n^m += (i k q) j_n(k rho) conj Y_n^m(rho^) */
static void p2m_c(long n, const double* xyz, const zc* q, const double c[3], zc k, int order,
                  zc* M) {
  zc* rad = (zc*)malloc(sizeof(zc) * (order + 1));
  zc* harm = (zc*)malloc(sizeof(zc) * nmdim(order));
  for (long b = 0; b < n; ++b) {
    const double rho[3] = {xyz[3 * b] - c[0], xyz[3 * b + 1] - c[1], xyz[3 * b + 2] - c[2]};
    radial_j(order, k * sqrt(rho[0] * rho[0] + rho[1] * rho[1] + rho[2] * rho[2]), rad);
    ynm_c(order, rho, harm);
    const zc w = I * k * q[b];
    for (int d = 0; d <= order; ++d)
      for (int m = -d; m <= d; ++m) M[nm(d, m)] += w * rad[d] * conj(harm[nm(d, m)]);
  }
  free(rad);
  free(harm);
}
void ho_p2m(long n, const double* xyz, const double* q, const double center[3], double k,
            int order, double* out) {
  memset(out, 0, sizeof(zc) * nmdim(order));
  p2m_c(n, xyz, (const zc*)q, center, k, order, (zc*)out);
}

/* ref: src/expansion.cpp:177-195 — sum coeff * (h_n or j_n)(k r) Y_n^m(r^) */
static zc eval_c(int local, int order, const zc* coeff, const double c[3], const double p[3],
                 zc k) {
  const double d[3] = {p[0] - c[0], p[1] - c[1], p[2] - c[2]};
  const double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  zc* harm = (zc*)malloc(sizeof(zc) * nmdim(order));
  zc* rad = (zc*)malloc(sizeof(zc) * (order + 1));
  ynm_c(order, d, harm);
  if (local)
    radial_j(order, k * r, rad);
  else
    sph_hn_c(order, k * r, rad);
  zc s = 0;
  for (int n = 0; n <= order; ++n)
    for (int m = -n; m <= n; ++m) s += coeff[nm(n, m)] * rad[n] * harm[nm(n, m)];
  free(harm);
  free(rad);
  return s;
}
void ho_eval_expansion(int local, int order, const double* coeff, const double center[3],
                       const double point[3], double k, double out[2]) {
  const zc v = eval_c(local, order, (const zc*)coeff, center, point, k);
  out[0] = creal(v);
  out[1] = cimag(v);
}

/* ------------------------------------------------------------------------------------------
 * octree
 * ---------------------------------------------------------------------------------------- */
typedef struct {
  int level;
  uint32_t ix, iy, iz;
  double c[3], radius;
  uint32_t body_first, body_count, child_first, child_count;
} cell_t;

struct ho_fmm {
  long n;
  double k, ki, theta, kd_max; /* wavenumber k + i ki */
  int order, ncrit;
  double lo[3], width;
  double* pos;    /* Morton order, 3n */
  uint64_t* key;  /* level-21 keys, Morton order */
  uint32_t* index; /* caller index per sorted slot */
  cell_t* cells;
  long ncells, cap_cells;
  uint32_t* leaves;
  long nleaves;
  int max_level;
  /* plan as CSR by target cell id */
  long n_m2l, n_p2p;
  uint32_t *m2l_t, *m2l_s, *p2p_t, *p2p_s; /* flat pairs, grouped by target ascending */
  /* expansions of the last matvec */
  zc *multipole, *local;
  double seconds[3];
};

/* ref: src/octree.cpp:25-51 — digitise at `level`, clamp the upper face, interleave x,y,z
 * (x highest) root-first */
static uint64_t morton_key(const double p[3], const double lo[3], double width, int level) {
  const uint64_t nside = (uint64_t)1 << level;
  const double scale = (double)nside / width;
  uint64_t g[3];
  for (int a = 0; a < 3; ++a) {
    int64_t i = (int64_t)((p[a] - lo[a]) * scale);
    if (i < 0) i = 0;
    if (i >= (int64_t)nside) i = (int64_t)nside - 1;
    g[a] = (uint64_t)i;
  }
  uint64_t key = 0;
  for (int b = level - 1; b >= 0; --b)
    key = key << 3 | ((g[0] >> b & 1) << 2) | ((g[1] >> b & 1) << 1) | (g[2] >> b & 1);
  return key;
}

typedef struct {
  uint64_t key;
  uint32_t idx;
} keyidx_t;
static int cmp_keyidx(const void* a, const void* b) {
  const keyidx_t *x = (const keyidx_t*)a, *y = (const keyidx_t*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

static long push_cell(ho_fmm* h, const cell_t* c) {
  if (h->ncells == h->cap_cells) {
    h->cap_cells = h->cap_cells ? 2 * h->cap_cells : 1024;
    h->cells = (cell_t*)realloc(h->cells, sizeof(cell_t) * h->cap_cells);
  }
  h->cells[h->ncells] = *c;
  return h->ncells++;
}

/* ref: src/octree.cpp:53-70 (cubified box, 1e-12 pad), :142-182 (key, sort by (key,index)),
 * :85-137 (split while count > capacity or diameter > cap; children contiguous; the reference's
 * recursion order is reproduced with an explicit stack so cell numbering is identical). */
static void build_tree(ho_fmm* h, const double* xyz, double leaf_cap) {
  const long n = h->n;
  double lo[3] = {xyz[0], xyz[1], xyz[2]}, hi[3] = {xyz[0], xyz[1], xyz[2]};
  for (long i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      if (xyz[3 * i + a] < lo[a]) lo[a] = xyz[3 * i + a];
      if (xyz[3 * i + a] > hi[a]) hi[a] = xyz[3 * i + a];
    }
  double w = hi[0] - lo[0];
  if (hi[1] - lo[1] > w) w = hi[1] - lo[1];
  if (hi[2] - lo[2] > w) w = hi[2] - lo[2];
  if (w <= 0) w = 1;
  w *= 1 + 1e-12;
  for (int a = 0; a < 3; ++a) h->lo[a] = (lo[a] + hi[a]) / 2.0 - w / 2;
  h->width = w;

  keyidx_t* ki = (keyidx_t*)malloc(sizeof(keyidx_t) * n);
  for (long i = 0; i < n; ++i) {
    ki[i].key = morton_key(xyz + 3 * i, h->lo, w, HO_MAXLEVEL);
    ki[i].idx = (uint32_t)i;
  }
  qsort(ki, n, sizeof(keyidx_t), cmp_keyidx);
  h->pos = (double*)malloc(sizeof(double) * 3 * n);
  h->key = (uint64_t*)malloc(sizeof(uint64_t) * n);
  h->index = (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (long i = 0; i < n; ++i) {
    h->key[i] = ki[i].key;
    h->index[i] = ki[i].idx;
    memcpy(h->pos + 3 * i, xyz + 3 * ki[i].idx, 3 * sizeof(double));
  }
  free(ki);

  cell_t root;
  memset(&root, 0, sizeof(root));
  for (int a = 0; a < 3; ++a) root.c[a] = h->lo[a] + w / 2;
  root.radius = w * sqrt(3.0) / 2;
  root.body_count = (uint32_t)n;
  push_cell(h, &root);

  long cap_stack = 64, top = 0;
  uint32_t* stack = (uint32_t*)malloc(sizeof(uint32_t) * cap_stack);
  long cap_leaf = 1024;
  h->leaves = (uint32_t*)malloc(sizeof(uint32_t) * cap_leaf);
  stack[top++] = 0;
  while (top) {
    const uint32_t ci = stack[--top];
    cell_t cell = h->cells[ci];
    if (cell.level > h->max_level) h->max_level = cell.level;
    const int over_cap = (int)cell.body_count > h->ncrit;
    const int over_diam = leaf_cap > 0 && 2 * cell.radius > leaf_cap && cell.body_count > 0;
    if ((!over_cap && !over_diam) || cell.level == HO_MAXLEVEL) {
      if (h->nleaves == cap_leaf) {
        cap_leaf *= 2;
        h->leaves = (uint32_t*)realloc(h->leaves, sizeof(uint32_t) * cap_leaf);
      }
      h->leaves[h->nleaves++] = ci;
      continue;
    }
    const int shift = 3 * (HO_MAXLEVEL - 1 - cell.level);
    uint32_t edge[9];
    uint32_t pos = cell.body_first;
    edge[0] = pos;
    for (uint32_t d = 0; d < 8; ++d) {
      while (pos < cell.body_first + cell.body_count && ((h->key[pos] >> shift) & 7) == d) ++pos;
      edge[d + 1] = pos;
    }
    const uint32_t first_child = (uint32_t)h->ncells;
    uint32_t nchild = 0;
    const double side = w / (double)((uint64_t)1 << (cell.level + 1));
    for (uint32_t d = 0; d < 8; ++d) {
      if (edge[d] == edge[d + 1]) continue;
      cell_t ch;
      memset(&ch, 0, sizeof(ch));
      ch.level = cell.level + 1;
      ch.ix = cell.ix << 1 | (d >> 2 & 1);
      ch.iy = cell.iy << 1 | (d >> 1 & 1);
      ch.iz = cell.iz << 1 | (d & 1);
      ch.c[0] = h->lo[0] + (ch.ix + 0.5) * side;
      ch.c[1] = h->lo[1] + (ch.iy + 0.5) * side;
      ch.c[2] = h->lo[2] + (ch.iz + 0.5) * side;
      ch.radius = side * sqrt(3.0) / 2;
      ch.body_first = edge[d];
      ch.body_count = edge[d + 1] - edge[d];
      push_cell(h, &ch);
      ++nchild;
    }
    h->cells[ci].child_first = first_child;
    h->cells[ci].child_count = nchild;
    if (top + nchild > cap_stack) {
      cap_stack = 2 * (top + nchild);
      stack = (uint32_t*)realloc(stack, sizeof(uint32_t) * cap_stack);
    }
    for (uint32_t j = nchild; j-- > 0;) stack[top++] = first_child + j; /* child 0 next */
  }
  free(stack);
}

/* ------------------------------------------------------------------------------------------
 * dual tree traversal
 * ---------------------------------------------------------------------------------------- */
typedef struct {
  uint32_t *t, *s;
  long n, cap;
} pairlist_t;
static void pl_push(pairlist_t* p, uint32_t t, uint32_t s) {
  if (p->n == p->cap) {
    p->cap = p->cap ? 2 * p->cap : 4096;
    p->t = (uint32_t*)realloc(p->t, sizeof(uint32_t) * p->cap);
    p->s = (uint32_t*)realloc(p->s, sizeof(uint32_t) * p->cap);
  }
  p->t[p->n] = t;
  p->s[p->n] = s;
  ++p->n;
}

/* ref: src/traversal.cpp:45-51 — wavenumber gate then centre-distance test */
static int admissible(const ho_fmm* h, const cell_t* a, const cell_t* b) {
  if (h->kd_max > 0 &&
      (hypot(h->k, h->ki) * 2 * a->radius > h->kd_max || hypot(h->k, h->ki) * 2 * b->radius > h->kd_max))
    return 0;
  const double d[3] = {a->c[0] - b->c[0], a->c[1] - b->c[1], a->c[2] - b->c[2]};
  return sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]) > (a->radius + b->radius) / h->theta;
}

/* ref: src/traversal.cpp:53-79 — admissible -> far; leaf-leaf -> near; else split the target iff
 * it is not a leaf and (source is a leaf or target radius is larger); ties open the source. */
static void walk(const ho_fmm* h, uint32_t ti, uint32_t si, pairlist_t* far, pairlist_t* near) {
  const cell_t* a = &h->cells[ti];
  const cell_t* b = &h->cells[si];
  if (admissible(h, a, b)) {
    pl_push(far, ti, si);
    return;
  }
  const int aleaf = a->child_count == 0, bleaf = b->child_count == 0;
  if (aleaf && bleaf) {
    pl_push(near, ti, si);
    return;
  }
  if (!aleaf && (bleaf || a->radius > b->radius)) {
    for (uint32_t c = 0; c < a->child_count; ++c) walk(h, a->child_first + c, si, far, near);
  } else {
    for (uint32_t c = 0; c < b->child_count; ++c) walk(h, ti, b->child_first + c, far, near);
  }
}

/* stable counting sort of discovery-ordered pairs by target: keeps each target's source order
 * (ref: traversal.hpp:20-22 "source order within a target follows the recorded traversal") */
static void group_by_target(const pairlist_t* in, long ncells, uint32_t** ot, uint32_t** os) {
  long* cnt = (long*)calloc(ncells + 1, sizeof(long));
  for (long i = 0; i < in->n; ++i) cnt[in->t[i] + 1]++;
  for (long c = 0; c < ncells; ++c) cnt[c + 1] += cnt[c];
  *ot = (uint32_t*)malloc(sizeof(uint32_t) * (in->n ? in->n : 1));
  *os = (uint32_t*)malloc(sizeof(uint32_t) * (in->n ? in->n : 1));
  for (long i = 0; i < in->n; ++i) {
    const long slot = cnt[in->t[i]]++;
    (*ot)[slot] = in->t[i];
    (*os)[slot] = in->s[i];
  }
  free(cnt);
}

ho_fmm* ho_fmm_create(long n, const double* xyz, double k, int order, int ncrit,
                      double leaf_cap, double theta, double kd_max) {
  return ho_fmm_create_complex_k(n, xyz, k, 0.0, order, ncrit, leaf_cap, theta, kd_max);
}
/* complex wavenumber kr + i ki (common.hpp:36-40); gates use |k| (traversal.cpp:86) */
ho_fmm* ho_fmm_create_complex_k(long n, const double* xyz, double k, double ki, int order, int ncrit,
                                double leaf_cap, double theta, double kd_max) {
  if (n < 1 || ncrit < 1 || !(theta > 0) || theta > 1 || order < 0) return NULL;
  ho_fmm* h = (ho_fmm*)calloc(1, sizeof(ho_fmm));
  h->n = n;
  h->k = k;
  h->ki = ki;
  h->order = order;
  h->ncrit = ncrit;
  h->theta = theta;
  h->kd_max = kd_max;
  build_tree(h, xyz, leaf_cap);
  pairlist_t far = {0}, near = {0};
  walk(h, 0, 0, &far, &near); /* ref: src/traversal.cpp:87-88 */
  h->n_m2l = far.n;
  h->n_p2p = near.n;
  group_by_target(&far, h->ncells, &h->m2l_t, &h->m2l_s);
  group_by_target(&near, h->ncells, &h->p2p_t, &h->p2p_s);
  free(far.t); free(far.s); free(near.t); free(near.s);
  return h;
}

void ho_fmm_destroy(ho_fmm* h) {
  if (!h) return;
  free(h->pos); free(h->key); free(h->index); free(h->cells); free(h->leaves);
  free(h->m2l_t); free(h->m2l_s); free(h->p2p_t); free(h->p2p_s);
  free(h->multipole); free(h->local);
  free(h);
}

static long count_groups(const uint32_t* t, long n, long* maxlen) {
  long g = 0, run = 0;
  *maxlen = 0;
  for (long i = 0; i < n; ++i) {
    if (i == 0 || t[i] != t[i - 1]) { ++g; run = 0; }
    if (++run > *maxlen) *maxlen = run;
  }
  return g;
}

void ho_fmm_counts(const ho_fmm* h, long long* c) {
  long mm, mp;
  c[0] = h->ncells;
  c[1] = h->nleaves;
  c[2] = h->n_m2l;
  c[3] = h->n_p2p;
  long long bp = 0;
  for (long i = 0; i < h->n_p2p; ++i)
    bp += (long long)h->cells[h->p2p_t[i]].body_count * h->cells[h->p2p_s[i]].body_count;
  c[4] = bp;
  c[5] = h->max_level;
  c[6] = count_groups(h->m2l_t, h->n_m2l, &mm);
  c[7] = count_groups(h->p2p_t, h->n_p2p, &mp);
  c[8] = mm;
  c[9] = mp;
}
void ho_fmm_cells(const ho_fmm* h, unsigned* out) {
  for (long i = 0; i < h->ncells; ++i) {
    const cell_t* c = &h->cells[i];
    unsigned* o = out + 8 * i;
    o[0] = (unsigned)c->level; o[1] = c->ix; o[2] = c->iy; o[3] = c->iz;
    o[4] = c->body_first; o[5] = c->body_count; o[6] = c->child_first; o[7] = c->child_count;
  }
}
void ho_fmm_box(const ho_fmm* h, double* lo_w) {
  lo_w[0] = h->lo[0]; lo_w[1] = h->lo[1]; lo_w[2] = h->lo[2]; lo_w[3] = h->width;
}
void ho_fmm_body_order(const ho_fmm* h, unsigned* out) {
  memcpy(out, h->index, sizeof(uint32_t) * h->n);
}
void ho_fmm_plan(const ho_fmm* h, int which, unsigned* targets, unsigned long long* offsets,
                 unsigned* sources) {
  const uint32_t* t = which ? h->p2p_t : h->m2l_t;
  const uint32_t* s = which ? h->p2p_s : h->m2l_s;
  const long n = which ? h->n_p2p : h->n_m2l;
  long g = 0;
  for (long i = 0; i < n; ++i) {
    if (i == 0 || t[i] != t[i - 1]) {
      targets[g] = t[i];
      offsets[g] = (unsigned long long)i;
      ++g;
    }
    sources[i] = s[i];
  }
  offsets[g] = (unsigned long long)n;
}

/* ------------------------------------------------------------------------------------------
 * pipeline
 * ---------------------------------------------------------------------------------------- */

/* ref: src/traversal.cpp:152-166 — exact lattice shift in half-side units at the finer level */
typedef struct {
  int64_t x, y, z;
  int32_t lmax;
  long pair;
} shiftkey_t;
static int cmp_shift(const void* a, const void* b) {
  const shiftkey_t *p = (const shiftkey_t*)a, *q = (const shiftkey_t*)b;
  if (p->lmax != q->lmax) return p->lmax < q->lmax ? -1 : 1;
  if (p->x != q->x) return p->x < q->x ? -1 : 1;
  if (p->y != q->y) return p->y < q->y ? -1 : 1;
  if (p->z != q->z) return p->z < q->z ? -1 : 1;
  return 0;
}

/* ref: src/expansion.cpp:200-222 — parent-minus-child half-side offsets, one matrix per
 * (level, octant); downward pass uses the negated shift */
static void shift_matrix(const ho_fmm* h, int level, int oct, int upward, zc* T) {
  const double hs = h->width / (double)((uint64_t)1 << level) / 2;
  double t[3] = {oct & 4 ? -hs : hs, oct & 2 ? -hs : hs, oct & 1 ? -hs : hs};
  if (!upward)
    for (int a = 0; a < 3; ++a) t[a] = -t[a];
  translation_matrix_c(h->k + I * h->ki, t, h->order, 0, T);
}

/* ref: src/traversal.cpp:175-204 + include/hfmm/kernel.hpp:16-23 — per target body, sources in
 * list order, skip R^2 == 0, accumulate in Real then add to trg */
static void near_field(const ho_fmm* h, const zc* src, zc* trg, int f32) {
  long g0 = 0;
  long ngroups = 0;
  long* gstart = (long*)malloc(sizeof(long) * (h->n_p2p + 1));
  for (long i = 0; i < h->n_p2p; ++i)
    if (i == 0 || h->p2p_t[i] != h->p2p_t[i - 1]) gstart[ngroups++] = i;
  gstart[ngroups] = h->n_p2p;
  (void)g0;
#pragma omp parallel for schedule(dynamic, 8)
  for (long g = 0; g < ngroups; ++g) {
    const cell_t* tc = &h->cells[h->p2p_t[gstart[g]]];
    for (uint32_t bi = tc->body_first; bi < tc->body_first + tc->body_count; ++bi) {
      const double* pt = h->pos + 3 * bi;
      if (f32) {
        float ar = 0, ai = 0;
        for (long e = gstart[g]; e < gstart[g + 1]; ++e) {
          const cell_t* sc = &h->cells[h->p2p_s[e]];
          for (uint32_t bj = sc->body_first; bj < sc->body_first + sc->body_count; ++bj) {
            const double* ps = h->pos + 3 * bj;
            const double ddx = pt[0] - ps[0], ddy = pt[1] - ps[1], ddz = pt[2] - ps[2];
            if (ddx * ddx + ddy * ddy + ddz * ddz == 0) continue;
            const float dx = (float)ddx, dy = (float)ddy, dz = (float)ddz;
            const float R = sqrtf(dx * dx + dy * dy + dz * dz);
            const float amp = expf((float)(-h->ki) * R) / ((float)(4.0 * HO_PI) * R);
            const float ph = (float)h->k * R;
            const float gr = amp * cosf(ph), gi = amp * sinf(ph);
            const float qr = (float)creal(src[bj]), qi = (float)cimag(src[bj]);
            ar += gr * qr - gi * qi;
            ai += gr * qi + gi * qr;
          }
        }
        trg[bi] += (double)ar + I * (double)ai;
      } else {
        zc acc = 0;
        for (long e = gstart[g]; e < gstart[g + 1]; ++e) {
          const cell_t* sc = &h->cells[h->p2p_s[e]];
          for (uint32_t bj = sc->body_first; bj < sc->body_first + sc->body_count; ++bj) {
            const double* ps = h->pos + 3 * bj;
            const double dx = pt[0] - ps[0], dy = pt[1] - ps[1], dz = pt[2] - ps[2];
            const double r2 = dx * dx + dy * dy + dz * dz;
            if (r2 == 0) continue;
            const double R = sqrt(r2);
            const double amp = exp(-h->ki * R) / (4.0 * HO_PI * R);
            acc += (amp * cos(h->k * R) + I * amp * sin(h->k * R)) * src[bj];
          }
        }
        trg[bi] += acc;
      }
    }
  }
  free(gstart);
}

/* ref: src/traversal.cpp:208-279 (execute_plan), src/expansion.cpp:226-301 (upward/downward) */
int ho_fmm_matvec(ho_fmm* h, const double* q, int f32_p2p, double* out) {
  const int dim = nmdim(h->order);
  const long nc = h->ncells, n = h->n;
  zc* src = (zc*)malloc(sizeof(zc) * n);
  zc* trg = (zc*)calloc(n, sizeof(zc));
  for (long i = 0; i < n; ++i) src[i] = q[2 * h->index[i]] + I * q[2 * h->index[i] + 1];
  free(h->multipole);
  free(h->local);
  h->multipole = (zc*)calloc((size_t)nc * dim, sizeof(zc));
  h->local = (zc*)calloc((size_t)nc * dim, sizeof(zc));

  /* upward: children before parents == descending cell index (parents precede children) */
  double t0 = now_s();
  zc* up[HO_MAXLEVEL + 1][8];
  memset(up, 0, sizeof(up));
  for (long i = nc; i-- > 0;) {
    const cell_t* c = &h->cells[i];
    zc* M = h->multipole + (size_t)i * dim;
    if (c->child_count == 0) {
      p2m_c(c->body_count, h->pos + 3 * c->body_first, src + c->body_first, c->c, h->k + I * h->ki, h->order, M);
    } else {
      for (uint32_t j = 0; j < c->child_count; ++j) {
        const cell_t* ch = &h->cells[c->child_first + j];
        const int oct = (ch->ix & 1) << 2 | (ch->iy & 1) << 1 | (ch->iz & 1);
        if (!up[ch->level][oct]) {
          up[ch->level][oct] = (zc*)malloc(sizeof(zc) * dim * dim);
          shift_matrix(h, ch->level, oct, 1, up[ch->level][oct]);
        }
        apply_dense(up[ch->level][oct], dim, h->multipole + (size_t)(c->child_first + j) * dim, M);
      }
    }
  }
  for (int l = 0; l <= HO_MAXLEVEL; ++l)
    for (int o = 0; o < 8; ++o) free(up[l][o]);
  double t1 = now_s();
  h->seconds[0] = t1 - t0;

  /* interaction: one dense matrix per distinct lattice shift, then per-target ordered sums */
  shiftkey_t* sk = (shiftkey_t*)malloc(sizeof(shiftkey_t) * (h->n_m2l ? h->n_m2l : 1));
  for (long e = 0; e < h->n_m2l; ++e) {
    const cell_t *a = &h->cells[h->m2l_t[e]], *b = &h->cells[h->m2l_s[e]];
    const int lmax = a->level > b->level ? a->level : b->level;
    const int ua = lmax - a->level, ub = lmax - b->level;
    sk[e].x = ((int64_t)(2 * (uint64_t)a->ix + 1) << ua) - ((int64_t)(2 * (uint64_t)b->ix + 1) << ub);
    sk[e].y = ((int64_t)(2 * (uint64_t)a->iy + 1) << ua) - ((int64_t)(2 * (uint64_t)b->iy + 1) << ub);
    sk[e].z = ((int64_t)(2 * (uint64_t)a->iz + 1) << ua) - ((int64_t)(2 * (uint64_t)b->iz + 1) << ub);
    sk[e].lmax = lmax;
    sk[e].pair = e;
  }
  qsort(sk, h->n_m2l, sizeof(shiftkey_t), cmp_shift);
  uint32_t* pair_shift = (uint32_t*)malloc(sizeof(uint32_t) * (h->n_m2l ? h->n_m2l : 1));
  long nshift = 0;
  long* shift_rep = (long*)malloc(sizeof(long) * (h->n_m2l ? h->n_m2l : 1));
  for (long e = 0; e < h->n_m2l; ++e) {
    if (e == 0 || cmp_shift(&sk[e], &sk[e - 1]) != 0) shift_rep[nshift++] = e;
    pair_shift[sk[e].pair] = (uint32_t)(nshift - 1);
  }
  zc* mats = (zc*)malloc(sizeof(zc) * (size_t)(nshift ? nshift : 1) * dim * dim);
#pragma omp parallel for schedule(dynamic, 4)
  for (long s = 0; s < nshift; ++s) {
    const shiftkey_t* r = &sk[shift_rep[s]];
    const double unit = h->width / (double)((uint64_t)1 << r->lmax) / 2;
    const double t[3] = {r->x * unit, r->y * unit, r->z * unit};
    translation_matrix_c(h->k + I * h->ki, t, h->order, 1, mats + (size_t)s * dim * dim);
  }
  {
    long ngroups = 0;
    long* gstart = (long*)malloc(sizeof(long) * (h->n_m2l + 1));
    for (long e = 0; e < h->n_m2l; ++e)
      if (e == 0 || h->m2l_t[e] != h->m2l_t[e - 1]) gstart[ngroups++] = e;
    gstart[ngroups] = h->n_m2l;
#pragma omp parallel for schedule(dynamic, 8)
    for (long g = 0; g < ngroups; ++g) {
      zc* L = h->local + (size_t)h->m2l_t[gstart[g]] * dim;
      for (long e = gstart[g]; e < gstart[g + 1]; ++e)
        apply_dense(mats + (size_t)pair_shift[e] * dim * dim, dim,
                    h->multipole + (size_t)h->m2l_s[e] * dim, L);
    }
    free(gstart);
  }
  free(mats); free(sk); free(pair_shift); free(shift_rep);
  near_field(h, src, trg, f32_p2p);
  double t2 = now_s();
  h->seconds[1] = t2 - t1;

  /* downward: parents before children == ascending index; then L2P at leaves */
  zc* dn[HO_MAXLEVEL + 1][8];
  memset(dn, 0, sizeof(dn));
  for (long i = 0; i < nc; ++i) {
    const cell_t* c = &h->cells[i];
    for (uint32_t j = 0; j < c->child_count; ++j) {
      const cell_t* ch = &h->cells[c->child_first + j];
      const int oct = (ch->ix & 1) << 2 | (ch->iy & 1) << 1 | (ch->iz & 1);
      if (!dn[ch->level][oct]) {
        dn[ch->level][oct] = (zc*)malloc(sizeof(zc) * dim * dim);
        shift_matrix(h, ch->level, oct, 0, dn[ch->level][oct]);
      }
      apply_dense(dn[ch->level][oct], dim, h->local + (size_t)i * dim,
                  h->local + (size_t)(c->child_first + j) * dim);
    }
  }
  for (int l = 0; l <= HO_MAXLEVEL; ++l)
    for (int o = 0; o < 8; ++o) free(dn[l][o]);
#pragma omp parallel for schedule(dynamic, 16)
  for (long li = 0; li < h->nleaves; ++li) {
    const cell_t* c = &h->cells[h->leaves[li]];
    const zc* L = h->local + (size_t)h->leaves[li] * dim;
    for (uint32_t b = c->body_first; b < c->body_first + c->body_count; ++b)
      trg[b] += eval_c(1, h->order, L, c->c, h->pos + 3 * b, h->k + I * h->ki);
  }
  h->seconds[2] = now_s() - t2;

  for (long i = 0; i < n; ++i) {
    out[2 * h->index[i]] = creal(trg[i]);
    out[2 * h->index[i] + 1] = cimag(trg[i]);
  }
  free(src);
  free(trg);
  return 0;
}
void ho_fmm_seconds(const ho_fmm* h, double s[3]) { memcpy(s, h->seconds, 3 * sizeof(double)); }
void ho_fmm_expansions(const ho_fmm* h, int which, double* out) {
  const zc* e = which ? h->local : h->multipole;
  const size_t cnt = (size_t)h->ncells * nmdim(h->order);
  if (e)
    memcpy(out, e, sizeof(zc) * cnt);
  else
    memset(out, 0, sizeof(zc) * cnt);
}

void ho_direct_sum(long n, const double* xyz, const double* q, double k, long nt,
                   const long long* target_index, double* out) {
#pragma omp parallel for schedule(static)
  for (long t = 0; t < nt; ++t) {
    const long long ti = target_index ? target_index[t] : t;
    const double* pt = xyz + 3 * ti;
    zc acc = 0;
    for (long j = 0; j < n; ++j) {
      const double dx = pt[0] - xyz[3 * j], dy = pt[1] - xyz[3 * j + 1], dz = pt[2] - xyz[3 * j + 2];
      const double r2 = dx * dx + dy * dy + dz * dz;
      if (r2 == 0) continue;
      const double R = sqrt(r2), amp = 1.0 / (4.0 * HO_PI * R);
      acc += (amp * cos(k * R) + I * amp * sin(k * R)) * (q[2 * j] + I * q[2 * j + 1]);
    }
    out[2 * t] = creal(acc);
    out[2 * t + 1] = cimag(acc);
  }
}

/* complex wavenumber k = kr + i ki (ref: include/hfmm/kernel.hpp:16-23: amp = exp(-ki R) / (4 pi R)) */
void ho_direct_sum_complex_k(long n, const double* xyz, const double* q, double kr, double ki, long nt,
                             const long long* target_index, double* out) {
#pragma omp parallel for schedule(static)
  for (long t = 0; t < nt; ++t) {
    const long long ti = target_index ? target_index[t] : t;
    const double* pt = xyz + 3 * ti;
    zc acc = 0;
    for (long j = 0; j < n; ++j) {
      const double dx = pt[0] - xyz[3 * j], dy = pt[1] - xyz[3 * j + 1], dz = pt[2] - xyz[3 * j + 2];
      const double r2 = dx * dx + dy * dy + dz * dz;
      if (r2 == 0) continue;
      const double R = sqrt(r2), amp = exp(-ki * R) / (4.0 * HO_PI * R), ph = kr * R;
      acc += (amp * cos(ph) + I * amp * sin(ph)) * (q[2 * j] + I * q[2 * j + 1]);
    }
    out[2 * t] = creal(acc);
    out[2 * t + 1] = cimag(acc);
  }
}

/* ------------------------------------------------------------------------------------------
 * GMRES — ref: src/gmres.cpp:35-174.  x0 = 0; modified Gram-Schmidt plus one unconditional
 * re-orthogonalisation pass; complex Givens; stop on |g_{j+1}| <= rtol*||b||; true residual
 * recomputed at restarts and on exit.
 * ---------------------------------------------------------------------------------------- */
static double vnorm(const zc* v, long n) {
  double s = 0;
  for (long i = 0; i < n; ++i) s += creal(v[i]) * creal(v[i]) + cimag(v[i]) * cimag(v[i]);
  return sqrt(s);
}
static zc vdot(const zc* a, const zc* b, long n) {
  zc s = 0;
  for (long i = 0; i < n; ++i) s += conj(a[i]) * b[i];
  return s;
}

int ho_gmres(ho_matvec_cb cb, void* user, long n, const double* rhs_d, double rtol, int restart,
             int max_iterations, double* x_d, double* report, double* residuals,
             int residual_cap) {
  if (!(rtol > 0 && rtol < 1) || restart < 1 || max_iterations < 1) return 1;
  const zc* rhs = (const zc*)rhs_d;
  zc* x = (zc*)x_d;
  const int m = restart;
  int iterations = 0, breakdown = 0, nres = 0;
  double last_est = -1;
  const double bnorm = vnorm(rhs, n);
  for (long i = 0; i < n; ++i) x[i] = 0;
  if (bnorm == 0) {
    report[0] = 0; report[1] = 1; report[2] = 0; report[3] = 0; report[4] = 0;
    return 0;
  }
  const double target = rtol * bnorm;
  zc* H = (zc*)calloc((size_t)(m + 1) * m, sizeof(zc));
#define HH(i, j) H[(size_t)(j) * (m + 1) + (i)]
  zc* cs = (zc*)calloc(m, sizeof(zc));
  zc* sn = (zc*)calloc(m, sizeof(zc));
  zc* g = (zc*)calloc(m + 1, sizeof(zc));
  zc** V = (zc**)calloc(m + 1, sizeof(zc*));
  for (int i = 0; i <= m; ++i) V[i] = (zc*)malloc(sizeof(zc) * n);
  zc* w = (zc*)malloc(sizeof(zc) * n);
  zc* res = (zc*)malloc(sizeof(zc) * n);
  memcpy(res, rhs, sizeof(zc) * n);
  int done = 0;
  while (!done) {
    const double beta = vnorm(res, n);
    if (beta <= target || iterations >= max_iterations) break;
    for (long i = 0; i < n; ++i) V[0][i] = res[i] / beta;
    for (int i = 0; i <= m; ++i) g[i] = 0;
    g[0] = beta;
    int cols = 0;
    for (int j = 0; j < m; ++j) {
      if (iterations >= max_iterations) break;
      cb(user, n, (const double*)V[j], (double*)w);
      const double wscale = vnorm(w, n);
      for (int pass = 0; pass < 2; ++pass)
        for (int i = 0; i <= j; ++i) {
          const zc c = vdot(V[i], w, n);
          if (pass == 0) HH(i, j) = c; else HH(i, j) += c;
          for (long r = 0; r < n; ++r) w[r] -= c * V[i][r];
        }
      double hnext = vnorm(w, n);
      const int broke = hnext <= 1e-14 * (wscale > 1e-300 ? wscale : 1e-300);
      if (broke) hnext = 0;
      for (int i = 0; i < j; ++i) {
        const zc a = HH(i, j), b = HH(i + 1, j);
        HH(i, j) = cs[i] * a + sn[i] * b;
        HH(i + 1, j) = -conj(sn[i]) * a + cs[i] * b;
      }
      const zc a = HH(j, j);
      const double b = hnext, rr = hypot(cabs(a), b);
      if (rr == 0) { cs[j] = 1; sn[j] = 0; }
      else if (cabs(a) == 0) { cs[j] = 0; sn[j] = 1; }
      else { cs[j] = cabs(a) / rr; sn[j] = (a / cabs(a)) * (b / rr); }
      HH(j, j) = cs[j] * a + sn[j] * b;
      g[j + 1] = -conj(sn[j]) * g[j];
      g[j] = cs[j] * g[j];
      ++iterations;
      cols = j + 1;
      last_est = cabs(g[j + 1]);
      if (nres < residual_cap) residuals[nres] = last_est / bnorm;
      ++nres;
      if (broke) { breakdown = 1; done = 1; break; }
      if (last_est <= target) { done = 1; break; }
      for (long r = 0; r < n; ++r) V[j + 1][r] = w[r] / hnext;
    }
    while (cols > 0 && cabs(HH(cols - 1, cols - 1)) == 0) --cols;
    zc* y = (zc*)calloc(cols ? cols : 1, sizeof(zc));
    for (int i = cols - 1; i >= 0; --i) {
      zc s = g[i];
      for (int l = i + 1; l < cols; ++l) s -= HH(i, l) * y[l];
      y[i] = cabs(HH(i, i)) == 0 ? 0 : s / HH(i, i);
    }
    for (int i = 0; i < cols; ++i)
      for (long r = 0; r < n; ++r) x[r] += y[i] * V[i][r];
    free(y);
    if (!done) {
      cb(user, n, (const double*)x, (double*)w);
      for (long r = 0; r < n; ++r) res[r] = rhs[r] - w[r];
    }
  }
  cb(user, n, (const double*)x, (double*)w);
  double s = 0;
  for (long r = 0; r < n; ++r) {
    const zc d = rhs[r] - w[r];
    s += creal(d) * creal(d) + cimag(d) * cimag(d);
  }
  const double final_res = sqrt(s) / bnorm;
  report[0] = iterations;
  report[1] = (final_res <= rtol || (nres > 0 && last_est / bnorm <= rtol)) ? 1 : 0;
  report[2] = breakdown;
  report[3] = bnorm;
  report[4] = final_res;
  for (int i = 0; i <= m; ++i) free(V[i]);
  free(V); free(w); free(res); free(H); free(cs); free(sn); free(g);
#undef HH
  return 0;
}

/* ref: src/solver.cpp:340-357 */
void ho_apply_corrections(long n, int ni, const double* patch_block, const unsigned* near_offset,
                          const unsigned* near_source, const double* near_delta, const double* xd,
                          double* yd) {
  const zc* x = (const zc*)xd;
  zc* y = (zc*)yd;
  if (patch_block) {
    const zc* B = (const zc*)patch_block;
    for (long p = 0; p < n / ni; ++p)
      for (int j = 0; j < ni; ++j) {
        zc acc = 0;
        for (int c = 0; c < ni; ++c) acc += B[((size_t)p * ni + j) * ni + c] * x[p * ni + c];
        y[p * ni + j] += acc;
      }
  }
  if (near_offset && near_delta) {
    const zc* D = (const zc*)near_delta;
    for (long r = 0; r < n; ++r) {
      zc acc = 0;
      for (unsigned e = near_offset[r]; e < near_offset[r + 1]; ++e) acc += D[e] * x[near_source[e]];
      y[r] += acc;
    }
  }
}

/* ref: src/solver.cpp:65-74 (lu_solve with recorded pivots), :376-382 (per-patch apply) */
void ho_block_lu_solve(long npatch, int ni, const double* block_lu, const int* block_piv,
                       double* xd) {
  zc* x = (zc*)xd;
  for (long p = 0; p < npatch; ++p) {
    const zc* a = (const zc*)block_lu + (size_t)p * ni * ni;
    const int* piv = block_piv + p * ni;
    zc* v = x + p * ni;
    for (int c = 0; c < ni; ++c) {
      if (piv[c] != c) { zc tmp = v[c]; v[c] = v[piv[c]]; v[piv[c]] = tmp; }
      for (int r = c + 1; r < ni; ++r) v[r] -= a[r * ni + c] * v[c];
    }
    for (int r = ni - 1; r >= 0; --r) {
      for (int c = r + 1; c < ni; ++c) v[r] -= a[r * ni + c] * v[c];
      v[r] /= a[r * ni + r];
    }
  }
}

/* ============================ correction builders ==========================================
 * ref: src/solver.cpp:78-230 (build_patch_blocks, build_near_corrections), src/geometry.cpp:9-45
 * (centroid, diameter, shape6, map_to_physical), include/hfmm/kernel.hpp:16-23 (green_t). */
typedef struct { double x, y, z; } v3;

/* ref: geometry.cpp:22-27, 40-45 */
static v3 hc_map(const double* node, double z, double e) {
  const double l1 = 1.0 - z - e, l2 = z, l3 = e;
  const double n[6] = {l1 * (2 * l1 - 1), l2 * (2 * l2 - 1), l3 * (2 * l3 - 1), 4 * l1 * l2, 4 * l2 * l3, 4 * l3 * l1};
  v3 r = {0, 0, 0};
  for (int k = 0; k < 6; ++k) {
    r.x += n[k] * node[3 * k];
    r.y += n[k] * node[3 * k + 1];
    r.z += n[k] * node[3 * k + 2];
  }
  return r;
}
/* ref: geometry.cpp:9-20 */
static double hc_diameter(const double* node) {
  v3 c = {0, 0, 0};
  for (int k = 0; k < 6; ++k) { c.x += node[3 * k]; c.y += node[3 * k + 1]; c.z += node[3 * k + 2]; }
  c.x /= 6.0; c.y /= 6.0; c.z /= 6.0;
  double r = 0;
  for (int k = 0; k < 6; ++k) {
    const double dx = node[3 * k] - c.x, dy = node[3 * k + 1] - c.y, dz = node[3 * k + 2] - c.z;
    const double d = sqrt(dx * dx + dy * dy + dz * dz);
    if (d > r) r = d;
  }
  return 2.0 * r;
}
/* ref: kernel.hpp:16-23 */
static zc hc_green(v3 a, v3 b, double kr, double ki) {
  const double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
  const double R = sqrt(dx * dx + dy * dy + dz * dz);
  const double amp = exp(-ki * R) / (4.0 * HO_PI * R);
  const double ph = kr * R;
  return amp * cos(ph) + I * (amp * sin(ph));
}
static double hc_norm2(v3 a, v3 b) {
  const double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
  return dx * dx + dy * dy + dz * dz;
}
/* ref: solver.cpp:40-43 */
static double hc_threshold(const ho_correction_rules* r, size_t patch) {
  return r->near_patch_distance < 0 ? 2.0 * hc_diameter(r->nodes + 18 * patch) : r->near_patch_distance;
}

void ho_correction_samples(const ho_correction_rules* r, double* xyz) {
  const int ni = r->basis_count;
  for (size_t p = 0; p < r->n_patches; ++p)
    for (int j = 0; j < ni; ++j) {
      const v3 v = hc_map(r->nodes + 18 * p, r->sample_ref[2 * j], r->sample_ref[2 * j + 1]);
      xyz[3 * (p * ni + j)] = v.x;
      xyz[3 * (p * ni + j) + 1] = v.y;
      xyz[3 * (p * ni + j) + 2] = v.z;
    }
}

/* ref: solver.cpp:45-62 */
static int hc_lu_factor(zc* a, int* piv, int n) {
  for (int c = 0; c < n; ++c) {
    int best = c;
    for (int r = c + 1; r < n; ++r)
      if (cabs(a[r * n + c]) > cabs(a[best * n + c])) best = r;
    piv[c] = best;
    if (best != c)
      for (int m = 0; m < n; ++m) { zc t = a[c * n + m]; a[c * n + m] = a[best * n + m]; a[best * n + m] = t; }
    if (a[c * n + c] == 0) return 1;
    for (int r = c + 1; r < n; ++r) {
      a[r * n + c] /= a[c * n + c];
      for (int m = c + 1; m < n; ++m) a[r * n + m] -= a[r * n + c] * a[c * n + m];
    }
  }
  return 0;
}

/* ref: solver.cpp:80-128 */
int ho_build_patch_blocks(const ho_correction_rules* r, double kr, double ki, double* patch_block,
                          double* block_lu, int* block_piv) {
  const int ni = r->basis_count;
  const int self_terms = r->mode != 0;
  zc* PB = (zc*)patch_block;
  zc* LU = (zc*)block_lu;
  int singular = 0;
  size_t* first = (size_t*)malloc(sizeof(size_t) * (ni + 1));
  first[0] = 0;
  for (int j = 0; j < ni; ++j) first[j + 1] = first[j] + (self_terms ? (size_t)r->self_npts[j] : 0);
  for (size_t p = 0; p < r->n_patches; ++p) {
    const double* node = r->nodes + 18 * p;
    zc* block = PB + p * ni * ni;
    v3 s[16];
    for (int j = 0; j < ni; ++j) s[j] = hc_map(node, r->sample_ref[2 * j], r->sample_ref[2 * j + 1]);
    for (int j = 0; j < ni; ++j) {
      for (int n = 0; n < ni; ++n) {
        block[j * ni + n] = 0;
        if (hc_norm2(s[j], s[n]) > 0.0) block[j * ni + n] -= hc_green(s[j], s[n], kr, ki) * r->far_weight[n];
      }
      if (!self_terms) continue;
      zc* row = LU + (p * (size_t)ni + j) * ni;
      for (int n = 0; n < ni; ++n) row[n] = 0;
      const v3 obs = s[j];
      for (size_t q = first[j]; q < first[j + 1]; ++q) {
        const v3 rp = hc_map(node, r->self_pts[3 * q], r->self_pts[3 * q + 1]);
        if (hc_norm2(obs, rp) == 0.0) continue;
        const zc g = hc_green(obs, rp, kr, ki);
        const double w = r->self_pts[3 * q + 2];
        for (int n = 0; n < ni; ++n) row[n] += w * r->self_basis[q * ni + n] * g;
      }
      for (int n = 0; n < ni; ++n) block[j * ni + n] += row[n];
    }
    if (self_terms) singular |= hc_lu_factor(LU + p * (size_t)ni * ni, block_piv + p * ni, ni);
  }
  free(first);
  return singular;
}

/* ref: solver.cpp:13-17 */
static unsigned long long hc_cell_key(long long cx, long long cy, long long cz) {
  const unsigned long long mask = (1ull << 21) - 1;
  return (((unsigned long long)cx & mask) << 42) | (((unsigned long long)cy & mask) << 21) | ((unsigned long long)cz & mask);
}
typedef struct { unsigned long long key; unsigned idx; } hc_entry;
static int hc_entry_cmp(const void* a, const void* b) {
  const hc_entry* x = (const hc_entry*)a; const hc_entry* y = (const hc_entry*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}
static int hc_u32_cmp(const void* a, const void* b) {
  const unsigned x = *(const unsigned*)a, y = *(const unsigned*)b;
  return x < y ? -1 : (x > y);
}

/* ref: solver.cpp:132-186 (the hash grid is replaced by a sorted key array: same candidate sets) */
long ho_build_near_lists(const ho_correction_rules* r, unsigned* near_offset, unsigned** near_source) {
  const int ni = r->basis_count;
  const size_t n = (size_t)r->n_patches * ni;
  for (size_t i = 0; i <= n; ++i) near_offset[i] = 0;
  *near_source = NULL;
  if (r->mode != 2) return 0;
  double* thr = (double*)malloc(sizeof(double) * (r->n_patches ? r->n_patches : 1));
  double h = 0;
  for (size_t p = 0; p < r->n_patches; ++p) { thr[p] = hc_threshold(r, p); if (thr[p] > h) h = thr[p]; }
  if (h <= 0.0) { free(thr); return 0; }
  double* xyz = (double*)malloc(sizeof(double) * 3 * (n ? n : 1));
  ho_correction_samples(r, xyz);
  hc_entry* grid = (hc_entry*)malloc(sizeof(hc_entry) * (n ? n : 1));
  for (size_t i = 0; i < n; ++i) {
    grid[i].key = hc_cell_key((long long)floor(xyz[3 * i] / h), (long long)floor(xyz[3 * i + 1] / h), (long long)floor(xyz[3 * i + 2] / h));
    grid[i].idx = (unsigned)i;
  }
  qsort(grid, n, sizeof(hc_entry), hc_entry_cmp);
  size_t cap = 1024, nnz = 0;
  unsigned* out = (unsigned*)malloc(sizeof(unsigned) * cap);
  for (size_t m = 0; m < n; ++m) {
    const size_t begin = nnz;
    const v3 t = {xyz[3 * m], xyz[3 * m + 1], xyz[3 * m + 2]};
    const long long cx = (long long)floor(t.x / h), cy = (long long)floor(t.y / h), cz = (long long)floor(t.z / h);
    for (long long dx = -1; dx <= 1; ++dx)
      for (long long dy = -1; dy <= 1; ++dy)
        for (long long dz = -1; dz <= 1; ++dz) {
          const unsigned long long key = hc_cell_key(cx + dx, cy + dy, cz + dz);
          size_t lo = 0, hi = n;
          while (lo < hi) { const size_t mid = (lo + hi) / 2; if (grid[mid].key < key) lo = mid + 1; else hi = mid; }
          for (size_t e = lo; e < n && grid[e].key == key; ++e) {
            const unsigned s = grid[e].idx;
            if (s / ni == m / ni) continue;
            const v3 sp = {xyz[3 * s], xyz[3 * s + 1], xyz[3 * s + 2]};
            const double r2 = hc_norm2(t, sp);
            if (r2 == 0.0) continue;
            const double th = thr[s / ni];
            if (th > 0.0 && r2 <= th * th) {
              if (nnz == cap) { cap *= 2; out = (unsigned*)realloc(out, sizeof(unsigned) * cap); }
              out[nnz++] = s;
            }
          }
        }
    qsort(out + begin, nnz - begin, sizeof(unsigned), hc_u32_cmp);
    near_offset[m + 1] = (unsigned)nnz;
  }
  free(thr); free(xyz); free(grid);
  *near_source = out;
  return (long)nnz;
}

/* ref: solver.cpp:194-230 */
void ho_build_near_deltas(const ho_correction_rules* r, double kr, double ki, const unsigned* near_offset,
                          const unsigned* near_source, double* near_delta) {
  const int ni = r->basis_count;
  const size_t n = (size_t)r->n_patches * ni;
  zc* D = (zc*)near_delta;
  double* xyz = (double*)malloc(sizeof(double) * 3 * (n ? n : 1));
  ho_correction_samples(r, xyz);
#pragma omp parallel for schedule(dynamic, 64)
  for (long m = 0; m < (long)n; ++m) {
    zc acc[16];
    const v3 t = {xyz[3 * m], xyz[3 * m + 1], xyz[3 * m + 2]};
    unsigned idx = near_offset[m];
    while (idx < near_offset[m + 1]) {
      const unsigned sp = near_source[idx] / (unsigned)ni;
      unsigned end = idx + 1;
      while (end < near_offset[m + 1] && near_source[end] / (unsigned)ni == sp) ++end;
      const double* node = r->nodes + 18 * (size_t)sp;
      for (int nn = 0; nn < ni; ++nn) acc[nn] = 0;
      for (int q = 0; q < r->near_npts; ++q) {
        const v3 rp = hc_map(node, r->near_pts[3 * q], r->near_pts[3 * q + 1]);
        const zc g = hc_green(t, rp, kr, ki);
        const double w = r->near_pts[3 * q + 2];
        for (int nn = 0; nn < ni; ++nn) acc[nn] += w * r->near_basis[q * ni + nn] * g;
      }
      for (; idx < end; ++idx) {
        const unsigned s = near_source[idx];
        const v3 sx = {xyz[3 * s], xyz[3 * s + 1], xyz[3 * s + 2]};
        D[idx] = acc[s % (unsigned)ni] - hc_green(t, sx, kr, ki) * r->far_weight[s % (unsigned)ni];
      }
    }
  }
  free(xyz);
}

void ho_free(void* p) { free(p); }

/* ============================ repartitioning loop ==========================================
 * ref: src/partition.cpp:143-163 (measure_weights), :175-227 (update_alpha) */
void ho_measure_weights(const ho_fmm* h, double* local, double* remote) {
  for (long i = 0; i < h->n; ++i) local[i] = remote[i] = 0.0;
  for (long e = 0; e < h->n_p2p;) {
    const uint32_t t = h->p2p_t[e];
    double partners = 0;
    long f = e;
    for (; f < h->n_p2p && h->p2p_t[f] == t; ++f) partners += (double)h->cells[h->p2p_s[f]].body_count;
    const cell_t* c = &h->cells[t];
    for (uint32_t b = c->body_first; b < c->body_first + c->body_count; ++b) local[h->index[b]] += partners;
    e = f;
  }
  for (long e = 0; e < h->n_m2l;) {
    const uint32_t t = h->m2l_t[e];
    long f = e;
    while (f < h->n_m2l && h->m2l_t[f] == t) ++f;
    const double pairs = (double)(f - e);
    const cell_t* c = &h->cells[t];
    for (uint32_t b = c->body_first; b < c->body_first + c->body_count; ++b) remote[h->index[b]] += pairs;
    e = f;
  }
}

int ho_update_alpha(const double* alpha, const double* runtime, int n, double alpha_max, double* next) {
  if (n < 1 || !(alpha_max > 0)) return 1;
  const double inv_phi = 0.6180339887498948;
  const int budget = 12;
  const double tol = 1e-12 * (alpha_max > 1.0 ? alpha_max : 1.0);
  char* used = (char*)calloc((size_t)n, 1);
#define HO_TAKE(a, out)                                              \
  do {                                                               \
    (out) = -1;                                                      \
    for (int i_ = 0; i_ < n; ++i_)                                   \
      if (!used[i_] && fabs(alpha[i_] - (a)) <= tol) {               \
        used[i_] = 1;                                                \
        (out) = i_;                                                  \
        break;                                                       \
      }                                                              \
  } while (0)
  double lo = 0, hi = alpha_max;
  double x1 = hi - inv_phi * (hi - lo), x2 = lo + inv_phi * (hi - lo);
  int s1, s2;
  HO_TAKE(x1, s1);
  if (s1 < 0) { *next = x1; free(used); return 0; }
  HO_TAKE(x2, s2);
  if (s2 < 0) { *next = x2; free(used); return 0; }
  for (int probes = 2; probes < budget && hi - lo > 1e-6 * alpha_max;) {
    if (runtime[s1] < runtime[s2]) {
      hi = x2; x2 = x1; s2 = s1;
      x1 = hi - inv_phi * (hi - lo);
      HO_TAKE(x1, s1);
      if (s1 < 0) { *next = x1; free(used); return 0; }
    } else {
      lo = x1; x1 = x2; s1 = s2;
      x2 = lo + inv_phi * (hi - lo);
      HO_TAKE(x2, s2);
      if (s2 < 0) { *next = x2; free(used); return 0; }
    }
    ++probes;
  }
#undef HO_TAKE
  int arg = 0;
  for (int i = 1; i < n; ++i)
    if (runtime[i] < runtime[arg]) arg = i;
  *next = alpha[arg];
  free(used);
  return 0;
}

