/* Seeded synthetic mesh generators for the BASELINE.json configs (host C).
 *
 * The reference measures no public dataset; BASELINE.json configs 1-5 are
 * synthetic meshes, generated here once on the host and fed unchanged to both
 * the GPU path and the CPU oracle. Connectivity and vertex order of the
 * icosphere and torus follow the reference's own generators
 * (proj/tests/test_meshes.hpp:94-129 icosphere_mesh, 132-153 torus_mesh) so
 * config 1 is exactly icosphere_mesh(5). Randomness: std::mt19937_64 restated
 * in C, uniform = (x >> 11) * 2^-53, normal = Box-Muller, so the arrays do not
 * depend on any library's distributions. Formulas and seeds: DESIGN.md §5.
 *
 * FMA contraction is disabled at build time (-ffp-contract=off) so positions
 * are identical however the file is compiled.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ---------------------------------------------------------------- mt19937_64 */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i) s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, MA = 0xB5026F5AA96619E9ULL;
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= MA;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

static double mt64_uniform(mt64* s) { return (double)(mt64_next(s) >> 11) * (1.0 / 9007199254740992.0); }
static double mt64_normal(mt64* s) {
  double u1 = 1.0 - mt64_uniform(s); /* (0, 1] */
  double u2 = mt64_uniform(s);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

uint64_t gh_gen_mt64_first(uint64_t seed) { /* self-test hook: 10000th output pinned in tests */
  mt64 s;
  mt64_seed(&s, seed);
  uint64_t x = 0;
  for (int i = 0; i < 10000; ++i) x = mt64_next(&s);
  return x;
}

void gh_gen_free(void* p) { free(p); }

/* ---------------------------------------------------------------- icosphere */
typedef struct {
  uint64_t* keys; /* (a << 32 | b) + 1, 0 = empty */
  int32_t* vals;
  uint64_t mask;
} midmap;

static uint64_t hash64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

static inline void normalize_scale(double* p, double radius) {
  /* Eigen normalized(): v / sqrt(squaredNorm); then * radius */
  double n2 = (p[0] * p[0] + p[1] * p[1]) + p[2] * p[2];
  if (n2 > 0.0) {
    double n = sqrt(n2);
    p[0] = p[0] / n; p[1] = p[1] / n; p[2] = p[2] / n;
  }
  p[0] = p[0] * radius; p[1] = p[1] * radius; p[2] = p[2] * radius;
}

/* icosphere_mesh (test_meshes.hpp:94-129): 10*4^k + 2 vertices. */
int gh_gen_icosphere(int32_t subdivisions, double radius, double** pos_out, int32_t* nv_out, int32_t** faces_out,
                     int32_t* nf_out) {
  const int64_t nv_final = 10LL * (1LL << (2 * subdivisions)) + 2;
  const int64_t nf_final = 20LL * (1LL << (2 * subdivisions));
  if (nv_final > 2147483647LL || nf_final * 3 > 2147483647LL) return 2;
  double* P = (double*)malloc(sizeof(double) * 3 * nv_final);
  int32_t* Fc = (int32_t*)malloc(sizeof(int32_t) * 3 * nf_final);
  int32_t* Fn = (int32_t*)malloc(sizeof(int32_t) * 3 * nf_final);
  if (!P || !Fc || !Fn) { free(P); free(Fc); free(Fn); return 3; }
  const double phi = (1.0 + sqrt(5.0)) / 2.0;
  const double base[12][3] = {{-1, phi, 0}, {1, phi, 0}, {-1, -phi, 0}, {1, -phi, 0}, {0, -1, phi}, {0, 1, phi},
                              {0, -1, -phi}, {0, 1, -phi}, {phi, 0, -1}, {phi, 0, 1}, {-phi, 0, -1}, {-phi, 0, 1}};
  const int32_t bf[20][3] = {{0, 11, 5}, {0, 5, 1}, {0, 1, 7}, {0, 7, 10}, {0, 10, 11}, {1, 5, 9}, {5, 11, 4},
                             {11, 10, 2}, {10, 7, 6}, {7, 1, 8}, {3, 9, 4}, {3, 4, 2}, {3, 2, 6}, {3, 6, 8},
                             {3, 8, 9}, {4, 9, 5}, {2, 4, 11}, {6, 2, 10}, {8, 6, 7}, {9, 8, 1}};
  for (int i = 0; i < 12; ++i) {
    memcpy(P + 3 * i, base[i], sizeof(double) * 3);
    normalize_scale(P + 3 * i, radius);
  }
  memcpy(Fc, bf, sizeof(bf));
  int64_t nv = 12, nf = 20;
  for (int level = 0; level < subdivisions; ++level) {
    int64_t ne = nf * 3 / 2 + 16;
    uint64_t cap = 1;
    while (cap < (uint64_t)ne * 2) cap <<= 1;
    midmap mm;
    mm.keys = (uint64_t*)calloc(cap, sizeof(uint64_t));
    mm.vals = (int32_t*)malloc(sizeof(int32_t) * cap);
    mm.mask = cap - 1;
    if (!mm.keys || !mm.vals) { free(mm.keys); free(mm.vals); free(P); free(Fc); free(Fn); return 3; }
    int64_t k = 0;
    for (int64_t f = 0; f < nf; ++f) {
      int32_t v[3] = {Fc[3 * f], Fc[3 * f + 1], Fc[3 * f + 2]};
      int32_t m[3];
      for (int e = 0; e < 3; ++e) { /* mid(f0,f1), mid(f1,f2), mid(f2,f0) */
        int32_t a = v[e], b = v[(e + 1) % 3];
        int32_t lo = a < b ? a : b, hi = a < b ? b : a;
        uint64_t key = (((uint64_t)lo << 32) | (uint32_t)hi) + 1;
        uint64_t slot = hash64(key) & mm.mask;
        while (mm.keys[slot] && mm.keys[slot] != key) slot = (slot + 1) & mm.mask;
        if (!mm.keys[slot]) {
          mm.keys[slot] = key;
          mm.vals[slot] = (int32_t)nv;
          double* q = P + 3 * nv;
          /* (0.5 * (p_a + p_b)).normalized() * radius */
          q[0] = 0.5 * (P[3 * a] + P[3 * b]);
          q[1] = 0.5 * (P[3 * a + 1] + P[3 * b + 1]);
          q[2] = 0.5 * (P[3 * a + 2] + P[3 * b + 2]);
          normalize_scale(q, radius);
          ++nv;
        }
        m[e] = mm.vals[slot];
      }
      int32_t a = m[0], b = m[1], c = m[2];
      int32_t* o = Fn + 3 * k;
      o[0] = v[0]; o[1] = a; o[2] = c;
      o[3] = v[1]; o[4] = b; o[5] = a;
      o[6] = v[2]; o[7] = c; o[8] = b;
      o[9] = a; o[10] = b; o[11] = c;
      k += 4;
    }
    free(mm.keys);
    free(mm.vals);
    nf = k;
    int32_t* t = Fc;
    Fc = Fn;
    Fn = t;
  }
  free(Fn);
  *pos_out = P;
  *nv_out = (int32_t)nv;
  *faces_out = Fc;
  *nf_out = (int32_t)nf;
  return 0;
}

/* ---------------------------------------------------------------- torus */
/* torus_mesh (test_meshes.hpp:132-153) plus optional seeded displacement along
 * the tube normal n = (cos phi cos theta, cos phi sin theta, sin phi) with
 * N(0, sigma^2) per vertex, drawn in vertex order after `nsources` distinct
 * uniform source draws. */
int gh_gen_torus(int32_t nu, int32_t nvv, double big_radius, double tube_radius, double sigma, uint64_t seed,
                 int32_t nsources, int32_t* sources_out, double** pos_out, int32_t* nv_out, int32_t** faces_out,
                 int32_t* nf_out) {
  const int64_t V = (int64_t)nu * nvv, F = 2 * V;
  if (V > 2147483647LL || 3 * F > 2147483647LL) return 2;
  double* P = (double*)malloc(sizeof(double) * 3 * V);
  int32_t* Fc = (int32_t*)malloc(sizeof(int32_t) * 3 * F);
  if (!P || !Fc) { free(P); free(Fc); return 3; }
  mt64 rng;
  mt64_seed(&rng, seed);
  for (int32_t s = 0; s < nsources; ++s) {
    for (;;) {
      int32_t c = (int32_t)(mt64_next(&rng) % (uint64_t)V);
      int dup = 0;
      for (int32_t q = 0; q < s; ++q) dup |= sources_out[q] == c;
      if (!dup) { sources_out[s] = c; break; }
    }
  }
  for (int64_t i = 0; i < nu; ++i) {
    const double theta = 2.0 * M_PI * (double)i / nu;
    const double ct = cos(theta), st = sin(theta);
    for (int64_t j = 0; j < nvv; ++j) {
      const double phi = 2.0 * M_PI * (double)j / nvv;
      const double cp = cos(phi), sp = sin(phi);
      const double w = big_radius + tube_radius * cp;
      double* p = P + 3 * (i * nvv + j);
      p[0] = w * ct;
      p[1] = w * st;
      p[2] = tube_radius * sp;
      if (sigma > 0.0) {
        const double d = sigma * mt64_normal(&rng);
        p[0] = p[0] + d * (cp * ct);
        p[1] = p[1] + d * (cp * st);
        p[2] = p[2] + d * sp;
      }
    }
  }
#define VID(a, b) ((int32_t)((((a) + nu) % nu) * (int64_t)nvv + ((b) + nvv) % nvv))
  int64_t k = 0;
  for (int64_t i = 0; i < nu; ++i)
    for (int64_t j = 0; j < nvv; ++j) {
      int32_t* o = Fc + 3 * k;
      o[0] = VID(i, j); o[1] = VID(i + 1, j); o[2] = VID(i + 1, j + 1);
      o[3] = VID(i, j); o[4] = VID(i + 1, j + 1); o[5] = VID(i, j + 1);
      k += 2;
    }
#undef VID
  *pos_out = P;
  *nv_out = (int32_t)V;
  *faces_out = Fc;
  *nf_out = (int32_t)F;
  return 0;
}

/* ---------------------------------------------------------------- jittered grid (config 2) */
/* n x n vertices on [0,1]^2, spacing h = 1/(n-1). Cell (i,j) splits along
 * (i,j)-(i+1,j+1) when i+j is even, else along (i+1,j)-(i,j+1). Interior
 * vertices get x,y jitter U(-jitter*h, jitter*h). z = amp * sum_{q<4}
 * sin(2 pi (a_q x + b_q y) + phi_q), a_q, b_q ~ U[1,4], phi_q ~ U[0, 2 pi).
 * Draw order: (a_q, b_q, phi_q) for q = 0..3, then (jx, jy) per interior vertex
 * in index order. */
int gh_gen_grid(int32_t n, double jitter, double amp, uint64_t seed, double** pos_out, int32_t* nv_out,
                int32_t** faces_out, int32_t* nf_out) {
  const int64_t V = (int64_t)n * n, F = 2LL * (n - 1) * (n - 1);
  if (n < 2 || V > 2147483647LL) return 2;
  double* P = (double*)malloc(sizeof(double) * 3 * V);
  int32_t* Fc = (int32_t*)malloc(sizeof(int32_t) * 3 * F);
  if (!P || !Fc) { free(P); free(Fc); return 3; }
  mt64 rng;
  mt64_seed(&rng, seed);
  double a[4], b[4], ph[4];
  for (int q = 0; q < 4; ++q) {
    a[q] = 1.0 + 3.0 * mt64_uniform(&rng);
    b[q] = 1.0 + 3.0 * mt64_uniform(&rng);
    ph[q] = 2.0 * M_PI * mt64_uniform(&rng);
  }
  const double h = 1.0 / (double)(n - 1);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) {
      double x = (double)i * h, y = (double)j * h;
      if (i > 0 && j > 0 && i < n - 1 && j < n - 1 && jitter > 0.0) {
        double jx = (2.0 * mt64_uniform(&rng) - 1.0) * jitter * h;
        double jy = (2.0 * mt64_uniform(&rng) - 1.0) * jitter * h;
        x = x + jx;
        y = y + jy;
      }
      double z = 0.0;
      if (amp != 0.0) {
        for (int q = 0; q < 4; ++q) z += sin(2.0 * M_PI * (a[q] * x + b[q] * y) + ph[q]);
        z = amp * z;
      }
      double* p = P + 3 * (j * n + i);
      p[0] = x; p[1] = y; p[2] = z;
    }
  int64_t k = 0;
  for (int64_t j = 0; j < n - 1; ++j)
    for (int64_t i = 0; i < n - 1; ++i) {
      int32_t v00 = (int32_t)(j * n + i), v10 = v00 + 1, v01 = (int32_t)((j + 1) * n + i), v11 = v01 + 1;
      int32_t* o = Fc + 3 * k;
      if (((i + j) & 1) == 0) {
        o[0] = v00; o[1] = v10; o[2] = v11;
        o[3] = v00; o[4] = v11; o[5] = v01;
      } else {
        o[0] = v00; o[1] = v10; o[2] = v01;
        o[3] = v10; o[4] = v11; o[5] = v01;
      }
      k += 2;
    }
  *pos_out = P;
  *nv_out = (int32_t)V;
  *faces_out = Fc;
  *nf_out = (int32_t)F;
  return 0;
}

/* ---------------------------------------------------------------- spherical-harmonic bump (config 4) */
/* Real spherical harmonics of degree <= lmax with N(0,1) coefficients (drawn
 * l = 0..lmax, m = -l..l); f scaled so max |f| over the vertices is 1; every
 * vertex p (on the unit sphere) becomes p * (1 + amplitude * f(p)). */
int gh_gen_sh_displace(double* P, int32_t nv, int32_t lmax, double amplitude, uint64_t seed) {
  if (lmax < 0 || lmax > 16) return 2;
  mt64 rng;
  mt64_seed(&rng, seed);
  double coef[17 * 17];
  int nc = 0;
  for (int l = 0; l <= lmax; ++l)
    for (int m = -l; m <= l; ++m) coef[nc++] = mt64_normal(&rng);
  double* f = (double*)malloc(sizeof(double) * (nv > 0 ? nv : 1));
  if (!f) return 3;
  double fmax = 0.0;
  for (int64_t v = 0; v < nv; ++v) {
    const double* p = P + 3 * v;
    double r = sqrt((p[0] * p[0] + p[1] * p[1]) + p[2] * p[2]);
    double ct = p[2] / r;
    if (ct > 1.0) ct = 1.0;
    if (ct < -1.0) ct = -1.0;
    double st = sqrt(1.0 - ct * ct);
    double az = atan2(p[1], p[0]);
    /* associated Legendre P_l^m(ct) (no Condon-Shortley phase), orthonormal scaling */
    double Plm[17][17];
    for (int m = 0; m <= lmax; ++m) {
      double pmm = 1.0;
      for (int q = 1; q <= m; ++q) pmm = pmm * (2.0 * q - 1.0) * st;
      Plm[m][m] = pmm;
      if (m + 1 <= lmax) Plm[m + 1][m] = ct * (2.0 * m + 1.0) * pmm;
      for (int l = m + 2; l <= lmax; ++l)
        Plm[l][m] = (ct * (2.0 * l - 1.0) * Plm[l - 1][m] - (double)(l + m - 1) * Plm[l - 2][m]) / (double)(l - m);
    }
    double val = 0.0;
    int c = 0;
    for (int l = 0; l <= lmax; ++l) {
      for (int m = -l; m <= l; ++m, ++c) {
        int am = m < 0 ? -m : m;
        double ratio = 1.0; /* (l-|m|)! / (l+|m|)! */
        for (int q = l - am + 1; q <= l + am; ++q) ratio = ratio / (double)q;
        double norm = sqrt((2.0 * l + 1.0) / (4.0 * M_PI) * ratio);
        double ang = m > 0 ? sqrt(2.0) * cos(m * az) : (m < 0 ? sqrt(2.0) * sin(am * az) : 1.0);
        val += coef[c] * norm * Plm[l][am] * ang;
      }
    }
    f[v] = val;
    double af = fabs(val);
    if (af > fmax) fmax = af;
  }
  if (fmax > 0.0)
    for (int64_t v = 0; v < nv; ++v) {
      double s = 1.0 + amplitude * (f[v] / fmax);
      P[3 * v] = P[3 * v] * s;
      P[3 * v + 1] = P[3 * v + 1] * s;
      P[3 * v + 2] = P[3 * v + 2] * s;
    }
  free(f);
  return 0;
}
