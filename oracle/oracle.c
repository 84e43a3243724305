/*
 * oracle.c — CPU restatement of the reference annealing hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h). Each function cites the reference
 * file:line it restates (paths relative to /root/reference/proj). Arithmetic is
 * written in the reference's evaluation order and must be compiled with
 * -ffp-contract=off (oracle/Makefile) so no multiply-add is fused, matching the
 * reference's x86-64 baseline build (proj/CMakeLists.txt:3-10, no -march, no FMA).
 * Complex products follow GCC's expansion of std::complex<double> operator*:
 * (a+bi)(c+di) = (ac - bd) + (ad + bc)i; complex*real and complex/real are
 * component-wise.
 */
#define _GNU_SOURCE
#include "oracle.h"


#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng.cpp */

/* rng.cpp:12-17 splitmix64 finalizer */
static uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.cpp:23-33 */
void tgo_stream_init(tgo_stream* st, uint64_t global_seed, uint64_t procedure_index) {
  uint64_t s = global_seed ^ mix64(procedure_index + 1);
  for (int w = 0; w < 4; ++w) {
    s += 0x9E3779B97F4A7C15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    st->s[w] = z ^ (z >> 31);
  }
  if ((st->s[0] | st->s[1] | st->s[2] | st->s[3]) == 0) st->s[0] = 1;
}

/* rng.cpp:35-45 xoshiro256++ */
uint64_t tgo_next_u64(tgo_stream* st) {
  uint64_t* s = st->s;
  const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}

/* rng.cpp:47-49 */
double tgo_uniform01(tgo_stream* st) { return (double)(tgo_next_u64(st) >> 11) * 0x1.0p-53; }

/* rng.cpp:51-59 (caller guarantees n >= 1) */
uint64_t tgo_uniform_index(tgo_stream* st, uint64_t n) {
  const uint64_t reject_below = (0 - n) % n;
  for (;;) {
    const uint64_t x = tgo_next_u64(st);
    if (x >= reject_below) return x % n;
  }
}

/* rng.cpp:61-67 Box-Muller; angle = (2*pi)*u2 with std::numbers::pi */
void tgo_normal_pair(tgo_stream* st, double* a, double* b) {
  const double u1 = 1.0 - tgo_uniform01(st);
  const double u2 = tgo_uniform01(st);
  const double r = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * 3.141592653589793 * u2;
  *a = r * cos(angle);
  *b = r * sin(angle);
}

/* ------------------------------------------------------------- spinmc.cpp */

/* spinmc.cpp:65-89: 16 normal pairs column-major into G, then modified Gram-Schmidt. */
void tgo_haar(tgo_stream* st, double* u) {
  double qr[16], qi[16]; /* element (i,j) at i + 4j */
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) tgo_normal_pair(st, &qr[i + 4 * j], &qi[i + 4 * j]);
  for (int j = 0; j < 4; ++j) {
    for (int prev = 0; prev < j; ++prev) {
      double pr = 0.0, pi = 0.0;
      for (int i = 0; i < 4; ++i) { /* proj += conj(q(i,prev)) * q(i,j) */
        const double ar = qr[i + 4 * prev], ai = -qi[i + 4 * prev];
        const double br = qr[i + 4 * j], bi = qi[i + 4 * j];
        const double tr = ar * br - ai * bi;
        const double ti = ar * bi + ai * br;
        pr += tr;
        pi += ti;
      }
      for (int i = 0; i < 4; ++i) { /* q(i,j) -= proj * q(i,prev) */
        const double br = qr[i + 4 * prev], bi = qi[i + 4 * prev];
        const double tr = pr * br - pi * bi;
        const double ti = pr * bi + pi * br;
        qr[i + 4 * j] -= tr;
        qi[i + 4 * j] -= ti;
      }
    }
    double nrm = 0.0;
    for (int i = 0; i < 4; ++i)
      nrm += qr[i + 4 * j] * qr[i + 4 * j] + qi[i + 4 * j] * qi[i + 4 * j];
    nrm = sqrt(nrm);
    for (int i = 0; i < 4; ++i) {
      qr[i + 4 * j] /= nrm;
      qi[i + 4 * j] /= nrm;
    }
  }
  for (int e = 0; e < 16; ++e) {
    u[2 * e] = qr[e];
    u[2 * e + 1] = qi[e];
  }
}

/* spinmc.cpp:91-136 */
int tgo_apply_gate(int spins, const double* psi, int site, const double* u, double* out) {
  if (site < 0 || site + 2 > spins) return -1;
  double ur[4][4], ui[4][4];
  for (int x = 0; x < 4; ++x)
    for (int y = 0; y < 4; ++y) {
      ur[x][y] = u[2 * (x + 4 * y)];
      ui[x][y] = u[2 * (x + 4 * y) + 1];
    }
  const uint64_t groups = (uint64_t)1 << (spins - 2);
  const uint64_t lo_mask = ((uint64_t)1 << site) - 1;
  const uint64_t bit0 = (uint64_t)1 << site;
  const uint64_t bit1 = (uint64_t)1 << (site + 1);
  for (uint64_t g = 0; g < groups; ++g) {
    const uint64_t base = ((g >> site) << (site + 2)) | (g & lo_mask);
    const uint64_t idx[4] = {base, base | bit0, base | bit1, base | bit0 | bit1};
    double vr[4], vi[4];
    for (int y = 0; y < 4; ++y) {
      vr[y] = psi[2 * idx[y]];
      vi[y] = psi[2 * idx[y] + 1];
    }
    for (int x = 0; x < 4; ++x) {
      double re = 0.0, im = 0.0;
      for (int y = 0; y < 4; ++y) {
        re += ur[x][y] * vr[y] - ui[x][y] * vi[y];
        im += ur[x][y] * vi[y] + ui[x][y] * vr[y];
      }
      out[2 * idx[x]] = re;
      out[2 * idx[x] + 1] = im;
    }
  }
  return 0;
}

/* spinmc.cpp:50-54 */
double tgo_state_norm(int spins, const double* psi) {
  const uint64_t n = (uint64_t)1 << spins;
  double sum = 0.0;
  for (uint64_t i = 0; i < n; ++i) sum += psi[2 * i] * psi[2 * i] + psi[2 * i + 1] * psi[2 * i + 1];
  return sqrt(sum);
}

/* spinmc.cpp:56-59 */
static void renormalize(int spins, double* psi) {
  const double inv = 1.0 / tgo_state_norm(spins, psi);
  const uint64_t n = (uint64_t)1 << spins;
  for (uint64_t i = 0; i < 2 * n; ++i) psi[i] *= inv;
}

/* ------------------------------------------------------------- linalg.cpp */

/* linalg.cpp:79-103 gemm_block over the whole output (linalg.cpp:105-113) */
void tgo_gemm(int m, int n, int k, const double* alpha, const double* a, const double* b,
              const double* beta, const double* c, double* out) {
  const double ar_ = alpha[0], ai_ = alpha[1], br_ = beta[0], bi_ = beta[1];
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < m; ++i) {
      double sr = 0.0, si = 0.0;
      for (int kk = 0; kk < k; ++kk) {
        const double avr = a[2 * (i + (size_t)kk * m)], avi = a[2 * (i + (size_t)kk * m) + 1];
        const double bvr = b[2 * (kk + (size_t)j * k)], bvi = b[2 * (kk + (size_t)j * k) + 1];
        const double tr = avr * bvr - avi * bvi;
        const double ti = avr * bvi + avi * bvr;
        sr += tr;
        si += ti;
      }
      const double cr = c[2 * (i + (size_t)j * m)], ci = c[2 * (i + (size_t)j * m) + 1];
      out[2 * (i + (size_t)j * m)] = ar_ * sr - ai_ * si + br_ * cr - bi_ * ci;
      out[2 * (i + (size_t)j * m) + 1] = ar_ * si + ai_ * sr + br_ * ci + bi_ * cr;
    }
  }
}

/* linalg.cpp:131-138 */
double tgo_frobenius(int rows, int cols, const double* a) {
  double sum = 0.0;
  const size_t cnt = (size_t)rows * cols;
  for (size_t idx = 0; idx < cnt; ++idx) sum += a[2 * idx] * a[2 * idx] + a[2 * idx + 1] * a[2 * idx + 1];
  return sqrt(sum);
}

/* linalg.cpp:146-158 */
static double off_diagonal_norm(int n, const double* w) {
  double sum = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      if (i == j) continue;
      const double re = w[2 * (i + j * n)], im = w[2 * (i + j * n) + 1];
      sum += re * re + im * im;
    }
  return sqrt(sum);
}

static int cmp_double(const void* x, const void* y) {
  const double a = *(const double*)x, b = *(const double*)y;
  return (a > b) - (a < b);
}

/* linalg.cpp:161-232 cyclic complex Jacobi */
int tgo_hermitian_eigenvalues(int n, const double* h, double* eig) {
#define W_RE(i, j) w[2 * ((i) + (size_t)(j) * n)]
#define W_IM(i, j) w[2 * ((i) + (size_t)(j) * n) + 1]
  const double h_norm = tgo_frobenius(n, n, h);
  double dev = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const double dr = h[2 * (i + j * n)] - h[2 * (j + i * n)];
      const double di = h[2 * (i + j * n) + 1] - (-h[2 * (j + i * n) + 1]);
      dev += dr * dr + di * di;
    }
  dev = sqrt(dev);
  if (dev > 1e-10 * h_norm) return -1;
  double* w = (double*)malloc(sizeof(double) * 2 * (size_t)n * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const double sr = h[2 * (i + j * n)] + h[2 * (j + i * n)];
      const double si = h[2 * (i + j * n) + 1] + (-h[2 * (j + i * n) + 1]);
      W_RE(i, j) = sr * 0.5;
      W_IM(i, j) = si * 0.5;
    }
  const double target = 1e-12 * h_norm;
  for (int sweep = 0; sweep < 30; ++sweep) {
    if (off_diagonal_norm(n, w) <= target) break;
    for (int p = 0; p + 1 < n; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const double betar = W_RE(p, q), betai = W_IM(p, q);
        const double beta_abs = hypot(betar, betai); /* std::abs(complex) = cabs = hypot */
        if (beta_abs == 0.0) continue;
        const double phr = betar / beta_abs, phi = betai / beta_abs;
        const double app = W_RE(p, p);
        const double aqq = W_RE(q, q);
        const double tau = (aqq - app) / (2.0 * beta_abs);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double cs = 1.0 / sqrt(1.0 + t * t);
        const double sn = t * cs;
        const double cpr = phr * cs, cpi = phi * cs; /* cs * phase */
        const double spr = phr * sn, spi = phi * sn; /* sn * phase */
        for (int i = 0; i < n; ++i) {
          const double wpr = W_RE(i, p), wpi = W_IM(i, p);
          const double wqr = W_RE(i, q), wqi = W_IM(i, q);
          /* (cs*phase)*wip - sn*wiq */
          const double ar = cpr * wpr - cpi * wpi, ai = cpr * wpi + cpi * wpr;
          const double br = wqr * sn, bi = wqi * sn;
          /* (sn*phase)*wip + cs*wiq */
          const double cr = spr * wpr - spi * wpi, ci = spr * wpi + spi * wpr;
          const double dr = wqr * cs, di = wqi * cs;
          W_RE(i, p) = ar - br;
          W_IM(i, p) = ai - bi;
          W_RE(i, q) = cr + dr;
          W_IM(i, q) = ci + di;
        }
        for (int jj = 0; jj < n; ++jj) {
          W_RE(p, jj) = W_RE(jj, p);
          W_IM(p, jj) = -W_IM(jj, p);
          W_RE(q, jj) = W_RE(jj, q);
          W_IM(q, jj) = -W_IM(jj, q);
        }
        const double new_pp = app * cs * cs - 2.0 * beta_abs * cs * sn + aqq * sn * sn;
        const double new_qq = app * sn * sn + 2.0 * beta_abs * cs * sn + aqq * cs * cs;
        W_RE(p, p) = new_pp;
        W_IM(p, p) = 0.0;
        W_RE(q, q) = new_qq;
        W_IM(q, q) = 0.0;
        W_RE(p, q) = 0.0;
        W_IM(p, q) = 0.0;
        W_RE(q, p) = 0.0;
        W_IM(q, p) = 0.0;
      }
    }
  }
  for (int i = 0; i < n; ++i) eig[i] = W_RE(i, i);
  free(w);
  qsort(eig, (size_t)n, sizeof(double), cmp_double);
  return 0;
#undef W_RE
#undef W_IM
}

/* spinmc.cpp:150-176. Psi = psi viewed d_a x d_b column-major (spinmc.cpp:145-148);
 * B = Psi^dagger materialised (linalg.cpp:43-51); rho = gemm(1, Psi, B, 0, zeros). */
int tgo_entropy(int spins, const double* psi, int kind, double* entropy_out) {
  const double nrm = tgo_state_norm(spins, psi);
  if (fabs(nrm - 1.0) > 1e-9) return -1;
  const int da = 1 << (spins / 2), db = 1 << (spins - spins / 2);
  double* b = (double*)malloc(sizeof(double) * 2 * (size_t)da * db);
  double* c = (double*)calloc(2 * (size_t)da * da, sizeof(double));
  double* rho = (double*)malloc(sizeof(double) * 2 * (size_t)da * da);
  for (int j = 0; j < db; ++j)
    for (int i = 0; i < da; ++i) { /* out(j, i) = conj(psi(i, j)) */
      b[2 * (j + (size_t)i * db)] = psi[2 * (i + (size_t)j * da)];
      b[2 * (j + (size_t)i * db) + 1] = -psi[2 * (i + (size_t)j * da) + 1];
    }
  const double one[2] = {1.0, 0.0}, zero[2] = {0.0, 0.0};
  tgo_gemm(da, da, db, one, psi, b, zero, c, rho);
  double entropy = 0.0;
  int rc = 0;
  if (kind == 0) {
    double* eig = (double*)malloc(sizeof(double) * da);
    rc = tgo_hermitian_eigenvalues(da, rho, eig);
    if (rc == 0)
      for (int i = 0; i < da; ++i)
        if (eig[i] > 1e-15) entropy -= eig[i] * log(eig[i]);
    free(eig);
  } else {
    const double f = tgo_frobenius(da, da, rho);
    entropy = -log(f * f);
  }
  free(b);
  free(c);
  free(rho);
  if (rc != 0) return -1;
  *entropy_out = (entropy < 0.0) ? 0.0 : entropy; /* std::max(entropy, 0.0) keeps -0.0 */
  return 0;
}

/* spinmc.cpp:178-184 */
double tgo_temperature(double t0, double t_min, uint64_t step, uint64_t total) {
  const double frac = (double)step / (double)total;
  return t0 * pow(t_min / t0, frac);
}

/* spinmc.cpp:186-191: std::min(x,0.0) then std::max(x,-745.0) */
double tgo_acceptance(double delta, double t) {
  double x = delta / t;
  x = (0.0 < x) ? 0.0 : x;
  x = (x < -745.0) ? -745.0 : x;
  return exp(x);
}

/* spinmc.cpp:37-48 */
static void random_state(int spins, tgo_stream* st, double* psi) {
  const uint64_t n = (uint64_t)1 << spins;
  for (uint64_t i = 0; i < n; ++i) tgo_normal_pair(st, &psi[2 * i], &psi[2 * i + 1]);
  renormalize(spins, psi);
}

/* spinmc.cpp:215-251 with metropolis_step (spinmc.cpp:193-213) inlined. */
int tgo_mc_procedure(const tgo_config* cfg, uint64_t p, double* initial_entropy,
                     double* entropies, uint8_t* accepted, uint8_t* sites, double* u_out,
                     double* p_out) {
  const int spins = cfg->spins;
  if (spins < 2 || spins > 30) return -1;
  if (cfg->t0 <= 0.0 || cfg->t_min <= 0.0 || cfg->t_min > cfg->t0) return -1;
  tgo_stream st;
  tgo_stream_init(&st, cfg->seed, p);
  const size_t n = (size_t)1 << spins;
  double* state = (double*)calloc(2 * n, sizeof(double));
  double* scratch = (double*)malloc(sizeof(double) * 2 * n);
  if (cfg->initial_state == 0)
    state[0] = 1.0;
  else
    random_state(spins, &st, state);
  int rc = 0;
  double current;
  if (tgo_entropy(spins, state, cfg->entropy_kind, &current) != 0) {
    rc = -2;
    goto done;
  }
  *initial_entropy = current;
  for (uint64_t s = 0; s < cfg->steps; ++s) {
    const int site = (int)tgo_uniform_index(&st, (uint64_t)(spins - 1));
    double u[32];
    tgo_haar(&st, u);
    tgo_apply_gate(spins, state, site, u, scratch);
    double proposed;
    if (tgo_entropy(spins, scratch, cfg->entropy_kind, &proposed) != 0) {
      rc = -2;
      goto done;
    }
    const double delta = cfg->objective == 0 ? proposed - current : current - proposed;
    const double t = tgo_temperature(cfg->t0, cfg->t_min, s, cfg->steps);
    const double prob = tgo_acceptance(delta, t);
    const double ud = tgo_uniform01(&st);
    const int acc = ud < prob;
    if (acc) {
      double* tmp = state;
      state = scratch;
      scratch = tmp;
      current = proposed;
    }
    entropies[s] = current;
    if (accepted) accepted[s] = (uint8_t)acc;
    if (sites) sites[s] = (uint8_t)site;
    if (u_out) u_out[s] = ud;
    if (p_out) p_out[s] = prob;
    if (cfg->renormalize_interval > 0 && (s + 1) % cfg->renormalize_interval == 0)
      renormalize(spins, state);
  }
done:
  free(state);
  free(scratch);
  return rc;
}

typedef struct {
  const tgo_config* cfg;
  uint64_t p0, count;
  atomic_ulong next;
  atomic_int rc;
  double *init, *ent;
  uint8_t *acc, *sites;
} pool_ctx;

static void* pool_worker(void* arg) {
  pool_ctx* c = (pool_ctx*)arg;
  const uint64_t steps = c->cfg->steps;
  for (;;) {
    const uint64_t r = atomic_fetch_add(&c->next, 1);
    if (r >= c->count) break;
    const int rc = tgo_mc_procedure(c->cfg, c->p0 + r, &c->init[r], c->ent + r * steps,
                                    c->acc ? c->acc + r * steps : NULL,
                                    c->sites ? c->sites + r * steps : NULL, NULL, NULL);
    if (rc != 0) {
      int zero = 0;
      atomic_compare_exchange_strong(&c->rc, &zero, rc);
    }
  }
  return NULL;
}

int tgo_run_pool(const tgo_config* cfg, uint64_t p0, uint64_t count, int threads,
                 double* initial_entropy, double* entropies, uint8_t* accepted, uint8_t* sites) {
  pool_ctx c;
  c.cfg = cfg;
  c.p0 = p0;
  c.count = count;
  atomic_init(&c.next, 0);
  atomic_init(&c.rc, 0);
  c.init = initial_entropy;
  c.ent = entropies;
  c.acc = accepted;
  c.sites = sites;
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, pool_worker, &c);
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  free(th);
  return atomic_load(&c.rc);
}

/* spinmc.cpp:253-269, bench.cpp:401-407 */
double tgo_average_entropy(uint64_t procedures, uint64_t steps, const double* initial_entropy,
                           const double* entropies) {
  double sum = 0.0;
  for (uint64_t p = 0; p < procedures; ++p)
    sum += steps > 0 ? entropies[p * steps + steps - 1] : initial_entropy[p];
  return sum / (double)procedures;
}
