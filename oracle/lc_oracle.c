/* TEST INFRASTRUCTURE ONLY — see lc_oracle.h.  fp64 restatement of the
 * reference algorithms; every function cites the reference file:line (paths
 * relative to /root/reference/proj) it restates.  Plain C11 + OpenMP over
 * independent channels (the reference's parallel_for, parallel.hpp:17-38). */
#include "lc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double re, im;
} cd;

static const double kPi = 3.14159265358979323846;

/* cmul: explicit complex multiply (types.hpp:17-20). */
static inline cd cmul(cd a, cd b) {
  cd r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}
static inline cd cadd(cd a, cd b) {
  cd r = {a.re + b.re, a.im + b.im};
  return r;
}
static inline cd cconj(cd a) {
  cd r = {a.re, -a.im};
  return r;
}
static inline cd cpolar(double theta) {
  cd r = {cos(theta), sin(theta)};
  return r;
}

/* ------------------------------------------------------------------------ */
/* RNG: xoshiro256++ seeded by splitmix64 (rng.cpp:12-69).                   */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t seed;
  uint64_t s[4];
  double cached;
  int has_cached;
} rng_t;

static uint64_t splitmix64(uint64_t* x) { /* rng.cpp:12-18 */
  *x += 0x9E3779B97F4A7C15ULL;
  uint64_t z = *x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static rng_t rng_make(uint64_t seed) { /* rng.cpp:29-33 */
  rng_t r;
  memset(&r, 0, sizeof(r));
  r.seed = seed;
  uint64_t x = seed;
  for (int i = 0; i < 4; ++i) r.s[i] = splitmix64(&x);
  if ((r.s[0] | r.s[1] | r.s[2] | r.s[3]) == 0) r.s[0] = 1;
  return r;
}
static rng_t rng_child(const rng_t* p, uint64_t stream) { /* rng.cpp:35-39 */
  uint64_t base = p->seed;
  uint64_t v = splitmix64(&base) + stream;
  uint64_t child_seed = splitmix64(&v); /* mix64(v) == splitmix64(copy of v) */
  return rng_make(child_seed);
}
static uint64_t rng_next(rng_t* r) { /* rng.cpp:41-51 */
  uint64_t* s = r->s;
  const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}
static double rng_uniform(rng_t* r) { /* rng.cpp:53-55 */
  return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}
static double rng_normal(rng_t* r) { /* rng.cpp:57-69 (Box-Muller, cached sine draw) */
  if (r->has_cached) {
    r->has_cached = 0;
    return r->cached;
  }
  const double u1 = 1.0 - rng_uniform(r);
  const double u2 = rng_uniform(r);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * kPi * u2;
  r->cached = radius * sin(angle);
  r->has_cached = 1;
  return radius * cos(angle);
}

int lco_normal_draws(uint64_t seed, uint64_t stream, size_t count, double* out) {
  if (count == 0) return 1; /* rng.cpp:72 */
  rng_t base = rng_make(seed);
  rng_t r = rng_child(&base, stream);
  for (size_t i = 0; i < count; ++i) out[i] = rng_normal(&r);
  return 0;
}
int lco_uniform_draws(uint64_t seed, uint64_t stream, size_t count, double* out) {
  rng_t base = rng_make(seed);
  rng_t r = rng_child(&base, stream);
  for (size_t i = 0; i < count; ++i) out[i] = rng_uniform(&r);
  return 0;
}

/* init_kernels + geometric_envelope (regularize.cpp:66-91). */
int lco_init_kernels(int kind, size_t H, size_t N, uint64_t seed, double* K, double* D) {
  if (H == 0 || N == 0) return 1;
  rng_t base = rng_make(seed);
  for (size_t h = 0; h < H; ++h) {
    rng_t st = rng_child(&base, h);
    const double decay = pow((double)H / 2.0, (double)h / (double)H);
    for (size_t i = 0; i < N; ++i) {
      double v = rng_normal(&st);
      if (kind) v *= exp(-((double)i / (double)N) * decay);
      K[h * N + i] = v;
    }
  }
  rng_t sk = rng_child(&base, H);
  for (size_t h = 0; h < H; ++h) D[h] = rng_normal(&sk);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Regularizers (regularize.cpp:12-64, 93-107).                              */
/* ------------------------------------------------------------------------ */
int lco_squash(const double* k, size_t n, double lambda, double* out) { /* :12-20 */
  if (lambda < 0.0) return 1;
  for (size_t i = 0; i < n; ++i) {
    const double mag = fabs(k[i]) - lambda;
    out[i] = mag > 0.0 ? copysign(mag, k[i]) : 0.0;
  }
  return 0;
}

int lco_smooth(const double* k, size_t n, size_t p, double* out) { /* :22-34 */
  const double inv_w = 1.0 / (double)(2 * p + 1);
  for (size_t i = 0; i < n; ++i) {
    double acc = 0.0;
    const size_t lo = (i >= p) ? i - p : 0;
    const size_t hi = (i + p < n - 1) ? i + p : n - 1;
    for (size_t j = lo; j <= hi; ++j) acc += k[j];
    out[i] = acc * inv_w;
  }
  return 0;
}

/* dft_naive / idft_naive (dft_reference.cpp:43-67). */
static void dft_naive_c(const cd* x, size_t n, int inverse, cd* y) {
  cd* roots = (cd*)malloc(sizeof(cd) * n);
  const double step = -2.0 * kPi / (double)n;
  for (size_t t = 0; t < n; ++t) roots[t] = cpolar(step * (double)t);
  const double inv_n = 1.0 / (double)n;
  for (size_t j = 0; j < n; ++j) {
    cd acc = {0.0, 0.0};
    for (size_t k = 0; k < n; ++k) {
      cd w = roots[(j * k) % n];
      if (inverse) w = cconj(w);
      acc = cadd(acc, cmul(x[k], w));
    }
    if (inverse) {
      acc.re *= inv_n;
      acc.im *= inv_n;
    }
    y[j] = acc;
  }
  free(roots);
}
int lco_dft_naive(const double* x, size_t n, int inverse, double* y) {
  dft_naive_c((const cd*)x, n, inverse, (cd*)y);
  return 0;
}

int lco_smooth_frequency(const double* k, size_t n, size_t p, double* out) { /* :36-53 */
  if (n == 0) return 0;
  cd* x = (cd*)calloc(n, sizeof(cd));
  cd* s = (cd*)malloc(sizeof(cd) * n);
  cd* t = (cd*)malloc(sizeof(cd) * n);
  for (size_t i = 0; i < n; ++i) x[i].re = k[i];
  dft_naive_c(x, n, 0, s);
  const double inv_w = 1.0 / (double)(2 * p + 1);
  for (size_t i = 0; i < n; ++i) {
    cd acc = {0.0, 0.0};
    for (size_t off = 0; off <= 2 * p; ++off) {
      long long j = ((long long)(i + off) - (long long)p) % (long long)n;
      if (j < 0) j += (long long)n;
      acc = cadd(acc, s[j]);
    }
    t[i].re = acc.re * inv_w;
    t[i].im = acc.im * inv_w;
  }
  dft_naive_c(t, n, 1, x);
  for (size_t i = 0; i < n; ++i) out[i] = x[i].re;
  free(x);
  free(s);
  free(t);
  return 0;
}

/* Dropout multiplier per element: 0 (dropped) or 1/(1-rate) (kept), drawn
 * from child stream h of SeededRng(seed), one uniform per element in order
 * (regularize.cpp:55-64, 96-100).  Identity (1.0) when !training or rate==0. */
int lco_dropout_mask(size_t H, size_t N, double rate, uint64_t seed, int training,
                     double* mask) {
  if (rate < 0.0 || rate >= 1.0) return 1;
  rng_t base = rng_make(seed);
  const double keep = 1.0 / (1.0 - rate);
  for (size_t h = 0; h < H; ++h) {
    rng_t st = rng_child(&base, h);
    for (size_t i = 0; i < N; ++i)
      mask[h * N + i] = (!training || rate == 0.0) ? 1.0
                        : (rng_uniform(&st) < rate) ? 0.0
                                                    : keep;
  }
  return 0;
}

/* regularize_bank: dropout -> smooth (time or frequency) -> squash
 * (regularize.cpp:93-107). */
int lco_regularize_bank(const double* K, size_t H, size_t N, double lambda, size_t p,
                        double rate, int domain, uint64_t seed, int training, double* Kout) {
  if (lambda < 0.0 || rate < 0.0 || rate >= 1.0) return 1;
  double* mask = (double*)malloc(sizeof(double) * H * N);
  lco_dropout_mask(H, N, rate, seed, training, mask);
  double* a = (double*)malloc(sizeof(double) * N);
  double* b = (double*)malloc(sizeof(double) * N);
  for (size_t h = 0; h < H; ++h) {
    for (size_t i = 0; i < N; ++i)
      a[i] = (mask[h * N + i] == 1.0) ? K[h * N + i] : K[h * N + i] * mask[h * N + i];
    if (domain)
      lco_smooth_frequency(a, N, p, b);
    else
      lco_smooth(a, N, p, b);
    lco_squash(b, N, lambda, Kout + h * N);
  }
  free(mask);
  free(a);
  free(b);
  return 0;
}

/* Chain rule of regularize_bank (time-domain smooth): smooth is a symmetric
 * zero-padded band (self-adjoint), squash' = 1[|s| > lambda], dropout' = mask. */
int lco_regularizer_backward(const double* K, size_t H, size_t N, double lambda, size_t p,
                             double rate, uint64_t seed, int training, const double* dKbar,
                             double* dK) {
  double* mask = (double*)malloc(sizeof(double) * H * N);
  if (lco_dropout_mask(H, N, rate, seed, training, mask)) {
    free(mask);
    return 1;
  }
  double* a = (double*)malloc(sizeof(double) * N);
  double* s = (double*)malloc(sizeof(double) * N);
  double* g = (double*)malloc(sizeof(double) * N);
  for (size_t h = 0; h < H; ++h) {
    for (size_t i = 0; i < N; ++i) a[i] = K[h * N + i] * mask[h * N + i];
    lco_smooth(a, N, p, s);
    for (size_t i = 0; i < N; ++i) g[i] = fabs(s[i]) > lambda ? dKbar[h * N + i] : 0.0;
    lco_smooth(g, N, p, s);
    for (size_t i = 0; i < N; ++i) dK[h * N + i] = s[i] * mask[h * N + i];
  }
  free(mask);
  free(a);
  free(s);
  free(g);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Butterfly plan (butterfly.cpp:11-118) and stage walk (:124-185).          */
/* ------------------------------------------------------------------------ */
typedef struct {
  size_t factor, segment, rest;
  cd* block;   /* factor x factor, entry (p,q) = exp(-2 pi i ((pq) mod f)/f)  (:13-20) */
  cd* twiddle; /* segment entries, (j,k) -> exp(-2 pi i jk / segment)         (:59-70) */
} stage_t;

typedef struct {
  size_t n, r, nstages;
  stage_t* st;
  uint32_t* output_map;
} plan_t;

static size_t greedy_factor(size_t L, size_t r) { /* :23-27 */
  for (size_t d = (L < r ? L : r); d >= 2; --d)
    if (L % d == 0) return d;
  return 0;
}

static void plan_free(plan_t* p) {
  for (size_t i = 0; i < p->nstages; ++i) {
    free(p->st[i].block);
    free(p->st[i].twiddle);
  }
  free(p->st);
  free(p->output_map);
  memset(p, 0, sizeof(*p));
}

static int plan_build(size_t n, size_t r, plan_t* p) { /* build_plan :72-118 */
  memset(p, 0, sizeof(*p));
  if (n == 0 || r < 2 || n > 0xFFFFFFFFull) return 2;
  p->n = n;
  p->r = r;
  p->st = (stage_t*)calloc(64, sizeof(stage_t));
  size_t seg = n;
  while (seg > 1) {
    const size_t f = (seg <= r) ? seg : greedy_factor(seg, r);
    if (f == 0) {
      plan_free(p);
      return 2;
    }
    stage_t* s = &p->st[p->nstages++];
    s->factor = f;
    s->segment = seg;
    s->rest = seg / f;
    s->block = (cd*)malloc(sizeof(cd) * f * f);
    const double bstep = -2.0 * kPi / (double)f;
    for (size_t a = 0; a < f; ++a)
      for (size_t b = 0; b < f; ++b) s->block[a * f + b] = cpolar(bstep * (double)((a * b) % f));
    s->twiddle = (cd*)malloc(sizeof(cd) * seg);
    const double tstep = -2.0 * kPi / (double)seg;
    for (size_t j = 0; j < f; ++j)
      for (size_t k = 0; k < s->rest; ++k)
        s->twiddle[j * s->rest + k] = cpolar(tstep * (double)(j * k));
    seg = s->rest;
  }
  /* composed trailing transposes (:103-116) */
  p->output_map = (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (size_t i = 0; i < n; ++i) p->output_map[i] = (uint32_t)i;
  for (size_t d = 0; d + 1 < p->nstages; ++d) {
    const size_t L = p->st[d].segment, f = p->st[d].factor, rest = L / f;
    for (size_t i = 0; i < n; ++i) {
      const size_t off = (p->output_map[i] / L) * L;
      const size_t local = p->output_map[i] % L;
      /* transpose(f, rest).map[local]: local = j2*f + j1 -> j1*rest + j2 */
      const size_t j2 = local / f, j1 = local % f;
      p->output_map[i] = (uint32_t)(off + j1 * rest + j2);
    }
  }
  return 0;
}

/* apply_stages (butterfly.cpp:124-163) with blocks[s] (NULL => plan DFT
 * blocks); optionally saves each stage's gathered block input.  gather map of
 * transpose(f, rest): out[i] = in[(i % f) * rest + i / f]; scatter (inverse):
 * out[i] = in[(i % rest) * f + i / rest]. */
static void apply_stages(const plan_t* p, cd* const* blocks, const cd* x, cd* out, cd* work,
                         cd* tmp, cd** saved) {
  const size_t n = p->n;
  memcpy(work, x, sizeof(cd) * n);
  for (size_t si = 0; si < p->nstages; ++si) {
    const stage_t* st = &p->st[si];
    const cd* blk = blocks ? blocks[si] : st->block;
    const size_t L = st->segment, f = st->factor, rest = st->rest;
    for (size_t off = 0; off < n; off += L)
      for (size_t i = 0; i < L; ++i) tmp[off + i] = work[off + (i % f) * rest + i / f];
    if (saved) memcpy(saved[si], tmp, sizeof(cd) * n);
    for (size_t base = 0; base < n; base += f)
      for (size_t a = 0; a < f; ++a) {
        cd acc = {0.0, 0.0};
        for (size_t q = 0; q < f; ++q) acc = cadd(acc, cmul(blk[a * f + q], tmp[base + q]));
        work[base + a] = acc;
      }
    for (size_t off = 0; off < n; off += L)
      for (size_t i = 0; i < L; ++i)
        tmp[off + i] = cmul(work[off + (i % rest) * f + i / rest], st->twiddle[i]);
    memcpy(work, tmp, sizeof(cd) * n);
  }
  for (size_t i = 0; i < n; ++i) out[i] = work[p->output_map[i]];
}

/* apply_plan (butterfly.cpp:173-185): inverse = conj(F conj(x)) / n. */
static void apply_plan_c(const plan_t* p, const cd* x, int inverse, cd* y, cd* w1, cd* w2,
                         cd* w3) {
  const size_t n = p->n;
  if (!inverse) {
    apply_stages(p, NULL, x, y, w1, w2, NULL);
    return;
  }
  for (size_t i = 0; i < n; ++i) w3[i] = cconj(x[i]);
  apply_stages(p, NULL, w3, y, w1, w2, NULL);
  const double inv_n = 1.0 / (double)n;
  for (size_t i = 0; i < n; ++i) {
    y[i].re = y[i].re * inv_n;
    y[i].im = -y[i].im * inv_n;
  }
}

int lco_plan_factors(size_t n, size_t r, size_t* factors, size_t* count) {
  plan_t p;
  int rc = plan_build(n, r, &p);
  if (rc) return rc;
  *count = p.nstages;
  for (size_t i = 0; i < p.nstages; ++i) factors[i] = p.st[i].factor;
  plan_free(&p);
  return 0;
}

int lco_apply_plan(size_t n, size_t r, const double* x, int inverse, double* y) {
  plan_t p;
  int rc = plan_build(n, r, &p);
  if (rc) return rc;
  cd* w = (cd*)malloc(sizeof(cd) * 3 * n);
  apply_plan_c(&p, (const cd*)x, inverse, (cd*)y, w, w + n, w + 2 * n);
  free(w);
  plan_free(&p);
  return 0;
}

/* conv_butterfly (butterfly.cpp:187-210) using a prebuilt plan of length
 * n = N (circular) or 2N (causal).  ws: 6n complex scratch. */
static void conv_plan(const plan_t* p, const cd* u, const cd* k, size_t N, int mode, cd* y,
                      cd* ws) {
  const size_t n = p->n;
  cd *pu = ws, *pk = ws + n, *su = ws + 2 * n, *sk = ws + 3 * n, *w1 = ws + 4 * n,
     *w2 = ws + 5 * n;
  memset(pu, 0, sizeof(cd) * n);
  memset(pk, 0, sizeof(cd) * n);
  memcpy(pu, u, sizeof(cd) * N);
  memcpy(pk, k, sizeof(cd) * N);
  apply_plan_c(p, pu, 0, su, w1, w2, NULL);
  apply_plan_c(p, pk, 0, sk, w1, w2, NULL);
  for (size_t i = 0; i < n; ++i) su[i] = cmul(su[i], sk[i]);
  apply_plan_c(p, su, 1, pu, w1, w2, pk);
  memcpy(y, pu, sizeof(cd) * N);
  (void)mode;
}

int lco_conv_butterfly(const double* u, const double* k, size_t N, int mode, double* y) {
  plan_t p;
  int rc = plan_build(mode ? 2 * N : N, 16, &p);
  if (rc) return rc;
  cd* ws = (cd*)malloc(sizeof(cd) * 6 * p.n);
  conv_plan(&p, (const cd*)u, (const cd*)k, N, mode, (cd*)y, ws);
  free(ws);
  plan_free(&p);
  return 0;
}

/* conv_{causal,circular}_naive_real (dft_reference.cpp:93-117). */
int lco_conv_naive_real(const double* u, const double* k, size_t N, int mode, double* y) {
  for (size_t i = 0; i < N; ++i) {
    double acc = 0.0;
    if (mode)
      for (size_t j = 0; j <= i; ++j) acc += k[j] * u[i - j];
    else
      for (size_t j = 0; j < N; ++j) acc += u[j] * k[(i + N - j) % N];
    y[i] = acc;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Layer forward (regularize.cpp:149-190, butterfly engine) and backward.    */
/* ------------------------------------------------------------------------ */

/* Spectra of the regularized kernels, one length-n transform per head
 * (butterfly.cpp:205 recomputes it per channel; the result is identical). */
static cd* kernel_spectra(const plan_t* p, const double* Kbar, size_t H, size_t N) {
  const size_t n = p->n;
  cd* kf = (cd*)malloc(sizeof(cd) * H * n);
#pragma omp parallel
  {
    cd* ws = (cd*)malloc(sizeof(cd) * 3 * n);
#pragma omp for schedule(static)
    for (size_t h = 0; h < H; ++h) {
      memset(ws, 0, sizeof(cd) * n);
      for (size_t i = 0; i < N; ++i) ws[i].re = Kbar[h * N + i];
      apply_plan_c(p, ws, 0, kf + h * n, ws + n, ws + 2 * n, NULL);
    }
    free(ws);
  }
  return kf;
}

/* y[b,h] = Re conv(u[b,h], Kbar[h]) + D[h] u[b,h] (regularize.cpp:177-188). */
int lco_long_conv_forward(const double* u, size_t B, size_t H, size_t N, const double* Kbar,
                          const double* D, int mode, double* y) {
  plan_t p;
  int rc = plan_build(mode ? 2 * N : N, 16, &p);
  if (rc) return rc;
  const size_t n = p.n;
  cd* kf = kernel_spectra(&p, Kbar, H, N);
#pragma omp parallel
  {
    cd* ws = (cd*)malloc(sizeof(cd) * 5 * n);
#pragma omp for schedule(static)
    for (size_t task = 0; task < B * H; ++task) {
      const size_t h = task % H;
      const double* uc = u + task * N;
      cd *a = ws, *s = ws + n, *w1 = ws + 2 * n, *w2 = ws + 3 * n, *w3 = ws + 4 * n;
      memset(a, 0, sizeof(cd) * n);
      for (size_t i = 0; i < N; ++i) a[i].re = uc[i];
      apply_plan_c(&p, a, 0, s, w1, w2, NULL);
      for (size_t i = 0; i < n; ++i) s[i] = cmul(s[i], kf[h * n + i]);
      apply_plan_c(&p, s, 1, a, w1, w2, w3);
      for (size_t i = 0; i < N; ++i) y[task * N + i] = a[i].re + D[h] * uc[i];
    }
    free(ws);
  }
  free(kf);
  plan_free(&p);
  return 0;
}

int lco_regularized_long_conv(const double* u, size_t B, size_t H, size_t N, const double* K,
                              const double* D, double lambda, size_t p, double rate,
                              int domain, uint64_t seed, int mode, int training, double* y) {
  double* kbar = (double*)malloc(sizeof(double) * H * N);
  int rc = lco_regularize_bank(K, H, N, lambda, p, rate, domain, seed, training, kbar);
  if (!rc) rc = lco_long_conv_forward(u, B, H, N, kbar, D, mode, y);
  free(kbar);
  return rc;
}

/* Backward, restated in the frequency domain on the same transform length:
 *   du    = IFFT(conj(Kf) . DY)[:N] + D dy         (correlation with Kbar)
 *   dKbar = Re IFFT(sum_b conj(U_b) . DY_b)[:N]     (correlation of dy with u)
 *   dD    = sum_{b,t} dy u
 * The 2N zero-pad makes both correlations exact for the causal layer
 * (circular mode: length-N circular correlations). */
int lco_long_conv_backward(const double* u, const double* dy, size_t B, size_t H, size_t N,
                           const double* Kbar, const double* D, int mode, double* du,
                           double* dKbar, double* dD) {
  plan_t p;
  int rc = plan_build(mode ? 2 * N : N, 16, &p);
  if (rc) return rc;
  const size_t n = p.n;
  cd* kf = kernel_spectra(&p, Kbar, H, N);
#pragma omp parallel
  {
    cd* ws = (cd*)malloc(sizeof(cd) * 7 * n);
#pragma omp for schedule(static)
    for (size_t h = 0; h < H; ++h) {
      cd *a = ws, *sdy = ws + n, *su = ws + 2 * n, *acc = ws + 3 * n, *w1 = ws + 4 * n,
         *w2 = ws + 5 * n, *w3 = ws + 6 * n;
      memset(acc, 0, sizeof(cd) * n);
      double dd = 0.0;
      for (size_t b = 0; b < B; ++b) {
        const double* uc = u + (b * H + h) * N;
        const double* gc = dy + (b * H + h) * N;
        memset(a, 0, sizeof(cd) * n);
        for (size_t i = 0; i < N; ++i) a[i].re = gc[i];
        apply_plan_c(&p, a, 0, sdy, w1, w2, NULL);
        memset(a, 0, sizeof(cd) * n);
        for (size_t i = 0; i < N; ++i) {
          a[i].re = uc[i];
          dd += gc[i] * uc[i];
        }
        apply_plan_c(&p, a, 0, su, w1, w2, NULL);
        for (size_t i = 0; i < n; ++i) {
          acc[i] = cadd(acc[i], cmul(cconj(su[i]), sdy[i]));
          su[i] = cmul(cconj(kf[h * n + i]), sdy[i]);
        }
        apply_plan_c(&p, su, 1, a, w1, w2, w3);
        for (size_t i = 0; i < N; ++i) du[(b * H + h) * N + i] = a[i].re + D[h] * gc[i];
      }
      apply_plan_c(&p, acc, 1, a, w1, w2, w3);
      for (size_t i = 0; i < N; ++i) dKbar[h * N + i] = a[i].re;
      dD[h] = dd;
    }
    free(ws);
  }
  free(kf);
  plan_free(&p);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Three-pass (three_pass.cpp:82-122, 183-254).                              */
/* ------------------------------------------------------------------------ */

/* d_k[a*l + tau] = l * K_hat[tau*m + a], K_hat = F_n k (three_pass.cpp:197-203). */
static int three_pass_dk_c(const cd* k, size_t n, size_t l, size_t m, cd* dk) {
  plan_t full;
  int rc = plan_build(n, 16, &full);
  if (rc) return rc;
  cd* w = (cd*)malloc(sizeof(cd) * 3 * n);
  apply_plan_c(&full, k, 0, w, w + n, w + 2 * n, NULL);
  for (size_t a = 0; a < m; ++a)
    for (size_t tau = 0; tau < l; ++tau) {
      dk[a * l + tau].re = w[tau * m + a].re * (double)l;
      dk[a * l + tau].im = w[tau * m + a].im * (double)l;
    }
  free(w);
  plan_free(&full);
  return 0;
}

int lco_three_pass_dk(const double* k, size_t n, size_t l, size_t m, double* dk) {
  if (l == 0 || m == 0 || l * m != n) return 1;
  return three_pass_dk_c((const cd*)k, n, l, m, (cd*)dk);
}

/* Circular conv of length n = l*m through the three passes:
 * pass 1 = B^T (entry (j,k,tau) = w_n^{k (j l + tau)} with (j,k) swapped by
 * the transpose: y[j l + tau] = sum_k w_n^{j (k l + tau)} x[k l + tau]);
 * pass 2 = m middle blocks, each an l-point FFT conv against its d_k slice
 * (three_pass.cpp:211-221); pass 3 = (B^-1)^T = conj(B)/m transposed-back
 * (three_pass.cpp:138-147, 253). */
int lco_conv_three_pass(const double* u_, const double* k_, size_t n, size_t l, size_t m,
                        double* y_) {
  if (l == 0 || m == 0 || l * m != n) return 1;
  const cd* u = (const cd*)u_;
  cd* y = (cd*)y_;
  cd* dk = (cd*)malloc(sizeof(cd) * n);
  int rc = three_pass_dk_c((const cd*)k_, n, l, m, dk);
  if (rc) {
    free(dk);
    return rc;
  }
  plan_t inner;
  rc = plan_build(l, 16, &inner);
  if (rc) {
    free(dk);
    return rc;
  }
  cd* roots = (cd*)malloc(sizeof(cd) * n);
  const double step = -2.0 * kPi / (double)n;
  for (size_t t = 0; t < n; ++t) roots[t] = cpolar(step * (double)t);
  cd* buf = (cd*)malloc(sizeof(cd) * n);
  /* pass 1: mixer.transpose().apply -> entry(j,k,tau) of the transposed
   * matrix = base entry with (j,k) swapped = roots[(j*(k*l+tau)) % n]. */
  for (size_t tau = 0; tau < l; ++tau)
    for (size_t j = 0; j < m; ++j) {
      cd acc = {0.0, 0.0};
      for (size_t kk = 0; kk < m; ++kk)
        acc = cadd(acc, cmul(roots[(j * (kk * l + tau)) % n], u[kk * l + tau]));
      buf[j * l + tau] = acc;
    }
  /* pass 2 */
  cd* ws = (cd*)malloc(sizeof(cd) * 5 * l);
  const double inv_l = 1.0 / (double)l;
  for (size_t a = 0; a < m; ++a) {
    cd *z = ws, *w1 = ws + l, *w2 = ws + 2 * l, *w3 = ws + 3 * l, *bk = ws + 4 * l;
    apply_plan_c(&inner, buf + a * l, 0, z, w1, w2, NULL);
    for (size_t tau = 0; tau < l; ++tau) {
      cd t = cmul(z[tau], dk[a * l + tau]);
      z[tau].re = t.re * inv_l;
      z[tau].im = t.im * inv_l;
    }
    apply_plan_c(&inner, z, 1, bk, w1, w2, w3);
    memcpy(buf + a * l, bk, sizeof(cd) * l);
  }
  /* pass 3: mixer_inv.transpose(): inv = conj, transposed, scale 1/m; its
   * transpose swaps back: entry(j,k,tau) = conj(roots[(k*(j*l+tau)) % n]) / m
   * applied as y[j l + tau] = sum_k entry(j,k,tau) buf[k l + tau]. */
  const double inv_m = 1.0 / (double)m;
  for (size_t tau = 0; tau < l; ++tau)
    for (size_t j = 0; j < m; ++j) {
      cd acc = {0.0, 0.0};
      for (size_t kk = 0; kk < m; ++kk) {
        cd e = cconj(roots[(kk * (j * l + tau)) % n]);
        e.re *= inv_m;
        e.im *= inv_m;
        acc = cadd(acc, cmul(e, buf[kk * l + tau]));
      }
      y[j * l + tau] = acc;
    }
  free(ws);
  free(buf);
  free(roots);
  free(dk);
  plan_free(&inner);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* conv_real_packed (three_pass.cpp:294-371).                                */
/* ------------------------------------------------------------------------ */
static void real_packed_circular(const double* u, const double* k, size_t n, double* y) {
  const size_t half = n / 2;
  plan_t p;
  plan_build(half, 16, &p);
  cd* w = (cd*)malloc(sizeof(cd) * 9 * (half + 1));
  cd *zu = w, *zk = w + half, *su = w + 2 * half, *sk = w + 3 * half, *w1 = w + 4 * half,
     *w2 = w + 5 * half, *spec_u = w + 6 * half, *spec_k = spec_u + half + 1,
     *prod = spec_k + half + 1;
  for (size_t t = 0; t < half; ++t) {
    zu[t].re = u[2 * t];
    zu[t].im = u[2 * t + 1];
    zk[t].re = k[2 * t];
    zk[t].im = k[2 * t + 1];
  }
  apply_plan_c(&p, zu, 0, su, w1, w2, NULL);
  apply_plan_c(&p, zk, 0, sk, w1, w2, NULL);
  for (int which = 0; which < 2; ++which) {
    const cd* z = which ? sk : su;
    cd* spec = which ? spec_k : spec_u;
    for (size_t j = 0; j < half; ++j) {
      const cd zc = cconj(z[(half - j) % half]);
      const cd even = {0.5 * (z[j].re + zc.re), 0.5 * (z[j].im + zc.im)};
      const cd dz = {z[j].re - zc.re, z[j].im - zc.im};
      const cd odd = cmul((cd){0.0, -0.5}, dz);
      const cd wj = cpolar(-2.0 * kPi * (double)j / (double)n);
      spec[j] = cadd(even, cmul(wj, odd));
      if (j == 0) spec[half] = (cd){even.re - odd.re, even.im - odd.im};
    }
  }
  for (size_t j = 0; j <= half; ++j) prod[j] = cmul(spec_u[j], spec_k[j]);
  for (size_t j = 0; j < half; ++j) {
    const cd yc = cconj(prod[half - j]);
    const cd even = {0.5 * (prod[j].re + yc.re), 0.5 * (prod[j].im + yc.im)};
    const cd wc = cpolar(2.0 * kPi * (double)j / (double)n);
    const cd odd = cmul((cd){0.5 * (prod[j].re - yc.re), 0.5 * (prod[j].im - yc.im)}, wc);
    zu[j] = cadd(even, cmul((cd){0.0, 1.0}, odd));
  }
  apply_plan_c(&p, zu, 1, su, w1, w2, zk);
  for (size_t t = 0; t < half; ++t) {
    y[2 * t] = su[t].re;
    y[2 * t + 1] = su[t].im;
  }
  free(w);
  plan_free(&p);
}

int lco_conv_real_packed(const double* u, const double* k, size_t N, int mode, double* y) {
  if (N == 0 || N % 2) return 1;
  if (!mode) {
    real_packed_circular(u, k, N, y);
    return 0;
  }
  double* pu = (double*)calloc(2 * N, sizeof(double));
  double* pk = (double*)calloc(2 * N, sizeof(double));
  double* full = (double*)malloc(sizeof(double) * 2 * N);
  memcpy(pu, u, sizeof(double) * N);
  memcpy(pk, k, sizeof(double) * N);
  real_packed_circular(pu, pk, 2 * N, full);
  memcpy(y, full, sizeof(double) * N);
  free(pu);
  free(pk);
  free(full);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Learned butterfly (butterfly.cpp:221-307).                                */
/* ------------------------------------------------------------------------ */
int lco_learned_param_count(size_t n, size_t r, size_t* count) {
  plan_t p;
  int rc = plan_build(n, r, &p);
  if (rc) return rc;
  size_t c = 0;
  for (size_t i = 0; i < p.nstages; ++i) c += p.st[i].factor * p.st[i].factor;
  *count = c;
  plan_free(&p);
  return 0;
}

int lco_learned_init(size_t n, size_t r, double* blocks) { /* from_plan :221-227 */
  plan_t p;
  int rc = plan_build(n, r, &p);
  if (rc) return rc;
  cd* b = (cd*)blocks;
  for (size_t i = 0; i < p.nstages; ++i) {
    const size_t ff = p.st[i].factor * p.st[i].factor;
    memcpy(b, p.st[i].block, sizeof(cd) * ff);
    b += ff;
  }
  plan_free(&p);
  return 0;
}

static void split_blocks(const plan_t* p, const cd* blocks, cd** out) {
  for (size_t i = 0; i < p->nstages; ++i) {
    out[i] = (cd*)blocks;
    blocks += p->st[i].factor * p->st[i].factor;
  }
}

int lco_learned_forward(size_t n, size_t r, const double* blocks, const double* x,
                        double* y) { /* :235-246 */
  plan_t p;
  int rc = plan_build(n, r, &p);
  if (rc) return rc;
  cd* bl[64] = {0};
  split_blocks(&p, (const cd*)blocks, bl);
  cd* w = (cd*)malloc(sizeof(cd) * 2 * n);
  apply_stages(&p, bl, (const cd*)x, (cd*)y, w, w + n, NULL);
  free(w);
  plan_free(&p);
  return 0;
}

int lco_learned_gradients(size_t n, size_t r, const double* blocks, const double* x,
                          const double* up, double* dblocks, double* dx) { /* :248-307 */
  plan_t p;
  int rc = plan_build(n, r, &p);
  if (rc) return rc;
  cd* bl[64] = {0};
  split_blocks(&p, (const cd*)blocks, bl);
  cd* saved[64];
  for (size_t i = 0; i < p.nstages; ++i) saved[i] = (cd*)malloc(sizeof(cd) * n);
  cd* w = (cd*)malloc(sizeof(cd) * 4 * n);
  cd *yo = w, *g = w + n, *tmp = w + 2 * n;
  apply_stages(&p, bl, (const cd*)x, yo, w + n, w + 2 * n, saved);
  cd* G = (cd*)dblocks;
  {
    size_t c = 0;
    for (size_t i = 0; i < p.nstages; ++i) c += p.st[i].factor * p.st[i].factor;
    memset(G, 0, sizeof(cd) * c);
  }
  cd* Gs[64];
  split_blocks(&p, G, Gs);
  const cd* ups = (const cd*)up;
  for (size_t i = 0; i < n; ++i) g[p.output_map[i]] = ups[i]; /* :268-269 */
  for (size_t si = p.nstages; si-- > 0;) {
    const stage_t* st = &p.st[si];
    const size_t L = st->segment, f = st->factor, rest = st->rest;
    const cd* v = saved[si];
    /* twiddle adjoint, then scatter adjoint (:279-281) */
    for (size_t off = 0; off < n; off += L)
      for (size_t i = 0; i < L; ++i)
        tmp[off + (i % rest) * f + i / rest] = cmul(g[off + i], cconj(st->twiddle[i]));
    for (size_t base = 0; base < n; base += f) { /* :284-296 */
      for (size_t a = 0; a < f; ++a) {
        const cd wp = tmp[base + a];
        for (size_t q = 0; q < f; ++q)
          Gs[si][a * f + q] = cadd(Gs[si][a * f + q], cmul(wp, cconj(v[base + q])));
      }
      for (size_t q = 0; q < f; ++q) {
        cd acc = {0.0, 0.0};
        for (size_t a = 0; a < f; ++a)
          acc = cadd(acc, cmul(cconj(bl[si][a * f + q]), tmp[base + a]));
        g[base + q] = acc;
      }
    }
    /* gather adjoint (:300-302) */
    for (size_t off = 0; off < n; off += L)
      for (size_t i = 0; i < L; ++i) tmp[off + (i % f) * rest + i / f] = g[off + i];
    memcpy(g, tmp, sizeof(cd) * n);
  }
  memcpy(dx, g, sizeof(cd) * n);
  for (size_t i = 0; i < p.nstages; ++i) free(saved[i]);
  free(w);
  plan_free(&p);
  return 0;
}

/* Synthetic signal batch of SURVEY.md §8d: channel (b,h) holds
 * standard_normal_draws(SeededRng(seed).child(b*H + h), N) (rng.cpp:35-77). */
int lco_signal_batch(uint64_t seed, size_t B, size_t H, size_t N, double* out) {
  if (N == 0) return 1;
  rng_t base = rng_make(seed);
#pragma omp parallel for schedule(static)
  for (size_t c = 0; c < B * H; ++c) {
    rng_t r = rng_child(&base, c);
    for (size_t i = 0; i < N; ++i) out[c * N + i] = rng_normal(&r);
  }
  return 0;
}
