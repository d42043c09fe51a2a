/*
 * oracle/rbm_oracle.c -- plain, slow, single-threaded CPU ORACLE for one
 * Random Batch Method time step (Jin, Li & Liu, arXiv:1812.10575).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * path under paper_1812_10575_b200/ (and neither includes the other).
 *
 * Citations:  P:n = line n of the paper's LaTeX source;
 *             D:x = reading x in DESIGN.md section "Readings of the paper".
 *
 * Every function follows the paper's algorithm in its own order:
 *   Alg. 1 (RBM-1): for each step m, divide {1..N} into batches
 *     randomly (here: the (key,id)-sorted order, D:6), then for every batch
 *     evolve Eq. (2.2) for one step tau with forward
 *     Euler-Maruyama.
 *   Alg. 2/3 (RBM-r', RBM-r) in the Jacobi-additive reading D:8.
 *   Splitting with exact pair flow for singular K (P:225-232, P:922-943,
 *     P:1029-1045) with the 1/2 factor of reading D:3.
 * Arithmetic is IEEE double throughout; where the working precision of the
 * product is fp32 the oracle reproduces only the two decisions that depend on
 * it (the fp32 uniform map, D:13, and the bounded-confidence window test, D:10).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* configuration (the oracle's own struct; mirrored field-by-field by  */
/* oracle/oracle.py with ctypes)                                        */
/* ------------------------------------------------------------------ */
typedef struct {
  uint32_t d;          /* spatial dimension, 1..3 */
  uint32_t p;          /* batch size */
  uint64_t n;          /* number of particles N */
  int32_t scheme;      /* 0 RBM-1, 1 RBM-r (Jacobi sweep) */
  int32_t integrator;  /* 0 Euler-Maruyama, 1 split with exact pair flow, 2 Verlet (second order) */
  int32_t kernel;      /* see ok_kernel() */
  int32_t potential;   /* 0 none, 1 harmonic beta|x|^2/2 */
  int32_t constraint;  /* 0 none, 1 unit sphere */
  int32_t fp32;        /* 1: product works in fp32 (uniform map + window test) */
  int32_t init_kind;   /* 1 normal, 2 box, 3 sphere, 4 gaussian mixture */
  uint32_t replica;
  int32_t noise;       /* 0 additive sigma dB; 1 multiplicative sigma X dB (Sec. 5.2.1) */
  int32_t state_form;  /* Verlet: 0 the state is (X_0, V_0), 1 it is (X_n, X_{n-1}) */
  int32_t pad1;
  double kparam[4];
  double vparam[2];
  double iparam[8];
  double sigma, dt;
  uint64_t seed;
  /* clustering model (Sec. 5.3, K_ADJ): symmetric adjacency a_ij in CSR,
   * rows sorted by column; kparam = {alpha, beta, edge_restricted} */
  const uint32_t* adj_rp;  /* n+1 row starts */
  const uint32_t* adj_ci;  /* nnz column indices */
  const double* adj_v;     /* nnz values a_ij >= 0 */
  uint64_t adj_nnz;
} oracle_cfg;

enum { K_ZERO = 0, K_DYSON = 1, K_COULOMB = 2, K_BOUNDED_CONF = 3,
       K_GAUSS_AR = 4, K_COULOMB_REG = 5, K_SMOOTH = 6, K_LINEAR = 7, K_ADJ = 8 };
enum { TAG_KEY = 0, TAG_NOISE = 1, TAG_INIT = 2, TAG_INIT_AUX = 3,
       TAG_SLOT = 4, TAG_NOISE_SLOT = 5 };

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al. 2011), written from the published round */
/* description: two 32x32->64 multiplies per round, Weyl key schedule.  */
/* Reading D:13 (the paper uses MATLAB randn / randperm).        */
/* ------------------------------------------------------------------ */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                          uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void philox_block(const oracle_cfg* c, uint32_t c0, uint32_t c1,
                         uint64_t m, uint32_t tag, uint32_t w[4]) {
  uint32_t ctr[4] = {c0, c1, (uint32_t)m, tag | (c->replica << 8)};
  uint32_t key[2] = {(uint32_t)c->seed, (uint32_t)(c->seed >> 32)};
  oracle_philox4x32_10(ctr, key, w);
}

/* uniform maps onto the open interval (0,1), D:13 */
float oracle_u01_f32(uint32_t w) {
  return (float)((w >> 9) * 2u + 1u) * 0x1p-24f;
}
double oracle_u01_f64(uint32_t a, uint32_t b) {
  uint64_t k = ((((uint64_t)a) << 32) | (uint64_t)b) >> 12;
  return (double)(2u * k + 1u) * 0x1p-53;
}

/* Box-Muller pair (D:13): r = sqrt(-2 ln u1), (r cos 2 pi u2, r sin 2 pi u2) */
static void box_muller(double u1, double u2, double* z0, double* z1) {
  double r = sqrt(-2.0 * log(u1));
  *z0 = r * cos(2.0 * M_PI * u2);
  *z1 = r * sin(2.0 * M_PI * u2);
}

/* d standard normals for counter (c0, m, tag).
 * fp32 product: one block, pairs (w0,w1) and (w2,w3), fp32 uniforms.
 * fp64 product: block b gives one pair from (w0,w1),(w2,w3) fp64 uniforms;
 *   d=3 takes z0,z1 of block 0 and z0 of block 1.                      */
static void normals(const oracle_cfg* c, int fp32, uint32_t c0, uint64_t m,
                    uint32_t tag, double* z) {
  uint32_t w[4];
  if (fp32) {
    philox_block(c, c0, 0, m, tag, w);
    double a, b, e, f;
    box_muller((double)oracle_u01_f32(w[0]), (double)oracle_u01_f32(w[1]), &a, &b);
    box_muller((double)oracle_u01_f32(w[2]), (double)oracle_u01_f32(w[3]), &e, &f);
    double zz[4] = {a, b, e, f};
    for (uint32_t k = 0; k < c->d; ++k) z[k] = zz[k];
  } else {
    double zz[4];
    for (uint32_t blk = 0; blk < 2; ++blk) {
      philox_block(c, c0, blk, m, tag, w);
      box_muller(oracle_u01_f64(w[0], w[1]), oracle_u01_f64(w[2], w[3]),
                 &zz[2 * blk], &zz[2 * blk + 1]);
    }
    /* d=1: z0; d=2: z0,z1; d=3: z0,z1 (blk 0) and z0 of blk 1 */
    double sel[3] = {zz[0], zz[1], zz[2]};
    for (uint32_t k = 0; k < c->d; ++k) z[k] = sel[k];
  }
}

/* exported for tests: Brownian increment normals z^i of particle id at step m
 * (P:31 sigma dB^i; P:943 z ~ N(0,1)) */
void oracle_noise(const oracle_cfg* c, uint32_t id, uint64_t m, double* z) {
  normals(c, c->fp32, id, m, TAG_NOISE, z);
}

/* ------------------------------------------------------------------ */
/* model registry: K and grad V                           */
/* ------------------------------------------------------------------ */
/* interaction kernel K(z), z = X^i - X^j  (Eq. 1.2; reading D:1) */
static void ok_kernel(const oracle_cfg* c, const double* z, double* out) {
  uint32_t d = c->d;
  double r2 = 0.0;
  for (uint32_t k = 0; k < d; ++k) r2 += z[k] * z[k];
  double s = 0.0; /* K(z) = s * z for every registry entry */
  switch (c->kernel) {
    case K_ZERO: s = 0.0; break;
    case K_DYSON: /* 1/x, d=1 (Eq. 4.4); K(0):=0 (D:12) */
      s = (r2 == 0.0) ? 0.0 : 1.0 / r2; break;
    case K_COULOMB: /* x/|x|^3; K(0):=0 (D:12) */
      s = (r2 == 0.0) ? 0.0 : 1.0 / (r2 * sqrt(r2)); break;
    case K_BOUNDED_CONF: { /* -alpha x 1{|x|<r} (Eq. 5.12; D:10);
                            kparam[2] != 0: the paper's closed window phi = chi_[0,1] */
      double alpha = c->kparam[0], rad = c->kparam[1];
      int closed = c->kparam[2] != 0.0;
      int inside;
      if (c->fp32 && d == 1) {
        float zf = (float)z[0];  /* z already holds fl32(x_i - x_j), D:10 */
        inside = closed ? fabsf(zf) <= (float)rad : fabsf(zf) < (float)rad;
      } else {
        inside = closed ? sqrt(r2) <= rad : sqrt(r2) < rad;
      }
      s = inside ? -alpha : 0.0;
      break;
    }
    case K_GAUSS_AR: /* z e^{-|z|^2/2} - z e^{-|z|^2/8}/4 (BASELINE.json C4) */
      s = exp(-0.5 * r2) - 0.25 * exp(-0.125 * r2); break;
    case K_COULOMB_REG: { /* z/(|z|^2+eps)^{3/2} (BASELINE.json C5) */
      double q = r2 + c->kparam[0];
      s = 1.0 / (q * sqrt(q));
      break;
    }
    case K_SMOOTH: /* z/(1+|z|^2) */
      s = 1.0 / (1.0 + r2); break;
    case K_LINEAR: /* -kappa z: quadratic trading potential phi = y^2/2 */
      s = -c->kparam[0]; break;
    default: s = NAN;
  }
  for (uint32_t k = 0; k < d; ++k) out[k] = s * z[k];
}

void oracle_kernel_eval(const oracle_cfg* c, const double* z, double* out) {
  ok_kernel(c, z, out);
}

/* grad V(x); harmonic V = beta |x|^2/2 */
static void grad_v(const oracle_cfg* c, const double* x, double* g) {
  for (uint32_t k = 0; k < c->d; ++k)
    g[k] = (c->potential == 1) ? c->vparam[0] * x[k] : 0.0;
}

/* difference z = x_i - x_j in IEEE double.  The one decision that follows
 * the product's working precision is the bounded-confidence window test
 * (reading D:10): in fp32 mode that kernel's z is fl32(x_i - x_j), so the
 * strict |z| < r test sees the same value as an fp32 product.  Every other
 * kernel takes the exact difference. */
static void diff(const oracle_cfg* c, const double* xi, const double* xj, double* z) {
  for (uint32_t k = 0; k < c->d; ++k) {
    if (c->fp32 && c->kernel == K_BOUNDED_CONF) z[k] = (double)((float)xi[k] - (float)xj[k]);
    else z[k] = xi[k] - xj[k];
  }
}

/* ------------------------------------------------------------------ */
/* initial data X_0^i ~ nu iid, reading D:13/D:14             */
/* ------------------------------------------------------------------ */
int oracle_init(const oracle_cfg* c, double* x) {
  uint32_t d = c->d;
  uint64_t n = c->n;
  double cent[64][3];
  int K = 0;
  if (c->init_kind == 4) {
    K = (int)c->iparam[0];
    if (K < 1 || K > 64) return 1;
    double lo = c->iparam[2], hi = c->iparam[3];
    for (int k = 0; k < K; ++k) {
      uint32_t w[4];
      philox_block(c, (uint32_t)k, 0, 0, TAG_INIT_AUX, w);
      cent[k][0] = lo + (hi - lo) * oracle_u01_f64(w[0], w[1]);
      cent[k][1] = lo + (hi - lo) * oracle_u01_f64(w[2], w[3]);
      philox_block(c, (uint32_t)k, 2, 0, TAG_INIT_AUX, w);
      cent[k][2] = lo + (hi - lo) * oracle_u01_f64(w[0], w[1]);
    }
  }
  for (uint64_t i = 0; i < n; ++i) {
    double* xi = x + i * d;
    double z[3];
    switch (c->init_kind) {
      case 1: /* normal(mean, std) */
        normals(c, 0, (uint32_t)i, 0, TAG_INIT, z);
        for (uint32_t k = 0; k < d; ++k) xi[k] = c->iparam[0] + c->iparam[1] * z[k];
        break;
      case 2: { /* uniform box [a,b]^d */
        double u[4];
        uint32_t w[4];
        for (uint32_t blk = 0; blk < 2; ++blk) {
          philox_block(c, (uint32_t)i, blk, 0, TAG_INIT, w);
          u[2 * blk] = oracle_u01_f64(w[0], w[1]);
          u[2 * blk + 1] = oracle_u01_f64(w[2], w[3]);
        }
        for (uint32_t k = 0; k < d; ++k)
          xi[k] = c->iparam[0] + (c->iparam[1] - c->iparam[0]) * u[k];
        break;
      }
      case 3: { /* uniform on S^{d-1}: normalised Gaussian vector */
        normals(c, 0, (uint32_t)i, 0, TAG_INIT, z);
        double r2 = 0.0;
        for (uint32_t k = 0; k < d; ++k) r2 += z[k] * z[k];
        double r = sqrt(r2);
        for (uint32_t k = 0; k < d; ++k) xi[k] = z[k] / r;
        break;
      }
      case 5: /* |normal(mean, std)|: the wealth model's X = |Y|, Y ~ N(0,1) */
        normals(c, 0, (uint32_t)i, 0, TAG_INIT, z);
        for (uint32_t k = 0; k < d; ++k) xi[k] = fabs(c->iparam[0] + c->iparam[1] * z[k]);
        break;
      case 4: { /* equal-weight Gaussian mixture (D:14) */
        uint32_t w[4];
        philox_block(c, (uint32_t)i, 1, 0, TAG_INIT_AUX, w);
        int k = (int)floor((double)K * oracle_u01_f64(w[0], w[1]));
        if (k >= K) k = K - 1;
        normals(c, 0, (uint32_t)i, 0, TAG_INIT, z);
        for (uint32_t a = 0; a < d; ++a) xi[a] = cent[k][a] + c->iparam[1] * z[a];
        break;
      }
      default: return 1;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* random division (Alg. 1 line 2; P:129 any uniform shuffle):    */
/* order = ids sorted ascending by (key_m(id), id), reading D:6         */
/* ------------------------------------------------------------------ */
typedef struct { uint32_t key, id; } kv_t;
static int kv_cmp(const void* a, const void* b) {
  const kv_t* x = (const kv_t*)a;
  const kv_t* y = (const kv_t*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return 0;
}

uint32_t oracle_key(const oracle_cfg* c, uint32_t id, uint64_t m) {
  uint32_t w[4];
  philox_block(c, id, 0, m, TAG_KEY, w);
  return w[0];
}

/* key_m(id) for every id 0..N-1 (test helper for full-size property checks) */
void oracle_keys(const oracle_cfg* c, uint64_t m, uint32_t* keys) {
  for (uint64_t i = 0; i < c->n; ++i) keys[i] = oracle_key(c, (uint32_t)i, m);
}

int oracle_permutation(const oracle_cfg* c, uint64_t m, uint32_t* order) {
  uint64_t n = c->n;
  kv_t* a = (kv_t*)malloc(sizeof(kv_t) * (n ? n : 1));
  if (!a) return 2;
  for (uint64_t i = 0; i < n; ++i) { a[i].key = oracle_key(c, (uint32_t)i, m); a[i].id = (uint32_t)i; }
  qsort(a, n, sizeof(kv_t), kv_cmp);
  for (uint64_t q = 0; q < n; ++q) order[q] = a[q].id;
  free(a);
  return 0;
}

/* batch b of the division: sorted positions [start, end) (D:7):
 * b < floor(N/p) full batches; remainder r=N mod p >= 2 forms a last batch,
 * r = 1 joins the last full batch (size p+1). Returns number of batches. */
uint64_t oracle_batches(uint64_t n, uint32_t p, uint64_t* starts /* nb+1 or NULL */) {
  uint64_t nfull = n / p, r = n % p;
  uint64_t nb = nfull + (r >= 2 ? 1 : 0);
  if (starts) {
    for (uint64_t b = 0; b < nb; ++b) starts[b] = b * p;
    starts[nb] = n;
  }
  return nb;
}

/* interaction force of Eq. (2.2) for every particle given a division:
 * f_i = 1/(|B|-1) sum_{j in B, j != i} K(X^i - X^j), summed in ascending
 * sorted position.  x in id order, f in id order.            */
int oracle_batch_forces(const oracle_cfg* c, const double* x, const uint32_t* order,
                        const uint64_t* starts, uint64_t nb, double* f) {
  uint32_t d = c->d;
  for (uint64_t b = 0; b < nb; ++b) {
    uint64_t s = starts[b], e = starts[b + 1];
    double inv = 1.0 / (double)(e - s - 1);
    for (uint64_t q = s; q < e; ++q) {
      uint32_t i = order[q];
      double acc[3] = {0, 0, 0};
      for (uint64_t q2 = s; q2 < e; ++q2) {
        if (q2 == q) continue;
        uint32_t j = order[q2];
        double z[3], kz[3];
        diff(c, x + (uint64_t)i * d, x + (uint64_t)j * d, z);
        ok_kernel(c, z, kz);
        for (uint32_t k = 0; k < d; ++k) acc[k] += kz[k];
      }
      for (uint32_t k = 0; k < d; ++k) f[(uint64_t)i * d + k] = acc[k] * inv;
    }
  }
  return 0;
}

/* Euler-Maruyama update of one member:
 * x' = x + dt (-grad V(x) + f) + sigma sqrt(dt) z ; on the sphere the drift
 * and z are projected onto the tangent plane at x and x' is renormalised
 * (reading D:11). */
static void em_member(const oracle_cfg* c, const double* x, const double* f,
                      const double* z, double* xn) {
  uint32_t d = c->d;
  double g[3], drift[3], zz[3];
  grad_v(c, x, g);
  for (uint32_t k = 0; k < d; ++k) { drift[k] = -g[k] + f[k]; zz[k] = z[k]; }
  if (c->constraint == 1) {
    double a = 0.0, b = 0.0;
    for (uint32_t k = 0; k < d; ++k) { a += drift[k] * x[k]; b += zz[k] * x[k]; }
    for (uint32_t k = 0; k < d; ++k) { drift[k] -= a * x[k]; zz[k] -= b * x[k]; }
  }
  double sq = c->sigma * sqrt(c->dt);
  /* multiplicative noise sigma X dB: Ito Euler-Maruyama term sigma x sqrt(dt) z */
  for (uint32_t k = 0; k < d; ++k)
    xn[k] = x[k] + c->dt * drift[k] + sq * (c->noise == 1 ? x[k] * zz[k] : zz[k]);
}

static void renormalise(const oracle_cfg* c, double* x) {
  double r2 = 0.0;
  for (uint32_t k = 0; k < c->d; ++k) r2 += x[k] * x[k];
  double r = sqrt(r2);
  for (uint32_t k = 0; k < c->d; ++k) x[k] /= r;
}

/* exact pair flow of dX^i = K(X^i-X^j)dt, dX^j = K(X^j-X^i)dt over tau
 * (P:225-232), with the 1/2 of reading D:3:
 *   Dyson:   D' = sgn(D) sqrt(D^2 + 4 tau)
 *   Coulomb: D' = D/|D| (|D|^3 + 6 tau)^{1/3}
 *   y_i = mid + D'/2, y_j = mid - D'/2.  sgn(0) := +1, direction e1 at D=0 (D:12) */
void oracle_pair_flow(const oracle_cfg* c, const double* xi, const double* xj,
                      double tau, double* yi, double* yj) {
  uint32_t d = c->d;
  double D[3], mid[3], Dn[3];
  for (uint32_t k = 0; k < d; ++k) { D[k] = xi[k] - xj[k]; mid[k] = 0.5 * (xi[k] + xj[k]); }
  if (c->kernel == K_DYSON) {
    double s = D[0] >= 0.0 ? 1.0 : -1.0;
    Dn[0] = s * sqrt(D[0] * D[0] + 4.0 * tau);
  } else if (c->kernel == K_LINEAR) {
    /* dD/dt = K(D) - K(-D) = -2 kappa D (wealth trading): D' = D e^{-2 kappa tau} */
    double e = exp(-2.0 * c->kparam[0] * tau);
    for (uint32_t k = 0; k < d; ++k) Dn[k] = D[k] * e;
  } else { /* K_COULOMB */
    double r2 = 0.0;
    for (uint32_t k = 0; k < d; ++k) r2 += D[k] * D[k];
    double r = sqrt(r2);
    double rn = cbrt(r2 * r + 6.0 * tau);
    for (uint32_t k = 0; k < d; ++k) Dn[k] = (r == 0.0) ? (k == 0 ? rn : 0.0) : D[k] / r * rn;
  }
  for (uint32_t k = 0; k < d; ++k) { yi[k] = mid[k] + 0.5 * Dn[k]; yj[k] = mid[k] - 0.5 * Dn[k]; }
}

/* ------------------------------------------------------------------ */
/* clustering through the interacting particle system (Sec. 5.3,        */
/* P:1240-1264): dX^i/dt = alpha (a_{i theta} - beta)(X^theta - X^i)     */
/* for the picked pair, solved exactly (the update formula of P:1258-    */
/* 1264): D' = D exp(-2 alpha (a_ij - beta) tau), midpoint kept.         */
/* ------------------------------------------------------------------ */
double oracle_adj_value(const oracle_cfg* c, uint32_t i, uint32_t j) {
  uint32_t lo = c->adj_rp[i], hi = c->adj_rp[i + 1];  /* binary search of row i */
  while (lo < hi) {
    uint32_t mid = lo + (hi - lo) / 2;
    if (c->adj_ci[mid] < j) lo = mid + 1; else hi = mid;
  }
  return (lo < c->adj_rp[i + 1] && c->adj_ci[lo] == j) ? c->adj_v[lo] : 0.0;
}

void oracle_adj_pair_flow(const oracle_cfg* c, uint32_t i, uint32_t j, const double* xi,
                          const double* xj, double tau, double* yi, double* yj) {
  double e = exp(-2.0 * c->kparam[0] * (oracle_adj_value(c, i, j) - c->kparam[1]) * tau);
  for (uint32_t k = 0; k < c->d; ++k) {
    double D = xi[k] - xj[k], sum = xi[k] + xj[k];
    yi[k] = 0.5 * (sum + D * e);
    yj[k] = 0.5 * (sum - D * e);
  }
}

/* the pair flow of the configured kernel for members (i, j) */
static void pair_flow_ids(const oracle_cfg* c, uint32_t i, uint32_t j, const double* xi,
                          const double* xj, double* yi, double* yj) {
  if (c->kernel == K_ADJ) oracle_adj_pair_flow(c, i, j, xi, xj, c->dt, yi, yj);
  else oracle_pair_flow(c, xi, xj, c->dt, yi, yj);
}

/* split step, second half: x' = y - tau grad V(y) + sigma sqrt(tau) z;
 * multiplicative noise ("solved by the splitting strategy" P:1175):
 * the exact geometric Brownian motion step x' = w exp(sigma sqrt(tau) z - sigma^2 tau/2),
 * w = y - tau grad V(y) */
static void split_member(const oracle_cfg* c, const double* y, const double* z, double* xn) {
  double g[3];
  grad_v(c, y, g);
  double sq = c->sigma * sqrt(c->dt);
  for (uint32_t k = 0; k < c->d; ++k) {
    double w = y[k] - c->dt * g[k];
    xn[k] = (c->noise == 1) ? w * exp(sq * z[k] - 0.5 * c->sigma * c->sigma * c->dt) : w + sq * z[k];
  }
  if (c->constraint == 1) renormalise(c, xn);
}

/* Second-order system (Appendix A): X' = V, V' = -grad V(X) +
 * force, with a 1-D particle stored as d = 2 components (x, w).  Verlet in
 * the paper's position form:
 *   first step  (state_form 0, w = V_0):     X_1 = X_0 + V_0 tau + F_0 tau^2 / 2
 *   later steps (state_form 1, w = X_{n-1}): X_{n+1} = 2 X_n - X_{n-1} + F_n tau^2
 * with F the batch force (RBM-1) or the full force (direct); new state (X_{n+1}, X_n). */
static double verlet_pair_force(const oracle_cfg* c, double xi, double xj) {
  oracle_cfg c1 = *c;
  c1.d = 1;
  double z = xi - xj, kz;
  ok_kernel(&c1, &z, &kz);
  return kz;
}

static void verlet_member(const oracle_cfg* c, const double* x, double f, double* xn) {
  double g = (c->potential == 1) ? c->vparam[0] * x[0] : 0.0;  /* grad V on the position */
  double F = -g + f;
  double t = c->dt;
  xn[0] = (c->state_form == 0) ? x[0] + x[1] * t + 0.5 * F * t * t : 2.0 * x[0] - x[1] + F * t * t;
  xn[1] = x[0];
}

/* ------------------------------------------------------------------ */
/* one batch C_q of Alg. 1 line 4: members ids[0..b) in sorted  */
/* order with positions xb (b x d, X_m) -> xo (b x d, X_{m+1}).             */
/* EM: Eq. (2.2) with prefactor 1/(b-1), forward Euler-Maruyama.           */
/* split (b = 2): exact pair flow, then confinement + noise.   */
/* ------------------------------------------------------------------ */
int oracle_batch_update(const oracle_cfg* c, uint64_t m, const uint32_t* ids,
                        const double* xb, uint32_t b, double* xo) {
  uint32_t d = c->d;
  if (b < 2) return 1;
  if (c->integrator == 2) {  /* Verlet: batch force on the positions (component 0) */
    double inv = 1.0 / (double)(b - 1);
    for (uint32_t q = 0; q < b; ++q) {
      double acc = 0.0;
      for (uint32_t q2 = 0; q2 < b; ++q2) {  /* ascending sorted position */
        if (q2 == q) continue;
        acc += verlet_pair_force(c, xb[(uint64_t)q * d], xb[(uint64_t)q2 * d]);
      }
      verlet_member(c, xb + (uint64_t)q * d, acc * inv, xo + (uint64_t)q * d);
    }
    (void)ids; (void)m;
  } else if (c->integrator == 0) {
    double inv = 1.0 / (double)(b - 1);
    for (uint32_t q = 0; q < b; ++q) {
      double acc[3] = {0, 0, 0}, f[3], z[3];
      for (uint32_t q2 = 0; q2 < b; ++q2) {    /* ascending sorted position */
        if (q2 == q) continue;
        double zz[3], kz[3];
        diff(c, xb + (uint64_t)q * d, xb + (uint64_t)q2 * d, zz);
        ok_kernel(c, zz, kz);
        for (uint32_t k = 0; k < d; ++k) acc[k] += kz[k];
      }
      for (uint32_t k = 0; k < d; ++k) f[k] = acc[k] * inv;
      oracle_noise(c, ids[q], m, z);
      em_member(c, xb + (uint64_t)q * d, f, z, xo + (uint64_t)q * d);
      if (c->constraint == 1) renormalise(c, xo + (uint64_t)q * d);
    }
  } else {
    if (b != 2) return 1;
    double y[2][3], z[3];
    oracle_pair_flow(c, xb, xb + d, c->dt, y[0], y[1]);
    for (uint32_t q = 0; q < 2; ++q) {
      oracle_noise(c, ids[q], m, z);
      split_member(c, y[q], z, xo + (uint64_t)q * d);
    }
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* RBM-1 step m: X_m (id order) -> X_{m+1} (id order), Alg. 1 */
/* ------------------------------------------------------------------ */
int oracle_rbm1_step(const oracle_cfg* c, uint64_t m, double* x) {
  uint64_t n = c->n;
  uint32_t d = c->d;
  if (c->p < 2 || c->p > n) return 1;
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint64_t nb = oracle_batches(n, c->p, NULL);
  uint64_t* starts = (uint64_t*)malloc(sizeof(uint64_t) * (nb + 1));
  double* xn = (double*)malloc(sizeof(double) * n * d);
  uint32_t bmax = c->p + 1;
  double* xb = (double*)malloc(sizeof(double) * bmax * d);
  double* xo = (double*)malloc(sizeof(double) * bmax * d);
  if (!order || !starts || !xn || !xb || !xo) return 2;
  oracle_permutation(c, m, order);          /* line 2: random division */
  oracle_batches(n, c->p, starts);
  for (uint64_t b = 0; b < nb; ++b) {       /* lines 3-5: each batch */
    uint64_t s = starts[b];
    uint32_t sz = (uint32_t)(starts[b + 1] - s);
    for (uint32_t q = 0; q < sz; ++q)
      for (uint32_t k = 0; k < d; ++k) xb[q * d + k] = x[(uint64_t)order[s + q] * d + k];
    int rc = oracle_batch_update(c, m, order + s, xb, sz, xo);
    if (rc) return rc;
    for (uint32_t q = 0; q < sz; ++q)
      for (uint32_t k = 0; k < d; ++k) xn[(uint64_t)order[s + q] * d + k] = xo[q * d + k];
  }
  memcpy(x, xn, sizeof(double) * n * d);
  free(order); free(starts); free(xn); free(xb); free(xo);
  return 0;
}

/* direct O(N^2) Euler-Maruyama step of Eq. (1.2): the p=N check */
int oracle_direct_step(const oracle_cfg* c, uint64_t m, double* x) {
  uint64_t n = c->n;
  uint32_t d = c->d;
  double* xn = (double*)malloc(sizeof(double) * n * d);
  if (!xn) return 2;
  for (uint64_t i = 0; i < n; ++i) {
    double f[3] = {0, 0, 0}, z[3];
    if (c->integrator == 2) {  /* full-force Verlet (the reference of P:866-868) */
      double acc = 0.0;
      for (uint64_t j = 0; j < n; ++j)
        if (j != i) acc += verlet_pair_force(c, x[i * d], x[j * d]);
      verlet_member(c, x + i * d, acc / (double)(n - 1), xn + i * d);
      continue;
    }
    for (uint64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      double zz[3], kz[3];
      diff(c, x + i * d, x + j * d, zz);
      ok_kernel(c, zz, kz);
      for (uint32_t k = 0; k < d; ++k) f[k] += kz[k];
    }
    for (uint32_t k = 0; k < d; ++k) f[k] /= (double)(n - 1);
    oracle_noise(c, (uint32_t)i, m, z);
    em_member(c, x + i * d, f, z, xn + i * d);
    if (c->constraint == 1) renormalise(c, xn + i * d);
  }
  memcpy(x, xn, sizeof(double) * n * d);
  free(xn);
  return 0;
}

/* ------------------------------------------------------------------ */
/* RBM-r, one sweep of ceil(N/p) with-replacement batches (Alg. 2/3,    */
/* P:148-200) in the Jacobi-additive reading D:8; distinct members D:9. */
/* ------------------------------------------------------------------ */
uint32_t oracle_slot_draw(const oracle_cfg* c, uint64_t s, uint32_t t, uint64_t m) {
  uint32_t w[4];
  philox_block(c, (uint32_t)s, t, m, TAG_SLOT, w);
  uint64_t u = (((uint64_t)w[0]) << 32) | w[1];
  return (uint32_t)(((unsigned __int128)c->n * u) >> 64);
}

/* edge-restricted pick ("the random batch can be picked from those
 * with nonzeros of a_ij only"): edge e = floor(nnz U64 / 2^64) of the CSR,
 * i = its row, j = its column; redrawn (t += 1) on a diagonal entry */
static void edge_draw(const oracle_cfg* c, uint64_t s0, uint64_t m, uint32_t* i, uint32_t* j) {
  for (uint32_t t = 0;; ++t) {
    uint32_t w[4];
    philox_block(c, (uint32_t)s0, t, m, TAG_SLOT, w);
    uint64_t u = (((uint64_t)w[0]) << 32) | w[1];
    uint64_t e = (uint64_t)(((unsigned __int128)c->adj_nnz * u) >> 64);
    uint32_t lo = 0, hi = (uint32_t)c->n;  /* row: largest r with adj_rp[r] <= e */
    while (hi - lo > 1) {
      uint32_t mid = lo + (hi - lo) / 2;
      if (c->adj_rp[mid] <= e) lo = mid; else hi = mid;
    }
    *i = lo;
    *j = c->adj_ci[e];
    if (*i != *j) return;
  }
}

int oracle_rbmr_slots(const oracle_cfg* c, uint64_t m, uint32_t* js) {
  uint64_t n = c->n;
  uint32_t p = c->p;
  uint64_t nb = (n + p - 1) / p;
  if (c->kernel == K_ADJ && c->kparam[2] != 0.0) {
    if (p != 2) return 1;
    for (uint64_t b = 0; b < nb; ++b) edge_draw(c, b * p, m, &js[b * p], &js[b * p + 1]);
    return 0;
  }
  for (uint64_t b = 0; b < nb; ++b) {
    for (uint32_t l = 0; l < p; ++l) {
      uint64_t s = b * p + l;
      uint32_t t = 0, j;
      for (;;) {
        j = oracle_slot_draw(c, s, t, m);
        int dup = 0;
        for (uint32_t l2 = 0; l2 < l; ++l2) if (js[b * p + l2] == j) dup = 1;
        if (!dup) break;
        ++t;
      }
      js[s] = j;
    }
  }
  return 0;
}

int oracle_rbmr_step(const oracle_cfg* c, uint64_t m, double* x) {
  uint64_t n = c->n;
  uint32_t d = c->d, p = c->p;
  if (p < 2 || p > n) return 1;
  uint64_t nb = (n + p - 1) / p, ns = nb * p;
  uint32_t* js = (uint32_t*)malloc(sizeof(uint32_t) * ns);
  double* delta = (double*)malloc(sizeof(double) * ns * d);
  unsigned char* touched = (unsigned char*)calloc(n, 1);
  if (!js || !delta || !touched) return 2;
  oracle_rbmr_slots(c, m, js);
  double inv = 1.0 / (double)(p - 1);
  for (uint64_t b = 0; b < nb; ++b) {         /* every batch evolves from X_m */
    uint64_t s0 = b * p;
    if (c->integrator == 0) {
      for (uint32_t l = 0; l < p; ++l) {
        uint32_t i = js[s0 + l];
        double f[3] = {0, 0, 0}, z[3], xn[3];
        for (uint32_t l2 = 0; l2 < p; ++l2) {
          if (l2 == l) continue;
          double zz[3], kz[3];
          diff(c, x + (uint64_t)i * d, x + (uint64_t)js[s0 + l2] * d, zz);
          ok_kernel(c, zz, kz);
          for (uint32_t k = 0; k < d; ++k) f[k] += kz[k];
        }
        for (uint32_t k = 0; k < d; ++k) f[k] *= inv;
        normals(c, c->fp32, (uint32_t)(s0 + l), m, TAG_NOISE_SLOT, z);
        em_member(c, x + (uint64_t)i * d, f, z, xn);
        for (uint32_t k = 0; k < d; ++k) delta[(s0 + l) * d + k] = xn[k] - x[(uint64_t)i * d + k];
      }
    } else {
      uint32_t i = js[s0], j = js[s0 + 1];
      double yi[3], yj[3], z[3], xn[3];
      pair_flow_ids(c, i, j, x + (uint64_t)i * d, x + (uint64_t)j * d, yi, yj);
      normals(c, c->fp32, (uint32_t)s0, m, TAG_NOISE_SLOT, z);
      oracle_cfg c2 = *c; c2.constraint = 0;
      split_member(&c2, yi, z, xn);
      for (uint32_t k = 0; k < d; ++k) delta[s0 * d + k] = xn[k] - x[(uint64_t)i * d + k];
      normals(c, c->fp32, (uint32_t)(s0 + 1), m, TAG_NOISE_SLOT, z);
      split_member(&c2, yj, z, xn);
      for (uint32_t k = 0; k < d; ++k) delta[(s0 + 1) * d + k] = xn[k] - x[(uint64_t)j * d + k];
    }
  }
  for (uint64_t s = 0; s < ns; ++s) {          /* x_j += sum_{s: j_s=j} Delta_s, ascending s */
    uint32_t j = js[s];
    touched[j] = 1;
    for (uint32_t k = 0; k < d; ++k) x[(uint64_t)j * d + k] += delta[s * d + k];
  }
  if (c->constraint == 1)
    for (uint64_t i = 0; i < n; ++i) if (touched[i]) renormalise(c, x + i * d);
  free(js); free(delta); free(touched);
  return 0;
}

/* ------------------------------------------------------------------ */
/* RBM-r' exactly as Algorithm 2 is written: */
/* within step m, for k = 1 .. ceil(N/p) in order, the batch C_k (the     */
/* slot draws of oracle_rbmr_slots, D:9) is updated from the CURRENT      */
/* positions, "set X^i <- Y^i(tau)", before the next batch is drawn.      */
/* The per-batch solve is the same as RBM-1's (Eq. 2.2 + EM with noise    */
/* from counter (s, blk, m, TAG_NOISE_SLOT), or the split pair flow).     */
/* ------------------------------------------------------------------ */
int oracle_rbmr_seq_step(const oracle_cfg* c, uint64_t m, double* x) {
  uint64_t n = c->n;
  uint32_t d = c->d, p = c->p;
  if (p < 2 || p > n) return 1;
  uint64_t nb = (n + p - 1) / p, ns = nb * p;
  uint32_t* js = (uint32_t*)malloc(sizeof(uint32_t) * ns);
  double* xo = (double*)malloc(sizeof(double) * p * d);
  if (!js || !xo) return 2;
  oracle_rbmr_slots(c, m, js);
  double inv = 1.0 / (double)(p - 1);
  for (uint64_t b = 0; b < nb; ++b) {
    uint64_t s0 = b * p;
    if (c->integrator == 0) {
      for (uint32_t l = 0; l < p; ++l) {
        uint32_t i = js[s0 + l];
        double f[3] = {0, 0, 0}, z[3];
        for (uint32_t l2 = 0; l2 < p; ++l2) {
          if (l2 == l) continue;
          double zz[3], kz[3];
          diff(c, x + (uint64_t)i * d, x + (uint64_t)js[s0 + l2] * d, zz);
          ok_kernel(c, zz, kz);
          for (uint32_t k = 0; k < d; ++k) f[k] += kz[k];
        }
        for (uint32_t k = 0; k < d; ++k) f[k] *= inv;
        normals(c, c->fp32, (uint32_t)(s0 + l), m, TAG_NOISE_SLOT, z);
        em_member(c, x + (uint64_t)i * d, f, z, xo + (uint64_t)l * d);
        if (c->constraint == 1) renormalise(c, xo + (uint64_t)l * d);
      }
    } else {
      uint32_t i = js[s0], j = js[s0 + 1];
      double y[2][3], z[3];
      pair_flow_ids(c, i, j, x + (uint64_t)i * d, x + (uint64_t)j * d, y[0], y[1]);
      for (uint32_t l = 0; l < 2; ++l) {
        normals(c, c->fp32, (uint32_t)(s0 + l), m, TAG_NOISE_SLOT, z);
        split_member(c, y[l], z, xo + (uint64_t)l * d);
      }
    }
    for (uint32_t l = 0; l < p; ++l)  /* X^i <- Y^i(tau) for the batch's members */
      for (uint32_t k = 0; k < d; ++k) x[(uint64_t)js[s0 + l] * d + k] = xo[(uint64_t)l * d + k];
  }
  free(js); free(xo);
  return 0;
}

/* convenience: steps m0 .. m0+nsteps-1 of the configured scheme */
int oracle_run(const oracle_cfg* c, uint64_t m0, uint64_t nsteps, double* x) {
  oracle_cfg c2 = *c;
  for (uint64_t s = 0; s < nsteps; ++s) {
    int rc = (c2.scheme == 0) ? oracle_rbm1_step(&c2, m0 + s, x)
             : (c2.scheme == 1) ? oracle_rbmr_step(&c2, m0 + s, x) : oracle_rbmr_seq_step(&c2, m0 + s, x);
    if (rc) return rc;
    c2.state_form = 1;  /* Verlet: (X_0, V_0) -> (X_n, X_{n-1}) after the first step */
  }
  return 0;
}

/* nsteps direct (full-force) steps, same state-form convention */
int oracle_direct_run(const oracle_cfg* c, uint64_t m0, uint64_t nsteps, double* x) {
  oracle_cfg c2 = *c;
  for (uint64_t s = 0; s < nsteps; ++s) {
    int rc = oracle_direct_step(&c2, m0 + s, x);
    if (rc) return rc;
    c2.state_form = 1;
  }
  return 0;
}
