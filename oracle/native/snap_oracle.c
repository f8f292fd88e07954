/* CPU oracle: single-element SNAP energy / gradient / virial (TEST INFRASTRUCTURE).
 *
 * No reference implementation exists (the reference package has no SNAP and
 * LAMMPS is not in the container): this is an independent
 * plain-C restatement of the published bispectrum formalism (Thompson et al.
 * 2015; adjoint force form of Wood & Thompson 2018), written on FULL
 * (J+1)x(J+1) matrices so it shares no half-row bookkeeping with the GPU:
 *
 *   neighbour k at r (|r| < rcut):  theta0 = rfac0*pi*(r - rmin0)/(rcut - rmin0)
 *     a = cos(theta0) - i (z/r) sin(theta0),   b = sin(theta0) (y - i x)/r
 *   U^0 = 1;  U^J[ma][mb] = sqrt((J-ma)/(J-mb)) a* U^{J-1}[ma][mb]
 *                         - sqrt(ma/(J-mb))    b* U^{J-1}[ma-1][mb]   (mb < J)
 *             U^J[J-ma][J] = (-1)^ma conj(U^J[ma][0])                  (last row)
 *   Utot^J = wself*I + sum_k fc(r_k) U^J(r_k),  fc = (cos(pi (r-rmin0)/(rcut-rmin0)) + 1)/2
 *   Z^{j1 j2}_J[ma][mb] = sum C(j1 ma1, j2 ma2 | J ma) C(j1 mb1, j2 mb2 | J mb)
 *                              Utot^{j1}[ma1][mb1] Utot^{j2}[ma2][mb2]
 *   B_{j1 j2 J} = Re sum_{ma,mb} conj(Utot^J) Z^{j1 j2}_J,  j1 >= j2, J >= j1 (canonical)
 *   E_i = beta_0 + sum_b beta_b B_b(i)
 *   dE_i/dr_ik = Re sum_J sum_{ma,mb} conj(d(fc U^J)/dr) Y^J,
 *   Y^J = sum_b beta_b [ d(J=j) Z^{j1j2}_j + d(J=j1) (j+1)/(j1+1) Z^{j j2}_{j1}
 *                        + d(J=j2) (j+1)/(j2+1) Z^{j1 j}_{j2} ]
 * (indices are 2j integers; C are Condon-Shortley Clebsch-Gordan coefficients
 * from the Racah formula).  Gradient on atom a:
 *   dE/dr_a = sum_{k in N(a)} [ dE_k/dr_{ka} - dE_a/dr_{ak} ].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double re, im;
} cplx;

static double fact(int n) {
  double f = 1.0;
  for (int i = 2; i <= n; ++i) f *= (double)i;
  return f;
}

/* <j1 m1 j2 m2 | J M>, all arguments are twice the physical values */
double orc_cg(int j1, int m1, int j2, int m2, int J, int M) {
  if (m1 + m2 != M) return 0.0;
  if (abs(m1) > j1 || abs(m2) > j2 || abs(M) > J) return 0.0;
  if (J < abs(j1 - j2) || J > j1 + j2 || ((j1 + j2 + J) & 1)) return 0.0;
  if (((j1 + m1) & 1) || ((j2 + m2) & 1) || ((J + M) & 1)) return 0.0;
  double pre = sqrt((J + 1) * fact((j1 + j2 - J) / 2) * fact((j1 - j2 + J) / 2) *
                    fact((-j1 + j2 + J) / 2) / fact((j1 + j2 + J) / 2 + 1));
  pre *= sqrt(fact((J + M) / 2) * fact((J - M) / 2) * fact((j1 - m1) / 2) * fact((j1 + m1) / 2) *
              fact((j2 - m2) / 2) * fact((j2 + m2) / 2));
  double s = 0.0;
  for (int k = 0; k <= 64; ++k) {
    int d1 = (j1 + j2 - J) / 2 - k, d2 = (j1 - m1) / 2 - k, d3 = (j2 + m2) / 2 - k;
    int d4 = (J - j2 + m1) / 2 + k, d5 = (J - j1 - m2) / 2 + k;
    if (d1 < 0 || d2 < 0 || d3 < 0) break;
    if (d4 < 0 || d5 < 0) continue;
    double t = 1.0 / (fact(k) * fact(d1) * fact(d2) * fact(d3) * fact(d4) * fact(d5));
    s += (k & 1) ? -t : t;
  }
  return pre * s;
}

#define JMAX 14
static int moff[JMAX + 2]; /* offset of full layer J in a flat U array */

static void init_offsets(int twojmax) {
  int o = 0;
  for (int J = 0; J <= twojmax; ++J) {
    moff[J] = o;
    o += (J + 1) * (J + 1);
  }
  moff[twojmax + 1] = o;
}
#define UIDX(J, ma, mb) (moff[J] + (mb) * ((J) + 1) + (ma))

static cplx cmul(cplx x, cplx y) {
  cplx r = {x.re * y.re - x.im * y.im, x.re * y.im + x.im * y.re};
  return r;
}
static cplx conj_(cplx x) {
  cplx r = {x.re, -x.im};
  return r;
}

/* U (full layers) and dU/dr_k (3 components) of one neighbour vector */
static void u_and_du(int twojmax, double rfac0, double rmin0, double rcut, const double* rv,
                     cplx* U, cplx* dU /* [3][size] or NULL */, int size) {
  double x = rv[0], y = rv[1], z = rv[2];
  double r = sqrt(x * x + y * y + z * z);
  double kappa = rfac0 * M_PI / (rcut - rmin0);
  double th = kappa * (r - rmin0);
  double s = sin(th), c = cos(th);
  double u[3] = {x / r, y / r, z / r};
  cplx a = {c, -u[2] * s}, b = {u[1] * s, -u[0] * s};
  cplx da[3], db[3];
  for (int k = 0; k < 3; ++k) {
    double dxk = (k == 0) - u[0] * u[k], dyk = (k == 1) - u[1] * u[k], dzk = (k == 2) - u[2] * u[k];
    da[k].re = -s * kappa * u[k];
    da[k].im = -(c * kappa * u[k] * u[2] + s * dzk / r);
    db[k].re = c * kappa * u[k] * u[1] + s * dyk / r;
    db[k].im = -(c * kappa * u[k] * u[0] + s * dxk / r);
  }
  cplx ac = conj_(a), bc = conj_(b);
  U[0].re = 1.0;
  U[0].im = 0.0;
  if (dU)
    for (int k = 0; k < 3; ++k) dU[k * size].re = dU[k * size].im = 0.0;
  for (int J = 1; J <= twojmax; ++J) {
    for (int mb = 0; mb < J; ++mb) {
      for (int ma = 0; ma <= J; ++ma) {
        cplx v = {0, 0};
        cplx dv[3] = {{0, 0}, {0, 0}, {0, 0}};
        if (ma < J) {
          double A = sqrt((double)(J - ma) / (double)(J - mb));
          cplx p = U[UIDX(J - 1, ma, mb)];
          cplx t = cmul(ac, p);
          v.re += A * t.re;
          v.im += A * t.im;
          if (dU)
            for (int k = 0; k < 3; ++k) {
              cplx t1 = cmul(conj_(da[k]), p), t2 = cmul(ac, dU[k * size + UIDX(J - 1, ma, mb)]);
              dv[k].re += A * (t1.re + t2.re);
              dv[k].im += A * (t1.im + t2.im);
            }
        }
        if (ma > 0) {
          double Bc = sqrt((double)ma / (double)(J - mb));
          cplx p = U[UIDX(J - 1, ma - 1, mb)];
          cplx t = cmul(bc, p);
          v.re -= Bc * t.re;
          v.im -= Bc * t.im;
          if (dU)
            for (int k = 0; k < 3; ++k) {
              cplx t1 = cmul(conj_(db[k]), p), t2 = cmul(bc, dU[k * size + UIDX(J - 1, ma - 1, mb)]);
              dv[k].re -= Bc * (t1.re + t2.re);
              dv[k].im -= Bc * (t1.im + t2.im);
            }
        }
        U[UIDX(J, ma, mb)] = v;
        if (dU)
          for (int k = 0; k < 3; ++k) dU[k * size + UIDX(J, ma, mb)] = dv[k];
      }
    }
    /* last row mb = J from row 0 by the inversion symmetry */
    for (int ma = 0; ma <= J; ++ma) {
      double sg = (ma & 1) ? -1.0 : 1.0;
      cplx p = U[UIDX(J, ma, 0)];
      U[UIDX(J, J - ma, J)].re = sg * p.re;
      U[UIDX(J, J - ma, J)].im = -sg * p.im;
      if (dU)
        for (int k = 0; k < 3; ++k) {
          cplx dp = dU[k * size + UIDX(J, ma, 0)];
          dU[k * size + UIDX(J, J - ma, J)].re = sg * dp.re;
          dU[k * size + UIDX(J, J - ma, J)].im = -sg * dp.im;
        }
    }
  }
}

/* memoised CG table: cgt[j1][j2][J][ma1][ma2] (M = m1 + m2) */
#define CGN (JMAX + 1)
static double* cgt = NULL;
static int cgt_jmax = -1;
static size_t cgi(int j1, int j2, int J, int a1, int a2) {
  return ((((size_t)j1 * CGN + j2) * CGN + J) * CGN + a1) * CGN + a2;
}
static void cg_table(int twojmax) {
  if (cgt && cgt_jmax >= twojmax) return;
  free(cgt);
  cgt = (double*)calloc((size_t)CGN * CGN * CGN * CGN * CGN, sizeof(double));
  for (int j1 = 0; j1 <= twojmax; ++j1)
    for (int j2 = 0; j2 <= twojmax; ++j2)
      for (int J = 0; J <= twojmax; ++J)
        for (int a1 = 0; a1 <= j1; ++a1)
          for (int a2 = 0; a2 <= j2; ++a2) {
            int m1 = 2 * a1 - j1, m2 = 2 * a2 - j2;
            cgt[cgi(j1, j2, J, a1, a2)] = orc_cg(j1, m1, j2, m2, J, m1 + m2);
          }
  cgt_jmax = twojmax;
}

/* Z^{j1 j2}_J (full (J+1)^2 matrix) from Utot */
static void zmat(int j1, int j2, int J, const cplx* Ut, cplx* Z) {
  for (int mb = 0; mb <= J; ++mb)
    for (int ma = 0; ma <= J; ++ma) {
      cplx acc = {0, 0};
      int M = 2 * ma - J, Mp = 2 * mb - J;
      for (int ma1 = 0; ma1 <= j1; ++ma1) {
        int m1 = 2 * ma1 - j1, m2 = M - m1;
        if (abs(m2) > j2) continue;
        int ma2 = (m2 + j2) / 2;
        double ca = cgt[cgi(j1, j2, J, ma1, ma2)];
        if (ca == 0.0) continue;
        for (int mb1 = 0; mb1 <= j1; ++mb1) {
          int mp1 = 2 * mb1 - j1, mp2 = Mp - mp1;
          if (abs(mp2) > j2) continue;
          int mb2 = (mp2 + j2) / 2;
          double cb = cgt[cgi(j1, j2, J, mb1, mb2)];
          cplx t = cmul(Ut[UIDX(j1, ma1, mb1)], Ut[UIDX(j2, ma2, mb2)]);
          acc.re += ca * cb * t.re;
          acc.im += ca * cb * t.im;
        }
      }
      Z[mb * (J + 1) + ma] = acc;
    }
}

static double min_image(double dx, double L) {
  /* rint(dx * (1/L)): the device evaluates the same expression (neigh.cuh) */
  double inv = 1.0 / L;
  double k = rint(dx * inv);
  return dx - L * k;
}

int orc_neighbours(int n, const double* box, double rcut, const double* q, int maxn, int32_t* nbr,
                   int32_t* cnt);

/* Per-atom bispectrum (n x nb) and per-pair dE_i/dr_ik for one system.
 * Returns number of B components.  energy/grad/virial may be NULL. */
int orc_snap(int n, const double* box, int twojmax, double rcut, double rfac0, double rmin0,
             int switchflag, double wself, const double* beta, int nbeta, const double* q,
             double* energy, double* grad, double* virial, double* bispectrum) {
  if (twojmax > JMAX) return -1;
  init_offsets(twojmax);
  cg_table(twojmax);
  int size = moff[twojmax + 1];
  const int maxn = 128;
  int32_t* nbr = (int32_t*)malloc(sizeof(int32_t) * (size_t)n * maxn);
  int32_t* cnt = (int32_t*)malloc(sizeof(int32_t) * n);
  if (orc_neighbours(n, box, rcut, q, maxn, nbr, cnt) > maxn) return -2;
  /* canonical triples */
  int nb = 0;
  int tj1[512], tj2[512], tJ[512];
  for (int j1 = 0; j1 <= twojmax; ++j1)
    for (int j2 = 0; j2 <= j1; ++j2)
      for (int J = j1 - j2; J <= (twojmax < j1 + j2 ? twojmax : j1 + j2); J += 2)
        if (J >= j1) {
          tj1[nb] = j1;
          tj2[nb] = j2;
          tJ[nb] = J;
          ++nb;
        }
  if (nbeta != nb + 1) return -3;
  cplx* Ut = (cplx*)malloc(sizeof(cplx) * size);
  cplx* Y = (cplx*)malloc(sizeof(cplx) * size);
  cplx* U = (cplx*)malloc(sizeof(cplx) * size);
  cplx* dU = (cplx*)malloc(sizeof(cplx) * 3 * size);
  cplx* Z = (cplx*)malloc(sizeof(cplx) * (twojmax + 1) * (twojmax + 1));
  double* dEdr = (double*)malloc(sizeof(double) * 3 * (size_t)n * maxn);
  double E = 0.0;
  double V[6] = {0, 0, 0, 0, 0, 0};
  for (int i = 0; i < n; ++i) {
    memset(Ut, 0, sizeof(cplx) * size);
    for (int J = 0; J <= twojmax; ++J)
      for (int ma = 0; ma <= J; ++ma) Ut[UIDX(J, ma, ma)].re = wself;
    for (int s = 0; s < cnt[i]; ++s) {
      int j = nbr[(int64_t)i * maxn + s];
      double rv[3] = {min_image(q[3 * j] - q[3 * i], box[0]), min_image(q[3 * j + 1] - q[3 * i + 1], box[1]),
                      min_image(q[3 * j + 2] - q[3 * i + 2], box[2])};
      double r = sqrt(rv[0] * rv[0] + rv[1] * rv[1] + rv[2] * rv[2]);
      double fc = switchflag ? 0.5 * (cos(M_PI * (r - rmin0) / (rcut - rmin0)) + 1.0) : 1.0;
      u_and_du(twojmax, rfac0, rmin0, rcut, rv, U, NULL, size);
      for (int t = 0; t < size; ++t) {
        Ut[t].re += fc * U[t].re;
        Ut[t].im += fc * U[t].im;
      }
    }
    /* B, energy, Y */
    memset(Y, 0, sizeof(cplx) * size);
    double Ei = beta[0];
    for (int b = 0; b < nb; ++b) {
      int j1 = tj1[b], j2 = tj2[b], J = tJ[b];
      zmat(j1, j2, J, Ut, Z);
      double Bv = 0.0;
      for (int t = 0; t < (J + 1) * (J + 1); ++t) {
        cplx u = Ut[moff[J] + t];
        Bv += u.re * Z[t].re + u.im * Z[t].im;
      }
      if (bispectrum) bispectrum[(int64_t)i * nb + b] = Bv;
      Ei += beta[b + 1] * Bv;
      double bb = beta[b + 1];
      /* slot J = j */
      for (int t = 0; t < (J + 1) * (J + 1); ++t) {
        Y[moff[J] + t].re += bb * Z[t].re;
        Y[moff[J] + t].im += bb * Z[t].im;
      }
      /* slot j1: Z^{J j2}_{j1} * (J+1)/(j1+1) */
      zmat(J, j2, j1, Ut, Z);
      double f1 = (double)(J + 1) / (double)(j1 + 1);
      for (int t = 0; t < (j1 + 1) * (j1 + 1); ++t) {
        Y[moff[j1] + t].re += bb * f1 * Z[t].re;
        Y[moff[j1] + t].im += bb * f1 * Z[t].im;
      }
      /* slot j2: Z^{J j1}_{j2} * (J+1)/(j2+1) */
      zmat(J, j1, j2, Ut, Z);
      double f2 = (double)(J + 1) / (double)(j2 + 1);
      for (int t = 0; t < (j2 + 1) * (j2 + 1); ++t) {
        Y[moff[j2] + t].re += bb * f2 * Z[t].re;
        Y[moff[j2] + t].im += bb * f2 * Z[t].im;
      }
    }
    E += Ei;
    /* per-pair dE_i / dr_ik */
    for (int s = 0; s < cnt[i]; ++s) {
      int j = nbr[(int64_t)i * maxn + s];
      double rv[3] = {min_image(q[3 * j] - q[3 * i], box[0]), min_image(q[3 * j + 1] - q[3 * i + 1], box[1]),
                      min_image(q[3 * j + 2] - q[3 * i + 2], box[2])};
      double r = sqrt(rv[0] * rv[0] + rv[1] * rv[1] + rv[2] * rv[2]);
      double arg = M_PI * (r - rmin0) / (rcut - rmin0);
      double fc = switchflag ? 0.5 * (cos(arg) + 1.0) : 1.0;
      double dfc = switchflag ? -0.5 * M_PI / (rcut - rmin0) * sin(arg) : 0.0;
      u_and_du(twojmax, rfac0, rmin0, rcut, rv, U, dU, size);
      for (int k = 0; k < 3; ++k) {
        double uk = rv[k] / r, acc = 0.0;
        for (int t = 0; t < size; ++t) {
          double gre = fc * dU[k * size + t].re + dfc * uk * U[t].re;
          double gim = fc * dU[k * size + t].im + dfc * uk * U[t].im;
          acc += gre * Y[t].re + gim * Y[t].im;
        }
        dEdr[((int64_t)i * maxn + s) * 3 + k] = acc;
      }
      for (int a = 0; a < 3; ++a) {
        /* virial_ab = -sum dE/dr_a r_b (symmetrised storage xx yy zz xy xz yz) */
        (void)a;
      }
      double* g = &dEdr[((int64_t)i * maxn + s) * 3];
      V[0] -= g[0] * rv[0];
      V[1] -= g[1] * rv[1];
      V[2] -= g[2] * rv[2];
      V[3] -= 0.5 * (g[0] * rv[1] + g[1] * rv[0]);
      V[4] -= 0.5 * (g[0] * rv[2] + g[2] * rv[0]);
      V[5] -= 0.5 * (g[1] * rv[2] + g[2] * rv[1]);
    }
  }
  if (grad) {
    for (int a = 0; a < n; ++a) {
      double gx = 0, gy = 0, gz = 0;
      for (int s = 0; s < cnt[a]; ++s) {
        int k = nbr[(int64_t)a * maxn + s];
        /* slot of a in k's list */
        int sk = -1;
        for (int t = 0; t < cnt[k]; ++t)
          if (nbr[(int64_t)k * maxn + t] == a) sk = t;
        const double* ga = &dEdr[((int64_t)a * maxn + s) * 3];
        const double* gk = &dEdr[((int64_t)k * maxn + sk) * 3];
        gx += gk[0] - ga[0];
        gy += gk[1] - ga[1];
        gz += gk[2] - ga[2];
      }
      grad[3 * a] = gx;
      grad[3 * a + 1] = gy;
      grad[3 * a + 2] = gz;
    }
  }
  if (energy) *energy = E;
  if (virial) memcpy(virial, V, sizeof(V));
  free(nbr); free(cnt); free(Ut); free(Y); free(U); free(dU); free(Z); free(dEdr);
  return nb;
}

/* U^J (full layers J = 0..twojmax, [J][mb][ma] order, interleaved re/im) of one
 * neighbour vector rv, for the external pins of the recursion (tests only). */
int orc_ulist(int twojmax, double rfac0, double rmin0, double rcut, const double* rv, double* out) {
  if (twojmax > JMAX) return -1;
  init_offsets(twojmax);
  int size = moff[twojmax + 1];
  u_and_du(twojmax, rfac0, rmin0, rcut, rv, (cplx*)out, NULL, size);
  return size;
}
