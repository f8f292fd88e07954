/* CPU oracle: periodic neighbour lists + tabulated EAM (TEST INFRASTRUCTURE).
 *
 * No reference implementation exists for this component (the reference
 * package has no EAM): this is an independent plain-C
 * restatement of the Finnis-Sinclair EAM energy/gradient/virial on the same
 * cubic-Hermite tables the GPU uses, evaluated with a brute-force
 * minimum-image pair search.  Compiled with -ffp-contract=off so the cutoff
 * test (dx*dx + dy*dy + dz*dz < rc*rc after rint minimum image) rounds
 * exactly like the device builder: pair sets are compared bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static double min_image(double dx, double L) {
  /* rint(dx * (1/L)): the device evaluates the same expression (neigh.cuh) */
  double inv = 1.0 / L;
  double k = rint(dx * inv);
  return dx - L * k;
}

/* full neighbour list of system q (n atoms), ascending j; returns max count */
int orc_neighbours(int n, const double* box, double rcut, const double* q, int maxn,
                   int32_t* nbr, int32_t* cnt) {
  double rc2 = rcut * rcut;
  int worst = 0;
  for (int i = 0; i < n; ++i) {
    int c = 0;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      double dx = min_image(q[3 * j] - q[3 * i], box[0]);
      double dy = min_image(q[3 * j + 1] - q[3 * i + 1], box[1]);
      double dz = min_image(q[3 * j + 2] - q[3 * i + 2], box[2]);
      double r2 = dx * dx + dy * dy;
      r2 = r2 + dz * dz;
      if (r2 < rc2) {
        if (c < maxn) nbr[(int64_t)i * maxn + c] = j;
        ++c;
      }
    }
    cnt[i] = c < maxn ? c : maxn;
    if (c > worst) worst = c;
  }
  return worst;
}

static void tab(const double* c, int n, double dx, double x, double* f, double* df) {
  double p = x / dx;
  int k = (int)p;
  if (k < 0) k = 0;
  if (k > n - 1) k = n - 1;
  double t = p - (double)k;
  const double* a = c + 4 * (int64_t)k;
  *f = a[0] + t * (a[1] + t * (a[2] + t * a[3]));
  *df = (a[1] + t * (2.0 * a[2] + t * (3.0 * a[3]))) / dx;
}

/* energy, gradient (3n), virial (6) of one system */
int orc_eam(int n, const double* box, double rcut, int n_r, double dr, const double* rho_c,
            const double* phi_c, int n_rho, double drho, const double* F_c, const double* q,
            double* energy, double* grad, double* virial) {
  const int maxn = 256;
  int32_t* nbr = (int32_t*)malloc(sizeof(int32_t) * (size_t)n * maxn);
  int32_t* cnt = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  double* Fp = (double*)malloc(sizeof(double) * (size_t)n);
  double* Fe = (double*)malloc(sizeof(double) * (size_t)n);
  if (orc_neighbours(n, box, rcut, q, maxn, nbr, cnt) > maxn) return -1;
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int k = 0; k < cnt[i]; ++k) {
      int j = nbr[(int64_t)i * maxn + k];
      double dx = min_image(q[3 * j] - q[3 * i], box[0]);
      double dy = min_image(q[3 * j + 1] - q[3 * i + 1], box[1]);
      double dz = min_image(q[3 * j + 2] - q[3 * i + 2], box[2]);
      double r = sqrt(dx * dx + dy * dy + dz * dz);
      double f, df;
      tab(rho_c, n_r, dr, r, &f, &df);
      s += f;
    }
    tab(F_c, n_rho, drho, s, &Fe[i], &Fp[i]);
  }
  double E = 0.0;
  double V[6] = {0, 0, 0, 0, 0, 0};
  for (int i = 0; i < n; ++i) {
    double gx = 0, gy = 0, gz = 0, e = 0;
    for (int k = 0; k < cnt[i]; ++k) {
      int j = nbr[(int64_t)i * maxn + k];
      double dx = min_image(q[3 * j] - q[3 * i], box[0]);
      double dy = min_image(q[3 * j + 1] - q[3 * i + 1], box[1]);
      double dz = min_image(q[3 * j + 2] - q[3 * i + 2], box[2]);
      double r = sqrt(dx * dx + dy * dy + dz * dz);
      double rf, drf, pf, dpf;
      tab(rho_c, n_r, dr, r, &rf, &drf);
      tab(phi_c, n_r, dr, r, &pf, &dpf);
      double coef = (Fp[i] + Fp[j]) * drf + dpf;
      double s = coef / r;
      gx -= s * dx;
      gy -= s * dy;
      gz -= s * dz;
      e += 0.5 * pf;
      double hs = 0.5 * s;
      V[0] -= hs * dx * dx; V[1] -= hs * dy * dy; V[2] -= hs * dz * dz;
      V[3] -= hs * dx * dy; V[4] -= hs * dx * dz; V[5] -= hs * dy * dz;
    }
    if (grad) {
      grad[3 * i] = gx;
      grad[3 * i + 1] = gy;
      grad[3 * i + 2] = gz;
    }
    E += Fe[i] + e;
  }
  if (energy) *energy = E;
  if (virial) memcpy(virial, V, sizeof(V));
  free(nbr);
  free(cnt);
  free(Fp);
  free(Fe);
  return 0;
}
