// Cubic-Hermite table lookups shared by the EAM kernels (eam.cu) and the
// persistent coarse sweep (sweep.cu).
#pragma once

#include "neigh.cuh"
#include "pl_common.cuh"

namespace pl {

struct Table {
  const double* c;  // [n][4]
  int n;
  double dx;
  double inv_dx;  // 1/dx (host)
};

// every operation explicit (fma / _rn): the batched EAM kernels and the
// persistent sweep evaluate identical instruction sequences, so a coarse
// window is bitwise the same on either path (degenerate pair => jump = 0)
__device__ __forceinline__ void tab_eval(const Table& T, double x, double& f, double& df) {
  const double p = __dmul_rn(x, T.inv_dx);
  int k = (int)p;
  k = k < 0 ? 0 : (k > T.n - 1 ? T.n - 1 : k);
  const double t = __dsub_rn(p, (double)k);
  const double2 c01 = __ldg(reinterpret_cast<const double2*>(T.c + 4 * (int64_t)k));
  const double2 c23 = __ldg(reinterpret_cast<const double2*>(T.c + 4 * (int64_t)k + 2));
  const double4 c = make_double4(c01.x, c01.y, c23.x, c23.y);
  f = fma(t, fma(t, fma(t, c.w, c.z), c.y), c.x);
  df = __dmul_rn(fma(t, fma(t, __dmul_rn(3.0, c.w), __dmul_rn(2.0, c.z)), c.y), T.inv_dx);
}

// threads per atom of the EAM gather (same rule on every path): minimise
// rounds/tpa for `threads` cooperating threads
__host__ __device__ inline int eam_tpa(int n, int threads) {
  int best = 1;
  double bestc = 1e30;
  for (int t = 1; t <= 32; t *= 2) {
    const int groups = threads / t;
    const double c = (double)((n + groups - 1) / groups) / t + 0.02 * t;
    if (c < bestc) {
      bestc = c;
      best = t;
    }
  }
  return best;
}

// pair geometry (r_j - r_i, |r|) of list entry k: recomputed (batched path) or
// read from the cache the persistent sweep fills once per step; both give the
// same bits (pair_vec, r2_exact, __dsqrt_rn)
__device__ __forceinline__ void pair_geo(const double* qb, int i, int j, const Box& box, const double4* cache,
                                         int k, double& dx, double& dy, double& dz, double& r2, double& r) {
  if (cache) {
    const double4 c = cache[k];
    dx = c.x;
    dy = c.y;
    dz = c.z;
    r = c.w;
    r2 = 0.0;  // unused: cached entries are already within rc
  } else {
    pair_vec(qb, i, j, box, dx, dy, dz);
    r2 = r2_exact(dx, dy, dz);
    r = __dsqrt_rn(r2);
  }
}

// partial density of atom i over EXACT-list entries sub, sub+tpa, ...
__device__ __forceinline__ double eam_rho_part(const double* qb, int i, const int32_t* list, int nl, int sub,
                                               int tpa, const Box& box, double rc2, const Table& rho,
                                               const double4* cache = nullptr) {
  double s = 0.0;
  // unrolled so several independent table loads are in flight (the 5000-knot
  // tables do not fit in L1); the sum order is unchanged
#pragma unroll 4
  for (int k = sub; k < nl; k += tpa) {
    const int j = list[k];
    double dx, dy, dz, r2, r;
    pair_geo(qb, i, j, box, cache, k, dx, dy, dz, r2, r);
    if (!cache && !(r2 < rc2)) continue;
    double f, df;
    tab_eval(rho, r, f, df);
    s = __dadd_rn(s, f);
  }
  return s;
}

// fixed-order xor-tree over the tpa lanes of a group
__device__ __forceinline__ double group_sum(double v, int tpa) {
  for (int off = tpa >> 1; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

// partial gradient of atom i (and pair energy / virial partials when asked)
template <bool EV>
__device__ __forceinline__ void eam_force_part(const double* qb, const double* fpb, int i, const int32_t* list,
                                               int nl, int sub, int tpa, const Box& box, double rc2,
                                               const Table& rho, const Table& phi, double* g, double* e,
                                               double* v, const double4* cache = nullptr) {
  const double fpi = fpb[i];
#pragma unroll 4
  for (int k = sub; k < nl; k += tpa) {
    const int j = list[k];
    double dx, dy, dz, r2, r;
    pair_geo(qb, i, j, box, cache, k, dx, dy, dz, r2, r);
    if (!cache && !(r2 < rc2)) continue;
    double rf, drf, pf, dpf;
    tab_eval(rho, r, rf, drf);
    tab_eval(phi, r, pf, dpf);
    const double sc = __ddiv_rn(fma(__dadd_rn(fpi, fpb[j]), drf, dpf), r);
    g[0] = fma(-sc, dx, g[0]);
    g[1] = fma(-sc, dy, g[1]);
    g[2] = fma(-sc, dz, g[2]);
    if (EV) {
      *e += 0.5 * pf;
      const double hs = 0.5 * sc;  // pair virial shared by i and j
      v[0] -= hs * dx * dx; v[1] -= hs * dy * dy; v[2] -= hs * dz * dz;
      v[3] -= hs * dx * dy; v[4] -= hs * dx * dz; v[5] -= hs * dy * dz;
    }
  }
}

}  // namespace pl
