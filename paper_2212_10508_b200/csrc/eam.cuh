// Cubic-Hermite table lookups shared by the EAM kernels (eam.cu) and the
// persistent coarse sweep (sweep.cu).
#pragma once

#include "pl_common.cuh"

namespace pl {

struct Table {
  const double* c;  // [n][4]
  int n;
  double dx;
};

__device__ __forceinline__ void tab_eval(const Table& T, double x, double& f, double& df) {
  double p = x / T.dx;
  int k = (int)p;
  k = k < 0 ? 0 : (k > T.n - 1 ? T.n - 1 : k);
  double t = p - (double)k;
  const double4 c = *reinterpret_cast<const double4*>(T.c + 4 * (int64_t)k);
  f = c.x + t * (c.y + t * (c.z + t * c.w));
  df = (c.y + t * (2.0 * c.z + t * (3.0 * c.w))) / T.dx;
}

}  // namespace pl
