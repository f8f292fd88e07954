// Device forms of the reference's analytic potentials (potentials.py:62-214).
// Arithmetic order follows numpy's left-to-right evaluation with explicit
// round-to-nearest intrinsics (no FMA), so gradients are bitwise equal to the
// reference for Harmonic / DoubleWell / Perturbed.
#pragma once

#include "pl_common.cuh"

namespace pl {

// A potential tree of elementwise terms flattened to postfix form.
enum EwOpCode { EW_FREE = 0, EW_HARM = 1, EW_DW = 2, EW_PERT = 3 };
struct EwOp {
  int code;
  const double* c0;  // per-component coefficient or nullptr (then s0)
  const double* c1;
  double s0, s1, lam;
};
constexpr int EW_MAX = 8;
struct EwProg {
  int n;
  EwOp op[EW_MAX];
};

__device__ __forceinline__ double ew_grad(const EwProg& P, double q, int64_t i) {
  double st[EW_MAX];
  int sp = 0;
#pragma unroll 1
  for (int k = 0; k < P.n; ++k) {
    const EwOp& o = P.op[k];
    switch (o.code) {
      case EW_FREE:
        st[sp++] = 0.0;  // np.zeros_like (potentials.py:72)
        break;
      case EW_HARM: {
        double kk = o.c0 ? o.c0[i] : o.s0;
        st[sp++] = mul(kk, q);  // k * q (potentials.py:95)
        break;
      }
      case EW_DW: {
        double a = o.c0 ? o.c0[i] : o.s0;
        double b = o.c1 ? o.c1[i] : o.s1;
        // 4.0 * a * q * (q * q - b)  (potentials.py:128)
        st[sp++] = mul(mul(mul(4.0, a), q), sub(mul(q, q), b));
        break;
      }
      default: {  // EW_PERT: base + lam * delta (potentials.py:214)
        double d = st[--sp];
        double b = st[--sp];
        st[sp++] = add(b, mul(o.lam, d));
      }
    }
  }
  return st[0];
}

__device__ __forceinline__ double ew_energy_term(const EwProg& P, double q, int64_t i) {
  double st[EW_MAX];
  int sp = 0;
#pragma unroll 1
  for (int k = 0; k < P.n; ++k) {
    const EwOp& o = P.op[k];
    switch (o.code) {
      case EW_FREE:
        st[sp++] = 0.0;
        break;
      case EW_HARM: {
        double kk = o.c0 ? o.c0[i] : o.s0;
        st[sp++] = 0.5 * kk * q * q;
        break;
      }
      case EW_DW: {
        double a = o.c0 ? o.c0[i] : o.s0;
        double b = o.c1 ? o.c1[i] : o.s1;
        double w = q * q - b;
        st[sp++] = a * w * w;
        break;
      }
      default: {
        double d = st[--sp];
        double b = st[--sp];
        st[sp++] = b + o.lam * d;
      }
    }
  }
  return st[0];
}

// x^3 correctly rounded in all but double-rounding corner cases (numpy's
// `** 3` goes through pow(); x*x*x would round twice).
__device__ __forceinline__ double cube_cr(double x) {
  double p = x * x;
  double e = fma(x, x, -p);
  double h = p * x;
  double e2 = fma(p, x, -h);
  return __dadd_rn(h, fma(e, x, e2));
}

// LJ gradient of atom i, component c, in the reference's order:
// diff = x_i - x_j, r2 = sum_c diff^2 (sequential), u3 = (s^2/r2)^3,
// coeff = (24 eps u3 - 48 eps u3 u3)/r2, grad_i = sum_j coeff*diff (j order)
// (potentials.py:156-180).  `x` is the atom-major position block.
template <int D>
__device__ __forceinline__ void lj_grad_atom(const double* x, int n, int i, double eps,
                                             double sigma, double* g, int* coincident) {
  double xi[D];
#pragma unroll
  for (int c = 0; c < D; ++c) xi[c] = x[i * D + c];
  const double s2 = mul(sigma, sigma);
  const double e24 = mul(24.0, eps), e48 = mul(48.0, eps);
  double acc[D];
  for (int j = 0; j < n; ++j) {
    double diff[D];
    double r2 = 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      diff[c] = sub(xi[c], x[j * D + c]);
      r2 = (c == 0) ? mul(diff[c], diff[c]) : add(r2, mul(diff[c], diff[c]));
    }
    double coeff;
    if (j == i) {
      coeff = 0.0;
    } else {
      if (r2 == 0.0) *coincident = 1;
      double u3 = cube_cr(dvd(s2, r2));
      coeff = dvd(sub(mul(e24, u3), mul(mul(e48, u3), u3)), r2);
    }
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double t = mul(coeff, diff[c]);
      acc[c] = (j == 0) ? t : add(acc[c], t);
    }
  }
#pragma unroll
  for (int c = 0; c < D; ++c) g[c] = acc[c];
}

}  // namespace pl
