// Potential handles and the batched Potential.energy/gradient entry
// (potentials.py:39-214 plus the periodic EAM / SNAP additions).
#include <cmath>
#include <cstring>

#include "pl_common.cuh"
#include "toy.cuh"

namespace pl {

bool is_elementwise(const pl_pot* p) {
  switch (p->kind) {
    case POT_FREE:
    case POT_HARMONIC:
    case POT_DOUBLE_WELL:
      return true;
    case POT_PERTURBED:
      return p->lam == 0.0 ? is_elementwise(p->base)
                           : (is_elementwise(p->base) && is_elementwise(p->delta));
    default:
      return false;
  }
}

static int flatten(const pl_pot* p, EwProg& P) {
  if (P.n >= EW_MAX) return fail(PL_EARG, "potential tree too deep");
  switch (p->kind) {
    case POT_FREE:
      P.op[P.n++] = EwOp{EW_FREE, nullptr, nullptr, 0, 0, 0};
      return PL_OK;
    case POT_HARMONIC:
      P.op[P.n++] = EwOp{EW_HARM, p->d_c0, nullptr, p->s0, 0, 0};
      return PL_OK;
    case POT_DOUBLE_WELL:
      P.op[P.n++] = EwOp{EW_DW, p->d_c0, p->d_c1, p->s0, p->s1, 0};
      return PL_OK;
    case POT_PERTURBED:
      if (p->lam == 0.0) return flatten(p->base, P);  // bit-for-bit base (potentials.py:212)
      PL_TRY(flatten(p->base, P));
      PL_TRY(flatten(p->delta, P));
      if (P.n >= EW_MAX) return fail(PL_EARG, "potential tree too deep");
      P.op[P.n++] = EwOp{EW_PERT, nullptr, nullptr, 0, 0, p->lam};
      return PL_OK;
    default:
      return fail(PL_EARG, "not an elementwise potential");
  }
}

int ew_program(const pl_pot* p, EwProg* out) {
  std::memset(out, 0, sizeof(EwProg));
  return flatten(p, *out);
}

// ---------------------------------------------------------------- kernels
__global__ void k_ew_compute(EwProg P, int64_t B, int64_t d, const double* __restrict__ q,
                             double* __restrict__ grad, double* __restrict__ eterm) {
  int64_t n = B * d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t % d;
    double x = q[t];
    if (grad) grad[t] = ew_grad(P, x, i);
    if (eterm) eterm[t] = ew_energy_term(P, x, i);
  }
}

// deterministic per-system sum (fixed order tree inside one CTA)
__global__ void k_rowsum(int64_t B, int64_t d, const double* __restrict__ v, double* __restrict__ out) {
  __shared__ double sh[256];
  int64_t b = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) s += v[b * d + i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[b] = sh[0];
}

template <int D>
__global__ void k_lj_compute(int64_t B, int n, double eps, double sigma, const double* __restrict__ q,
                             double* __restrict__ grad, double* __restrict__ energy,
                             int* __restrict__ coincident) {
  extern __shared__ double sx[];
  int64_t b = blockIdx.x;
  const double* qb = q + b * (int64_t)n * D;
  for (int t = threadIdx.x; t < n * D; t += blockDim.x) sx[t] = qb[t];
  __syncthreads();
  int bad = 0;
  if (grad) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double g[D];
      lj_grad_atom<D>(sx, n, i, eps, sigma, g, &bad);
#pragma unroll
      for (int c = 0; c < D; ++c) grad[b * (int64_t)n * D + i * D + c] = g[c];
    }
  }
  if (energy) {
    // pair energy 4 eps (u3^2 - u3), i < j (potentials.py:165-170)
    __shared__ double sh[256];
    double e = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      for (int j = i + 1; j < n; ++j) {
        double r2 = 0.0;
        for (int c = 0; c < D; ++c) {
          double dd = sx[i * D + c] - sx[j * D + c];
          r2 += dd * dd;
        }
        if (r2 == 0.0) bad = 1;
        double u3 = cube_cr(sigma * sigma / r2);
        e += 4.0 * eps * (u3 * u3 - u3);
      }
    }
    sh[threadIdx.x] = e;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) energy[b] = sh[0];
  }
  if (bad) atomicExch(coincident, 1);
}

__global__ void k_axpy_lam(int64_t n, double lam, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    y[t] = add(y[t], mul(lam, x[t]));  // base + lam * delta
}

static unsigned grid_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

int lj_compute(pl_pot* pot, int64_t B, const double* q, double* energy, double* grad) {
  pl_ctx* ctx = pot->ctx;
  PL_TRY(pot->work[7].reserve(16));
  int* flag = (int*)pot->work[7].ptr;
  PL_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
  int n = pot->n_atoms;
  size_t smem = (size_t)n * pot->space_dim * sizeof(double);
  if (smem > 200 * 1024) return fail(PL_EARG, "LJ cluster too large for one CTA");
  switch (pot->space_dim) {
    case 1:
      cudaFuncSetAttribute(k_lj_compute<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_lj_compute<1><<<(unsigned)B, 256, smem, ctx->stream>>>(B, n, pot->eps, pot->sigma, q, grad, energy, flag);
      break;
    case 2:
      cudaFuncSetAttribute(k_lj_compute<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_lj_compute<2><<<(unsigned)B, 256, smem, ctx->stream>>>(B, n, pot->eps, pot->sigma, q, grad, energy, flag);
      break;
    case 3:
      cudaFuncSetAttribute(k_lj_compute<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_lj_compute<3><<<(unsigned)B, 256, smem, ctx->stream>>>(B, n, pot->eps, pot->sigma, q, grad, energy, flag);
      break;
    default:
      return fail(PL_EARG, "LJ space_dim must be 1, 2 or 3 on the device");
  }
  PL_CHECK_LAUNCH();
  return PL_OK;
}

int lj_check(pl_pot* pot) {
  int h = 0;
  PL_CUDA(cudaMemcpyAsync(&h, pot->work[7].ptr, sizeof(int), cudaMemcpyDeviceToHost, pot->ctx->stream));
  PL_CUDA(cudaStreamSynchronize(pot->ctx->stream));
  if (h) return fail(PL_EPOT, "coincident atoms: pair distance is zero");
  return PL_OK;
}

int compute(pl_pot* pot, int64_t B, int64_t d, const double* q, double* energy, double* grad,
            double* virial) {
  pl_ctx* ctx = pot->ctx;
  if (pot->dim && pot->dim != d)
    return fail(PL_EARG, "potential expects dimension " + std::to_string(pot->dim) +
                             ", got " + std::to_string(d));
  if (B == 0 || d == 0) return PL_OK;
  if (virial && !(pot->kind == POT_EAM || pot->kind == POT_SNAP || pot->kind == POT_PERTURBED))
    PL_CUDA(cudaMemsetAsync(virial, 0, sizeof(double) * 6 * B, ctx->stream));
  if (is_elementwise(pot)) {
    EwProg P;
    PL_TRY(ew_program(pot, &P));
    double* eterm = nullptr;
    if (energy) {
      PL_TRY(pot->work[6].reserve(sizeof(double) * B * d));
      eterm = (double*)pot->work[6].ptr;
    }
    k_ew_compute<<<grid_for(B * d), 256, 0, ctx->stream>>>(P, B, d, q, grad, eterm);
    PL_CHECK_LAUNCH();
    if (energy) {
      k_rowsum<<<(unsigned)B, 256, 0, ctx->stream>>>(B, d, eterm, energy);
      PL_CHECK_LAUNCH();
    }
    return PL_OK;
  }
  switch (pot->kind) {
    case POT_LJ:
      PL_TRY(lj_compute(pot, B, q, energy, grad));
      return PL_OK;
    case POT_EAM:
      return compute_eam(pot, B, q, energy, grad, virial);
    case POT_SNAP:
      return compute_snap(pot, B, q, energy, grad, virial);
    case POT_PERTURBED: {
      PL_TRY(compute(pot->base, B, d, q, energy, grad, virial));
      if (pot->lam == 0.0) return PL_OK;
      // delta into scratch, then y = y + lam * x (potentials.py:209, 214)
      size_t need = sizeof(double) * (B * d + B + 6 * B);
      PL_TRY(pot->work[5].reserve(need));
      double* g2 = (double*)pot->work[5].ptr;
      double* e2 = g2 + B * d;
      double* v2 = e2 + B;
      PL_TRY(compute(pot->delta, B, d, q, energy ? e2 : nullptr, grad ? g2 : nullptr,
                     virial ? v2 : nullptr));
      if (grad) k_axpy_lam<<<grid_for(B * d), 256, 0, ctx->stream>>>(B * d, pot->lam, g2, grad);
      if (energy) k_axpy_lam<<<grid_for(B), 256, 0, ctx->stream>>>(B, pot->lam, e2, energy);
      if (virial) k_axpy_lam<<<grid_for(6 * B), 256, 0, ctx->stream>>>(6 * B, pot->lam, v2, virial);
      PL_CHECK_LAUNCH();
      return PL_OK;
    }
    default:
      return fail(PL_EARG, "unknown potential kind");
  }
}

}  // namespace pl
