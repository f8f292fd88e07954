// Tabulated EAM / Finnis-Sinclair potential, batched over systems
// (the coarse potential of the parareal pair).
//
//   E   = sum_i F(rho_i) + 1/2 sum_i sum_j phi(r_ij),   rho_i = sum_j rho(r_ij)
//   dE/dr_i = -sum_j [ (F'(rho_i) + F'(rho_j)) rho'(r_ij) + phi'(r_ij) ] (r_j - r_i)/r_ij
//
// Two gather passes over a full neighbour list (density, then forces): no
// atomics, every sum in neighbour-list order, so results are deterministic
// and independent of launch shape.  The tables are cubic Hermite pieces; a
// piece lookup costs one divide, one conversion and a Horner chain.
#include <cmath>

#include "eam.cuh"
#include "neigh.cuh"
#include "pl_common.cuh"

namespace pl {

int eam_tpa_for(int n);

constexpr int EAM_MAXN = 96;

// tpa threads per atom (eam_tpa rule), one atom per group, groups strided over
// the batch; group-reduced in the same xor-tree as the persistent sweep
__global__ void k_eam_density(int64_t B, int N, int tpa, Box box, double rc2, Table rho, Table F,
                              const double* __restrict__ q, const int32_t* __restrict__ nbr,
                              const int32_t* __restrict__ cnt, int maxn, double* __restrict__ Fp,
                              double* __restrict__ Fe) {
  const int64_t gid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / tpa;
  const int sub = threadIdx.x % tpa;
  const int64_t t = gid < B * N ? gid : B * N - 1;  // keep whole groups alive for the shuffles
  const int64_t b = t / N;
  const int i = (int)(t - b * N);
  const double s = group_sum(eam_rho_part(q + b * (int64_t)N * 3, i, nbr + t * maxn, cnt[t], sub, tpa, box,
                                          rc2, rho), tpa);
  if (gid < B * N && sub == 0) {
    double f, df;
    tab_eval(F, s, f, df);
    Fp[t] = df;
    Fe[t] = f;
  }
}

__global__ void k_eam_force(int64_t B, int N, int tpa, Box box, double rc2, Table rho, Table phi,
                            const double* __restrict__ q, const int32_t* __restrict__ nbr,
                            const int32_t* __restrict__ cnt, int maxn, const double* __restrict__ Fp,
                            const double* __restrict__ Fe, double* __restrict__ grad,
                            double* __restrict__ eatom, double* __restrict__ vatom) {
  const int64_t gid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / tpa;
  const int sub = threadIdx.x % tpa;
  const int64_t t = gid < B * N ? gid : B * N - 1;
  const int64_t b = t / N;
  const int i = (int)(t - b * N);
  double g[3] = {0.0, 0.0, 0.0}, e = 0.0, v[6] = {0, 0, 0, 0, 0, 0};
  if (eatom || vatom)
    eam_force_part<true>(q + b * (int64_t)N * 3, Fp + b * (int64_t)N, i, nbr + t * maxn, cnt[t], sub, tpa, box,
                         rc2, rho, phi, g, &e, v);
  else
    eam_force_part<false>(q + b * (int64_t)N * 3, Fp + b * (int64_t)N, i, nbr + t * maxn, cnt[t], sub, tpa,
                          box, rc2, rho, phi, g, &e, v);
  g[0] = group_sum(g[0], tpa);
  g[1] = group_sum(g[1], tpa);
  g[2] = group_sum(g[2], tpa);
  if (eatom) e = group_sum(e, tpa);
  if (vatom)
    for (int c = 0; c < 6; ++c) v[c] = group_sum(v[c], tpa);
  if (gid < B * N && sub == 0) {
    if (grad) {
      grad[3 * t] = g[0];
      grad[3 * t + 1] = g[1];
      grad[3 * t + 2] = g[2];
    }
    if (eatom) eatom[t] = Fe[t] + e;
    if (vatom)
      for (int c = 0; c < 6; ++c) vatom[6 * t + c] = v[c];
  }
}

// per-system fixed-order reductions of per-atom energy (and virial)
__global__ void k_sys_reduce(int64_t B, int N, int width, const double* __restrict__ per_atom,
                             double* __restrict__ out) {
  __shared__ double sh[256];
  int64_t b = blockIdx.x;
  for (int c = 0; c < width; ++c) {
    double s = 0.0;
    for (int i = threadIdx.x; i < N; i += blockDim.x) s += per_atom[(b * N + i) * width + c];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[b * width + c] = sh[0];
    __syncthreads();
  }
}

int eam_prepare(pl_pot* pot, const double* rho, const double* phi, const double* F) {
  size_t nr = sizeof(double) * 4 * pot->n_r, nf = sizeof(double) * 4 * pot->n_rho;
  PL_CUDA(cudaMalloc(&pot->d_rho, nr));
  PL_CUDA(cudaMalloc(&pot->d_phi, nr));
  PL_CUDA(cudaMalloc(&pot->d_F, nf));
  PL_CUDA(cudaMemcpy(pot->d_rho, rho, nr, cudaMemcpyHostToDevice));
  PL_CUDA(cudaMemcpy(pot->d_phi, phi, nr, cudaMemcpyHostToDevice));
  PL_CUDA(cudaMemcpy(pot->d_F, F, nf, cudaMemcpyHostToDevice));
  // algorithmic flops per system: ~ (2 table evals + 25) per pair x 2 passes
  pot->flops = 0.0;
  return PL_OK;
}

int compute_eam(pl_pot* pot, int64_t B, const double* q, double* energy, double* grad, double* virial) {
  pl_ctx* ctx = pot->ctx;
  int N = pot->n_atoms;
  NeighList nl;
  PL_TRY(build_neighbours(pot, B, q, pot->rcut, EAM_MAXN, &nl));
  size_t na = (size_t)B * N;
  PL_TRY(pot->work[2].reserve(sizeof(double) * na * (2 + 1 + 6)));
  double* Fp = (double*)pot->work[2].ptr;
  double* Fe = Fp + na;
  double* ea = Fe + na;
  double* va = ea + na;
  Box box = make_box(pot->box);
  Table trho{pot->d_rho, pot->n_r, pot->dr, 1.0 / pot->dr}, tphi{pot->d_phi, pot->n_r, pot->dr, 1.0 / pot->dr},
      tF{pot->d_F, pot->n_rho, pot->drho, 1.0 / pot->drho};
  const int tpa = eam_tpa_for(N);  // the cluster sweep's rule (same lane partition and reduction tree)
  const double rc2 = pot->rcut * pot->rcut;
  unsigned g = (unsigned)((na * tpa + 127) / 128);
  prof_mark(ctx->stream, ST_EAM, true);
  k_eam_density<<<g, 128, 0, ctx->stream>>>(B, N, tpa, box, rc2, trho, tF, q, nl.nbr, nl.cnt, nl.maxn, Fp, Fe);
  PL_CHECK_LAUNCH();
  k_eam_force<<<g, 128, 0, ctx->stream>>>(B, N, tpa, box, rc2, trho, tphi, q, nl.nbr, nl.cnt, nl.maxn, Fp, Fe,
                                          grad, energy ? ea : nullptr, virial ? va : nullptr);
  PL_CHECK_LAUNCH();
  prof_mark(ctx->stream, ST_EAM, false);
  if (energy) {
    k_sys_reduce<<<(unsigned)B, 256, 0, ctx->stream>>>(B, N, 1, ea, energy);
    PL_CHECK_LAUNCH();
  }
  if (virial) {
    k_sys_reduce<<<(unsigned)B, 256, 0, ctx->stream>>>(B, N, 6, va, virial);
    PL_CHECK_LAUNCH();
  }
  return PL_OK;
}

}  // namespace pl
