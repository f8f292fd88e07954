// Batched steepest descent with Armijo backtracking (potentials.py:231-266
// _descend, used by local_minima 268-287): B independent descents in lockstep.
//
// Per outer iteration: one batched gradient evaluation, fixed-order |g|^2 per
// member; members with sqrt(|g|^2) <= tol stop.  The others double their step
// (capped at 1e3) and backtrack: trial = x - step*g (numpy order: the product
// first), one batched energy evaluation of all trials per round, accept when
// the energy is finite and E_trial <= E - 0.5*step*|g|^2, else halve the step
// (stall below 1e-18).  A trial the potential rejects (coincident atoms,
// neighbour overflow) counts as +inf, as the reference maps PotentialError.
// The accept / halve decisions are the reference's scalar arithmetic on the
// host; the vectors never leave the device.
#include <cmath>
#include <vector>

#include "pl_common.cuh"

namespace pl {

int compute(pl_pot* pot, int64_t B, int64_t d, const double* q, double* energy, double* grad, double* virial);
int lj_check(pl_pot* pot);
int neigh_check(pl_pot* pot);

constexpr int MIN_THREADS = 256;

// fixed-order |g|^2 per member: strided partials, then a tree over the CTA
__global__ void __launch_bounds__(MIN_THREADS) k_sqnorm(int64_t d, const double* __restrict__ g,
                                                        double* __restrict__ out) {
  __shared__ double part[MIN_THREADS];
  const double* gb = g + blockIdx.x * d;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < d; i += MIN_THREADS) s = fma(gb[i], gb[i], s);
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = MIN_THREADS / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = part[0];
}

// trial = x - step*g for members with step > 0, else trial = x
__global__ void k_trial(int64_t B, int64_t d, const double* __restrict__ x, const double* __restrict__ g,
                        const double* __restrict__ step, double* __restrict__ trial) {
  const int64_t n = B * d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const double st = step[t / d];
    trial[t] = st > 0.0 ? __dsub_rn(x[t], __dmul_rn(st, g[t])) : x[t];
  }
}

// x = trial for accepted members
__global__ void k_accept(int64_t B, int64_t d, const int32_t* __restrict__ acc, const double* __restrict__ trial,
                         double* __restrict__ x) {
  const int64_t n = B * d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    if (acc[t / d]) x[t] = trial[t];
}

static unsigned grid_of(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

// energies of B states; members the potential rejects get +inf
static int energies_or_inf(pl_pot* pot, int64_t B, int64_t d, const double* q, double* d_e, double* h_e) {
  cudaStream_t st = pot->ctx->stream;
  int rc = compute(pot, B, d, q, d_e, nullptr, nullptr);
  if (rc == PL_OK) rc = pot->kind == POT_LJ ? lj_check(pot) : neigh_check(pot);
  if (rc == PL_OK) {
    PL_CUDA(cudaMemcpyAsync(h_e, d_e, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
    PL_CUDA(cudaStreamSynchronize(st));
    return PL_OK;
  }
  if (rc != PL_EPOT) return rc;
  // a batch-wide rejection: find the offending members one by one
  for (int64_t b = 0; b < B; ++b) {
    int r = compute(pot, 1, d, q + b * d, d_e + b, nullptr, nullptr);
    if (r == PL_OK) r = pot->kind == POT_LJ ? lj_check(pot) : neigh_check(pot);
    if (r == PL_OK) {
      PL_CUDA(cudaMemcpyAsync(h_e + b, d_e + b, sizeof(double), cudaMemcpyDeviceToHost, st));
      PL_CUDA(cudaStreamSynchronize(st));
    } else if (r == PL_EPOT) {
      h_e[b] = INFINITY;
    } else {
      return r;
    }
  }
  return PL_OK;
}

int minimize(pl_ctx* ctx, pl_pot* pot, int64_t B, int64_t d, double* x, double tol, int64_t max_iter,
             int32_t* h_status, int64_t* h_iters, double* h_energy) {
  if (B < 1 || d < 1 || !(tol > 0.0) || max_iter < 0) return fail(PL_EARG, "need B, d >= 1, tol > 0, max_iter >= 0");
  cudaStream_t st = ctx->stream;
  Scratch buf;
  const size_t nd = (size_t)B * d;
  PL_TRY(buf.reserve(sizeof(double) * (2 * nd + 3 * B) + sizeof(int32_t) * B));
  double* g = (double*)buf.ptr;
  double* trial = g + nd;
  double* d_e = trial + nd;
  double* d_gn = d_e + B;
  double* d_step = d_gn + B;
  int32_t* d_acc = (int32_t*)(d_step + B);
  std::vector<double> E(B), Et(B), gn(B), step(B, 1.0), hstep(B);
  std::vector<int32_t> acc(B), done(B, 0);
  // initial energies: a rejection of a start is the caller's error (the reference lets it raise)
  PL_TRY(compute(pot, B, d, x, d_e, nullptr, nullptr));
  PL_TRY(pot->kind == POT_LJ ? lj_check(pot) : neigh_check(pot));
  PL_CUDA(cudaMemcpyAsync(E.data(), d_e, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
  for (int64_t b = 0; b < B; ++b) {
    h_status[b] = 2;  // no convergence unless proven otherwise
    h_iters[b] = max_iter;
  }
  int64_t active = B;
  for (int64_t it = 0; it < max_iter && active > 0; ++it) {
    PL_TRY(compute(pot, B, d, x, nullptr, g, nullptr));
    PL_TRY(pot->kind == POT_LJ ? lj_check(pot) : neigh_check(pot));
    k_sqnorm<<<(unsigned)B, MIN_THREADS, 0, st>>>(d, g, d_gn);
    PL_CHECK_LAUNCH();
    PL_CUDA(cudaMemcpyAsync(gn.data(), d_gn, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
    PL_CUDA(cudaStreamSynchronize(st));
    std::vector<int32_t> searching(B, 0);
    for (int64_t b = 0; b < B; ++b) {
      if (done[b]) continue;
      if (std::sqrt(gn[b]) <= tol) {
        done[b] = 1;
        h_status[b] = 0;
        h_iters[b] = it;
        --active;
        continue;
      }
      step[b] = std::min(step[b] * 2.0, 1e3);
      searching[b] = 1;
    }
    if (active == 0) break;
    for (int64_t b = 0; b < B; ++b) acc[b] = 0;
    for (;;) {
      bool any = false;
      for (int64_t b = 0; b < B; ++b) {
        hstep[b] = searching[b] ? step[b] : 0.0;
        any = any || searching[b];
      }
      if (!any) break;
      PL_CUDA(cudaMemcpyAsync(d_step, hstep.data(), sizeof(double) * B, cudaMemcpyHostToDevice, st));
      k_trial<<<grid_of((int64_t)nd), 256, 0, st>>>(B, d, x, g, d_step, trial);
      PL_CHECK_LAUNCH();
      PL_TRY(energies_or_inf(pot, B, d, trial, d_e, Et.data()));
      for (int64_t b = 0; b < B; ++b) {
        if (!searching[b]) continue;
        if (std::isfinite(Et[b]) && Et[b] <= E[b] - 0.5 * step[b] * gn[b]) {
          searching[b] = 0;
          acc[b] = 1;
        } else {
          step[b] *= 0.5;
          if (step[b] < 1e-18) {  // line search stalled
            searching[b] = 0;
            done[b] = 1;
            h_status[b] = 1;
            h_iters[b] = it;
            --active;
          }
        }
      }
      // the accepted trials of this round must land before the next round overwrites trial
      PL_CUDA(cudaMemcpyAsync(d_acc, acc.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice, st));
      k_accept<<<grid_of((int64_t)nd), 256, 0, st>>>(B, d, d_acc, trial, x);
      PL_CHECK_LAUNCH();
      for (int64_t b = 0; b < B; ++b)
        if (acc[b]) {
          E[b] = Et[b];
          acc[b] = 0;
        }
      PL_CUDA(cudaStreamSynchronize(st));  // acc is reused from the host
    }
  }
  if (h_energy)
    for (int64_t b = 0; b < B; ++b) h_energy[b] = E[b];
  PL_CUDA(cudaStreamSynchronize(st));
  return PL_OK;
}

}  // namespace pl
