// Corrected coarse sweep of parareal (parareal.py:289-299, 195-198, 425-445).
//
// The sweep is the sequential critical path: window m's coarse propagation
// needs cur[m], produced by window m-1.  States stay in HBM; per node only
// the running error (two scalars) is read back, which is what the adaptive
// engine's truncation decision needs (parareal.py:433-445).
#include <cmath>
#include <cstdlib>
#include <vector>

#include "pl_common.cuh"

namespace pl {

int propagate_windows(pl_ctx* ctx, pl_pot* pot, int64_t W, int64_t d, int L, const double* q0,
                      const double* p0, const double* noise, const double* h_amp,
                      const double* mass, double dt, double h, double hg, double* q1, double* p1,
                      int32_t* blow, double* s1 = nullptr, double* s2 = nullptr);

namespace {

constexpr int CT = 1024;

// deterministic block sum of squares (fixed tree order)
__device__ double block_sumsq(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int w = CT / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  double r = sh[0];
  __syncthreads();
  return r;
}

// acc = {num, den, delta, nonfinite}
__global__ void __launch_bounds__(CT)
k_combine(int64_t d, const double* __restrict__ base_q, const double* __restrict__ base_p,
          const double* __restrict__ jump_q, const double* __restrict__ jump_p,
          const double* __restrict__ prev_q, double* __restrict__ cur_q, double* __restrict__ cur_p,
          double* __restrict__ acc, double* __restrict__ hist) {
  __shared__ double sh[CT];
  double s1 = 0.0, s2 = 0.0;
  int bad = 0;
  for (int64_t i = threadIdx.x; i < d; i += CT) {
    // corrected value: coarse + jump, jump formed first (parareal.py:293); prev is
    // read before cur is written, so prev_q may alias cur_q (replica batches)
    const double pq = prev_q[i];
    double q = add(base_q[i], jump_q[i]);
    double p = add(base_p[i], jump_p[i]);
    cur_q[i] = q;
    cur_p[i] = p;
    if (!isfinite(q) || !isfinite(p)) bad = 1;
    double e = sub(q, pq);
    s1 += e * e;
    s2 += pq * pq;
  }
  bad = __syncthreads_or(bad);
  double n1 = sqrt(block_sumsq(s1, sh));
  double n2 = sqrt(block_sumsq(s2, sh));
  if (threadIdx.x == 0) {
    double num = acc[0] + n1;  // parareal.py:196-197
    double den = acc[1] + n2;
    acc[0] = num;
    acc[1] = den;
    acc[2] = num / den;
    acc[3] = bad ? 1.0 : 0.0;
    *hist = num / den;
  }
}

__global__ void __launch_bounds__(CT)
k_accumulate_node(int64_t d, const double* __restrict__ q, double* __restrict__ acc) {
  __shared__ double sh[CT];
  double s2 = 0.0;
  for (int64_t i = threadIdx.x; i < d; i += CT) s2 += q[i] * q[i];
  double n2 = sqrt(block_sumsq(s2, sh));
  if (threadIdx.x == 0) acc[1] += n2;  // num += ||q - q|| = 0
}

__global__ void k_sub(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                      double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = sub(a[t], b[t]);
}

}  // namespace

int sub_arrays(pl_ctx* ctx, int64_t n, const double* a, const double* b, double* out) {
  if (n <= 0) return PL_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_sub<<<(unsigned)blocks, 256, 0, ctx->stream>>>(n, a, b, out);
  PL_CHECK_LAUNCH();
  return PL_OK;
}

int sweep_cta(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t m0, int64_t m1, int include_m0,
              int mode, double* Q, double* P, const double* prevQ, double* baseQ, double* baseP,
              const double* jumpQ, const double* jumpP, const double* noise, const double* h_amp,
              const double* mass, double dt, double h, double hg, double expl, double* h_state,
              int64_t* h_out4, double* d_hist);

int sweep_cluster_batch(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t N, int R_act, const int32_t* h_ridx,
                        const int64_t* h_m0, const int64_t* h_m1, const int32_t* h_inc, int mode, double* Q,
                        double* P, double* baseQ, double* baseP, const double* jumpQ, const double* jumpP,
                        const double* noise, const double* h_amp, const double* mass, double dt, double h,
                        double hg, double expl, double* h_state, int64_t* h_out4, double* d_hist);

// one-slot cluster sweep (EAM coarse); -1 when not applicable
static int sweep_cluster_one(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t m0, int64_t m1, int inc,
                             int mode, double* Q, double* P, double* baseQ, double* baseP, const double* jumpQ,
                             const double* jumpP, const double* noise, const double* h_amp, const double* mass,
                             double dt, double h, double hg, double expl, double* h_state, int64_t* o4,
                             double* d_hist) {
  if (coarse->kind != POT_EAM || getenv("PL_SWEEP_NOCLUSTER")) return -1;
  const int32_t ridx = 0;
  const int32_t incl = inc;
  return sweep_cluster_batch(ctx, coarse, d, L, m1, 1, &ridx, &m0, &m1, &incl, mode, Q, P, baseQ, baseP, jumpQ,
                             jumpP, noise, h_amp, mass, dt, h, hg, expl, h_state, o4, d_hist);
}

static int cta_status(const int64_t* o4, int64_t* h_out, int32_t* h_blowup) {
  if (o4[3] == 1) {
    h_out[0] = o4[1];
    h_blowup[0] = (int32_t)o4[2];
    return fail(PL_EBLOWUP, "coarse window blew up");
  }
  if (o4[3] == 2) {
    h_out[0] = o4[1];
    h_blowup[0] = 0;
    return fail(PL_EBLOWUP, "corrected state is not finite");
  }
  h_out[0] = o4[0];
  return PL_OK;
}

int bootstrap(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t m0, int64_t m1, double* Q, double* P,
              double* baseQ, double* baseP, const double* noise_all, const double* h_amp, const double* mass,
              double dt, double h, double hg, int64_t* h_out, int32_t* h_blowup) {
  h_out[0] = 0;
  h_blowup[0] = 0;
  if (m1 <= m0) return PL_OK;
  if (coarse->dim && coarse->dim != d) return fail(PL_EARG, "potential dimension mismatch");
  int64_t o4[4];
  double state[2] = {0.0, 0.0};
  PL_TRY(ctx->work[6].reserve(sizeof(double) * (m1 - m0 + 1)));
  int rc = sweep_cluster_one(ctx, coarse, d, L, m0, m1, 0, 1, Q, P, baseQ, baseP, baseQ, baseP, noise_all, h_amp,
                             mass, dt, h, hg, 0.0, state, o4, (double*)ctx->work[6].ptr);
  if (rc == -1)
    rc = sweep_cta(ctx, coarse, d, L, m0, m1, 0, 1, Q, P, Q, baseQ, baseP, baseQ, baseP, noise_all, h_amp, mass, dt,
                   h, hg, 0.0, state, o4, (double*)ctx->work[6].ptr);
  if (rc != -1) {
    PL_TRY(rc);
    return cta_status(o4, h_out, h_blowup);
  }
  // generic: one batched-propagator call per window, first blow-up reported
  cudaStream_t st = ctx->stream;
  PL_TRY(ctx->work[6].reserve(sizeof(int32_t) * (m1 - m0 + 1)));
  int32_t* blows = (int32_t*)ctx->work[6].ptr;
  PL_CUDA(cudaMemsetAsync(blows, 0, sizeof(int32_t) * (m1 - m0), st));
  const int64_t nb = (int64_t)(L + 1) * d;
  for (int64_t m = m0; m < m1; ++m) {
    PL_TRY(propagate_windows(ctx, coarse, 1, d, L, Q + m * d, P + m * d, noise_all + m * nb, h_amp, mass, dt,
                             h, hg, baseQ + m * d, baseP + m * d, blows + (m - m0)));
    PL_CUDA(cudaMemcpyAsync(Q + (m + 1) * d, baseQ + m * d, sizeof(double) * d, cudaMemcpyDeviceToDevice, st));
    PL_CUDA(cudaMemcpyAsync(P + (m + 1) * d, baseP + m * d, sizeof(double) * d, cudaMemcpyDeviceToDevice, st));
  }
  std::vector<int32_t> hb(m1 - m0);
  PL_CUDA(cudaMemcpyAsync(hb.data(), blows, sizeof(int32_t) * (m1 - m0), cudaMemcpyDeviceToHost, st));
  PL_CUDA(cudaStreamSynchronize(st));
  for (int64_t k = 0; k < m1 - m0; ++k)
    if (hb[k]) {
      h_out[0] = m0 + k;
      h_blowup[0] = hb[k];
      return fail(PL_EBLOWUP, "coarse bootstrap blew up");
    }
  h_out[0] = m1 - m0;
  return PL_OK;
}

int sweep(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t m0, int64_t m1, int include_m0,
          double* traj_q, double* traj_p, const double* prev_q, double* base_q, double* base_p,
          const double* jump_q, const double* jump_p, const double* noise_all, const double* h_amp,
          const double* mass, double dt, double h, double hg, double expl, double* h_state,
          double* d_hist, int64_t* h_out, int32_t* h_blowup) {
  cudaStream_t st = ctx->stream;
  h_out[0] = 0;
  h_blowup[0] = 0;
  if (m1 <= m0) return PL_OK;
  if (coarse->dim && coarse->dim != d) return fail(PL_EARG, "potential dimension mismatch");
  if (!getenv("PL_SWEEP_GENERIC")) {
    int64_t o4[4];
    int rc = sweep_cluster_one(ctx, coarse, d, L, m0, m1, include_m0, 0, traj_q, traj_p, base_q, base_p, jump_q,
                               jump_p, noise_all, h_amp, mass, dt, h, hg, expl, h_state, o4, d_hist);
    if (rc == -1)
      rc = sweep_cta(ctx, coarse, d, L, m0, m1, include_m0, 0, traj_q, traj_p, prev_q, base_q, base_p, jump_q,
                     jump_p, noise_all, h_amp, mass, dt, h, hg, expl, h_state, o4, d_hist);
    if (rc != -1) {
      PL_TRY(rc);
      return cta_status(o4, h_out, h_blowup);
    }
  }
  PL_TRY(ctx->work[3].reserve(sizeof(double) * 8 + sizeof(int32_t) * 8));
  double* acc = (double*)ctx->work[3].ptr;
  int32_t* blow = (int32_t*)(acc + 4);
  if (!ctx->pinned) {
    PL_CUDA(cudaMallocHost(&ctx->pinned, 256));
    ctx->pinned_bytes = 256;
  }
  double* hacc = (double*)ctx->pinned;
  int32_t* hblow = (int32_t*)(hacc + 4);
  double init[4] = {h_state[0], h_state[1], 0.0, 0.0};
  PL_CUDA(cudaMemcpyAsync(acc, init, sizeof(init), cudaMemcpyHostToDevice, st));
  if (include_m0) {
    k_accumulate_node<<<1, CT, 0, st>>>(d, traj_q + m0 * d, acc);
    PL_CHECK_LAUNCH();
  }
  const int64_t nb = (int64_t)(L + 1) * d;
  for (int64_t m = m0; m < m1; ++m) {
    PL_TRY(propagate_windows(ctx, coarse, 1, d, L, traj_q + m * d, traj_p + m * d,
                             noise_all + m * nb, h_amp, mass, dt, h, hg, base_q + m * d,
                             base_p + m * d, blow));
    k_combine<<<1, CT, 0, st>>>(d, base_q + m * d, base_p + m * d, jump_q + m * d, jump_p + m * d,
                                prev_q + (m + 1) * d, traj_q + (m + 1) * d, traj_p + (m + 1) * d,
                                acc, d_hist + (m - m0));
    PL_CHECK_LAUNCH();
    PL_CUDA(cudaMemcpyAsync(hacc, acc, sizeof(double) * 4 + sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    PL_CUDA(cudaStreamSynchronize(st));
    h_state[0] = hacc[0];
    h_state[1] = hacc[1];
    if (hblow[0]) {
      h_out[0] = m;
      h_blowup[0] = hblow[0];
      return fail(PL_EBLOWUP, "coarse window blew up");
    }
    if (hacc[3] != 0.0) {
      h_out[0] = m;
      h_blowup[0] = 0;
      return fail(PL_EBLOWUP, "corrected state is not finite");
    }
    h_out[0] = m - m0 + 1;
    if (hacc[1] == 0.0) return PL_OK;  // caller raises DegenerateNormalizationError
    if (expl > 0.0 && hacc[2] > expl) return PL_OK;
  }
  return PL_OK;
}

// Replica batch through the per-window generic path (systems too large for the
// persistent sweeps, e.g. the 16,001-atom heavy config): slot by slot, with the
// pl_sweep_batch conventions (arrays with a leading replica dimension, out4 =
// {nodes done, window, substep, status 1 blow-up / 2 non-finite}).
int sweep_generic_batch(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t N, int R_act, const int32_t* h_ridx,
                        const int64_t* h_m0, const int64_t* h_m1, const int32_t* h_inc, int mode, double* Q,
                        double* P, double* baseQ, double* baseP, const double* jumpQ, const double* jumpP,
                        const double* noise, const double* h_amp, const double* mass, double dt, double h, double hg,
                        double expl, double* h_state, int64_t* h_out4, double* d_hist) {
  for (int s = 0; s < R_act; ++s) {
    const int64_t r = h_ridx[s];
    double* q = Q + r * (N + 1) * d;
    double* p = P + r * (N + 1) * d;
    double* bq = baseQ + r * N * d;
    double* bp = baseP + r * N * d;
    const double* nz = noise + r * N * (int64_t)(L + 1) * d;
    int64_t* o4 = h_out4 + 4 * s;
    int64_t out = 0;
    int32_t blow = 0;
    int rc;
    if (mode == 1) {
      rc = bootstrap(ctx, coarse, d, L, h_m0[s], h_m1[s], q, p, bq, bp, nz, h_amp, mass, dt, h, hg, &out, &blow);
    } else {
      rc = sweep(ctx, coarse, d, L, h_m0[s], h_m1[s], h_inc[s], q, p, q, bq, bp, jumpQ + r * N * d,
                 jumpP + r * N * d, nz, h_amp, mass, dt, h, hg, expl, h_state + 2 * s, d_hist + r * N, &out, &blow);
    }
    o4[0] = o4[1] = o4[2] = o4[3] = 0;
    if (rc == PL_EBLOWUP) {
      o4[1] = out;
      o4[2] = blow;
      o4[3] = blow ? 1 : 2;
      continue;
    }
    PL_TRY(rc);
    o4[0] = out;
  }
  return PL_OK;
}

}  // namespace pl

extern "C" int pl_bootstrap(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t m0, int64_t m1,
                            double* d_traj_q, double* d_traj_p, double* d_base_q, double* d_base_p,
                            const double* d_noise_all, const double* h_amp, const double* d_mass, double dt,
                            double half_dt, double half_dt_gamma, int64_t* h_out, int32_t* h_blowup) {
  if (!ctx || !coarse || !d_traj_q || !d_traj_p || !d_base_q || !d_base_p || !d_noise_all || !h_amp ||
      !h_out || !h_blowup)
    return pl::fail(PL_EARG, "NULL argument");
  if (d < 1 || L < 1 || m0 < 0) return pl::fail(PL_EARG, "need d >= 1, L >= 1, m0 >= 0");
  return pl::bootstrap(ctx, coarse, d, L, m0, m1, d_traj_q, d_traj_p, d_base_q, d_base_p, d_noise_all, h_amp,
                       d_mass, dt, half_dt, half_dt_gamma, h_out, h_blowup);
}

extern "C" int pl_sub(pl_ctx* ctx, int64_t n, const double* a, const double* b, double* out) {
  if (!ctx || (n > 0 && (!a || !b || !out))) return pl::fail(PL_EARG, "NULL argument");
  return pl::sub_arrays(ctx, n, a, b, out);
}
