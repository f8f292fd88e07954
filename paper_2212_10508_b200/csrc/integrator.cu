// Batched modified-BBK window propagation (integrator.py:173-308).
//
// Per window of L substeps (block l of the window's noise = G_l):
//   open  s:  p_half = p - h*grad - hg*p_ref + (a_{s-1} sqrt m) G_{s-1}
//             q      = q + dt*(p_half/m)          p_ref = p (s=1), p_half_prev (s>1)
//   force:    grad   = dV(q)
//   close s:  p      = p_half - h*grad - hg*p_half + (a_s sqrt m) G_s
//             blow-up check on (q, p)
// with h = 0.5*dt and hg = 0.5*dt*gamma formed as Python forms them.  All
// operations use explicit round-to-nearest intrinsics in numpy's order, so a
// window is bitwise equal to the reference for a bitwise-equal gradient.
//
// Three execution shapes:
//   * elementwise potentials (Free/Harmonic/DoubleWell/Perturbed of those):
//     one thread owns one component of one window for all L substeps;
//   * Lennard-Jones clusters: one CTA owns one window, positions in shared
//     memory, all L substeps in one launch;
//   * periodic many-body (EAM/SNAP/mixtures): per substep, the batched force
//     pipeline over all W windows, then one fused close(s)+open(s+1) kernel.
#include <climits>

#include "pl_common.cuh"
#include "toy.cuh"

namespace pl {

int ew_program(const pl_pot* p, EwProg* out);
int lj_compute(pl_pot* pot, int64_t B, const double* q, double* energy, double* grad);
int lj_check(pl_pot* pot);

struct StepConsts {
  double dt, h, hg;
  int L;
};

struct AmpTable {
  const double* d_amp;  // L+1 scalar amplitudes (device)
};

__device__ __forceinline__ void record_blowup(int32_t* blow, int64_t w, int s) {
  // keep the smallest non-zero substep (first failure)
  int32_t old = blow[w];
  while (old == 0 || old > s) {
    int32_t prev = atomicCAS((int*)&blow[w], old, s);
    if (prev == old) break;
    old = prev;
  }
}

__device__ __forceinline__ bool bounded(double a) { return fabs(a) <= BLOWUP_LIMIT; }

// running momentum moments of the full steps (integrator.py:359-361: s1 += p,
// s2 += p * p, numpy order), one slot per (window, substep, component)
__device__ __forceinline__ void moment(double* s1, double* s2, int64_t k, double p) {
  s1[k] = add(s1[k], p);
  s2[k] = add(s2[k], mul(p, p));
}

// ------------------------------------------------------------ elementwise
__global__ void k_window_ew(EwProg P, int64_t W, int64_t d, StepConsts K,
                            const double* __restrict__ amp, const double* __restrict__ q0,
                            const double* __restrict__ p0, const double* __restrict__ noise,
                            const double* __restrict__ mass, double* __restrict__ q1,
                            double* __restrict__ p1, int32_t* __restrict__ blow, double* __restrict__ s1,
                            double* __restrict__ s2) {
  int64_t n = W * d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t w = t / d, i = t - w * d;
    double m = mass ? mass[i] : 1.0;
    double sm = mass ? __dsqrt_rn(m) : 1.0;
    const double* g = noise + w * (K.L + 1) * d + i;
    double q = q0[t], p = p0[t];
    double grad = ew_grad(P, q, i);
    double pref = p, ph = 0.0;
    int failed = 0;
    double gl = g[0];
    double al = mul(amp[0], sm);
    for (int s = 1; s <= K.L; ++s) {
      ph = add(sub(sub(p, mul(K.h, grad)), mul(K.hg, pref)), mul(al, gl));
      q = add(q, mul(K.dt, dvd(ph, m)));
      grad = ew_grad(P, q, i);
      gl = g[(int64_t)s * d];
      al = mul(amp[s], sm);
      p = add(sub(sub(ph, mul(K.h, grad)), mul(K.hg, ph)), mul(al, gl));
      if (!failed && !(bounded(q) && bounded(p))) failed = s;
      if (s1) moment(s1, s2, (w * K.L + (s - 1)) * d + i, p);
      pref = ph;
    }
    q1[t] = q;
    p1[t] = p;
    if (failed) record_blowup(blow, w, failed);
  }
}

// ------------------------------------------------------------ LJ, CTA per window
template <int D>
__global__ void __launch_bounds__(256)
k_window_lj(int64_t W, int n, double eps, double sigma, StepConsts K,
            const double* __restrict__ amp, const double* __restrict__ q0,
            const double* __restrict__ p0, const double* __restrict__ noise,
            const double* __restrict__ mass, double* __restrict__ q1, double* __restrict__ p1,
            int32_t* __restrict__ blow, int* __restrict__ coincident, double* __restrict__ s1,
            double* __restrict__ s2) {
  extern __shared__ double sm_[];
  const int d = n * D;
  double* sq = sm_;          // positions
  double* sg = sm_ + d;      // gradient
  __shared__ int s_fail;
  int64_t w = blockIdx.x;
  const double* qw = q0 + w * d;
  const double* pw = p0 + w * d;
  const double* gw = noise + w * (int64_t)(K.L + 1) * d;
  if (threadIdx.x == 0) s_fail = 0;
  // each thread owns components t = threadIdx.x + k*blockDim (<= 8 per thread)
  constexpr int PER = 16;
  double p[PER], ph[PER], pref[PER];
  for (int t = threadIdx.x; t < d; t += blockDim.x) sq[t] = qw[t];
  __syncthreads();
  int bad = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) lj_grad_atom<D>(sq, n, i, eps, sigma, sg + i * D, &bad);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    int t = threadIdx.x + k * blockDim.x;
    if (t < d) { p[k] = pw[t]; pref[k] = p[k]; }
  }
  for (int s = 1; s <= K.L; ++s) {
    // open substep s
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      int t = threadIdx.x + k * blockDim.x;
      if (t < d) {
        double m = mass ? mass[t] : 1.0;
        double smm = mass ? __dsqrt_rn(m) : 1.0;
        double al = mul(amp[s - 1], smm);
        ph[k] = add(sub(sub(p[k], mul(K.h, sg[t])), mul(K.hg, pref[k])), mul(al, gw[(int64_t)(s - 1) * d + t]));
        sq[t] = add(sq[t], mul(K.dt, dvd(ph[k], m)));
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) lj_grad_atom<D>(sq, n, i, eps, sigma, sg + i * D, &bad);
    __syncthreads();
    int f = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      int t = threadIdx.x + k * blockDim.x;
      if (t < d) {
        double m = mass ? mass[t] : 1.0;
        double smm = mass ? __dsqrt_rn(m) : 1.0;
        (void)m;
        double al = mul(amp[s], smm);
        p[k] = add(sub(sub(ph[k], mul(K.h, sg[t])), mul(K.hg, ph[k])), mul(al, gw[(int64_t)s * d + t]));
        if (!(bounded(sq[t]) && bounded(p[k]))) f = 1;
        if (s1) moment(s1, s2, (w * K.L + (s - 1)) * d + t, p[k]);
        pref[k] = ph[k];
      }
    }
    if (f) atomicCAS(&s_fail, 0, s);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    int t = threadIdx.x + k * blockDim.x;
    if (t < d) { q1[w * d + t] = sq[t]; p1[w * d + t] = p[k]; }
  }
  if (threadIdx.x == 0 && s_fail) blow[w] = s_fail;
  if (bad) atomicExch(coincident, 1);
}

// ------------------------------------------------------------ generic many-body
__global__ void k_open(int64_t W, int64_t d, int s, bool first, StepConsts K,
                       const double* __restrict__ amp, const double* __restrict__ noise,
                       const double* __restrict__ mass, const double* __restrict__ grad,
                       const double* __restrict__ p, double* __restrict__ ph,
                       double* __restrict__ q) {
  griddep_wait();
  int64_t n = W * d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t w = t / d, i = t - w * d;
    double m = mass ? mass[i] : 1.0;
    double smm = mass ? __dsqrt_rn(m) : 1.0;
    double al = mul(amp[s - 1], smm);
    double gl = noise[(w * (K.L + 1) + (s - 1)) * d + i];
    double pref = first ? p[t] : ph[t];
    double h = add(sub(sub(p[t], mul(K.h, grad[t])), mul(K.hg, pref)), mul(al, gl));
    ph[t] = h;
    q[t] = add(q[t], mul(K.dt, dvd(h, m)));
  }
}

__global__ void k_close(int64_t W, int64_t d, int s, StepConsts K, const double* __restrict__ amp,
                        const double* __restrict__ noise, const double* __restrict__ mass,
                        const double* __restrict__ grad, const double* __restrict__ ph,
                        const double* __restrict__ q, double* __restrict__ p,
                        int32_t* __restrict__ blow, double* __restrict__ s1, double* __restrict__ s2) {
  griddep_wait();
  int64_t n = W * d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t w = t / d, i = t - w * d;
    double smm = mass ? __dsqrt_rn(mass[i]) : 1.0;
    double al = mul(amp[s], smm);
    double gl = noise[(w * (K.L + 1) + s) * d + i];
    double h = ph[t];
    double pn = add(sub(sub(h, mul(K.h, grad[t])), mul(K.hg, h)), mul(al, gl));
    p[t] = pn;
    if (!(bounded(q[t]) && bounded(pn))) record_blowup(blow, w, s);
    if (s1) moment(s1, s2, (w * K.L + (s - 1)) * d + i, pn);
  }
}

// close substep s and open substep s+1 in one pass: both read noise block s
// (block s closes s and reopens s+1, integrator.py:281-288) and the same grad
// and p_half, so one kernel moves 56 B per component instead of 96 B for
// k_close + k_open.  Same operations in the same order as the two kernels.
__global__ void k_close_open(int64_t W, int64_t d, int s, StepConsts K, const double* __restrict__ amp,
                             const double* __restrict__ noise, const double* __restrict__ mass,
                             const double* __restrict__ grad, double* __restrict__ ph,
                             double* __restrict__ q, double* __restrict__ p, int32_t* __restrict__ blow,
                             double* __restrict__ s1, double* __restrict__ s2) {
  griddep_wait();
  int64_t n = W * d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t w = t / d, i = t - w * d;
    const double m = mass ? mass[i] : 1.0;
    const double smm = mass ? __dsqrt_rn(m) : 1.0;
    const double al = mul(amp[s], smm);
    const double gl = noise[(w * (K.L + 1) + s) * d + i];
    const double g = grad[t];
    const double h = ph[t];
    const double qv = q[t];
    const double pn = add(sub(sub(h, mul(K.h, g)), mul(K.hg, h)), mul(al, gl));
    p[t] = pn;
    if (!(bounded(qv) && bounded(pn))) record_blowup(blow, w, s);
    if (s1) moment(s1, s2, (w * K.L + (s - 1)) * d + i, pn);
    // open s + 1: p_ref = p_half of substep s
    const double hn = add(sub(sub(pn, mul(K.h, g)), mul(K.hg, h)), mul(al, gl));
    ph[t] = hn;
    q[t] = add(qv, mul(K.dt, dvd(hn, m)));
  }
}

static unsigned grid_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

int propagate_windows(pl_ctx* ctx, pl_pot* pot, int64_t W, int64_t d, int L, const double* q0,
                      const double* p0, const double* noise, const double* h_amp,
                      const double* mass, double dt, double h, double hg, double* q1, double* p1,
                      int32_t* blow, double* s1, double* s2) {
  if (W < 0 || d < 1 || L < 1) return fail(PL_EARG, "need W >= 0, d >= 1, L >= 1");
  if (pot->dim && pot->dim != d)
    return fail(PL_EARG, "potential expects dimension " + std::to_string(pot->dim) + ", got " +
                             std::to_string(d));
  if (W == 0) return PL_OK;
  cudaStream_t st = ctx->stream;
  // amplitudes -> device (pinned-free small copy through the context scratch)
  // speculative windows (ctx->spec, second stream) use their own scratch slots
  pl::Scratch& w_amp = ctx->work[ctx->spec ? 8 : 1];
  pl::Scratch& w_grad = ctx->work[ctx->spec ? 9 : 2];
  PL_TRY(w_amp.reserve(sizeof(double) * (L + 1)));
  double* amp = (double*)w_amp.ptr;
  PL_CUDA(cudaMemcpyAsync(amp, h_amp, sizeof(double) * (L + 1), cudaMemcpyHostToDevice, st));
  PL_CUDA(cudaMemsetAsync(blow, 0, sizeof(int32_t) * W, st));
  StepConsts K{dt, h, hg, L};

  if (is_elementwise(pot)) {
    EwProg P;
    PL_TRY(ew_program(pot, &P));
    k_window_ew<<<grid_for(W * d), 256, 0, st>>>(P, W, d, K, amp, q0, p0, noise, mass, q1, p1, blow, s1, s2);
    PL_CHECK_LAUNCH();
    // the amplitude upload is ordered on the stream, but h_amp is pageable:
    // cudaMemcpyAsync from pageable memory is synchronous w.r.t. the host.
    return PL_OK;
  }
  if (pot->kind == POT_LJ && pot->n_atoms * pot->space_dim <= 16 * 256) {
    PL_TRY(pot->work[7].reserve(16));
    int* flag = (int*)pot->work[7].ptr;
    PL_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    size_t smem = sizeof(double) * 2 * d;
    if (smem > 200 * 1024) return fail(PL_EARG, "LJ cluster too large for one CTA");
#define LJ_CASE(DD)                                                                          \
  case DD:                                                                                   \
    cudaFuncSetAttribute(k_window_lj<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    k_window_lj<DD><<<(unsigned)W, 256, smem, st>>>(W, pot->n_atoms, pot->eps, pot->sigma, K, amp, \
                                                   q0, p0, noise, mass, q1, p1, blow, flag, s1, s2); \
    break;
    switch (pot->space_dim) {
      LJ_CASE(1)
      LJ_CASE(2)
      LJ_CASE(3)
      default:
        return fail(PL_EARG, "LJ space_dim must be 1, 2 or 3 on the device");
    }
#undef LJ_CASE
    PL_CHECK_LAUNCH();
    return lj_check(pot);
  }

  // generic: batched force pipeline per substep; SNAP keeps Verlet-skin lists over
  // the window's substeps, rebuilt from the window's start state (so a window's
  // result is a function of its start state alone)
  struct SkinScope {
    pl_pot* p;
    SkinScope(pl_pot* p_) : p(p_) {
      if (p && p->kind == POT_SNAP) {
        p->skin_on = true;
        p->skin_force = true;
      }
    }
    ~SkinScope() {
      if (p) p->skin_on = false;
    }
  } skin_scope(pot);
  size_t nd = (size_t)W * d;
  PL_TRY(w_grad.reserve(sizeof(double) * 2 * nd));
  double* grad = (double*)w_grad.ptr;
  double* ph = grad + nd;
  if (q1 != q0) PL_CUDA(cudaMemcpyAsync(q1, q0, sizeof(double) * nd, cudaMemcpyDeviceToDevice, st));
  if (p1 != p0) PL_CUDA(cudaMemcpyAsync(p1, p0, sizeof(double) * nd, cudaMemcpyDeviceToDevice, st));
  PL_TRY(compute(pot, W, d, q1, nullptr, grad, nullptr));
  unsigned g = grid_for((int64_t)nd);
  prof_mark(st, ST_INT, true);
  PL_CUDA(launch_pdl(k_open, dim3(g), dim3(256), 0, st, W, d, 1, true, K, amp, noise, mass, grad, p1, ph, q1));
  PL_CHECK_LAUNCH();
  prof_mark(st, ST_INT, false);
  for (int s = 1; s <= L; ++s) {
    PL_TRY(compute(pot, W, d, q1, nullptr, grad, nullptr));
    prof_mark(st, ST_INT, true);
    if (s < L)
      PL_CUDA(launch_pdl(k_close_open, dim3(g), dim3(256), 0, st, W, d, s, K, amp, noise, mass, grad, ph, q1, p1,
                         blow, s1, s2));
    else
      PL_CUDA(launch_pdl(k_close, dim3(g), dim3(256), 0, st, W, d, s, K, amp, noise, mass, grad, ph, q1, p1, blow,
                         s1, s2));
    PL_CHECK_LAUNCH();
    prof_mark(st, ST_INT, false);
  }
  if (pot->kind == POT_LJ) return lj_check(pot);
  return neigh_check(pot);
}

}  // namespace pl
