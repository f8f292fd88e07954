// Persistent single-CTA coarse sweep (parareal.py:289-299, 195-198, 404-405, 425-445).
//
// The corrected sweep is the sequential critical path of parareal: window m
// needs cur[m], produced by window m-1.  For the small systems of the
// BASELINE configs (129 / 1025 atoms) one CTA holds the whole state in shared
// memory and runs every window of the sweep -- L BBK substeps each, EAM (or
// elementwise) forces, the corrected update, the running relative error and
// the adaptive truncation test -- in ONE launch.  Per substep there is no
// kernel boundary, only __syncthreads.
//
// Modes: 0 = corrected sweep (cur[m+1] = C(cur[m]) + jump[m]); 1 = coarse
// bootstrap (cur[m+1] = C(cur[m]) exactly).  Both cache base[m] = C(cur[m]).
// Integrator arithmetic = integrator.cu (explicit round-to-nearest, numpy
// order); EAM sums in neighbour order; every reduction in a fixed tree:
// the sweep is bitwise deterministic.
#include <cstdlib>

#include "eam.cuh"
#include "neigh.cuh"
#include "pl_common.cuh"
#include "toy.cuh"

namespace pl {

constexpr int SW_THREADS = 1024;
constexpr int SW_MAXN = 128;      // Verlet candidates per atom (rc + skin)
constexpr double SW_SKIN = 0.4;   // Angstrom

struct SweepArgs {
  int64_t d;
  int n_atoms, L, mode, include_m0, tpa, use_ew;
  int64_t m0, m1;
  double* Q;
  double* P;
  const double* prevQ;
  double* baseQ;
  double* baseP;
  const double* jumpQ;
  const double* jumpP;
  const double* noise;
  const double* amp;
  const double* mass;
  double dt, h, hg, expl;
  double* acc;    // {num, den}
  double* hist;   // running error after each node
  int64_t* out;   // {nodes done, fail window, fail substep, fail kind (1 blow-up, 2 non-finite)}
  // EAM
  Box box;
  double rc2, rl2;  // cutoff^2, (cutoff + skin)^2
  Table rho, phi, F;
  int32_t* cand;    // [n_atoms][SW_MAXN] Verlet candidates (rc + skin)
  int32_t* ncand;   // [n_atoms]
  double4* geo;     // [slots][n_atoms][SW_MAXN] pair geometry cache
  int* overflow;
  // elementwise
  EwProg ew;
  // replica batch (grid = slots): per-slot replica index and slab, NULL for a single run
  const int32_t* b_ridx;
  const int64_t* b_m0;
  const int64_t* b_m1;
  const int32_t* b_inc;
  int64_t s_traj, s_win, s_noise, s_hist;  // per-replica strides (elements)
};

__device__ __forceinline__ double block_sum(double v, double* red) {
  // fixed-order: warp xor-tree, then warp 0 over the 32 warp sums
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    r = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    for (int off = 16; off > 0; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
    if (lane == 0) red[32] = r;
  }
  __syncthreads();
  r = red[32];
  __syncthreads();
  return r;
}

struct Slot {  // per-CTA (replica slot) view of the arrays, kept in registers
  double* Q;
  double* P;
  const double* prevQ;
  double* baseQ;
  double* baseP;
  const double* jumpQ;
  const double* jumpP;
  const double* noise;
  double* hist;
  double* acc;
  int64_t* out;
  int64_t m0, m1;
  int include_m0;
  int32_t* cand;
  int32_t* ncand;
  int32_t* nbr;   // exact list of the current step (compacted candidates)
  int32_t* nnbr;
  double4* geo;   // cached (dx, dy, dz, r) of the exact-list pairs
};

// Verlet candidate lists (ascending j, rc + skin) of the current positions
__device__ void sw_build(const SweepArgs& A, const Slot& S, const double* q, double* qref) {
  const int n = A.n_atoms;
  // one warp per atom, lanes over j, ballot compaction in ascending j (the
  // lists of a serial scan, with a 32x shorter dependent chain)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int i = warp; i < n; i += nwarps) {
    const double xi = q[3 * i], yi = q[3 * i + 1], zi = q[3 * i + 2];
    int c = 0;
    int32_t* my = S.cand + (int64_t)i * SW_MAXN;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      bool hit = false;
      if (j < n && j != i) {
        const double dx = min_image(sub(q[3 * j], xi), A.box.L[0], A.box.inv[0]);
        const double dy = min_image(sub(q[3 * j + 1], yi), A.box.L[1], A.box.inv[1]);
        const double dz = min_image(sub(q[3 * j + 2], zi), A.box.L[2], A.box.inv[2]);
        hit = r2_exact(dx, dy, dz) < A.rl2;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const int pos = c + __popc(bal & ((1u << lane) - 1u));
        if (pos < SW_MAXN) my[pos] = j;
      }
      c += __popc(bal);
    }
    if (lane == 0) {
      S.ncand[i] = c < SW_MAXN ? c : SW_MAXN;
      if (c > SW_MAXN) *A.overflow = 1;
    }
  }
  for (int t = threadIdx.x; t < 3 * n; t += blockDim.x) qref[t] = q[t];
}

// EAM gradient of the CTA's system into g: tpa lanes per atom over the Verlet
// candidates (r < rc filter inside); the j % tpa lane partition and the
// xor-tree equal k_eam_density / k_eam_force on exact lists, so the gradient
// is bitwise the batched one
__device__ void sw_eam(const SweepArgs& A, const Slot& S, const double* q, double* g, double* fp, double* qref,
                       bool force_rebuild) {
  const int n = A.n_atoms;
  int moved = 0;
  if (!force_rebuild) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double dx = q[3 * i] - qref[3 * i], dy = q[3 * i + 1] - qref[3 * i + 1];
      const double dz = q[3 * i + 2] - qref[3 * i + 2];
      if (!(dx * dx + dy * dy + dz * dz <= 0.25 * SW_SKIN * SW_SKIN)) moved = 1;
    }
  }
  if (__syncthreads_or(moved) || force_rebuild) {
    sw_build(A, S, q, qref);
    __syncthreads();
  }
  // exact list of this step: tpa lanes per atom filter the candidates in
  // chunks, ballots keep the ascending-j order, and the pair geometry of every
  // kept pair is cached for both passes
  const int tpa = A.tpa;
  const int groups = blockDim.x / tpa;
  const int gi0 = threadIdx.x / tpa, sub = threadIdx.x % tpa;
  const int lane = threadIdx.x & 31;
  const unsigned gmask = (tpa == 32 ? 0xffffffffu : ((1u << tpa) - 1u)) << (lane & ~(tpa - 1));
  for (int base = 0; base < n; base += groups) {
    const int i = base + gi0;
    const bool live = i < n;
    const int nc = live ? S.ncand[i] : 0;
    const int32_t* cl = S.cand + (int64_t)(live ? i : 0) * SW_MAXN;
    int32_t* el = S.nbr + (int64_t)(live ? i : 0) * SW_MAXN;
    double4* geo = S.geo + (int64_t)(live ? i : 0) * SW_MAXN;
    int c = 0;
    for (int k0 = 0; k0 < SW_MAXN; k0 += tpa) {
      const int k = k0 + sub;
      bool keep = false;
      double dx = 0.0, dy = 0.0, dz = 0.0, r2 = 0.0;
      int j = 0;
      if (k < nc) {
        j = cl[k];
        pair_vec(q, i, j, A.box, dx, dy, dz);
        r2 = r2_exact(dx, dy, dz);
        keep = r2 < A.rc2;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep) & gmask;
      if (keep) {
        const int pos = c + __popc(bal & ((1u << lane) - 1u));
        el[pos] = j;
        geo[pos] = make_double4(dx, dy, dz, __dsqrt_rn(r2));
      }
      c += __popc(bal);
      if (!__any_sync(0xffffffffu, k0 + tpa < nc)) break;
    }
    if (live && sub == 0) S.nnbr[i] = c;
  }
  __syncthreads();
  for (int base = 0; base < n; base += groups) {
    const int i = base + gi0;
    const bool live = i < n;
    const int ii = live ? i : 0;
    const double s = group_sum(eam_rho_part(q, ii, S.nbr + (int64_t)ii * SW_MAXN, live ? S.nnbr[ii] : 0, sub, tpa,
                                            A.box, A.rc2, A.rho, S.geo + (int64_t)ii * SW_MAXN), tpa);
    if (live && sub == 0) {
      double f, df;
      tab_eval(A.F, s, f, df);
      fp[i] = df;
    }
  }
  __syncthreads();
  for (int base = 0; base < n; base += groups) {
    const int i = base + gi0;
    const bool live = i < n;
    const int ii = live ? i : 0;
    double gg[3] = {0.0, 0.0, 0.0}, e = 0.0, v[6];
    eam_force_part<false>(q, fp, ii, S.nbr + (int64_t)ii * SW_MAXN, live ? S.nnbr[ii] : 0, sub, tpa, A.box, A.rc2,
                          A.rho, A.phi, gg, &e, v, S.geo + (int64_t)ii * SW_MAXN);
    gg[0] = group_sum(gg[0], tpa);
    gg[1] = group_sum(gg[1], tpa);
    gg[2] = group_sum(gg[2], tpa);
    if (live && sub == 0) {
      g[3 * i] = gg[0];
      g[3 * i + 1] = gg[1];
      g[3 * i + 2] = gg[2];
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void sw_force(const SweepArgs& A, const Slot& S, const double* q, double* g,
                                         double* fp, double* qref, bool force_rebuild) {
  if (A.use_ew) {
    for (int64_t t = threadIdx.x; t < A.d; t += blockDim.x) g[t] = ew_grad(A.ew, q[t], t);
    __syncthreads();
  } else {
    sw_eam(A, S, q, g, fp, qref, force_rebuild);
  }
}

__global__ void __launch_bounds__(SW_THREADS) k_sweep_cta(const __grid_constant__ SweepArgs A) {
  extern __shared__ double sm[];
  Slot S{A.Q, A.P, A.prevQ, A.baseQ, A.baseP, A.jumpQ, A.jumpP, A.noise, A.hist, A.acc, A.out,
         A.m0, A.m1, A.include_m0, A.cand, A.ncand, A.cand, A.ncand, A.geo};
  if (A.b_ridx) {
    // replica slot: offset every per-replica array, take this slot's slab
    const int slot = blockIdx.x;
    const int64_t r = A.b_ridx[slot];
    S.Q += r * A.s_traj;
    S.P += r * A.s_traj;
    S.prevQ += r * A.s_traj;
    S.baseQ += r * A.s_win;
    S.baseP += r * A.s_win;
    S.jumpQ += r * A.s_win;
    S.jumpP += r * A.s_win;
    S.noise += r * A.s_noise;
    S.hist += r * A.s_hist;
    S.acc += 2 * slot;
    S.out += 4 * slot;
    S.m0 = A.b_m0[slot];
    S.m1 = A.b_m1[slot];
    S.include_m0 = A.b_inc[slot];
    if (!A.use_ew) {
      S.cand += (int64_t)slot * 2 * ((int64_t)A.n_atoms * (SW_MAXN + 1) + 8);
      S.geo += (int64_t)slot * A.n_atoms * SW_MAXN;
    }
  }
  if (!A.use_ew) {
    // per slot: [candidates][counts][exact list][counts]
    S.ncand = S.cand + (int64_t)A.n_atoms * SW_MAXN;
    S.nbr = S.ncand + A.n_atoms + 8;
    S.nnbr = S.nbr + (int64_t)A.n_atoms * SW_MAXN;
  }
  const int64_t d = A.d;
  double* q = sm;
  double* p = q + d;
  double* ph = p + d;
  double* g = ph + d;
  double* fp = g + d;  // n doubles (EAM)
  double* qref = fp + (A.use_ew ? 0 : A.n_atoms);
  __shared__ double red[33];
  __shared__ int s_fail;
  __shared__ double s_num, s_den;
  if (threadIdx.x == 0) {
    s_num = S.acc[0];
    s_den = S.acc[1];
    S.out[0] = 0;
    S.out[1] = -1;
    S.out[2] = 0;
    S.out[3] = 0;
  }
  const int64_t m0 = S.m0;
  for (int64_t t = threadIdx.x; t < d; t += blockDim.x) {
    q[t] = S.Q[m0 * d + t];
    p[t] = S.P[m0 * d + t];
  }
  __syncthreads();
  if (S.include_m0) {
    double s2 = 0.0;
    for (int64_t t = threadIdx.x; t < d; t += blockDim.x) s2 += q[t] * q[t];
    const double tot = block_sum(s2, red);
    if (threadIdx.x == 0) s_den += sqrt(tot);  // num += ||q - q|| = 0
  }
  const double h = A.h, hg = A.hg, dt = A.dt;
  const double* mass = A.mass;
  const int L = A.L;
  int64_t done = 0;
  for (int64_t m = m0; m < S.m1; ++m) {
    const double* G = S.noise + m * (int64_t)(L + 1) * d;
    if (threadIdx.x == 0) s_fail = 0;
    sw_force(A, S, q, g, fp, qref, true);
    for (int s = 1; s <= L; ++s) {
      // open substep s (integrator.py:174-175, 182-183)
      for (int64_t t = threadIdx.x; t < d; t += blockDim.x) {
        const double mm = mass ? mass[t] : 1.0;
        const double smm = mass ? __dsqrt_rn(mm) : 1.0;
        const double al = mul(A.amp[s - 1], smm);
        const double pref = (s == 1) ? p[t] : ph[t];
        const double hv = add(sub(sub(p[t], mul(h, g[t])), mul(hg, pref)), mul(al, G[(int64_t)(s - 1) * d + t]));
        ph[t] = hv;
        q[t] = add(q[t], mul(dt, dvd(hv, mm)));
      }
      __syncthreads();
      sw_force(A, S, q, g, fp, qref, false);
      // close substep s (integrator.py:177, 185) + blow-up check (163-170)
      int bad = 0;
      for (int64_t t = threadIdx.x; t < d; t += blockDim.x) {
        const double smm = mass ? __dsqrt_rn(mass[t]) : 1.0;
        const double al = mul(A.amp[s], smm);
        const double hv = ph[t];
        const double pn = add(sub(sub(hv, mul(h, g[t])), mul(hg, hv)), mul(al, G[(int64_t)s * d + t]));
        p[t] = pn;
        if (!(fabs(q[t]) <= BLOWUP_LIMIT && fabs(pn) <= BLOWUP_LIMIT)) bad = 1;
      }
      if (__syncthreads_or(bad) && threadIdx.x == 0 && s_fail == 0) s_fail = s;
    }
    __syncthreads();
    // base[m] = C(cur[m])
    for (int64_t t = threadIdx.x; t < d; t += blockDim.x) {
      S.baseQ[m * d + t] = q[t];
      S.baseP[m * d + t] = p[t];
    }
    if (s_fail) {
      if (threadIdx.x == 0) {
        S.out[1] = m;
        S.out[2] = s_fail;
        S.out[3] = 1;
      }
      break;
    }
    if (A.mode == 1) {
      for (int64_t t = threadIdx.x; t < d; t += blockDim.x) {
        S.Q[(m + 1) * d + t] = q[t];
        S.P[(m + 1) * d + t] = p[t];
      }
      ++done;
      continue;
    }
    // corrected value base + jump (jump formed first, parareal.py:293) and the
    // running relative error (parareal.py:196-197)
    double e1 = 0.0, e2 = 0.0;
    int nonfinite = 0;
    for (int64_t t = threadIdx.x; t < d; t += blockDim.x) {
      // prev[m+1] is read before cur[m+1] overwrites it (prevQ may alias Q)
      const double pv = S.prevQ[(m + 1) * d + t];
      const double cq = add(q[t], S.jumpQ[m * d + t]);
      const double cp = add(p[t], S.jumpP[m * d + t]);
      S.Q[(m + 1) * d + t] = cq;
      S.P[(m + 1) * d + t] = cp;
      q[t] = cq;
      p[t] = cp;
      if (!isfinite(cq) || !isfinite(cp)) nonfinite = 1;
      const double e = sub(cq, pv);
      e1 += e * e;
      e2 += pv * pv;
    }
    nonfinite = __syncthreads_or(nonfinite);
    const double n1 = sqrt(block_sum(e1, red));
    const double n2 = sqrt(block_sum(e2, red));
    ++done;
    bool stop = false;
    if (threadIdx.x == 0) {
      s_num = s_num + n1;
      s_den = s_den + n2;
      S.hist[m - m0] = s_num / s_den;
    }
    __syncthreads();
    if (nonfinite) {
      if (threadIdx.x == 0) {
        S.out[1] = m;
        S.out[3] = 2;
      }
      break;
    }
    if (s_den == 0.0) stop = true;
    else if (A.expl > 0.0 && s_num / s_den > A.expl) stop = true;
    if (stop) break;
  }
  if (threadIdx.x == 0) {
    S.acc[0] = s_num;
    S.acc[1] = s_den;
    S.out[0] = done;
  }
}

int ew_program(const pl_pot* p, EwProg* out);

// returns PL_OK if handled, -1 if this coarse potential needs the generic path
int sweep_cta(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t m0, int64_t m1, int include_m0,
              int mode, double* Q, double* P, const double* prevQ, double* baseQ, double* baseP,
              const double* jumpQ, const double* jumpP, const double* noise, const double* h_amp,
              const double* mass, double dt, double h, double hg, double expl, double* h_state,
              int64_t* h_out4, double* d_hist) {
  SweepArgs A{};
  const bool ew = is_elementwise(coarse);
  if (!ew && coarse->kind != POT_EAM) return -1;
  const int n = ew ? 0 : coarse->n_atoms;
  const size_t smem = sizeof(double) * (4 * (size_t)d + (ew ? 0 : (size_t)n + 3 * (size_t)n));
  if (smem > 200 * 1024) return -1;
  A.d = d;
  A.n_atoms = n;
  A.L = L;
  A.mode = mode;
  A.include_m0 = include_m0;
  A.use_ew = ew ? 1 : 0;
  A.m0 = m0;
  A.m1 = m1;
  A.Q = Q; A.P = P; A.prevQ = prevQ; A.baseQ = baseQ; A.baseP = baseP; A.jumpQ = jumpQ; A.jumpP = jumpP;
  A.noise = noise;
  A.mass = mass;
  A.dt = dt; A.h = h; A.hg = hg; A.expl = expl;
  cudaStream_t st = ctx->stream;
  // device scratch: amp, acc, out, (EAM lists)
  size_t lists = ew ? 0 : 2 * sizeof(int32_t) * ((size_t)n * (SW_MAXN + 1) + 8) + 128;
  PL_TRY(ctx->work[4].reserve(sizeof(double) * (L + 1 + 2) + sizeof(int64_t) * 4 + 64 + lists));
  char* w = (char*)ctx->work[4].ptr;
  double* amp = (double*)w;
  double* acc = amp + (L + 1);
  int64_t* out = (int64_t*)(acc + 2);
  char* lw = (char*)(out + 4);
  A.amp = amp;
  A.acc = acc;
  A.out = out;
  A.hist = d_hist;
  if (ew) {
    PL_TRY(ew_program(coarse, &A.ew));
  } else {
    A.box = make_box(coarse->box);
    A.rc2 = coarse->rcut * coarse->rcut;
    A.rl2 = (coarse->rcut + SW_SKIN) * (coarse->rcut + SW_SKIN);
    A.rho = Table{coarse->d_rho, coarse->n_r, coarse->dr, 1.0 / coarse->dr};
    A.phi = Table{coarse->d_phi, coarse->n_r, coarse->dr, 1.0 / coarse->dr};
    A.F = Table{coarse->d_F, coarse->n_rho, coarse->drho, 1.0 / coarse->drho};
    // scratch: [overflow flag][pad][candidates n x SW_MAXN][counts n]
    A.overflow = (int*)lw;
    A.cand = (int32_t*)(((uintptr_t)(A.overflow + 4) + 15) & ~(uintptr_t)15);
    A.ncand = A.cand + (size_t)n * SW_MAXN;
    A.tpa = eam_tpa(n, SW_THREADS);
    PL_TRY(ctx->work[7].reserve(sizeof(double4) * (size_t)n * SW_MAXN));
    A.geo = (double4*)ctx->work[7].ptr;
    PL_CUDA(cudaMemsetAsync(A.overflow, 0, sizeof(int), st));
  }
  double init[2] = {h_state[0], h_state[1]};
  PL_CUDA(cudaMemcpyAsync(amp, h_amp, sizeof(double) * (L + 1), cudaMemcpyHostToDevice, st));
  PL_CUDA(cudaMemcpyAsync(acc, init, sizeof(init), cudaMemcpyHostToDevice, st));
  static std::atomic<uint64_t> attr_devs{0};
  if (first_on_device(attr_devs)) {
    cudaFuncSetAttribute(k_sweep_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  k_sweep_cta<<<1, SW_THREADS, smem, st>>>(A);
  PL_CHECK_LAUNCH();
  double hacc[2];
  int ovf = 0;
  PL_CUDA(cudaMemcpyAsync(hacc, acc, sizeof(hacc), cudaMemcpyDeviceToHost, st));
  PL_CUDA(cudaMemcpyAsync(h_out4, out, sizeof(int64_t) * 4, cudaMemcpyDeviceToHost, st));
  if (!ew) PL_CUDA(cudaMemcpyAsync(&ovf, A.overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
  PL_CUDA(cudaStreamSynchronize(st));
  if (ovf) return fail(PL_EPOT, "neighbour capacity exceeded in the coarse sweep");
  h_state[0] = hacc[0];
  h_state[1] = hacc[1];
  return PL_OK;
}

int sweep_cluster_batch(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t N, int R_act, const int32_t* h_ridx,
                        const int64_t* h_m0, const int64_t* h_m1, const int32_t* h_inc, int mode, double* Q,
                        double* P, double* baseQ, double* baseP, const double* jumpQ, const double* jumpP,
                        const double* noise, const double* h_amp, const double* mass, double dt, double h,
                        double hg, double expl, double* h_state, int64_t* h_out4, double* d_hist);

int sweep_generic_batch(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t N, int R_act, const int32_t* h_ridx,
                        const int64_t* h_m0, const int64_t* h_m1, const int32_t* h_inc, int mode, double* Q,
                        double* P, double* baseQ, double* baseP, const double* jumpQ, const double* jumpP,
                        const double* noise, const double* h_amp, const double* mass, double dt, double h, double hg,
                        double expl, double* h_state, int64_t* h_out4, double* d_hist);

// R_act replica slots in one launch (grid = R_act CTAs); arrays carry a leading
// replica dimension: Q/P (R, N+1, d), base/jump (R, N, d), noise (R, N, L+1, d),
// d_hist (R, N).  h_state (2 R_act) and h_out4 (4 R_act) per slot.
int sweep_cta_batch(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t N, int R_act, const int32_t* h_ridx,
                    const int64_t* h_m0, const int64_t* h_m1, const int32_t* h_inc, int mode, double* Q, double* P,
                    double* baseQ, double* baseP, const double* jumpQ, const double* jumpP, const double* noise,
                    const double* h_amp, const double* mass, double dt, double h, double hg, double expl,
                    double* h_state, int64_t* h_out4, double* d_hist) {
  if (R_act <= 0) return PL_OK;
  if (!getenv("PL_SWEEP_NOCLUSTER")) {
    const int rc = sweep_cluster_batch(ctx, coarse, d, L, N, R_act, h_ridx, h_m0, h_m1, h_inc, mode, Q, P, baseQ,
                                       baseP, jumpQ, jumpP, noise, h_amp, mass, dt, h, hg, expl, h_state, h_out4,
                                       d_hist);
    if (rc != -1) return rc;
  }
  SweepArgs A{};
  const bool ew = is_elementwise(coarse);
  if (!ew && coarse->kind != POT_EAM) return fail(PL_EARG, "batched sweep needs an EAM or elementwise coarse potential");
  const int n = ew ? 0 : coarse->n_atoms;
  const size_t smem = sizeof(double) * (4 * (size_t)d + (ew ? 0 : (size_t)n + 3 * (size_t)n));
  if (smem > 200 * 1024)  // positions do not fit one CTA: per-window generic path, replica by replica
    return sweep_generic_batch(ctx, coarse, d, L, N, R_act, h_ridx, h_m0, h_m1, h_inc, mode, Q, P, baseQ, baseP,
                               jumpQ, jumpP, noise, h_amp, mass, dt, h, hg, expl, h_state, h_out4, d_hist);
  A.d = d; A.n_atoms = n; A.L = L; A.mode = mode; A.use_ew = ew ? 1 : 0;
  A.Q = Q; A.P = P; A.prevQ = Q; A.baseQ = baseQ; A.baseP = baseP; A.jumpQ = jumpQ; A.jumpP = jumpP;
  A.noise = noise; A.mass = mass; A.dt = dt; A.h = h; A.hg = hg; A.expl = expl;
  A.s_traj = (N + 1) * d;
  A.s_win = N * d;
  A.s_noise = N * (int64_t)(L + 1) * d;
  A.s_hist = N;
  cudaStream_t st = ctx->stream;
  const size_t per_slot_lists = ew ? 0 : 2 * sizeof(int32_t) * ((size_t)n * (SW_MAXN + 1) + 8);
  const size_t hdr = sizeof(double) * (L + 1) + sizeof(double) * 2 * R_act + sizeof(int64_t) * 4 * R_act +
                     sizeof(int64_t) * 2 * R_act + sizeof(int32_t) * 2 * R_act + 256;
  PL_TRY(ctx->work[4].reserve(hdr + per_slot_lists * R_act + 256));
  char* w = (char*)ctx->work[4].ptr;
  double* amp = (double*)w;
  double* acc = amp + (L + 1);
  int64_t* out = (int64_t*)(acc + 2 * R_act);
  int64_t* m0 = out + 4 * R_act;
  int64_t* m1 = m0 + R_act;
  int32_t* ridx = (int32_t*)(m1 + R_act);
  int32_t* inc = ridx + R_act;
  int* ovf = (int*)(inc + R_act);
  char* lists = (char*)(((uintptr_t)(ovf + 4) + 255) & ~(uintptr_t)255);
  A.amp = amp; A.acc = acc; A.out = out; A.hist = d_hist;
  A.b_ridx = ridx; A.b_m0 = m0; A.b_m1 = m1; A.b_inc = inc;
  if (ew) {
    PL_TRY(ew_program(coarse, &A.ew));
  } else {
    A.box = make_box(coarse->box);
    A.rc2 = coarse->rcut * coarse->rcut;
    A.rl2 = (coarse->rcut + SW_SKIN) * (coarse->rcut + SW_SKIN);
    A.rho = Table{coarse->d_rho, coarse->n_r, coarse->dr, 1.0 / coarse->dr};
    A.phi = Table{coarse->d_phi, coarse->n_r, coarse->dr, 1.0 / coarse->dr};
    A.F = Table{coarse->d_F, coarse->n_rho, coarse->drho, 1.0 / coarse->drho};
    A.cand = (int32_t*)lists;
    A.ncand = A.cand + (size_t)n * SW_MAXN;  // slot 0; the kernel offsets per slot
    A.overflow = ovf;
    A.tpa = eam_tpa(n, SW_THREADS);
    PL_TRY(ctx->work[7].reserve(sizeof(double4) * (size_t)n * SW_MAXN * R_act));
    A.geo = (double4*)ctx->work[7].ptr;
    PL_CUDA(cudaMemsetAsync(ovf, 0, sizeof(int), st));
  }
  PL_CUDA(cudaMemcpyAsync(amp, h_amp, sizeof(double) * (L + 1), cudaMemcpyHostToDevice, st));
  PL_CUDA(cudaMemcpyAsync(acc, h_state, sizeof(double) * 2 * R_act, cudaMemcpyHostToDevice, st));
  PL_CUDA(cudaMemcpyAsync(m0, h_m0, sizeof(int64_t) * R_act, cudaMemcpyHostToDevice, st));
  PL_CUDA(cudaMemcpyAsync(m1, h_m1, sizeof(int64_t) * R_act, cudaMemcpyHostToDevice, st));
  PL_CUDA(cudaMemcpyAsync(ridx, h_ridx, sizeof(int32_t) * R_act, cudaMemcpyHostToDevice, st));
  PL_CUDA(cudaMemcpyAsync(inc, h_inc, sizeof(int32_t) * R_act, cudaMemcpyHostToDevice, st));
  static std::atomic<uint64_t> attr_devs{0};
  if (first_on_device(attr_devs)) {
    cudaFuncSetAttribute(k_sweep_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  k_sweep_cta<<<R_act, SW_THREADS, smem, st>>>(A);
  PL_CHECK_LAUNCH();
  int hovf = 0;
  PL_CUDA(cudaMemcpyAsync(h_state, acc, sizeof(double) * 2 * R_act, cudaMemcpyDeviceToHost, st));
  PL_CUDA(cudaMemcpyAsync(h_out4, out, sizeof(int64_t) * 4 * R_act, cudaMemcpyDeviceToHost, st));
  if (!ew) PL_CUDA(cudaMemcpyAsync(&hovf, ovf, sizeof(int), cudaMemcpyDeviceToHost, st));
  PL_CUDA(cudaStreamSynchronize(st));
  if (hovf) return fail(PL_EPOT, "neighbour capacity exceeded in the coarse sweep");
  return PL_OK;
}

}  // namespace pl

extern "C" int pl_sweep_batch(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t N, int R_act,
                              const int32_t* h_ridx, const int64_t* h_m0, const int64_t* h_m1,
                              const int32_t* h_include_m0, int mode, double* d_Q, double* d_P, double* d_baseQ,
                              double* d_baseP, const double* d_jumpQ, const double* d_jumpP,
                              const double* d_noise, const double* h_amp, const double* d_mass, double dt,
                              double half_dt, double half_dt_gamma, double expl, double* h_state,
                              int64_t* h_out4, double* d_hist) {
  if (!ctx || !coarse || !h_ridx || !h_m0 || !h_m1 || !h_include_m0 || !d_Q || !d_P || !d_baseQ || !d_baseP ||
      !d_noise || !h_amp || !h_state || !h_out4 || !d_hist)
    return pl::fail(PL_EARG, "NULL argument");
  if (mode == 0 && (!d_jumpQ || !d_jumpP)) return pl::fail(PL_EARG, "NULL jumps");
  return pl::sweep_cta_batch(ctx, coarse, d, L, N, R_act, h_ridx, h_m0, h_m1, h_include_m0, mode, d_Q, d_P,
                             d_baseQ, d_baseP, mode == 0 ? d_jumpQ : d_baseQ, mode == 0 ? d_jumpP : d_baseP,
                             d_noise, h_amp, d_mass, dt, half_dt, half_dt_gamma, expl, h_state, h_out4, d_hist);
}
