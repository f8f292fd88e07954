// Cluster-parallel persistent coarse sweep (EAM), one thread-block cluster per
// replica slot.
//
// The single-CTA sweep (sweep_cta.cu) is latency bound: one SM walks every
// pair of every atom through global-memory lists each substep.  Here the
// system's atoms are split over C CTAs of one cluster (C <= 16, one SM each):
//   * every CTA keeps the full positions q and embedding derivatives F' in
//     shared memory and updates its own atom slice; slices are pushed to the
//     peers through distributed shared memory, then cluster.sync() (two per
//     substep: after the position update, after the density pass);
//   * Verlet candidates, the exact per-step list and the pair distances of the
//     own atoms live in shared memory;
//   * running-error partial sums, blow-up and rebuild flags are reduced over
//     the cluster in rank order, so every CTA takes the same decision.
// The per-atom arithmetic is the batched EAM path's (eam.cuh, same threads per
// atom, same lane partition): coarse windows are bitwise those of
// k_eam_density / k_eam_force + k_open / k_close.
#include <cooperative_groups.h>
#include <stdlib.h>

#include <algorithm>


#include "eam.cuh"
#include "neigh.cuh"
#include "pl_common.cuh"

namespace cg = cooperative_groups;

namespace pl {

constexpr int CL_THREADS = 1024;
constexpr int CL_MAXC = 128;   // Verlet candidates per atom (rc + skin)
constexpr int CL_MAXN = 80;    // exact neighbours per atom
constexpr double CL_SKIN = 0.4;

// cluster size and threads per atom of an n-atom system (also used by the
// batched EAM kernels so both paths share the lane partition)
static int cluster_own_max() {  // atoms per CTA before the cluster grows (env PL_SWEEP_OWN, default 32: 15.0 vs 17.2 us per substep at 129 atoms)
  static const int v = [] {
    const char* e = getenv("PL_SWEEP_OWN");
    const int x = e ? atoi(e) : 32;
    return x < 8 ? 8 : x;
  }();
  return v;
}

inline void cluster_layout(int n, int& C, int& tpa) {
  const int own_max = cluster_own_max();
  C = 1;
  while (C < 16 && (n + C - 1) / C > own_max) C *= 2;
  const int own = (n + C - 1) / C;
  tpa = 1;
  while (tpa < 32 && own * tpa * 2 <= CL_THREADS) tpa *= 2;
}

struct ClArgs {
  int64_t d;
  int n_atoms, L, mode, C, tpa;
  int cache;  // table derivatives cached by the density pass: 0 none, 1 drho/dr, 2 drho/dr and dphi/dr
  double* Q;
  double* P;
  double* baseQ;
  double* baseP;
  const double* jumpQ;
  const double* jumpP;
  const double* noise;
  const double* amp;
  const double* mass;
  double dt, h, hg, expl;
  double* acc;    // 2 per slot
  double* hist;
  int64_t* out;   // 4 per slot
  Box box;
  double rc2, rl2;
  Table rho, phi, F;
  const int32_t* b_ridx;
  const int64_t* b_m0;
  const int64_t* b_m1;
  const int32_t* b_inc;
  int64_t s_traj, s_win, s_noise, s_hist;
  int* overflow;
  int64_t* progress;  // host-mapped: windows finished (single-slot sweeps), or null
};

struct ClSmem {  // carve-up of the dynamic shared memory of one CTA
  double* q;       // 3n full positions (two buffers: substeps alternate)
  double* q2;
  double* fp;      // n full F'
  double* p;       // own momenta
  double* ph;      // own half-step momenta
  double* g;       // own gradient
  double* qref;    // own positions at the last list build
  double* rr;      // own exact-pair distances [own][CL_MAXN]
  double* drf;     // d rho/dr of the exact pairs [own][CL_MAXN] (cache >= 1)
  double* dpf;     // d phi/dr of the exact pairs [own][CL_MAXN] (cache == 2)
  int32_t* cand;   // [own][CL_MAXC]
  int32_t* ncand;  // [own]
  int32_t* nbr;    // [own][CL_MAXN]
  int32_t* nnbr;   // [own]
};

__host__ __device__ inline size_t cl_smem_bytes(int n, int own, int cache = 0) {
  return sizeof(double) * (6 * (size_t)n + n + 4 * 3 * (size_t)own + (size_t)(1 + cache) * own * CL_MAXN) +
         sizeof(int32_t) * ((size_t)own * CL_MAXC + own + (size_t)own * CL_MAXN + own) + 64;
}

// Distributed shared memory through its own state space: mapa gives the peer's
// shared::cluster address, st.shared::cluster writes it, and the cluster barrier
// (release / acquire at cluster scope) orders those stores.  Generic pointers from
// map_shared_rank made every exchange a generic store and the barrier a
// GPU-scope membar (MEMBAR.ALL.GPU + ERRBAR in the SASS).
__device__ __forceinline__ uint32_t dsmem_addr(const void* local, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((uint32_t)__cvta_generic_to_shared(local)), "r"(rank));
  return r;
}
__device__ __forceinline__ void dsmem_st(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// own slice [c0, c0 + cnt) of a shared array -> the same range of every peer:
// one (peer, element) item per thread, so only threads with work run
__device__ __forceinline__ void dsmem_push(const double* arr, int c0, int cnt, int C) {
  for (int t = threadIdx.x; t < C * cnt; t += blockDim.x) {
    const int pr = t / cnt, k = t - pr * cnt;
    dsmem_st(dsmem_addr(arr + c0 + k, pr), arr[c0 + k]);
  }
}

// fixed-order sum of one double per CTA over the cluster: every CTA pushes its
// value to slot [rank] of every peer, then sums slots 0..C-1
__device__ __forceinline__ double cluster_sum(cg::cluster_group& cl, double v, double* slots, int C, int rank) {
  if (threadIdx.x < (unsigned)C) dsmem_st(dsmem_addr(slots + rank, (int)threadIdx.x), v);
  cluster_barrier();
  double s = 0.0;
  for (int r = 0; r < C; ++r) s += slots[r];
  return s;
}

// MAXT: launch bound of the instantiation.  The CTA runs only the threads its
// atoms use (own x tpa, rounded to warps): the lane partition (tpa) is the
// 1024-thread rule shared with the batched EAM kernels, and the per-CTA error
// sums see the same per-thread terms (at most one component per thread) plus
// zeros, so every result is bitwise that of a 1024-thread CTA
template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_sweep_cluster(const __grid_constant__ ClArgs A) {
  extern __shared__ double sm[];
  __shared__ double red[33];
  __shared__ double slots_a[16], slots_b[16], slots_c[16];
  __shared__ int s_fail;
  cg::cluster_group cl = cg::this_cluster();
  const int C = A.C;
  const int rank = (int)cl.block_rank();
  const int slot = blockIdx.x / C;
  const int n = A.n_atoms;
  const int own = (n + C - 1) / C;
  const int a0 = min(n, rank * own), a1 = min(n, a0 + own), nown = a1 - a0;
  const int64_t d = A.d;
  const int c0 = 3 * a0, dn = 3 * nown;
  // per-slot arrays
  const int64_t r = A.b_ridx[slot];
  double* Q = A.Q + r * A.s_traj;
  double* P = A.P + r * A.s_traj;
  double* baseQ = A.baseQ + r * A.s_win;
  double* baseP = A.baseP + r * A.s_win;
  const double* jumpQ = A.jumpQ + r * A.s_win;
  const double* jumpP = A.jumpP + r * A.s_win;
  const double* noise = A.noise + r * A.s_noise;
  double* hist = A.hist + r * A.s_hist;
  const int64_t m0 = A.b_m0[slot], m1 = A.b_m1[slot];
  // shared memory carve-up
  ClSmem M;
  M.q = sm;
  M.q2 = M.q + 3 * n;
  M.fp = M.q2 + 3 * n;
  M.p = M.fp + n;
  M.ph = M.p + 3 * own;
  M.g = M.ph + 3 * own;
  M.qref = M.g + 3 * own;
  M.rr = M.qref + 3 * own;
  M.drf = M.rr + (size_t)own * CL_MAXN;
  M.dpf = M.drf + (A.cache >= 1 ? (size_t)own * CL_MAXN : 0);
  M.cand = reinterpret_cast<int32_t*>(M.dpf + (A.cache == 2 ? (size_t)own * CL_MAXN : 0));
  M.ncand = M.cand + (size_t)own * CL_MAXC;
  M.nbr = M.ncand + own;
  M.nnbr = M.nbr + (size_t)own * CL_MAXN;
  const int tpa = A.tpa;
  const int groups = blockDim.x / tpa;
  const int gi0 = threadIdx.x / tpa, sl = threadIdx.x % tpa;
  const int lane = threadIdx.x & 31;
  const unsigned gmask = (tpa == 32 ? 0xffffffffu : ((1u << tpa) - 1u)) << (lane & ~(tpa - 1));

  // positions of the current substep (q) and the buffer the next open writes
  // (qn): a peer still reading q in its force pass never sees our next slice,
  // so one cluster barrier per position exchange suffices
  double* q = M.q;
  double* qn = M.q2;
  auto push_q_slice = [&]() { dsmem_push(q, c0, dn, C); };  // own positions -> every peer's current buffer

  // ---------------------------------------------------------------- force
  auto eam_force = [&](bool any) {
    // rebuild (any CTA saw an atom move by more than half the skin): own atoms'
    // candidates from the full positions
    if (any) {
      // one warp per own atom, lanes over j: ballot compaction keeps ascending j,
      // so the candidate lists are the serial scan's (32x shorter chain; the
      // serial scan of n atoms by one thread per own atom held every other warp
      // at the barrier: ~half of the sweep's time at 1025 atoms)
      const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
      for (int i = warp; i < nown; i += nwarps) {
        const int ai = a0 + i;
        const double xi = q[3 * ai], yi = q[3 * ai + 1], zi = q[3 * ai + 2];
        int c = 0;
        int32_t* my = M.cand + (size_t)i * CL_MAXC;
        for (int j0 = 0; j0 < n; j0 += 32) {
          const int j = j0 + lane;
          bool hit = false;
          if (j < n && j != ai) {
            const double dx = min_image(sub(q[3 * j], xi), A.box.L[0], A.box.inv[0]);
            const double dy = min_image(sub(q[3 * j + 1], yi), A.box.L[1], A.box.inv[1]);
            const double dz = min_image(sub(q[3 * j + 2], zi), A.box.L[2], A.box.inv[2]);
            hit = r2_exact(dx, dy, dz) < A.rl2;
          }
          const unsigned bal = __ballot_sync(0xffffffffu, hit);
          if (hit) {
            const int pos = c + __popc(bal & ((1u << lane) - 1u));
            if (pos < CL_MAXC) my[pos] = j;
          }
          c += __popc(bal);
        }
        if (lane == 0) {
          M.ncand[i] = c < CL_MAXC ? c : CL_MAXC;
          if (c > CL_MAXC) *A.overflow = 1;
          M.qref[3 * i] = xi;
          M.qref[3 * i + 1] = yi;
          M.qref[3 * i + 2] = zi;
        }
      }
      __syncthreads();
    }
    // exact list + distances of this step (ballot-ordered, ascending j)
    for (int base = 0; base < nown; base += groups) {
      const int i = base + gi0;
      const bool live = i < nown;
      const int nc = live ? M.ncand[i] : 0;
      const int ii = live ? i : 0;
      const int ai = a0 + ii;
      int c = 0;
      for (int k0 = 0; k0 < CL_MAXC; k0 += tpa) {
        const int k = k0 + sl;
        bool keep = false;
        double r2 = 0.0;
        int j = 0;
        if (k < nc) {
          j = M.cand[(size_t)ii * CL_MAXC + k];
          double dx, dy, dz;
          pair_vec(q, ai, j, A.box, dx, dy, dz);
          r2 = r2_exact(dx, dy, dz);
          keep = r2 < A.rc2;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep) & gmask;
        if (keep) {
          const int pos = c + __popc(bal & ((1u << lane) - 1u));
          if (pos < CL_MAXN) {
            M.nbr[(size_t)ii * CL_MAXN + pos] = j;
            M.rr[(size_t)ii * CL_MAXN + pos] = __dsqrt_rn(r2);
          }
        }
        c += __popc(bal);
        if (!__any_sync(0xffffffffu, k0 + tpa < nc)) break;
      }
      if (live && sl == 0) {
        M.nnbr[i] = c < CL_MAXN ? c : CL_MAXN;
        if (c > CL_MAXN) *A.overflow = 1;
      }
    }
    __syncthreads();
    // density pass (eam_rho_part semantics with cached r)
    for (int base = 0; base < nown; base += groups) {
      const int i = base + gi0;
      const bool live = i < nown;
      const int ii = live ? i : 0;
      const int nl = live ? M.nnbr[ii] : 0;
      double s = 0.0;
      for (int k = sl; k < nl; k += tpa) {
        // the force pass's table values for the same pair: d rho/dr is this
        // lookup's derivative, d phi/dr an independent lookup issued alongside
        const size_t ix = (size_t)ii * CL_MAXN + k;
        double f, df;
        tab_eval(A.rho, M.rr[ix], f, df);
        s = __dadd_rn(s, f);
        if (A.cache >= 1) M.drf[ix] = df;
        if (A.cache == 2) {
          double pf, dpf;
          tab_eval(A.phi, M.rr[ix], pf, dpf);
          M.dpf[ix] = dpf;
        }
      }
      s = group_sum(s, tpa);
      if (live && sl == 0) {
        double f, df;
        tab_eval(A.F, s, f, df);
        M.fp[a0 + i] = df;
      }
    }
    __syncthreads();
    dsmem_push(M.fp, a0, nown, C);  // own F' -> every peer
    cluster_barrier();
    // force pass (eam_force_part semantics with cached r)
    for (int base = 0; base < nown; base += groups) {
      const int i = base + gi0;
      const bool live = i < nown;
      const int ii = live ? i : 0;
      const int ai = a0 + ii;
      const int nl = live ? M.nnbr[ii] : 0;
      const double fpi = M.fp[ai];
      double gx = 0.0, gy = 0.0, gz = 0.0;
      for (int k = sl; k < nl; k += tpa) {
        const int j = M.nbr[(size_t)ii * CL_MAXN + k];
        double dx, dy, dz;
        pair_vec(q, ai, j, A.box, dx, dy, dz);
        const double rr = M.rr[(size_t)ii * CL_MAXN + k];
        double rf, drf, pf, dpf;
        if (A.cache >= 1)
          drf = M.drf[(size_t)ii * CL_MAXN + k];
        else
          tab_eval(A.rho, rr, rf, drf);
        if (A.cache == 2)
          dpf = M.dpf[(size_t)ii * CL_MAXN + k];
        else
          tab_eval(A.phi, rr, pf, dpf);
        const double sc = __ddiv_rn(fma(__dadd_rn(fpi, M.fp[j]), drf, dpf), rr);
        gx = fma(-sc, dx, gx);
        gy = fma(-sc, dy, gy);
        gz = fma(-sc, dz, gz);
      }
      gx = group_sum(gx, tpa);
      gy = group_sum(gy, tpa);
      gz = group_sum(gz, tpa);
      if (live && sl == 0) {
        M.g[3 * i] = gx;
        M.g[3 * i + 1] = gy;
        M.g[3 * i + 2] = gz;
      }
    }
    __syncthreads();
  };

  // ---------------------------------------------------------------- sweep
  double num = A.acc[2 * slot], den = A.acc[2 * slot + 1];
  for (int64_t t = threadIdx.x; t < 3 * (int64_t)n; t += blockDim.x) q[t] = Q[m0 * d + t];
  for (int t = threadIdx.x; t < dn; t += blockDim.x) M.p[t] = P[m0 * d + c0 + t];
  __syncthreads();
  cl.sync();
  if (A.b_inc[slot]) {
    double s2 = 0.0;
    for (int t = threadIdx.x; t < dn; t += blockDim.x) s2 += q[c0 + t] * q[c0 + t];
    for (int off = 16; off > 0; off >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, off);
    if (lane == 0) red[threadIdx.x >> 5] = s2;
    __syncthreads();
    double blk = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) blk += red[w];
    __syncthreads();
    den += sqrt(cluster_sum(cl, blk, slots_a, C, rank));  // num += ||q - q|| = 0
  }
  int64_t done = 0;
  int64_t fail_m = -1, fail_kind = 0;
  int fail_sub = 0;
  for (int64_t m = m0; m < m1; ++m) {
    const double* G = noise + m * (int64_t)(A.L + 1) * d;
    if (threadIdx.x == 0) s_fail = 0;
    eam_force(true);
    for (int s = 1; s <= A.L; ++s) {
      for (int t = threadIdx.x; t < dn; t += blockDim.x) {  // open (own components)
        const int gc = c0 + t;
        const double mm = A.mass ? A.mass[gc] : 1.0;
        const double smm = A.mass ? __dsqrt_rn(mm) : 1.0;
        const double al = mul(A.amp[s - 1], smm);
        const double pref = (s == 1) ? M.p[t] : M.ph[t];
        const double hv = add(sub(sub(M.p[t], mul(A.h, M.g[t])), mul(A.hg, pref)), mul(al, G[(int64_t)(s - 1) * d + gc]));
        M.ph[t] = hv;
        qn[gc] = add(q[gc], mul(A.dt, dvd(hv, mm)));
      }
      __syncthreads();
      {  // swap buffers; own moved-by-half-skin flag travels with the slice
        double* tq = q;
        q = qn;
        qn = tq;
      }
      int moved = 0;
      for (int i = threadIdx.x; i < nown; i += blockDim.x) {
        const double dx = q[c0 + 3 * i] - M.qref[3 * i], dy = q[c0 + 3 * i + 1] - M.qref[3 * i + 1];
        const double dz = q[c0 + 3 * i + 2] - M.qref[3 * i + 2];
        if (!(dx * dx + dy * dy + dz * dz <= 0.25 * CL_SKIN * CL_SKIN)) moved = 1;
      }
      moved = __syncthreads_or(moved);
      push_q_slice();
      if (threadIdx.x < (unsigned)C) dsmem_st(dsmem_addr(slots_c + rank, (int)threadIdx.x), moved ? 1.0 : 0.0);
      cluster_barrier();
      bool any = false;
      for (int rr_ = 0; rr_ < C; ++rr_) any = any || slots_c[rr_] > 0.0;
      eam_force(any);
      int bad = 0;
      for (int t = threadIdx.x; t < dn; t += blockDim.x) {  // close + blow-up check
        const int gc = c0 + t;
        const double smm = A.mass ? __dsqrt_rn(A.mass[gc]) : 1.0;
        const double al = mul(A.amp[s], smm);
        const double hv = M.ph[t];
        const double pn = add(sub(sub(hv, mul(A.h, M.g[t])), mul(A.hg, hv)), mul(al, G[(int64_t)s * d + gc]));
        M.p[t] = pn;
        if (!(fabs(q[gc]) <= BLOWUP_LIMIT && fabs(pn) <= BLOWUP_LIMIT)) bad = 1;
      }
      if (__syncthreads_or(bad) && threadIdx.x == 0 && s_fail == 0) s_fail = s;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < dn; t += blockDim.x) {
      baseQ[m * d + c0 + t] = q[c0 + t];
      baseP[m * d + c0 + t] = M.p[t];
    }
    // first failing substep over the cluster (0 = none): min over ranks
    {
      const double f = cluster_sum(cl, 0.0, slots_b, C, rank);  // barrier only
      (void)f;
      if (threadIdx.x < (unsigned)C) {
        dsmem_st(dsmem_addr(slots_a + rank, (int)threadIdx.x), (double)s_fail);
      }
      cluster_barrier();
      int mn = 0;
      for (int rr = 0; rr < C; ++rr) {
        const int v = (int)slots_a[rr];
        if (v && (!mn || v < mn)) mn = v;
      }
      cl.sync();
      if (mn) {
        fail_m = m;
        fail_sub = mn;
        fail_kind = 1;
        break;
      }
    }
    if (A.mode == 1) {
      for (int t = threadIdx.x; t < dn; t += blockDim.x) {
        Q[(m + 1) * d + c0 + t] = q[c0 + t];
        P[(m + 1) * d + c0 + t] = M.p[t];
      }
      ++done;
      continue;
    }
    double e1 = 0.0, e2 = 0.0;
    int nonfinite = 0;
    for (int t = threadIdx.x; t < dn; t += blockDim.x) {
      const int gc = c0 + t;
      const double pv = Q[(m + 1) * d + gc];  // prev[m+1], read before cur[m+1] overwrites it
      const double cq = add(q[gc], jumpQ[m * d + gc]);
      const double cp = add(M.p[t], jumpP[m * d + gc]);
      Q[(m + 1) * d + gc] = cq;
      P[(m + 1) * d + gc] = cp;
      q[gc] = cq;
      M.p[t] = cp;
      if (!isfinite(cq) || !isfinite(cp)) nonfinite = 1;
      const double e = sub(cq, pv);
      e1 += e * e;
      e2 += pv * pv;
    }
    nonfinite = __syncthreads_or(nonfinite);
    for (int off = 16; off > 0; off >>= 1) {
      e1 += __shfl_xor_sync(0xffffffffu, e1, off);
      e2 += __shfl_xor_sync(0xffffffffu, e2, off);
    }
    if (lane == 0) red[threadIdx.x >> 5] = e1;
    __syncthreads();
    double b1 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b1 += red[w];
    __syncthreads();
    if (lane == 0) red[threadIdx.x >> 5] = e2;
    __syncthreads();
    double b2 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b2 += red[w];
    __syncthreads();
    push_q_slice();  // corrected positions are the next window's start
    const double t1 = cluster_sum(cl, b1, slots_a, C, rank);
    const double t2 = cluster_sum(cl, b2, slots_b, C, rank);
    const double nf = cluster_sum(cl, nonfinite ? 1.0 : 0.0, slots_c, C, rank);
    cl.sync();
    num = num + sqrt(t1);
    den = den + sqrt(t2);
    ++done;
    if (rank == 0 && threadIdx.x == 0) {
      hist[m - m0] = num / den;
      if (A.progress) {  // node m+1 of every CTA is stored (cluster barrier above): publish it
        __threadfence_system();
        *(volatile int64_t*)A.progress = done;
      }
    }
    if (nf > 0.0) {
      fail_m = m;
      fail_kind = 2;
      break;
    }
    if (den == 0.0) break;
    if (A.expl > 0.0 && num / den > A.expl) break;
  }
  if (rank == 0 && threadIdx.x == 0) {
    A.acc[2 * slot] = num;
    A.acc[2 * slot + 1] = den;
    int64_t* o = A.out + 4 * slot;
    o[0] = done;
    o[1] = fail_m;
    o[2] = fail_sub;
    o[3] = fail_kind;
  }
  cl.sync();  // peers must not exit while DSMEM traffic to them is pending
}

// R_act slots, each one cluster; EAM coarse only.  Same contract as
// sweep_cta_batch.
int sweep_cluster_batch(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t N, int R_act, const int32_t* h_ridx,
                        const int64_t* h_m0, const int64_t* h_m1, const int32_t* h_inc, int mode, double* Q,
                        double* P, double* baseQ, double* baseP, const double* jumpQ, const double* jumpP,
                        const double* noise, const double* h_amp, const double* mass, double dt, double h,
                        double hg, double expl, double* h_state, int64_t* h_out4, double* d_hist) {
  if (R_act <= 0) return PL_OK;
  if (coarse->kind != POT_EAM) return -1;
  const int n = coarse->n_atoms;
  int C, tpa;
  cluster_layout(n, C, tpa);
  const int own = (n + C - 1) / C;
  if (cl_smem_bytes(n, own) > 220 * 1024) return -1;
  // cache as many table derivatives as shared memory allows (values bitwise the same)
  static const int cache_env = [] {
    const char* e = getenv("PL_SWEEP_CACHE");
    return e ? atoi(e) : 2;
  }();
  int cache = cache_env;
  while (cache > 0 && cl_smem_bytes(n, own, cache) > 220 * 1024) --cache;
  const size_t smem = cl_smem_bytes(n, own, cache);
  ClArgs A{};
  A.d = d; A.n_atoms = n; A.L = L; A.mode = mode; A.C = C; A.tpa = tpa; A.cache = cache;
  A.Q = Q; A.P = P; A.baseQ = baseQ; A.baseP = baseP;
  A.jumpQ = mode == 0 ? jumpQ : baseQ;
  A.jumpP = mode == 0 ? jumpP : baseP;
  A.noise = noise; A.mass = mass; A.dt = dt; A.h = h; A.hg = hg; A.expl = expl;
  A.box = make_box(coarse->box);
  A.rc2 = coarse->rcut * coarse->rcut;
  A.rl2 = (coarse->rcut + CL_SKIN) * (coarse->rcut + CL_SKIN);
  A.rho = Table{coarse->d_rho, coarse->n_r, coarse->dr, 1.0 / coarse->dr};
  A.phi = Table{coarse->d_phi, coarse->n_r, coarse->dr, 1.0 / coarse->dr};
  A.F = Table{coarse->d_F, coarse->n_rho, coarse->drho, 1.0 / coarse->drho};
  A.s_traj = (N + 1) * d;
  A.s_win = N * d;
  A.s_noise = N * (int64_t)(L + 1) * d;
  A.s_hist = N;
  cudaStream_t st = ctx->stream;
  const size_t bytes = sizeof(double) * (L + 1 + 2 * R_act) + sizeof(int64_t) * (4 + 2) * R_act +
                       sizeof(int32_t) * 2 * R_act + 256;
  PL_TRY(ctx->work[5].reserve(bytes));
  char* w = (char*)ctx->work[5].ptr;
  double* amp = (double*)w;
  double* acc = amp + (L + 1);
  int64_t* out = (int64_t*)(acc + 2 * R_act);
  int64_t* m0 = out + 4 * R_act;
  int64_t* m1 = m0 + R_act;
  int32_t* ridx = (int32_t*)(m1 + R_act);
  int32_t* inc = ridx + R_act;
  int* ovf = (int*)(inc + R_act);
  A.amp = amp; A.acc = acc; A.out = out; A.hist = d_hist;
  A.b_ridx = ridx; A.b_m0 = m0; A.b_m1 = m1; A.b_inc = inc; A.overflow = ovf;
  A.progress = (R_act == 1 && mode == 0) ? ctx->progress_dev : nullptr;
  if (A.progress) *(volatile int64_t*)ctx->progress = 0;
  PL_CUDA(cudaMemsetAsync(ovf, 0, sizeof(int), st));
  PL_CUDA(cudaMemcpyAsync(amp, h_amp, sizeof(double) * (L + 1), cudaMemcpyHostToDevice, st));
  PL_CUDA(cudaMemcpyAsync(acc, h_state, sizeof(double) * 2 * R_act, cudaMemcpyHostToDevice, st));
  PL_CUDA(cudaMemcpyAsync(m0, h_m0, sizeof(int64_t) * R_act, cudaMemcpyHostToDevice, st));
  PL_CUDA(cudaMemcpyAsync(m1, h_m1, sizeof(int64_t) * R_act, cudaMemcpyHostToDevice, st));
  PL_CUDA(cudaMemcpyAsync(ridx, h_ridx, sizeof(int32_t) * R_act, cudaMemcpyHostToDevice, st));
  PL_CUDA(cudaMemcpyAsync(inc, h_inc, sizeof(int32_t) * R_act, cudaMemcpyHostToDevice, st));
  static std::atomic<uint64_t> attr_devs{0};
  if (first_on_device(attr_devs)) {
    cudaFuncSetAttribute(k_sweep_cluster<CL_THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_sweep_cluster<CL_THREADS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_sweep_cluster<640>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_sweep_cluster<640>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(C * R_act));
  // threads the atoms use (and >= the own components, so every thread holds at
  // most one component in the error sums, as with 1024 threads)
  int threads = std::max(own * tpa, 3 * own);
  threads = std::min(CL_THREADS, (threads + 31) / 32 * 32);
  if (getenv("PL_SWEEP_FULL")) threads = CL_THREADS;
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (threads <= 640)
    PL_CUDA(cudaLaunchKernelEx(&cfg, k_sweep_cluster<640>, A));
  else
    PL_CUDA(cudaLaunchKernelEx(&cfg, k_sweep_cluster<CL_THREADS>, A));
  int hovf = 0;
  PL_CUDA(cudaMemcpyAsync(h_state, acc, sizeof(double) * 2 * R_act, cudaMemcpyDeviceToHost, st));
  PL_CUDA(cudaMemcpyAsync(h_out4, out, sizeof(int64_t) * 4 * R_act, cudaMemcpyDeviceToHost, st));
  PL_CUDA(cudaMemcpyAsync(&hovf, ovf, sizeof(int), cudaMemcpyDeviceToHost, st));
  PL_CUDA(cudaStreamSynchronize(st));
  if (hovf) return fail(PL_EPOT, "neighbour capacity exceeded in the coarse sweep");
  return PL_OK;
}

// 2 when a single-replica sweep of this coarse potential runs as the persistent
// cluster kernel (the path that publishes progress), else 0
int sweep_path(const pl_pot* coarse) {
  if (!coarse || coarse->kind != POT_EAM || getenv("PL_SWEEP_NOCLUSTER") || getenv("PL_SWEEP_GENERIC")) return 0;
  int C, tpa;
  cluster_layout(coarse->n_atoms, C, tpa);
  const int own = (coarse->n_atoms + C - 1) / C;
  return cl_smem_bytes(coarse->n_atoms, own) > 220 * 1024 ? 0 : 2;
}

int eam_tpa_for(int n) {
  int C, tpa;
  cluster_layout(n, C, tpa);
  return tpa;
}

}  // namespace pl

extern "C" int pl_sweep_path(pl_pot* coarse) {
  if (!coarse) return pl::fail(PL_EARG, "NULL argument");
  return pl::sweep_path(coarse);
}
