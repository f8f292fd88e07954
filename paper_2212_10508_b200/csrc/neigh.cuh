// Periodic neighbour lists for batches of systems (B x N atoms, flat AoS q).
//
// Positions stay UNWRAPPED in the state (the reference's Euclidean error
// metric, parareal.py:196-197, must see continuous coordinates); the minimum
// image is applied here only.  The box must be >= 2*rcut, so every pair has at
// most one image inside the cutoff.  Lists are ordered by ascending j: the
// force sums are then in a fixed order, which keeps every kernel run-to-run
// deterministic and lets the C oracle reproduce the same pair set bit for bit
// (the cutoff test uses explicit round-to-nearest ops, no FMA).
#pragma once

#include "pl_common.cuh"

namespace pl {

struct Box {
  double L[3];
  double inv[3];  // 1/L, formed on the host (the C oracle forms the same quotient)
};

inline Box make_box(const double* L) {
  Box b;
  for (int c = 0; c < 3; ++c) {
    b.L[c] = L[c];
    b.inv[c] = 1.0 / L[c];
  }
  return b;
}

// image index rint(dx / L) evaluated as rint(dx * (1/L)): no divide on the hot
// path; the oracle uses the identical expression, so pair sets stay bit-exact
__device__ __forceinline__ double min_image(double dx, double L, double inv) {
  double k = rint(mul(dx, inv));
  return sub(dx, mul(L, k));
}

__device__ __forceinline__ double r2_exact(double dx, double dy, double dz) {
  return add(add(mul(dx, dx), mul(dy, dy)), mul(dz, dz));
}

constexpr int NB_THREADS = 128;

// one thread per atom i of system b; j tiles staged in shared memory
static __global__ void __launch_bounds__(NB_THREADS)
k_neigh_brute(int64_t B, int N, Box box, double rc2, int maxn, const double* __restrict__ q,
              int32_t* __restrict__ nbr, int32_t* __restrict__ cnt, int* __restrict__ overflow) {
  __shared__ double sx[NB_THREADS * 3];
  int64_t b = blockIdx.y;
  int i = blockIdx.x * NB_THREADS + threadIdx.x;
  const double* qb = q + b * (int64_t)N * 3;
  double xi = 0, yi = 0, zi = 0;
  if (i < N) {
    xi = qb[3 * i];
    yi = qb[3 * i + 1];
    zi = qb[3 * i + 2];
  }
  int c = 0;
  int32_t* my = nbr + (b * N + (i < N ? i : 0)) * (int64_t)maxn;
  for (int j0 = 0; j0 < N; j0 += NB_THREADS) {
    __syncthreads();
    for (int t = threadIdx.x; t < NB_THREADS * 3; t += NB_THREADS) {
      int jj = j0 * 3 + t;
      sx[t] = jj < N * 3 ? qb[jj] : 0.0;
    }
    __syncthreads();
    if (i < N) {
      int jmax = min(NB_THREADS, N - j0);
      for (int jj = 0; jj < jmax; ++jj) {
        int j = j0 + jj;
        if (j == i) continue;
        double dx = min_image(sub(sx[3 * jj], xi), box.L[0], box.inv[0]);
        double dy = min_image(sub(sx[3 * jj + 1], yi), box.L[1], box.inv[1]);
        double dz = min_image(sub(sx[3 * jj + 2], zi), box.L[2], box.inv[2]);
        double r2 = r2_exact(dx, dy, dz);
        if (r2 < rc2) {
          if (c < maxn) my[c] = j;
          ++c;
        }
      }
    }
  }
  if (i < N) {
    cnt[b * N + i] = c < maxn ? c : maxn;
    if (c > maxn) atomicExch(overflow, 1);
  }
}

// one warp per atom i: lanes test 32 candidates j at a time, hits are written
// in ascending j by ballot/popc (the same list as k_neigh_brute, for small
// systems where one thread per atom leaves the latency of N serial tests)
static __global__ void __launch_bounds__(NB_THREADS)
k_neigh_brute_w(int64_t B, int N, Box box, double rc2, int maxn, const double* __restrict__ q,
                int32_t* __restrict__ nbr, int32_t* __restrict__ cnt, int* __restrict__ overflow,
                const int* __restrict__ go) {
  griddep_wait();
  if (go && *go == 0) return;
  const int64_t t = (blockIdx.x * (int64_t)NB_THREADS + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= B * N) return;
  const int64_t b = t / N;
  const int i = (int)(t - b * N);
  const double* qb = q + b * (int64_t)N * 3;
  const double xi = qb[3 * i], yi = qb[3 * i + 1], zi = qb[3 * i + 2];
  int32_t* my = nbr + t * (int64_t)maxn;
  int c = 0;
  for (int j0 = 0; j0 < N; j0 += 32) {
    const int j = j0 + lane;
    bool hit = false;
    if (j < N && j != i) {
      const double dx = min_image(sub(qb[3 * j], xi), box.L[0], box.inv[0]);
      const double dy = min_image(sub(qb[3 * j + 1], yi), box.L[1], box.inv[1]);
      const double dz = min_image(sub(qb[3 * j + 2], zi), box.L[2], box.inv[2]);
      hit = r2_exact(dx, dy, dz) < rc2;
    }
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    const int slot = c + __popc(m & ((1u << lane) - 1u));
    if (hit && slot < maxn) my[slot] = j;
    c += __popc(m);
  }
  if (lane == 0) {
    cnt[t] = c < maxn ? c : maxn;
    if (c > maxn) atomicExch(overflow, 1);
  }
}

// displacement r_j - r_i under the minimum image (same ops as the builder)
__device__ __forceinline__ void pair_vec(const double* qb, int i, int j, const Box& box, double& dx,
                                         double& dy, double& dz) {
  dx = min_image(sub(qb[3 * j], qb[3 * i]), box.L[0], box.inv[0]);
  dy = min_image(sub(qb[3 * j + 1], qb[3 * i + 1]), box.L[1], box.inv[1]);
  dz = min_image(sub(qb[3 * j + 2], qb[3 * i + 2]), box.L[2], box.inv[2]);
}

struct NeighList {
  int32_t* nbr = nullptr;
  int32_t* cnt = nullptr;
  int* overflow = nullptr;
  int maxn = 0;
};

// builds into pot->work[0] (lists) / work[1] (counts + flag)
// go (device flag, optional): every build kernel returns at entry when *go == 0
// (Verlet-skin lists that are still valid; the lists are left as they are)
int build_neighbours(pl_pot* pot, int64_t B, const double* q, double rcut, int maxn, NeighList* out,
                     const int* go = nullptr);
// Verlet skin (snap.cu): *flag = 1 when an atom moved more than skin/2 since qref;
// qref = q where *flag (both on pot's stream, no host synchronisation)
int skin_check(pl_pot* pot, int64_t na, const double* q, const double* qref, int* flag);
int skin_ref(pl_pot* pot, int64_t na, const double* q, double* qref, const int* flag);
// exact pair test of the list builders (r < rc on the minimum image)
__device__ __forceinline__ bool pair_exact(const double* qb, int i, int j, const Box& box, double rc2);

__device__ __forceinline__ bool pair_exact(const double* qb, int i, int j, const Box& box, double rc2) {
  double dx, dy, dz;
  pair_vec(qb, i, j, box, dx, dy, dz);
  return r2_exact(dx, dy, dz) < rc2;
}

}  // namespace pl
