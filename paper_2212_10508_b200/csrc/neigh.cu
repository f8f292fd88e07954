// Periodic neighbour lists: brute force for small systems, cell lists above
// CELL_MIN_ATOMS.  Both produce the same lists bit for bit: ascending j, pair
// test r^2 < rc^2 on the exactly rounded minimum-image displacement
// (neigh.cuh), so every force sum downstream sees the same pairs in the same
// order regardless of the builder.
#include <cub/block/block_scan.cuh>

#include "neigh.cuh"
#include "pl_common.cuh"

namespace pl {

constexpr int CELL_MIN_ATOMS = 512;
constexpr int CELL_MAXN = 128;  // per-thread collection buffer (local memory)

struct CellGrid {
  int n[3];
  double inv[3];  // cells per Angstrom
};

// cell of a (possibly unwrapped) position component
__device__ __forceinline__ int cell_of(double x, double L, double inv, int n) {
  double w = x - L * floor(x / L);  // wrap into [0, L)
  int c = (int)(w * inv);
  return c < 0 ? 0 : (c >= n ? n - 1 : c);
}

__global__ void k_cell_count(int64_t B, int N, Box box, CellGrid g, const double* __restrict__ q,
                             int32_t* __restrict__ cell_of_atom, int32_t* __restrict__ ccount,
                             const int* __restrict__ go) {
  griddep_wait();
  if (go && *go == 0) return;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= B * N) return;
  int64_t b = t / N;
  const double* x = q + 3 * t;
  int cx = cell_of(x[0], box.L[0], g.inv[0], g.n[0]);
  int cy = cell_of(x[1], box.L[1], g.inv[1], g.n[1]);
  int cz = cell_of(x[2], box.L[2], g.inv[2], g.n[2]);
  int c = (cz * g.n[1] + cy) * g.n[0] + cx;
  int64_t gc = b * (int64_t)g.n[0] * g.n[1] * g.n[2] + c;
  cell_of_atom[t] = (int32_t)gc;
  atomicAdd(&ccount[gc], 1);  // integer: the counts are order independent
}

// exclusive scan of cell counts (single CTA, chunked)
__global__ void __launch_bounds__(1024) k_cell_scan(int64_t ncell, const int32_t* __restrict__ ccount,
                                                   int32_t* __restrict__ cstart, int32_t* __restrict__ cfill,
                                                   const int* __restrict__ go) {
  griddep_wait();
  if (go && *go == 0) return;
  typedef cub::BlockScan<int32_t, 1024> S;
  __shared__ typename S::TempStorage tmp;
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < ncell; base += 1024) {
    int64_t i = base + threadIdx.x;
    int32_t v = i < ncell ? ccount[i] : 0, ex, tot;
    S(tmp).ExclusiveSum(v, ex, tot);
    if (i < ncell) {
      cstart[i] = carry + ex;
      cfill[i] = carry + ex;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) cstart[ncell] = carry;
}

__global__ void k_cell_fill(int64_t natoms, int N, const int32_t* __restrict__ cell_of_atom,
                            int32_t* __restrict__ cfill, int32_t* __restrict__ catoms, const int* __restrict__ go) {
  griddep_wait();
  if (go && *go == 0) return;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= natoms) return;
  int slot = atomicAdd(&cfill[cell_of_atom[t]], 1);
  catoms[slot] = (int32_t)(t % N);  // order inside a cell is arbitrary: lists are sorted below
}

__global__ void __launch_bounds__(128)
k_neigh_cell(int64_t B, int N, Box box, CellGrid g, double rc2, int maxn, const double* __restrict__ q,
             const int32_t* __restrict__ cell_of_atom, const int32_t* __restrict__ cstart,
             const int32_t* __restrict__ catoms, int32_t* __restrict__ nbr, int32_t* __restrict__ cnt,
             int* __restrict__ overflow, const int* __restrict__ go) {
  if (go && *go == 0) return;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= B * N) return;
  int64_t b = t / N;
  int i = (int)(t - b * N);
  const double* qb = q + b * (int64_t)N * 3;
  const int64_t cells = (int64_t)g.n[0] * g.n[1] * g.n[2];
  const int c = (int)(cell_of_atom[t] - b * cells);
  const int cx = c % g.n[0], cy = (c / g.n[0]) % g.n[1], cz = c / (g.n[0] * g.n[1]);
  const double xi = qb[3 * i], yi = qb[3 * i + 1], zi = qb[3 * i + 2];
  int32_t found[CELL_MAXN];
  int nf = 0;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int ex = (cx + dx + g.n[0]) % g.n[0], ey = (cy + dy + g.n[1]) % g.n[1], ez = (cz + dz + g.n[2]) % g.n[2];
        int64_t cc = b * cells + (ez * g.n[1] + ey) * g.n[0] + ex;
        for (int s = cstart[cc]; s < cstart[cc + 1]; ++s) {
          int j = catoms[s];
          if (j == i) continue;
          double ddx = min_image(sub(qb[3 * j], xi), box.L[0], box.inv[0]);
          double ddy = min_image(sub(qb[3 * j + 1], yi), box.L[1], box.inv[1]);
          double ddz = min_image(sub(qb[3 * j + 2], zi), box.L[2], box.inv[2]);
          if (r2_exact(ddx, ddy, ddz) < rc2) {
            if (nf < CELL_MAXN) found[nf] = j;
            ++nf;
          }
        }
      }
  int keep = nf < CELL_MAXN ? nf : CELL_MAXN;
  // ascending j (insertion sort of a few dozen entries)
  for (int a = 1; a < keep; ++a) {
    int v = found[a], k = a - 1;
    while (k >= 0 && found[k] > v) {
      found[k + 1] = found[k];
      --k;
    }
    found[k + 1] = v;
  }
  int outn = keep < maxn ? keep : maxn;
  int32_t* my = nbr + t * maxn;
  for (int a = 0; a < outn; ++a) my[a] = found[a];
  cnt[t] = outn;
  if (nf > outn) atomicExch(overflow, 1);  // also when nf exceeds the CELL_MAXN buffer
}

// one warp per atom: lane c < 27 owns neighbour cell c, a warp scan of the cell
// counts flattens the ~200 candidates over the lanes (all loads of a pass in
// flight together), hits are collected by ballot and ranked into ascending j
// (the same list as k_neigh_cell, without one thread's serial 27-cell walk)
constexpr int NC_WARPS = 4;
__global__ void __launch_bounds__(NC_WARPS * 32)
k_neigh_cell_w(int64_t B, int N, Box box, CellGrid g, double rc2, int maxn, const double* __restrict__ q,
               const int32_t* __restrict__ cell_of_atom, const int32_t* __restrict__ cstart,
               const int32_t* __restrict__ catoms, int32_t* __restrict__ nbr, int32_t* __restrict__ cnt,
               int* __restrict__ overflow, const int* __restrict__ go) {
  griddep_wait();
  if (go && *go == 0) return;
  __shared__ int32_t s_found[NC_WARPS][CELL_MAXN];
  __shared__ int32_t s_off[NC_WARPS][32], s_beg[NC_WARPS][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * NC_WARPS + warp;
  if (t >= B * N) return;
  const int64_t b = t / N;
  const int i = (int)(t - b * N);
  const double* qb = q + b * (int64_t)N * 3;
  const int64_t cells = (int64_t)g.n[0] * g.n[1] * g.n[2];
  const int c = (int)(cell_of_atom[t] - b * cells);
  const int cx = c % g.n[0], cy = (c / g.n[0]) % g.n[1], cz = c / (g.n[0] * g.n[1]);
  const double xi = qb[3 * i], yi = qb[3 * i + 1], zi = qb[3 * i + 2];
  int beg = 0, num = 0;
  if (lane < 27) {  // same cell order as k_neigh_cell (dz, dy, dx)
    const int dz = lane / 9 - 1, dy = (lane / 3) % 3 - 1, dx = lane % 3 - 1;
    const int ex = (cx + dx + g.n[0]) % g.n[0], ey = (cy + dy + g.n[1]) % g.n[1], ez = (cz + dz + g.n[2]) % g.n[2];
    const int64_t cc = b * cells + (ez * g.n[1] + ey) * g.n[0] + ex;
    beg = cstart[cc];
    num = cstart[cc + 1] - beg;
  }
  int incl = num;  // inclusive warp scan of the cell counts
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  s_off[warp][lane] = incl - num;
  s_beg[warp][lane] = beg;
  __syncwarp();
  int nf = 0;
#pragma unroll 4
  for (int base = 0; base < total; base += 32) {
    const int idx = base + lane;
    bool hit = false;
    int j = -1;
    if (idx < total) {
      int lo = 0, hi = 26;  // last cell with off <= idx (empty cells share offsets: take the last)
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_off[warp][mid] <= idx) lo = mid; else hi = mid - 1;
      }
      j = catoms[s_beg[warp][lo] + idx - s_off[warp][lo]];
      if (j != i) {
        const double ddx = min_image(sub(qb[3 * j], xi), box.L[0], box.inv[0]);
        const double ddy = min_image(sub(qb[3 * j + 1], yi), box.L[1], box.inv[1]);
        const double ddz = min_image(sub(qb[3 * j + 2], zi), box.L[2], box.inv[2]);
        hit = r2_exact(ddx, ddy, ddz) < rc2;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    const int slot = nf + __popc(m & ((1u << lane) - 1u));
    if (hit && slot < CELL_MAXN) s_found[warp][slot] = j;
    nf += __popc(m);
  }
  __syncwarp();
  const int keep = nf < CELL_MAXN ? nf : CELL_MAXN;
  const int outn = keep < maxn ? keep : maxn;
  int32_t* my = nbr + t * maxn;
  for (int e = lane; e < keep; e += 32) {  // rank = number of smaller j (j distinct)
    const int v = s_found[warp][e];
    int r = 0;
    for (int f = 0; f < keep; ++f) r += s_found[warp][f] < v;
    if (r < outn) my[r] = v;
  }
  if (lane == 0) {
    cnt[t] = outn;
    if (nf > outn) atomicExch(overflow, 1);  // also when nf exceeds the CELL_MAXN buffer
  }
}

__global__ void k_or_flag(const int* __restrict__ src, int32_t* __restrict__ dst) { *dst |= *src; }

// Verlet skin: *flag = 1 when an atom moved more than skin/2 since the last build
// (positions are unwrapped and continuous: no minimum image)
__global__ void k_skin_check(int64_t n3, const double* __restrict__ q, const double* __restrict__ qref, double h2,
                             int* __restrict__ flag) {
  griddep_wait();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (3 * t >= n3) return;
  const double dx = q[3 * t] - qref[3 * t], dy = q[3 * t + 1] - qref[3 * t + 1], dz = q[3 * t + 2] - qref[3 * t + 2];
  if (!(dx * dx + dy * dy + dz * dz <= h2)) *flag = 1;  // every writer stores 1 (non-finite moves rebuild too)
}

// the reference positions follow a rebuild
__global__ void k_skin_ref(int64_t n3, const double* __restrict__ q, double* __restrict__ qref,
                           const int* __restrict__ flag) {
  griddep_wait();
  if (*flag == 0) return;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n3; t += (int64_t)gridDim.x * blockDim.x)
    qref[t] = q[t];
}

int skin_check(pl_pot* pot, int64_t na, const double* q, const double* qref, int* flag) {
  cudaStream_t st = pot->ctx->stream;
  PL_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
  const double h = 0.5 * pot->skin;
  PL_CUDA(launch_pdl(k_skin_check, dim3((unsigned)((na + 255) / 256)), dim3(256), 0, st, 3 * na, q, qref, h * h, flag));
  PL_CHECK_LAUNCH();
  return PL_OK;
}

int skin_ref(pl_pot* pot, int64_t na, const double* q, double* qref, const int* flag) {
  cudaStream_t st = pot->ctx->stream;
  int64_t blocks = (3 * na + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  PL_CUDA(launch_pdl(k_skin_ref, dim3((unsigned)blocks), dim3(256), 0, st, 3 * na, q, qref, flag));
  PL_CHECK_LAUNCH();
  return PL_OK;
}

int build_neighbours(pl_pot* pot, int64_t B, const double* q, double rcut, int maxn, NeighList* out,
                     const int* go) {
  int N = pot->n_atoms;
  size_t lists = sizeof(int32_t) * (size_t)B * N * maxn;
  size_t counts = sizeof(int32_t) * (size_t)B * N;
  PL_TRY(pot->work[0].reserve(lists));
  void* const cnt_before = pot->work[1].ptr;
  PL_TRY(pot->work[1].reserve(counts + 64));
  out->nbr = (int32_t*)pot->work[0].ptr;
  out->cnt = (int32_t*)pot->work[1].ptr;
  out->overflow = (int*)((char*)pot->work[1].ptr + ((counts + 15) & ~(size_t)15));
  out->maxn = maxn;
  pot->nb_overflow = out->overflow;
  if (B > 65535) return fail(PL_EARG, "at most 65535 systems per call");
  Box box = make_box(pot->box);
  double rc2 = rcut * rcut;
  cudaStream_t st = pot->ctx->stream;
  // the flag is sticky between checks: every build of a window (one per substep)
  // can raise it, and neigh_check at the end of the call sees any of them
  if (pot->nb_armed || pot->work[1].ptr != cnt_before) PL_CUDA(cudaMemsetAsync(out->overflow, 0, sizeof(int), st));
  pot->nb_armed = false;
  CellGrid g;
  bool cells_ok = N >= CELL_MIN_ATOMS && !getenv("PL_NEIGH_BRUTE");
  for (int c = 0; c < 3; ++c) {
    g.n[c] = (int)(pot->box[c] / rcut);
    if (g.n[c] < 3) cells_ok = false;
    g.inv[c] = g.n[c] / pot->box[c];
  }
  prof_mark(st, ST_NEIGH, true);
  if (!cells_ok) {
    const int64_t warps = B * N;
    PL_CUDA(launch_pdl(k_neigh_brute_w, dim3((unsigned)((warps * 32 + NB_THREADS - 1) / NB_THREADS)), dim3(NB_THREADS),
                       0, st, B, N, box, rc2, maxn, q, out->nbr, out->cnt, out->overflow, go));
    PL_CHECK_LAUNCH();
  } else {
    int64_t cells = (int64_t)g.n[0] * g.n[1] * g.n[2];
    int64_t nc = B * cells;
    int64_t na = B * N;
    size_t bytes = sizeof(int32_t) * (na + 3 * (nc + 1) + na) + 256;
    PL_TRY(pot->work[3].reserve(bytes));
    int32_t* cell_of_atom = (int32_t*)pot->work[3].ptr;
    int32_t* ccount = cell_of_atom + na;
    int32_t* cstart = ccount + (nc + 1);
    int32_t* cfill = cstart + (nc + 1);
    int32_t* catoms = cfill + (nc + 1);
    PL_CUDA(cudaMemsetAsync(ccount, 0, sizeof(int32_t) * nc, st));
    unsigned ga = (unsigned)((na + 255) / 256);
    PL_CUDA(launch_pdl(k_cell_count, dim3(ga), dim3(256), 0, st, B, N, box, g, q, cell_of_atom, ccount, go));
    PL_CUDA(launch_pdl(k_cell_scan, dim3(1), dim3(1024), 0, st, nc, ccount, cstart, cfill, go));
    PL_CUDA(launch_pdl(k_cell_fill, dim3(ga), dim3(256), 0, st, na, N, cell_of_atom, cfill, catoms, go));
    static const bool warp_cells = !getenv("PL_NEIGH_THREAD");
    if (warp_cells)
      PL_CUDA(launch_pdl(k_neigh_cell_w, dim3((unsigned)((na + NC_WARPS - 1) / NC_WARPS)), dim3(NC_WARPS * 32), 0, st,
                         B, N, box, g, rc2, maxn, q, cell_of_atom, cstart, catoms, out->nbr, out->cnt,
                         out->overflow, go));
    else
      k_neigh_cell<<<(unsigned)((na + 127) / 128), 128, 0, st>>>(B, N, box, g, rc2, maxn, q, cell_of_atom,
                                                                cstart, catoms, out->nbr, out->cnt, out->overflow,
                                                                go);
    PL_CHECK_LAUNCH();
  }
  prof_mark(st, ST_NEIGH, false);
  return PL_OK;
}

int neigh_check(pl_pot* pot) {
  switch (pot->kind) {
    case POT_PERTURBED:
      PL_TRY(neigh_check(pot->base));
      return pot->lam != 0.0 ? neigh_check(pot->delta) : PL_OK;
    case POT_EAM:
    case POT_SNAP:
      break;
    default:
      return PL_OK;
  }
  if (!pot->nb_overflow) return PL_OK;
  if (pot->ctx->spec) return PL_OK;  // deferred: pl_pot_overflow_async
  int h = 0;
  PL_CUDA(cudaMemcpyAsync(&h, pot->nb_overflow, sizeof(int), cudaMemcpyDeviceToHost, pot->ctx->stream));
  PL_CUDA(cudaStreamSynchronize(pot->ctx->stream));
  pot->nb_armed = true;
  if (h) return fail(PL_EPOT, "neighbour capacity exceeded (atoms too close / dense)");
  return PL_OK;
}

// stream-ordered copy of the overflow flag (accumulated since the last check)
// into d_out, OR-ed over the parts of a perturbed potential; re-arms the flag
int overflow_async(pl_pot* pot, int32_t* d_out, bool first) {
  cudaStream_t st = pot->ctx->stream;
  if (pot->kind == POT_PERTURBED) {
    PL_TRY(overflow_async(pot->base, d_out, first));
    return pot->lam != 0.0 ? overflow_async(pot->delta, d_out, false) : PL_OK;
  }
  if ((pot->kind != POT_EAM && pot->kind != POT_SNAP) || !pot->nb_overflow) {
    if (first) PL_CUDA(cudaMemsetAsync(d_out, 0, sizeof(int32_t), st));
    return PL_OK;
  }
  if (first) {
    PL_CUDA(cudaMemcpyAsync(d_out, pot->nb_overflow, sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  } else {
    k_or_flag<<<1, 1, 0, st>>>(pot->nb_overflow, d_out);
    PL_CHECK_LAUNCH();
  }
  pot->nb_armed = true;
  return PL_OK;
}


}  // namespace pl

extern "C" int pl_pot_overflow_async(pl_ctx* ctx, pl_pot* pot, int32_t* d_out) {
  if (!ctx || !pot || !d_out) return pl::fail(PL_EARG, "NULL argument");
  if (pot->ctx != ctx) return pl::fail(PL_EARG, "potential belongs to another context");
  return pl::overflow_async(pot, d_out, true);
}
