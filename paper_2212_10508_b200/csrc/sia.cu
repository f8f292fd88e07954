// Self-interstitial site detection by Wigner-Seitz occupancy.
//
// The reference labels basins by the nearest catalogued minimum in the full
// configuration space (analysis.py:90-111), which cannot scale to the ~2n^3
// equivalent SIA positions of a W lattice.  Here every atom is assigned to its
// nearest perfect-BCC site (two simple-cubic sublattices, periodic box); with
// N = 2n^3 + 1 atoms at least one site is doubly occupied, and the smallest
// such site index labels the node.  A hop is a change of label between nodes.
// One CTA per configuration, integer shared-memory counts: deterministic.
#include "pl_common.cuh"

namespace pl {

__global__ void k_sia_sites(int64_t B, int N, int n, double a, const double* __restrict__ q,
                            int32_t* __restrict__ label) {
  extern __shared__ int cnt[];
  const int sites = 2 * n * n * n;
  const double L = a * n;
  for (int s = threadIdx.x; s < sites; s += blockDim.x) cnt[s] = 0;
  __syncthreads();
  const double* qb = q + blockIdx.x * (int64_t)N * 3;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    int c[3], h[3];
    double dc = 0.0, dh = 0.0;
    for (int k = 0; k < 3; ++k) {
      const double x = qb[3 * i + k];
      const double xw = x - L * floor(x / L);  // wrap into [0, L)
      const double u = xw / a;
      const double rc = rint(u), fh = floor(u) + 0.5;
      double e1 = (u - rc) * a, e2 = (u - fh) * a;
      dc += e1 * e1;
      dh += e2 * e2;
      c[k] = ((int)rc % n + n) % n;
      h[k] = ((int)floor(u) % n + n) % n;
    }
    const int site = dc <= dh ? (c[0] * n + c[1]) * n + c[2] : n * n * n + (h[0] * n + h[1]) * n + h[2];
    atomicAdd(&cnt[site], 1);
  }
  __syncthreads();
  __shared__ int best;
  if (threadIdx.x == 0) best = 0x7fffffff;
  __syncthreads();
  for (int s = threadIdx.x; s < sites; s += blockDim.x)
    if (cnt[s] >= 2) atomicMin(&best, s);
  __syncthreads();
  if (threadIdx.x == 0) label[blockIdx.x] = best == 0x7fffffff ? -1 : best;
}

}  // namespace pl

extern "C" int pl_sia_sites(pl_ctx* ctx, int64_t B, int n_atoms, int n_cells, double a, const double* d_q,
                            int32_t* d_label) {
  if (!ctx || !d_q || !d_label) return pl::fail(PL_EARG, "NULL argument");
  if (B < 0 || n_atoms < 1 || n_cells < 1 || !(a > 0.0)) return pl::fail(PL_EARG, "bad SIA-site arguments");
  if (B == 0) return PL_OK;
  const size_t smem = sizeof(int) * 2 * (size_t)n_cells * n_cells * n_cells;
  if (smem > 200 * 1024) return pl::fail(PL_EARG, "lattice too large for one CTA");
  cudaFuncSetAttribute(pl::k_sia_sites, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  pl::k_sia_sites<<<(unsigned)B, 256, smem, ctx->stream>>>(B, n_atoms, n_cells, a, d_q, d_label);
  PL_CHECK_LAUNCH();
  return PL_OK;
}
