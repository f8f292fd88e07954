// SNAP Z/Y contraction at twojmax = 8: k_snap_yi_p ("P form").
//
// For a triple (X, Y, J) (X >= Y) and a half row mb of layer J,
//   Z[ma][mb] = sum_{a, mb1} C(ma; a) C(mb; mb1) U^X[a][mb1] U^Y[b][mb2],
//   b = ma + SH - a,  mb2 = mb + SH - mb1,  SH = (X + Y - J) / 2.
// The kernel sums over mb1 FIRST, per cell (a, b) of the CG band
// (SH <= a + b <= SH + J):
//   P[a][b] = sum_mb1 U^X[a][mb1] (C(mb; mb1) U^Y[b][mb2])          4 DFMA / product
//   Z[ma]   = sum_a C(ma; a) P[a][ma + SH - a]                      once per cell
// so the a-side CG weight leaves the inner loop (the previous "box" kernel
// applied it per product: 2 DMUL + 4 DFMA, and spent ~40 % of its products on
// the zero corners of the (X+1)(Y+1) box; this form issues only band products,
// 1.83x fewer FP64 instructions per atom).  The band is compile-time, so P
// lives in registers: one body per triple, ptri<X, Y, J> (125 bodies).
//
// Lanes = atoms (32 per CTA; U^J of all layers expanded to full matrices in
// shared memory, [element][atom], conflict-free), warps own (J, mb) half rows.
// Code size: 125 bodies are ~5x the box kernel's, more than the instruction
// cache holds.  The CTA therefore walks the triples in PHASES (consecutive
// triples in (X, Y, J) order within a code budget) separated by
// __syncthreads(): only one phase's bodies are live at a time, and the rows are re-assigned to warps per phase (host LPT +
// local search on a cost model), which also balances each phase.  A row's
// items are summed in (X, Y) order whatever warp or phase takes them, so Y
// does not depend on the schedule or on the batch (bitwise).
//
// Symmetries (as in the box kernel): middle rows (2 mb = J) sum mb1 <= X/2 and
// are folded once at the end (U[J-ma][J-mb] = (-1)^(ma+mb) conj U[ma][mb]);
// for X = Y the other rows sum mb1 <= mb2 with weight 2 off the diagonal.
// Energy by Euler's identity E = beta0 + (1/3) sum_J <U^J, Y^J>.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <utility>
#include <vector>

#ifdef PL_CHECKS
#include <cassert>
#define PL_DASSERT(cond) assert(cond)
#else
#define PL_DASSERT(cond) ((void)0)
#endif

namespace pl {

double snap_clebsch(int j1, int m1, int j2, int m2, int J, int M);  // snap.cu

__device__ __forceinline__ void griddep_wait_yi() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl_yi(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                 Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

namespace yib {
constexpr int TJ = 8;
constexpr int NT = 125;        // (X >= Y, J) triples at twojmax 8
constexpr int NFULL = 285;     // sum (J+1)^2
constexpr int NHALF = 155;     // sum (J+1)(J/2+1)
constexpr int ATOMS = 32;
constexpr int BOX_MAX = 4098;  // sum over triples of (X+1)(Y+1)
constexpr int ROWS = 25;       // (J, mb <= J/2) half rows
constexpr int NPH = 24;        // max phases (host: consecutive triples, code budget per phase)
constexpr int foff(int J) { return J * (J + 1) * (2 * J + 1) / 6; }
constexpr int rowoff(int J) { return (J / 2 + 1) * (J / 2 + 1) - (J % 2 == 0 ? J / 2 + 1 : 0); }  // rows of layers < J
constexpr int hoff(int J) {
  int h = 0;
  for (int j = 0; j < J; ++j) h += (j + 1) * (j / 2 + 1);
  return h;
}
// offset of triple (X, Y, J) in the box table, triples in (x, y <= x, J) order
constexpr int box_off(int X, int Y, int J) {
  int o = 0;
  for (int x = 0; x <= TJ; ++x)
    for (int y = 0; y <= x; ++y)
      for (int j = x - y; j <= (TJ < x + y ? TJ : x + y); j += 2) {
        if (x == X && y == Y && j == J) return o;
        o += (x + 1) * (y + 1);
      }
  return -1;
}
}  // namespace yib

__constant__ double c_box[yib::BOX_MAX];  // per triple: [Y+1][X+1], C(ma = a + b - SH; X a, Y b)

// full-matrix element f -> its source in the half-row storage: (src << 2) |
// (mirrored << 1) | (odd ma + mb); U[ma][mb] for 2 mb > J is (-1)^(ma+mb)
// conj(U[J-ma][J-mb]).  One warp expands one element f for its 32 atoms, so the
// lookup is a uniform constant-bank read.
struct BoxExpand {
  int e[yib::NFULL];
  constexpr BoxExpand() : e() {
    int f = 0;
    for (int J = 0; J <= yib::TJ; ++J)
      for (int mb = 0; mb <= J; ++mb)
        for (int ma = 0; ma <= J; ++ma, ++f) {
          const bool mir = 2 * mb > J;
          const int src = yib::hoff(J) + (mir ? (J - mb) * (J + 1) + (J - ma) : mb * (J + 1) + ma);
          e[f] = (src << 2) | (mir ? 2 : 0) | ((ma + mb) & 1);
        }
  }
};
__constant__ BoxExpand c_box_exp = BoxExpand();
// Y^dagger element o = hoff(J) + ma (J/2 + 1) + mb (column-interleaved half rows) ->
// (source half element << 12) | (half element of (mb, ma) << 2) | (mirrored << 1) | (odd ma + mb)
struct YtMap {
  int e[yib::NHALF];
  constexpr YtMap() : e() {
    for (int J = 0; J <= yib::TJ; ++J)
      for (int ma = 0; ma <= J; ++ma)
        for (int mb = 0; 2 * mb <= J; ++mb) {
          const int base = yib::hoff(J);
          const bool mir = 2 * ma > J;  // element (row ma, column mb) of the full matrix
          const int src = mir ? base + (J - ma) * (J + 1) + (J - mb) : base + ma * (J + 1) + mb;
          e[base + ma * (J / 2 + 1) + mb] =
              (src << 12) | ((base + mb * (J + 1) + ma) << 2) | (mir ? 2 : 0) | ((ma + mb) & 1);
        }
  }
};
__constant__ YtMap c_yt_map = YtMap();
__constant__ int c_box_code[yib::NT];  // X*100 + Y*10 + J
// compiled variants: (warps per CTA, CTAs per 32-atom block).  A block's rows
// are split over S CTAs when the batch has fewer blocks than SMs (latency of
// small systems); a row stays with one CTA for the whole kernel.
// (warps, CTAs per block): 1 CTA per block for large batches; a block's rows split
// over 2 CTAs below 148 blocks, over 4 below 37 (one CTA per SM either way)
constexpr int P_NV = 3;
constexpr int P_NW[P_NV] = {8, 8, 8};   // 2 warps per SMSP, 255 registers (12 warps: 168, measured slower)
constexpr int P_NS[P_NV] = {1, 2, 4};
constexpr int P_MAX_VW = 32;
constexpr int P_MAX_ITEMS = 400;  // (row, triple) items: 375 at twojmax 8
__constant__ int c_p_iseg[P_NV][yib::NPH][P_MAX_VW + 1];  // items of virtual warp w in phase p
// per item, decoded on the host: {tid, Y-row offset (elements), lo | hi << 8 | mb << 16 | mid << 24 | swap << 25, 0}
// The items live in global memory next to the potential's coefficients, 32 bytes each:
// the descriptor above and cy = coef[tid], so an item costs two independent 16-byte
// loads through L1 instead of an indexed constant load followed by a dependent global
// load (the per-item dispatch was 8.6 % of the kernel's stall samples, and the constant
// cache shares the GPC-level cache with the instruction fetches)
constexpr int P_REC_OFF = 2 * yib::NT + 2 * yib::NHALF;  // doubles before the records in the coefficient buffer
static std::vector<int4> g_items4;  // host copy of the schedule (device independent)
__constant__ int c_p_rowsplit[P_NV][yib::ROWS];          // CTA of the block that owns row r
__constant__ int c_p_nph;                                // phases in use

struct Cx {
  double re, im;
};

struct PItem {
  const Cx* Ul;  // full U matrices, this lane's atom
  Cx* yrow;      // Y half row (J, mb), this lane's atom
  double cy;     // coefficient of Z^{XY}_J in Y^J
  int mb, lo, hi;
  bool mid, swap;
  unsigned zaddr;  // shared-memory address of 16 zero bytes
};

// rows a in [A0, A1] of the band (the whole band except for (8, 8, 8), whose 61
// cells do not fit 255 registers and run as two halves)
template <int X, int Y, int J, int A0 = 0, int A1 = X>
__device__ __forceinline__ void ptri(const PItem& A) {
  constexpr int SH = (X + Y - J) / 2;
  constexpr int OFF = yib::box_off(X, Y, J);
  constexpr int FX = yib::foff(X), FY = yib::foff(Y);
  constexpr int AT = yib::ATOMS;
  Cx P[X + 1][Y + 1];
  const Cx* __restrict__ Ul = A.Ul;
  // one mb1 step; with PL_YI_PEEL the first one initialises P (P = ux uy exactly
  // as fma(ux, uy, 0) rounds: no zero fill), else P starts from zeros
  auto step = [&](const int mb1, const bool first) {
    const int mb2 = A.mb + SH - mb1;
    const double w = A.mid ? (2 * mb1 == X ? 0.5 : 1.0) : (A.swap ? (mb1 == mb2 ? 1.0 : 2.0) : 1.0);
    const double cbv = w * c_box[OFF + mb2 * (X + 1) + mb1];  // w C(mb; mb1), w exact
    const Cx* px = Ul + (FX + mb1 * (X + 1)) * AT;
    const Cx* py = Ul + (FY + mb2 * (Y + 1)) * AT;
    Cx ux[X + 1];
#pragma unroll
    for (int a = A0; a <= A1; ++a) ux[a] = px[a * AT];
#pragma unroll
    for (int b = 0; b <= Y; ++b) {
      const Cx v = py[b * AT];
      const Cx uy{cbv * v.re, cbv * v.im};
#pragma unroll
      for (int a = A0; a <= A1; ++a) {
        if (a + b < SH || a + b > SH + J) continue;  // outside the CG band (compile time)
        if (first) {
          P[a][b].re = ux[a].re * uy.re;
          P[a][b].im = ux[a].re * uy.im;
        } else {
          P[a][b].re = fma(ux[a].re, uy.re, P[a][b].re);
          P[a][b].im = fma(ux[a].re, uy.im, P[a][b].im);
        }
        P[a][b].re = fma(-ux[a].im, uy.im, P[a][b].re);
        P[a][b].im = fma(ux[a].im, uy.re, P[a][b].im);
      }
    }
  };
#ifdef PL_YI_PEEL
  if (A.lo > A.hi) return;  // no admissible mb1: no contribution
  step(A.lo, true);
#pragma unroll 1
  for (int mb1 = A.lo + 1; mb1 <= A.hi; ++mb1) step(mb1, false);
#else
  // P = 0: one 16-byte shared-memory load of zeros per band cell instead of two CS2R per
  // cell (the zero fill was 16 % of the kernel's static code, executed once per fetch;
  // volatile, or ptxas merges the loads and copies registers): 33.5 k -> 31.2 k
  // instructions, 1.638 -> 1.620 ms; corners are never read: no registers
#pragma unroll
  for (int a = A0; a <= A1; ++a)
#pragma unroll
    for (int b = 0; b <= Y; ++b) {
      if (a + b < SH || a + b > SH + J) continue;
      asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(P[a][b].re), "=d"(P[a][b].im) : "r"(A.zaddr));
    }
#pragma unroll 1
  for (int mb1 = A.lo; mb1 <= A.hi; ++mb1) step(mb1, false);
#endif
  // Z[ma] = sum_a C(ma; a) P[a][ma + SH - a], then Y[ma] += cy Z[ma] (the warp owns the row)
  Cx* yo = A.yrow;
#pragma unroll
  for (int ma = 0; ma <= J; ++ma) {
    Cx z{0.0, 0.0};
#pragma unroll
    for (int a = A0; a <= A1; ++a) {
      const int b = ma + SH - a;
      if (b < 0 || b > Y) continue;
      const double c = c_box[OFF + b * (X + 1) + a];
      z.re = fma(c, P[a][b].re, z.re);
      z.im = fma(c, P[a][b].im, z.im);
    }
    Cx y = yo[ma * AT];
    y.re = fma(A.cy, z.re, y.re);
    y.im = fma(A.cy, z.im, y.im);
    yo[ma * AT] = y;
  }
}

template <int NW>
__device__ __forceinline__ void ptri_dispatch(int tid, const PItem& A) {
  switch (tid) {
    // one case per triple, in (x, y <= x, J) order (generated)
#include "snap_yi8_cases.inc"
    default: break;
  }
}

#ifdef PL_YI_TIMING
// per (block, phase, warp): cycles from the phase start to the warp's arrival at the
// phase barrier (diagnostic build, scripts/probe_yi_phases.py)
constexpr int YT_BLOCKS = 4096;
__device__ long long g_yi_timing[YT_BLOCKS][yib::NPH][P_MAX_VW];
__device__ unsigned long long g_yi_item_cyc[yib::NT][5];  // per (triple, mb): summed cycles, and counts
__device__ unsigned long long g_yi_item_cnt[yib::NT][5];
#endif

template <int NW, int V, int S>
__global__ void __launch_bounds__(NW * 32, 1)
k_snap_yi_p(int64_t natoms, double beta0, const double* __restrict__ coef, const double* __restrict__ vs,
            const Cx* __restrict__ utot, Cx* __restrict__ ylist, double* __restrict__ eatom,
            double* __restrict__ erow_g, Cx* __restrict__ ytlist) {
  griddep_wait_yi();
  extern __shared__ double smem[];
  Cx* Uf = reinterpret_cast<Cx*>(smem);                 // [NFULL][32] full U matrices
  Cx* Ys = Uf + yib::NFULL * yib::ATOMS;               // [NHALF][32] Y half rows
  double* erow = reinterpret_cast<double*>(Ys + yib::NHALF * yib::ATOMS);  // [ROWS][32] energy per row
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t blk = blockIdx.x / S;
  const int split = (int)(blockIdx.x - blk * S);
  const int64_t a0 = blk * yib::ATOMS;
  const int na_blk = (int)min((int64_t)yib::ATOMS, natoms - a0);
  // the block's U_tot half rows are one contiguous range: one bulk async copy
  // (TMA engine) into the Y area, which is free until the expansion is done
  __shared__ __align__(8) uint64_t mbar;
  const Cx* Ust = reinterpret_cast<const Cx*>(Ys);
  {
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&mbar);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // the block this SM most likely runs next (one CTA per SM, blocks dispatched in
      // order): its U_tot towards L2 while this block computes
      const int64_t nxt = blk + 148;
#ifndef PL_NO_YI_PF
      if (S == 1 && nxt * yib::ATOMS < natoms) {
#else
      if (false) {
#endif
        const int64_t nn = min((int64_t)yib::ATOMS, natoms - nxt * yib::ATOMS);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(utot + nxt * yib::ATOMS * yib::NHALF),
                     "r"((unsigned)(sizeof(Cx) * yib::NHALF * nn))
                     : "memory");
      }
      const unsigned bytes = (unsigned)(sizeof(Cx) * yib::NHALF * na_blk);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              (unsigned)__cvta_generic_to_shared(Ys)),
          "l"(utot + a0 * yib::NHALF), "r"(bytes), "r"(bar)
          : "memory");
    }
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(bar)
        : "memory");
  }
  for (int f = warp; f < yib::NFULL; f += NW) {  // one full-matrix element per warp, lanes = atoms
    const int code = c_box_exp.e[f];
    Cx v{0.0, 0.0};
    if (lane < na_blk) {
      const Cx w = Ust[lane * yib::NHALF + (code >> 2)];
      v = !(code & 2) ? w : ((code & 1) ? Cx{-w.re, w.im} : Cx{w.re, -w.im});
    }
    Uf[f * yib::ATOMS + lane] = v;
  }
  __syncthreads();  // staged U_tot consumed before Y is cleared
  for (int t = threadIdx.x; t < yib::NHALF * yib::ATOMS; t += blockDim.x) Ys[t] = Cx{0.0, 0.0};
  for (int t = threadIdx.x; t < yib::ROWS * yib::ATOMS; t += blockDim.x) erow[t] = 0.0;
  __syncthreads();
  const int vw = split * NW + warp;  // virtual warp of the block's schedule
  const int nph = c_p_nph;
  for (int ph = 0; ph < nph; ++ph) {
#ifdef PL_YI_TIMING
    const long long t_ph = clock64();
#endif
    // (the bound in a register: read from constant memory in the loop condition it was
    // re-loaded after every body, whose asm statements clobber memory)
    const int it_end = c_p_iseg[V][ph][vw + 1];
    for (int it = c_p_iseg[V][ph][vw]; it < it_end; ++it) {
      PL_DASSERT(it < P_MAX_ITEMS);
      const double* rec = coef + P_REC_OFF + 4 * (V * P_MAX_ITEMS + it);
      const int4 item = __ldg(reinterpret_cast<const int4*>(rec));  // host-decoded descriptor
      const double cy = __ldg(rec + 2);
      const int tid = item.x;
      PL_DASSERT(tid < yib::NT && item.y >= 0 && item.y < yib::NHALF);
      PItem A;
      A.Ul = Uf + lane;
      A.yrow = Ys + item.y * yib::ATOMS + lane;
      A.cy = cy;
      A.zaddr = (unsigned)__cvta_generic_to_shared(erow);  // zero until the energy pass
      A.lo = item.z & 0xff;
      A.hi = (item.z >> 8) & 0xff;
      A.mb = (item.z >> 16) & 0xff;
      A.mid = (item.z >> 24) & 1;
      A.swap = (item.z >> 25) & 1;
#ifdef PL_YI_TIMING
      const long long t_it = clock64();
#endif
      ptri_dispatch<NW>(tid, A);
#ifdef PL_YI_TIMING
      if (lane == 0) {
        atomicAdd(&g_yi_item_cyc[tid][A.mb], (unsigned long long)(clock64() - t_it));
        atomicAdd(&g_yi_item_cnt[tid][A.mb], 1ull);
      }
#endif
    }
#ifdef PL_YI_TIMING
    if (lane == 0 && blockIdx.x < YT_BLOCKS) g_yi_timing[blockIdx.x][ph][vw] = clock64() - t_ph;
#endif
    __syncthreads();  // next phase: rows change owners
  }
  // middle rows: Y[ma] += (-1)^(J/2+ma) conj(Y[J-ma]) for ma <= J/2 (the images of
  // the mb1 > X/2 terms), then the upper half is cleared
  for (int t = threadIdx.x; t < 5 * yib::ATOMS; t += blockDim.x) {
    const int J = 2 * (t >> 5), at = t & 31, mb = J / 2;
    if (S > 1 && c_p_rowsplit[V][yib::rowoff(J) + mb] != split) continue;
    Cx* y = Ys + (yib::hoff(J) + mb * (J + 1)) * yib::ATOMS + at;
    for (int ma = 0; ma < mb; ++ma) {
      Cx lo = y[ma * yib::ATOMS];
      const Cx up = y[(J - ma) * yib::ATOMS];
      const bool neg = ((mb + ma) & 1) != 0;
      lo.re += neg ? -up.re : up.re;
      lo.im += neg ? up.im : -up.im;
      y[ma * yib::ATOMS] = lo;
      y[(J - ma) * yib::ATOMS] = Cx{0.0, 0.0};
    }
    Cx c = y[mb * yib::ATOMS];
    y[mb * yib::ATOMS] = Cx{c.re + c.re, 0.0};
  }
  __syncthreads();
  // energy: E - beta0 is cubic in U and Y = dE/dU, so E = beta0 + (1/3) sum_J <U^J, Y^J>
  // (half rows with the full-matrix weights); per row, rows summed in row order
  for (int t = threadIdx.x; t < yib::ROWS * yib::ATOMS; t += blockDim.x) {
    const int r = t >> 5, at = t & 31;
    if (S > 1 && c_p_rowsplit[V][r] != split) continue;
    int J = 0;
    while (J < yib::TJ && r >= yib::rowoff(J + 1)) ++J;
    const int mb = r - yib::rowoff(J);
    const Cx* u = Uf + (yib::foff(J) + mb * (J + 1)) * yib::ATOMS + at;
    const Cx* y = Ys + (yib::hoff(J) + mb * (J + 1)) * yib::ATOMS + at;
    double e = 0.0;
    for (int ma = 0; ma <= J; ++ma) {
      const double w = (2 * mb < J || 2 * ma < J) ? 2.0 : (2 * ma == J ? 1.0 : 0.0);
      const Cx uu = u[ma * yib::ATOMS], yy = y[ma * yib::ATOMS];
      e = fma(w, fma(uu.re, yy.re, uu.im * yy.im), e);
    }
    erow[t] = e * (1.0 / 3.0);
  }
  __syncthreads();
  // rows owned by this CTA -> global (all rows when S = 1), as S (.) Y: the force
  // kernels propagate the coefficient-free V = U / S (snap.cu, vstep), and
  // Re<U, Y> = Re<V, S (.) Y>
  if constexpr (S == 1) {
    // The block's Y is one contiguous range of ylist ([atom][h]).  It is transposed into
    // that layout in shared memory (the U area is dead after the energy pass; [h][atom]
    // reads and [atom][h] writes are both conflict-free: 155 x 16 B per atom puts the 32
    // lanes on 8 x 4 distinct banks) and leaves as ONE bulk async store (TMA engine),
    // instead of 16-byte stores to 8 atoms' rows per warp.  S (.) Y^dagger for the pair
    // force kernel (k_snap_ytrans' arithmetic, bit for bit: the stored S (.) Y element,
    // mirrored through the inversion symmetry for ma > J/2, times vs2 = S^2, conjugated;
    // column-interleaved [J][ma][mb <= J/2]) is built from the transposed copy into the Y
    // area and leaves the same way: no k_snap_ytrans launch re-reading Y from HBM.
    double2* T = reinterpret_cast<double2*>(Uf);
    const double2* Y2 = reinterpret_cast<const double2*>(Ys);
#pragma unroll 5
    for (int h = warp; h < yib::NHALF; h += NW) {
      const double sc = __ldg(vs + h);
      const double2 y = Y2[h * yib::ATOMS + lane];
      T[lane * yib::NHALF + h] = make_double2(y.x * sc, y.y * sc);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const unsigned bytes = (unsigned)(sizeof(Cx) * yib::NHALF * na_blk);
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(ylist + a0 * yib::NHALF),
                   "r"((unsigned)__cvta_generic_to_shared(T)), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (ytlist) {
      const double* vs2 = vs + yib::NHALF;
      double2* T2 = reinterpret_cast<double2*>(Ys);  // Y fully consumed above
#pragma unroll 5
      for (int o = warp; o < yib::NHALF; o += NW) {
        const int code = c_yt_map.e[o];
        PL_DASSERT((code >> 12) >= 0 && (code >> 12) < yib::NHALF && ((code >> 2) & 0x3ff) < yib::NHALF);
        double2 v = T[lane * yib::NHALF + (code >> 12)];
        if (code & 2) v = (code & 1) ? make_double2(-v.x, v.y) : make_double2(v.x, -v.y);
        const double f = __ldg(vs2 + ((code >> 2) & 0x3ff));
        T2[lane * yib::NHALF + o] = make_double2(f * v.x, -(f * v.y));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(ytlist + a0 * yib::NHALF),
                     "r"((unsigned)__cvta_generic_to_shared(T2)), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
  } else {
    // 8 consecutive threads take 8 consecutive atoms of one element h: conflict-free
    // shared-memory reads ([h][atom] layout), 16-byte global stores
    for (int t = threadIdx.x; t < yib::ATOMS * yib::NHALF; t += blockDim.x) {
      const int rest = t >> 3, h = rest % yib::NHALF, at = (rest / yib::NHALF) * 8 + (t & 7);
      if (at >= na_blk) continue;
      int J = 0;
      while (J < yib::TJ && h >= yib::hoff(J + 1)) ++J;
      const int r = yib::rowoff(J) + (h - yib::hoff(J)) / (J + 1);
      if (c_p_rowsplit[V][r] != split) continue;
      const Cx y = Ys[h * yib::ATOMS + at];
      const double sc = __ldg(vs + h);
      ylist[(a0 + at) * yib::NHALF + h] = Cx{y.re * sc, y.im * sc};
    }
  }
  if (S == 1) {
    if (warp == 0 && lane < na_blk) {
      double e = beta0;
      for (int r = 0; r < yib::ROWS; ++r) e += erow[r * yib::ATOMS + lane];
      eatom[a0 + lane] = e;
    }
    // the staging areas stay valid until the bulk stores have read them (.read: the writes
    // complete with the grid; a full wait_group costs a CCTL.IVALL and the drain, ~1 us per CTA)
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  } else {
    for (int t = threadIdx.x; t < yib::ROWS * na_blk; t += blockDim.x) {
      const int r = t / na_blk, at = t - r * na_blk;
      if (c_p_rowsplit[V][r] == split) erow_g[(int64_t)r * natoms + a0 + at] = erow[r * yib::ATOMS + at];
    }
  }
}

// split mode: E_i = beta0 + sum over rows in row order (the S = 1 arithmetic)
__global__ void k_box_energy(int64_t natoms, double beta0, const double* __restrict__ erow_g,
                             double* __restrict__ eatom) {
  griddep_wait_yi();
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < natoms; a += (int64_t)gridDim.x * blockDim.x) {
    double e = beta0;
    for (int r = 0; r < yib::ROWS; ++r) e += erow_g[(int64_t)r * natoms + a];
    eatom[a] = e;
  }
}

// ------------------------------------------------------------------ host schedule
namespace {

struct Triple {
  int X, Y, J;
};

std::vector<Triple> triples8() {
  std::vector<Triple> t;
  for (int x = 0; x <= yib::TJ; ++x)
    for (int y = 0; y <= x; ++y)
      for (int J = x - y; J <= std::min(yib::TJ, x + y); J += 2) t.push_back({x, y, J});
  return t;
}

int row_index(int J, int mb) { return yib::rowoff(J) + mb; }

// cost of item (triple, mb) for the k_snap_yi_p body: per summed mb1, band
// products (4 DFMA) + the C(mb; mb1) scaling + the column loads; epilogue per
// band cell and per Y element.  (Per-item cycles measured in a PL_YI_TIMING build
// correlate at 0.88 with this model, but scheduling by them balanced the phases
// worse, 0.921 vs 0.944: an item's cost depends on what runs beside it.)
double item_cost(const Triple& t, int mb) {
  const int SH = (t.X + t.Y - t.J) / 2;
  const bool mid = 2 * mb == t.J, swap = (t.X == t.Y) && !mid;
  const int lo = std::max(0, mb + SH - t.Y);
  const int hi = mid ? t.X / 2 : (swap ? (mb + SH) / 2 : std::min(t.X, mb + SH));
  int K = 0;
  for (int mb1 = lo; mb1 <= hi; ++mb1) K += (mb + SH - mb1 >= 0 && mb + SH - mb1 <= t.Y);
  int band = 0;
  for (int a = 0; a <= t.X; ++a)
    for (int b = 0; b <= t.Y; ++b) band += (a + b >= SH && a + b <= SH + t.J);
  return K * (4.0 * band + 2.0 * (t.Y + 1) + 3.0 * (t.X + t.Y + 2) + 12.0) + 2.0 * band + 5.0 * (t.J + 1) + 40.0;
}

// jobs (cost, id) -> NB bins: LPT, then deterministic local search (single moves
// and pairwise swaps) that lowers the makespan, ties broken by the sum of squares.
// Returns bin[id] (ids < max id + 1; unused ids map to -1).
std::vector<int> balance(const std::vector<std::pair<double, int>>& jobs_in, int NB) {
  std::vector<std::pair<double, int>> jobs(jobs_in);
  std::stable_sort(jobs.begin(), jobs.end(), [](auto& a, auto& b) { return a.first > b.first; });
  const int nj = (int)jobs.size();
  std::vector<int> asg(nj);
  std::vector<double> wl(NB, 0.0);
  for (int i = 0; i < nj; ++i) {
    const int w = (int)(std::min_element(wl.begin(), wl.end()) - wl.begin());
    asg[i] = w;
    wl[w] += jobs[i].first;
  }
  auto score = [](const std::vector<double>& l) {
    double mx = 0.0, sq = 0.0;
    for (double v : l) {
      mx = std::max(mx, v);
      sq += v * v;
    }
    return std::make_pair(mx, sq);
  };
  for (bool improved = true; improved;) {
    improved = false;
    auto cur = score(wl);
    for (int i = 0; i < nj; ++i)
      for (int w = 0; w < NB; ++w) {
        if (w == asg[i]) continue;
        std::vector<double> nl(wl);
        nl[asg[i]] -= jobs[i].first;
        nl[w] += jobs[i].first;
        auto sc = score(nl);
        if (sc < cur) {
          wl = nl;
          asg[i] = w;
          cur = sc;
          improved = true;
        }
      }
    for (int i = 0; i < nj; ++i)
      for (int j = i + 1; j < nj; ++j) {
        const int a = asg[i], b = asg[j];
        if (a == b) continue;
        std::vector<double> nl(wl);
        nl[a] += jobs[j].first - jobs[i].first;
        nl[b] += jobs[i].first - jobs[j].first;
        auto sc = score(nl);
        if (sc < cur) {
          wl = nl;
          std::swap(asg[i], asg[j]);
          cur = sc;
          improved = true;
        }
      }
  }
  int maxid = -1;
  for (auto& j : jobs_in) maxid = std::max(maxid, j.second);
  std::vector<int> out(maxid + 1, -1);
  for (int i = 0; i < nj; ++i) out[jobs[i].second] = asg[i];
  return out;
}

}  // namespace

// Upload the CG box table, the triple codes and the per-variant phase schedules
// (twojmax 8; call once per device).  *balance_out: work-weighted mean / max warp
// load of the S = 1 schedule over the phases (cost model).
cudaError_t snap_yi8_setup(double* balance_out) {
  const auto T = triples8();
  if ((int)T.size() != yib::NT) return cudaErrorInvalidValue;
  std::vector<double> box;
  std::vector<int> code;
  for (const auto& t : T) {
    const int sh = (t.X + t.Y - t.J) / 2;
    if ((int)box.size() != yib::box_off(t.X, t.Y, t.J)) return cudaErrorInvalidValue;
    for (int b = 0; b <= t.Y; ++b)
      for (int a = 0; a <= t.X; ++a) {
        const int ma = a + b - sh;
        box.push_back(ma >= 0 && ma <= t.J ? snap_clebsch(t.X, 2 * a - t.X, t.Y, 2 * b - t.Y, t.J, 2 * ma - t.J) : 0.0);
      }
    code.push_back(t.X * 100 + t.Y * 10 + t.J);
  }
  // phases: consecutive triples (code order, ascending X) whose bodies fit the
  // budget (estimated SASS bytes; PL_YI_PHASE_KB, default 90 KB; round 2 first measured
  // 1.70 ms at 100-140 KB vs 1.79 at 60 and 2.5-2.6 at 170 KB-1 phase, larger config)
  // (re-scanned on the final kernel, larger config: 70-128 KB give 1.58, 1.56, 1.52 (80),
  // 1.55 (84), 1.517 (88), 1.491 (90, 91), 1.555 (92), 1.516 (94), 1.518 (100), 1.508 (110),
  // 1.53-1.55 (120-128) ms: the budget decides which triples share a phase, hence the balance)
  double budget = 90.0 * 1024.0;
  if (const char* e = getenv("PL_YI_PHASE_KB")) budget = atof(e) * 1024.0;
  std::vector<int> tphase(yib::NT, 0);
  int nph = 1;
  {
    double acc = 0.0;
    for (int tid = 0; tid < yib::NT; ++tid) {
      const Triple& t = T[tid];
      const int SH = (t.X + t.Y - t.J) / 2;
      int band = 0;
      for (int a = 0; a <= t.X; ++a)
        for (int b = 0; b <= t.Y; ++b) band += (a + b >= SH && a + b <= SH + t.J);
      const double bytes = 21.3 * (6.0 * band + 3.0 * (t.Y + 1) + (t.X + 1) + 5.0 * (t.J + 1) + 30.0);
      if (acc > 0.0 && acc + bytes > budget) {
        if (nph == yib::NPH) return cudaErrorInvalidValue;
        ++nph;
        acc = 0.0;
      }
      acc += bytes;
      tphase[tid] = nph - 1;
    }
  }
  // items per (row, phase)
  std::vector<std::vector<std::vector<int>>> ritems(yib::ROWS, std::vector<std::vector<int>>(yib::NPH));
  std::vector<std::vector<double>> rcost(yib::ROWS, std::vector<double>(yib::NPH, 0.0));
  for (int tid = 0; tid < yib::NT; ++tid) {
    const Triple& t = T[tid];
    for (int mb = 0; 2 * mb <= t.J; ++mb) {
      const int r = row_index(t.J, mb), ph = tphase[tid];
      ritems[r][ph].push_back((tid << 16) | (t.J << 8) | mb);
      rcost[r][ph] += item_cost(t, mb);
    }
  }
  std::vector<int> iseg(P_NV * yib::NPH * (P_MAX_VW + 1), 0), items(P_NV * P_MAX_ITEMS, 0),
      rowsplit(P_NV * yib::ROWS, 0);
  double bal_num = 0.0, bal_den = 0.0;
  for (int v = 0; v < P_NV; ++v) {
    const int NW = P_NW[v], NS = P_NS[v];
    // rows -> CTAs of the block (fixed for the whole kernel)
    std::vector<int> cta(yib::ROWS, 0);
    if (NS > 1) {
      std::vector<std::pair<double, int>> jobs;
      for (int r = 0; r < yib::ROWS; ++r) {
        double c = 0.0;
        for (int ph = 0; ph < yib::NPH; ++ph) c += rcost[r][ph];
        jobs.push_back({c, r});
      }
      cta = balance(jobs, NS);
    }
    for (int r = 0; r < yib::ROWS; ++r) rowsplit[v * yib::ROWS + r] = cta[r];
    int n = 0;
    for (int ph = 0; ph < yib::NPH; ++ph) {
      std::vector<int> vwarp(yib::ROWS, -1);
      if (ph >= nph) {
        for (int w = 0; w <= P_MAX_VW; ++w) iseg[(v * yib::NPH + ph) * (P_MAX_VW + 1) + w] = n;
        continue;
      }
      for (int s = 0; s < NS; ++s) {
        std::vector<std::pair<double, int>> jobs;
        for (int r = 0; r < yib::ROWS; ++r)
          if (cta[r] == s && rcost[r][ph] > 0.0) jobs.push_back({rcost[r][ph], r});
        if (jobs.empty()) continue;
        const auto bin = balance(jobs, NW);
        std::vector<double> load(NW, 0.0);
        for (auto& j : jobs) {
          vwarp[j.second] = s * NW + bin[j.second];
          load[bin[j.second]] += j.first;
        }
        if (v == 0) {
          double sum = 0.0, mx = 0.0;
          for (double l : load) {
            sum += l;
            mx = std::max(mx, l);
          }
          bal_num += sum / NW;
          bal_den += mx;
        }
      }
      for (int w = 0; w <= P_MAX_VW; ++w) {
        iseg[(v * yib::NPH + ph) * (P_MAX_VW + 1) + w] = n;
        if (w == P_MAX_VW) break;
        std::vector<std::pair<int, int>> mine;  // ((X, Y, J, mb) key, item)
        for (int r = 0; r < yib::ROWS; ++r)
          if (vwarp[r] == w)
            for (int it : ritems[r][ph]) {
              const Triple& t = T[it >> 16];
              mine.push_back({((t.X * 10 + t.Y) * 10 + t.J) * 10 + (it & 0xff), it});
            }
        std::sort(mine.begin(), mine.end());
        for (auto& m : mine) {
          if (n >= P_MAX_ITEMS) return cudaErrorInvalidValue;
          items[v * P_MAX_ITEMS + n++] = m.second;
        }
      }
    }
  }
  if (balance_out) *balance_out = bal_den > 0.0 ? bal_num / bal_den : 1.0;
  cudaError_t e;
  if ((e = cudaMemcpyToSymbol(c_box, box.data(), sizeof(double) * box.size())) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(c_box_code, code.data(), sizeof(int) * code.size())) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(c_p_nph, &nph, sizeof(int))) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(c_p_iseg, iseg.data(), sizeof(int) * iseg.size())) != cudaSuccess) return e;
  std::vector<int4> items4(items.size());
  for (size_t i = 0; i < items.size(); ++i) {
    const int it = items[i], tid = it >> 16, J = (it >> 8) & 0xff, mb = it & 0xff;
    const Triple& t = T[tid];
    const int SH = (t.X + t.Y - J) / 2;
    const bool mid = 2 * mb == J, swap = (t.X == t.Y) && !mid;
    const int lo = std::max(0, mb + SH - t.Y);
    const int hi = mid ? t.X / 2 : (swap ? (mb + SH) / 2 : std::min(t.X, mb + SH));
    items4[i] = make_int4(tid, yib::hoff(J) + mb * (J + 1),
                          lo | (hi << 8) | (mb << 16) | ((mid ? 1 : 0) << 24) | ((swap ? 1 : 0) << 25), 0);
  }
  g_items4 = items4;
  if ((e = cudaMemcpyToSymbol(c_p_rowsplit, rowsplit.data(), sizeof(int) * rowsplit.size())) != cudaSuccess)
    return e;
  return cudaSuccess;
}

// item records {descriptor, cy = coef[tid], 0} of the three variants, appended to the
// potential's coefficient buffer (after coef, beta, vs, vs2: P_REC_OFF doubles)
bool snap_yi8_append_records(const double* coef, std::vector<double>& out) {
  if ((int)out.size() != P_REC_OFF || g_items4.size() != (size_t)P_NV * P_MAX_ITEMS) return false;
  for (const int4& it : g_items4) {
    double d[4] = {0.0, 0.0, 0.0, 0.0};
    static_assert(sizeof(int4) == 2 * sizeof(double), "record layout");
    memcpy(d, &it, sizeof(int4));
    d[2] = (it.x >= 0 && it.x < yib::NT) ? coef[it.x] : 0.0;
    out.insert(out.end(), d, d + 4);
  }
  return true;
}

template <int NW, int V, int S>
static cudaError_t p_launch(cudaStream_t st, int64_t natoms, double beta0, const double* coef, const double* vs,
                            const void* utot, void* ylist, double* eatom, double* erow_g, void* ytlist) {
  const size_t sm = sizeof(Cx) * (yib::NFULL + yib::NHALF) * yib::ATOMS + sizeof(double) * yib::ROWS * yib::ATOMS;
  static std::atomic<uint64_t> attr_devs{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_devs.load() & bit)) {  // exactly the dynamic size: the static mbarrier counts against the 227 KB too
    cudaError_t e = cudaFuncSetAttribute(k_snap_yi_p<NW, V, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    attr_devs.fetch_or(bit);
  }
  const unsigned grid = (unsigned)(S * ((natoms + yib::ATOMS - 1) / yib::ATOMS));
  cudaError_t e = launch_pdl_yi(k_snap_yi_p<NW, V, S>, dim3(grid), dim3(NW * 32), sm, st, natoms, beta0, coef,
                                vs, (const Cx*)utot, (Cx*)ylist, eatom, erow_g, (Cx*)ytlist);
  if (e != cudaSuccess) return e;
  if (S > 1)
    e = launch_pdl_yi(k_box_energy, dim3((unsigned)((natoms + 255) / 256)), dim3(256), 0, st, natoms, beta0,
                      (const double*)erow_g, eatom);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// split rows over 2 CTAs per block when the batch has fewer blocks than SMs
// (erow_g: 25 x natoms doubles of scratch).  ytlist (optional): S (.) Y^dagger, written
// by the unsplit kernel; *yt_done tells the caller whether it was (else k_snap_ytrans).
cudaError_t snap_box_launch(cudaStream_t st, int64_t natoms, double beta0, const double* coef, const double* vs,
                            const void* utot, void* ylist, double* eatom, double* erow_g, void* ytlist,
                            bool* yt_done) {
  const int64_t blocks = (natoms + yib::ATOMS - 1) / yib::ATOMS;
  const bool split = blocks < 148 && erow_g;
  static const int max_split = [] {  // PL_YI_SPLIT_MAX=2: no 4-way split (A/B)
    const char* e = getenv("PL_YI_SPLIT_MAX");
    return e ? atoi(e) : 4;
  }();
  static const bool fuse_yt = [] {  // PL_YI_YT=0: separate k_snap_ytrans at every size (A/B, tests)
    const char* e = getenv("PL_YI_YT");
    return !(e && e[0] == '0');
  }();
  if (yt_done) *yt_done = false;
  if (split && max_split >= 4 && 4 * blocks <= 148)
    return p_launch<8, 2, 4>(st, natoms, beta0, coef, vs, utot, ylist, eatom, erow_g, nullptr);
  if (split) return p_launch<8, 1, 2>(st, natoms, beta0, coef, vs, utot, ylist, eatom, erow_g, nullptr);
  void* yt = fuse_yt ? ytlist : nullptr;
  if (yt_done) *yt_done = yt != nullptr;
  return p_launch<8, 0, 1>(st, natoms, beta0, coef, vs, utot, ylist, eatom, erow_g, yt);
}

}  // namespace pl

// diagnostic: per (block, phase, warp) cycle counts of the last Y launch (only in a
// build with -DPL_YI_TIMING; PL_EARG otherwise).  h_out: 4096 x 24 x 24 int64.
extern "C" int pl_yi_timing(int64_t* h_out) {
#ifdef PL_YI_TIMING
  if (!h_out) return 1;
  if (cudaMemcpyFromSymbol(h_out, pl::g_yi_timing, sizeof(pl::g_yi_timing)) != cudaSuccess) return 2;
  // then per (triple, mb) summed item cycles and counts (125 x 5 each)
  int64_t* p = h_out + sizeof(pl::g_yi_timing) / sizeof(int64_t);
  if (cudaMemcpyFromSymbol(p, pl::g_yi_item_cyc, sizeof(pl::g_yi_item_cyc)) != cudaSuccess) return 2;
  return cudaMemcpyFromSymbol(p + pl::yib::NT * 5, pl::g_yi_item_cnt, sizeof(pl::g_yi_item_cnt)) == cudaSuccess ? 0 : 2;
#else
  (void)h_out;
  return 1;
#endif
}
