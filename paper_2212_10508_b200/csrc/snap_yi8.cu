// SNAP Z/Y contraction, twojmax = 8, "box" form (k_snap_yi_box).
//
// Lanes = atoms (32 per CTA, U^J of all layers expanded to full matrices in
// shared memory, as k_snap_yi_six); warps own (J, mb) half rows by an LPT
// schedule.  For every triple (X, Y, J) of a row and every admissible mb1,
// both U columns U^X[.][mb1] and U^Y[.][mb2] are loaded into registers (the
// b-side CG factor C(mb, mb1) folded into U^Y) and ALL (X+1)(Y+1) products are
// accumulated on their anti-diagonal s = ma1 + ma2 (compile-time register
// index), weighted by the box table C(ma = s - SH, ma1) that is zero outside
// the CG band.  The code per (X, Y) is one branch-free block of independent
// FMA chains with constant-bank coefficients at compile-time offsets; the
// corner products it spends on zeros (~40%) are cheaper than the per-product
// index arithmetic and predication of the banded loops (k_snap_yi_six).  The
// diagonals are mapped to the z row (runtime shift SH) through the warp's
// shared strip once per (triple, row).
//
// Separate translation unit: the box table (32.8 KB) has its own constant
// bank next to snap.cu's CG blocks.
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace pl {

__device__ __forceinline__ void griddep_wait_yi() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// programmatic dependent launch (see pl_common.cuh launch_pdl)
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
constexpr int foff(int J) { return J * (J + 1) * (2 * J + 1) / 6; }
constexpr int rowoff(int J) { return (J / 2 + 1) * (J / 2 + 1) - (J % 2 == 0 ? J / 2 + 1 : 0); }  // rows of layers < J
constexpr int hoff(int J) {
  int h = 0;
  for (int j = 0; j < J; ++j) h += (j + 1) * (j / 2 + 1);
  return h;
}
}  // namespace yib

__constant__ double c_box[yib::BOX_MAX];  // per triple: [Y+1][X+1]

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
__constant__ int c_box_off[yib::NT];
__constant__ int c_box_code[yib::NT];         // X*100 + Y*10 + J
constexpr int BOX_MAX_ITEMS = 400;            // (row, triple) pairs: 375 at twojmax 8
// compiled variants: (warps per CTA, CTAs per 32-atom block).  A block's
// (J, mb) rows are split over S CTAs when the batch has fewer blocks than SMs
// (latency of small systems); each row stays with one warp.  (3 warps per SM
// sub-partition leave 168 registers per thread; 4 would force 128 and spill.)
constexpr int BOX_NV = 3;
constexpr int BOX_NW[BOX_NV] = {12, 8, 12};
constexpr int BOX_NS[BOX_NV] = {1, 1, 2};
constexpr int BOX_ROWS = 25;                              // (J, mb <= J/2) half rows at twojmax 8
__constant__ int c_box_iseg[BOX_NV][BOX_ROWS + 1];        // items of virtual warp w: [iseg[w], iseg[w+1])
__constant__ int c_box_items[BOX_NV][BOX_MAX_ITEMS];     // tid << 16 | J << 8 | mb
__constant__ int c_box_rowsplit[BOX_NV][BOX_ROWS];       // CTA of the block that owns row r

struct Cx {
  double re, im;
};

// The middle row (2 mb = J): the terms of mb1 and X - mb1 are images of each
// other under U[J-ma][J-mb] = (-1)^(ma+mb) conj(U[ma][mb]) (CG included), so
// only mb1 <= X/2 is summed (the self-image X/2 with weight 1/2, exact) over the
// whole band ma = 0..J; the kernel folds the row's upper half onto the lower
// half once all items are in (fold_middle_rows).
template <int X>
__device__ __forceinline__ void box_x(const Cx* __restrict__ Ul, int Y, int SH, int J, bool mid, int mb, int boff,
                                      double cy, Cx* __restrict__ yrow) {
  const int jtop = J;
  constexpr int S = X + yib::TJ;
  constexpr int FX = yib::foff(X);
  Cx d[S + 1];
#pragma unroll
  for (int s = 0; s <= S; ++s) d[s] = Cx{0.0, 0.0};
  const double* cb = c_box + boff;  // [Y+1][X+1]: cb[b * (X + 1) + a] = C(ma = a + b - SH, ma1 = a)
  const int FY = yib::foff(Y);
  // X = Y (other rows): the (mb1, ma1) and (mb2, ma2) factors swap roles with an
  // unchanged CG product, so mb1 <= mb2 is summed with weight 2 off the diagonal
  const bool swap = (Y == X) && !mid;
  const int lo = max(0, mb + SH - Y);
  const int hi = mid ? X / 2 : (swap ? (mb + SH) / 2 : min(X, mb + SH));
#pragma unroll 1
  for (int mb1 = lo; mb1 <= hi; ++mb1) {
    const int mb2 = mb + SH - mb1;
    const double w = mid ? (2 * mb1 == X ? 0.5 : 1.0) : (swap ? (mb1 == mb2 ? 1.0 : 2.0) : 1.0);
    const double cbv = w * cb[mb2 * (X + 1) + mb1];  // w C(mb, mb1), w exact
    const Cx* px = Ul + (FX + mb1 * (X + 1)) * yib::ATOMS;
    const Cx* py = Ul + (FY + mb2 * (Y + 1)) * yib::ATOMS;
    Cx ux[X + 1];
#pragma unroll
    for (int a = 0; a <= X; ++a) ux[a] = px[a * yib::ATOMS];
    // element b of the U^Y column times row block b of the box: X+1 independent
    // diagonals (skipping the zero corners per product costs more than it saves)
#pragma unroll
    for (int b = 0; b <= yib::TJ; ++b) {
      if (b > Y) break;
      const Cx v = py[b * yib::ATOMS];
      const Cx uy{cbv * v.re, cbv * v.im};
#pragma unroll
      for (int a = 0; a <= X; ++a) {
        const double c = cb[b * (X + 1) + a];
        const double tr = c * ux[a].re, ti = c * ux[a].im;
        d[a + b].re = fma(tr, uy.re, d[a + b].re);
        d[a + b].im = fma(tr, uy.im, d[a + b].im);
        d[a + b].re = fma(-ti, uy.im, d[a + b].re);
        d[a + b].im = fma(ti, uy.re, d[a + b].im);
      }
    }
  }
  // diagonal s -> element ma = s - SH of the Y row (the warp owns the row)
  Cx* yo = yrow - SH * yib::ATOMS;
#pragma unroll
  for (int s = 0; s <= S; ++s) {
    if (s >= SH && s <= SH + jtop) {
      Cx y = yo[s * yib::ATOMS];
      y.re = fma(cy, d[s].re, y.re);
      y.im = fma(cy, d[s].im, y.im);
      yo[s * yib::ATOMS] = y;
    }
  }
}

constexpr int box_regs(int nw) { return nw <= 8 ? 255 : 168; }

template <int NW, int V, int S>
__global__ void __maxnreg__(box_regs(NW))
k_snap_yi_box(int64_t natoms, double beta0, const double* __restrict__ coef, const Cx* __restrict__ utot,
              Cx* __restrict__ ylist, double* __restrict__ eatom, double* __restrict__ erow_g) {
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
  for (int t = threadIdx.x; t < BOX_ROWS * yib::ATOMS; t += blockDim.x) erow[t] = 0.0;
  __syncthreads();
  const Cx* Ul = Uf + lane;
  const int vw = split * NW + warp;  // virtual warp of the block's schedule
  // the warp's (row, triple) items in ascending X: all warps sweep the X
  // instantiations in the same order, so the live code stays small
  for (int it = c_box_iseg[V][vw]; it < c_box_iseg[V][vw + 1]; ++it) {
    const int item = c_box_items[V][it];
    const int tid = item >> 16, J = (item >> 8) & 0xff, mb = item & 0xff;
    const int code = c_box_code[tid];
    const int X = code / 100, Y = (code / 10) % 10;
    const int SH = (X + Y - J) / 2;
    const bool mid = (2 * mb == J);
    const int boff = c_box_off[tid];
    const double cy = coef[tid];
    Cx* yrow = Ys + (yib::hoff(J) + mb * (J + 1)) * yib::ATOMS + lane;
    switch (X) {
      case 0: box_x<0>(Ul, Y, SH, J, mid, mb, boff, cy, yrow); break;
      case 1: box_x<1>(Ul, Y, SH, J, mid, mb, boff, cy, yrow); break;
      case 2: box_x<2>(Ul, Y, SH, J, mid, mb, boff, cy, yrow); break;
      case 3: box_x<3>(Ul, Y, SH, J, mid, mb, boff, cy, yrow); break;
      case 4: box_x<4>(Ul, Y, SH, J, mid, mb, boff, cy, yrow); break;
      case 5: box_x<5>(Ul, Y, SH, J, mid, mb, boff, cy, yrow); break;
      case 6: box_x<6>(Ul, Y, SH, J, mid, mb, boff, cy, yrow); break;
      case 7: box_x<7>(Ul, Y, SH, J, mid, mb, boff, cy, yrow); break;
      default: box_x<8>(Ul, Y, SH, J, mid, mb, boff, cy, yrow); break;
    }
  }
  __syncthreads();
  // middle rows: Y[ma] += (-1)^(J/2+ma) conj(Y[J-ma]) for ma <= J/2 (the images of
  // the mb1 > X/2 terms), then the upper half is cleared
  for (int t = threadIdx.x; t < 5 * yib::ATOMS; t += blockDim.x) {
    const int J = 2 * (t >> 5), at = t & 31, mb = J / 2;
    if (S > 1 && c_box_rowsplit[V][yib::rowoff(J) + mb] != split) continue;
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
  for (int t = threadIdx.x; t < BOX_ROWS * yib::ATOMS; t += blockDim.x) {
    const int r = t >> 5, at = t & 31;
    if (S > 1 && c_box_rowsplit[V][r] != split) continue;
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
  // rows owned by this CTA -> global (all rows when S = 1)
  // 8 consecutive threads take 8 consecutive atoms of one element h: conflict-free
  // shared-memory reads ([h][atom] layout), 16-byte global stores
  for (int t = threadIdx.x; t < yib::ATOMS * yib::NHALF; t += blockDim.x) {
    const int rest = t >> 3, h = rest % yib::NHALF, at = (rest / yib::NHALF) * 8 + (t & 7);
    if (at >= na_blk) continue;
    if (S > 1) {
      int J = 0;
      while (J < yib::TJ && h >= yib::hoff(J + 1)) ++J;
      const int r = yib::rowoff(J) + (h - yib::hoff(J)) / (J + 1);
      if (c_box_rowsplit[V][r] != split) continue;
    }
    ylist[(a0 + at) * yib::NHALF + h] = Ys[h * yib::ATOMS + at];
  }
  if (S == 1) {
    if (warp == 0 && lane < na_blk) {
      double e = beta0;
      for (int r = 0; r < BOX_ROWS; ++r) e += erow[r * yib::ATOMS + lane];
      eatom[a0 + lane] = e;
    }
  } else {
    for (int t = threadIdx.x; t < BOX_ROWS * na_blk; t += blockDim.x) {
      const int r = t / na_blk, at = t - r * na_blk;
      if (c_box_rowsplit[V][r] == split) erow_g[(int64_t)r * natoms + a0 + at] = erow[r * yib::ATOMS + at];
    }
  }
}

// split mode: E_i = beta0 + sum over rows in row order (the S = 1 arithmetic)
__global__ void k_box_energy(int64_t natoms, double beta0, const double* __restrict__ erow_g,
                             double* __restrict__ eatom) {
  griddep_wait_yi();
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < natoms; a += (int64_t)gridDim.x * blockDim.x) {
    double e = beta0;
    for (int r = 0; r < BOX_ROWS; ++r) e += erow_g[(int64_t)r * natoms + a];
    eatom[a] = e;
  }
}

// Upload the box table, the per-virtual-warp item lists and the row owners
// (process-wide; twojmax 8 only).  iseg: [BOX_NV][ROWS+1], items: [BOX_NV][nitems],
// rowsplit: [BOX_NV][ROWS].
cudaError_t snap_box_setup(const double* box, int nbox, const int* off, const int* code, const int* iseg,
                           const int* items, int nitems, const int* rowsplit) {
  if (nbox > yib::BOX_MAX || nitems > BOX_MAX_ITEMS) return cudaErrorInvalidValue;
  cudaError_t e;
  if ((e = cudaMemcpyToSymbol(c_box, box, sizeof(double) * nbox)) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(c_box_off, off, sizeof(int) * yib::NT)) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(c_box_code, code, sizeof(int) * yib::NT)) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(c_box_iseg, iseg, sizeof(int) * BOX_NV * (BOX_ROWS + 1))) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(c_box_rowsplit, rowsplit, sizeof(int) * BOX_NV * BOX_ROWS)) != cudaSuccess) return e;
  for (int v = 0; v < BOX_NV; ++v)
    if ((e = cudaMemcpyToSymbol(c_box_items, items + (size_t)v * nitems, sizeof(int) * nitems,
                                sizeof(int) * BOX_MAX_ITEMS * v)) != cudaSuccess)
      return e;
  return cudaSuccess;
}

// (warps, splits) of every variant; returns the count
int snap_box_variants(int* nw, int* ns) {
  for (int v = 0; v < BOX_NV; ++v) {
    nw[v] = BOX_NW[v];
    ns[v] = BOX_NS[v];
  }
  return BOX_NV;
}

template <int NW, int V, int S>
static cudaError_t box_launch(cudaStream_t st, int64_t natoms, double beta0, const double* coef, const void* utot,
                              void* ylist, double* eatom, double* erow_g) {
  const size_t sm = sizeof(Cx) * (yib::NFULL + yib::NHALF) * yib::ATOMS + sizeof(double) * BOX_ROWS * yib::ATOMS;
  static std::atomic<uint64_t> attr_devs{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_devs.load() & bit)) {  // exactly the dynamic size: the static mbarrier counts against the 227 KB too
    cudaError_t e = cudaFuncSetAttribute(k_snap_yi_box<NW, V, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    attr_devs.fetch_or(bit);
  }
  const unsigned grid = (unsigned)(S * ((natoms + yib::ATOMS - 1) / yib::ATOMS));
  cudaError_t e = launch_pdl_yi(k_snap_yi_box<NW, V, S>, dim3(grid), dim3(NW * 32), sm, st, natoms, beta0, coef,
                                (const Cx*)utot, (Cx*)ylist, eatom, erow_g);
  if (e != cudaSuccess) return e;
  if (S > 1)
    e = launch_pdl_yi(k_box_energy, dim3((unsigned)((natoms + 255) / 256)), dim3(256), 0, st, natoms, beta0,
                      (const double*)erow_g, eatom);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// split rows over 2 CTAs per block when the batch has fewer blocks than SMs
// (erow_g: 25 x natoms doubles of scratch)
cudaError_t snap_box_launch(cudaStream_t st, int64_t natoms, double beta0, const double* coef,
                            const void* utot, void* ylist, double* eatom, double* erow_g) {
  const int64_t blocks = (natoms + yib::ATOMS - 1) / yib::ATOMS;
  if (blocks < 148 && erow_g) return box_launch<12, 2, 2>(st, natoms, beta0, coef, utot, ylist, eatom, erow_g);
  return box_launch<12, 0, 1>(st, natoms, beta0, coef, utot, ylist, eatom, erow_g);
}

}  // namespace pl
