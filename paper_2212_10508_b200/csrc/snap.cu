// fp64 SNAP (single element) batched over systems x atoms, sm_100a.
//
// Formalism (2j-integer indices J = 0..twojmax; see oracle/native/snap_oracle.c
// for the full-matrix statement this file is checked against):
//   U^J of a neighbour from the Cayley-Klein pair (a, b) by the recursion
//     U^J[ma][mb] = sqrt((J-ma)/(J-mb)) a* U^{J-1}[ma][mb] - sqrt(ma/(J-mb)) b* U^{J-1}[ma-1][mb]
//   Utot = wself I + sum_k fc(r_k) U(r_k);  Z^{xy}_J = CG (x) CG contraction of Utot^x Utot^y
//   E_i = beta_0 + sum_b beta_b B_b,  B_{j1j2J} = Re <Utot^J, Z^{j1j2}_J>
//   dE_i/dr_ik = Re sum_J <d(fc U^J)/dr, Y^J>,  Y^J = sum coefY(x,y,J) Z^{xy}_J
// Only the half rows mb <= J/2 of every layer are computed and stored: the
// other half follows from U[J-ma][J-mb] = (-1)^(ma+mb) conj(U[ma][mb]), and
// the full-matrix sums are recovered with weights w(ma,mb) in {0,1,2}.
//
// Kernels (one force evaluation of B systems of N atoms):
//   k_snap_ui      CTA per atom, one warp per neighbour slot: U recursion with
//                  lanes over the elements of a layer (layers ping-pong in
//                  shared memory), per-warp partial Utot, fixed-order combine.
//   k_snap_yi      CTA per atom: Utot expanded to full matrices in shared
//                  memory, the Z/Y contraction split into cost-balanced work
//                  units (host schedule), fixed-order segmented reduction to
//                  Y (half rows) and the atom energy.
//   k_snap_deidrj  CTA per atom, one warp per neighbour slot: U and dU/dr
//                  recursion contracted on the fly with Y (shared memory).
//   k_snap_gather  thread per atom: dE/dr_a = sum_k dE_k/dr_ka - dE_a/dr_ak
//                  (reverse slot by binary search; no atomics), energies and
//                  virials reduced per system in a fixed order.
// Everything is deterministic (no floating-point atomics): reruns are bitwise
// identical, as parareal's convergence test requires (SURVEY.md finding 4).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <tuple>
#include <vector>

#include "neigh.cuh"
#include "pl_common.cuh"

namespace pl {

constexpr int SNAP_MAXN = 64;
constexpr int SNAP_JMAX = 14;
constexpr int UI_WARPS = 4;
constexpr int DE_WARPS = 4;
constexpr int YI_THREADS = 256;
constexpr int YI_ATOMS = 32;                 // lanes = atoms in k_snap_yi
constexpr int YI_WARPS = YI_THREADS / 32;

struct SnapItem {      // one half-row element of one Z^{xy}_J
  int16_t x, y, J, ma, mb;
  int16_t ma1lo, na, mb1lo, nb;
  int16_t bidx;        // canonical B index or -1
  int32_t cga, cgb;    // offsets into the CG pool (na, nb values)
  double coefY;        // weight of this Z element in Y^J (0 if none)
  double coefE;        // beta_b * w(ma,mb) if canonical, else 0
  double w;            // half-row weight
};

struct SnapUnit {      // a contiguous run of items of one target half index
  int32_t target, i0, i1;
};

struct SnapIndex {
  int tj = 0, nhalf = 0, nfull = 0, nB = 0, nitems = 0, nunits = 0;
  int hoff[SNAP_JMAX + 2], foff[SNAP_JMAX + 2];
  SnapItem* d_items = nullptr;
  SnapUnit* d_units = nullptr;
  int32_t* d_useg = nullptr;   // units of target h: [useg[h], useg[h+1])
  int32_t* d_tseg = nullptr;   // items of target h: [tseg[h], tseg[h+1])
  int32_t* d_wtarget = nullptr;  // targets owned by warp w of k_snap_yi: [wseg[w], wseg[w+1])
  int32_t* d_wseg = nullptr;
  double* d_cg = nullptr;
  double beta0 = 0.0;
  double flops_ui_pair = 0, flops_yi_atom = 0, flops_de_pair = 0;
  double flops_de_pair_adj = 0, flops_yi_atom_reg = 0, flops_ui_pair_v = 0;
  bool yi_reg = false;  // box-form Y tables set up (twojmax = 8)
  double* d_yi5 = nullptr;  // [2][NT]: coefY(X,Y,J), beta_b of canonical triples (else 0)
};

struct SnapDev {  // POD view passed to kernels
  int tj, nhalf, nfull, nB, nunits;
  int hoff[SNAP_JMAX + 2], foff[SNAP_JMAX + 2];
  const SnapItem* items;
  const SnapUnit* units;
  const int32_t* useg;
  const int32_t* tseg;
  const int32_t* wtarget;
  const int32_t* wseg;
  const double* yi5;  // [2][NT]
  const double* vs;   // twojmax 8: [2][nhalf] S^J[ma][mb] = N(J, ma) / N(J, mb) and its square (V recursion)
  const double* cg;
  double beta0, rcut, rfac0, rmin0, wself;
  double kappa, pi_span, half_pi_span;  // rfac0*pi/(rcut-rmin0), pi/(rcut-rmin0), 0.5*pi/(rcut-rmin0)
  int switchflag;
  int lists_exact;  // 1: the neighbour lists hold exactly the pairs r < rcut (no skin pairs to skip)
};

__constant__ double c_rootpq[SNAP_JMAX + 2][SNAP_JMAX + 2];  // sqrt(p/q)
// layer offsets depend on J only (not on twojmax): half rows and full matrices
__constant__ int c_hoff[SNAP_JMAX + 2];

// layer J and its half-storage offset of element t at twojmax 8, from
// immediate constants (a lane-divergent c_hoff search serialises on the
// constant cache)
constexpr int hoff8(int J) {
  int h = 0;
  for (int j = 0; j < J; ++j) h += (j + 1) * (j / 2 + 1);
  return h;
}
__device__ __forceinline__ void half_layer8(int t, int& J, int& base) {
  J = 0;
  base = 0;
#pragma unroll
  for (int j = 1; j <= 8; ++j)
    if (t >= hoff8(j)) {
      J = j;
      base = hoff8(j);
    }
}
__constant__ int c_foff[SNAP_JMAX + 2];
// box-form Z/Y kernel (snap_yi8.cu, own constant bank)
cudaError_t snap_yi8_setup(double* balance_out);
bool snap_yi8_append_records(const double* coef, std::vector<double>& out);  // snap_yi8.cu
cudaError_t snap_box_launch(cudaStream_t st, int64_t natoms, double beta0, const double* coef, const double* vs,
                            const void* utot, void* ylist, double* eatom, double* erow_g, void* ytlist,
                            bool* yt_done);

// ------------------------------------------------------------------ host setup
static double fact(int n) {
  double f = 1.0;
  for (int i = 2; i <= n; ++i) f *= (double)i;
  return f;
}

// Condon-Shortley <j1 m1 j2 m2 | J M> (Racah formula), arguments are 2j / 2m
double snap_clebsch(int j1, int m1, int j2, int m2, int J, int M) {
  if (m1 + m2 != M || std::abs(m1) > j1 || std::abs(m2) > j2 || std::abs(M) > J) return 0.0;
  if (J < std::abs(j1 - j2) || J > j1 + j2 || ((j1 + j2 + J) & 1)) return 0.0;
  double pre = std::sqrt((J + 1) * fact((j1 + j2 - J) / 2) * fact((j1 - j2 + J) / 2) *
                         fact((-j1 + j2 + J) / 2) / fact((j1 + j2 + J) / 2 + 1));
  pre *= std::sqrt(fact((J + M) / 2) * fact((J - M) / 2) * fact((j1 - m1) / 2) *
                   fact((j1 + m1) / 2) * fact((j2 - m2) / 2) * fact((j2 + m2) / 2));
  double s = 0.0;
  for (int k = 0;; ++k) {
    int d1 = (j1 + j2 - J) / 2 - k, d2 = (j1 - m1) / 2 - k, d3 = (j2 + m2) / 2 - k;
    int d4 = (J - j2 + m1) / 2 + k, d5 = (J - j1 - m2) / 2 + k;
    if (d1 < 0 || d2 < 0 || d3 < 0) break;
    if (d4 < 0 || d5 < 0) continue;
    double t = 1.0 / (fact(k) * fact(d1) * fact(d2) * fact(d3) * fact(d4) * fact(d5));
    s += (k & 1) ? -t : t;
  }
  return pre * s;
}

static double half_weight(int J, int ma, int mb) {
  if (2 * mb < J) return 2.0;
  if (2 * ma < J) return 2.0;
  if (2 * ma == J) return 1.0;
  return 0.0;
}

int snap_prepare(pl_pot* pot, const double* beta) {
  const int tj = pot->twojmax;
  SnapIndex* S = new SnapIndex();
  S->tj = tj;
  int h = 0, f = 0;
  for (int J = 0; J <= tj + 1; ++J) {
    S->hoff[J] = h;
    S->foff[J] = f;
    h += (J + 1) * (J / 2 + 1);
    f += (J + 1) * (J + 1);
  }
  S->nhalf = S->hoff[tj + 1];
  S->nfull = S->foff[tj + 1];
  // canonical triples (j1 >= j2, J >= j1) -> B index
  std::map<std::tuple<int, int, int>, int> bindex;
  std::vector<std::tuple<int, int, int>> canon;
  for (int j1 = 0; j1 <= tj; ++j1)
    for (int j2 = 0; j2 <= j1; ++j2)
      for (int J = j1 - j2; J <= std::min(tj, j1 + j2); J += 2)
        if (J >= j1) {
          bindex[{j1, j2, J}] = (int)canon.size();
          canon.push_back({j1, j2, J});
        }
  S->nB = (int)canon.size();
  if (pot->nbeta != S->nB + 1) {
    delete S;
    return fail(PL_EARG, "beta must have 1 + n_B(twojmax) = " + std::to_string(S->nB + 1) +
                             " entries, got " + std::to_string(pot->nbeta));
  }
  S->beta0 = beta[0];
  // Y coefficients per Z^{xy}_z (x >= y) from the three slots of every canonical triple
  std::map<std::tuple<int, int, int>, double> coefY;
  for (size_t b = 0; b < canon.size(); ++b) {
    int j1, j2, J;
    std::tie(j1, j2, J) = canon[b];
    double bb = beta[b + 1];
    coefY[{j1, j2, J}] += bb;                                        // slot J
    coefY[{J, j2, j1}] += bb * (double)(J + 1) / (double)(j1 + 1);   // slot j1
    coefY[{J, j1, j2}] += bb * (double)(J + 1) / (double)(j2 + 1);   // slot j2
  }
  // box-form Y (snap_yi8.cu, twojmax = 8): per-triple coefficients, rows by J,
  // schedule of the (J, mb) rows over the CTA's warps
  S->yi_reg = false;
  if (tj == 8) {
    std::vector<double> cy, be;
    std::vector<int> code;
    std::vector<std::vector<int>> byJ(tj + 1);
    for (int x = 0; x <= tj; ++x)
      for (int y = 0; y <= x; ++y)
        for (int J = x - y; J <= std::min(tj, x + y); J += 2) {
          int tid = (int)code.size();
          auto itc = coefY.find({x, y, J});
          cy.push_back(itc == coefY.end() ? 0.0 : itc->second);
          auto itb = bindex.find({x, y, J});
          be.push_back(itb == bindex.end() ? 0.0 : beta[itb->second + 1]);
          code.push_back(x * 100 + y * 10 + J);
          byJ[J].push_back(tid);
        }
    static std::atomic<uint64_t> yi_devs{0};  // __constant__ tables are per device
    if (first_on_device(yi_devs)) {
      double bal = 0.0;
      PL_CUDA(snap_yi8_setup(&bal));
    }
    std::vector<double> cb2(cy);
    cb2.insert(cb2.end(), be.begin(), be.end());
    // scale of the V recursion per half element (J, mb, ma): S = N(J, ma) / N(J, mb),
    // N(J, x) = sqrt(x! (J - x)!); then S^2 (exact ratio of integers, rounded once)
    std::vector<double> vs, vs2;
    for (int J = 0; J <= tj; ++J)
      for (int mb = 0; 2 * mb <= J; ++mb)
        for (int ma = 0; ma <= J; ++ma) {
          const double r = (fact(ma) * fact(J - ma)) / (fact(mb) * fact(J - mb));
          vs.push_back(std::sqrt(r));
          vs2.push_back(r);
        }
    if ((int)vs.size() != S->nhalf || (int)code.size() != 125) {
      delete S;
      return fail(PL_EARG, "twojmax-8 index sizes");
    }
    cb2.insert(cb2.end(), vs.begin(), vs.end());
    cb2.insert(cb2.end(), vs2.begin(), vs2.end());
    if (!snap_yi8_append_records(cy.data(), cb2)) {  // the Y kernel's item records with cy folded in
      delete S;
      return fail(PL_EARG, "twojmax-8 item records");
    }
    PL_CUDA(cudaMalloc(&S->d_yi5, sizeof(double) * cb2.size()));
    PL_CUDA(cudaMemcpy(S->d_yi5, cb2.data(), sizeof(double) * cb2.size(), cudaMemcpyHostToDevice));
    S->yi_reg = true;
  }
  // items grouped by target half index
  std::vector<std::vector<SnapItem>> per_target(S->nhalf);
  std::vector<double> pool;
  for (int x = 0; x <= tj; ++x)
    for (int y = 0; y <= x; ++y)
      for (int J = x - y; J <= std::min(tj, x + y); J += 2) {
        auto itc = coefY.find({x, y, J});
        double cy = itc == coefY.end() ? 0.0 : itc->second;
        auto itb = bindex.find({x, y, J});
        int bidx = itb == bindex.end() ? -1 : itb->second;
        for (int mb = 0; 2 * mb <= J; ++mb)
          for (int ma = 0; ma <= J; ++ma) {
            SnapItem it{};
            it.x = x; it.y = y; it.J = J; it.ma = ma; it.mb = mb;
            int M = 2 * ma - J, Mp = 2 * mb - J;
            // ma1 range with ma2 = (M - m1 + y)/2 in [0, y]
            std::vector<double> ca, cb;
            int lo = -1;
            for (int ma1 = 0; ma1 <= x; ++ma1) {
              int m2 = M - (2 * ma1 - x);
              if (std::abs(m2) > y) continue;
              if (lo < 0) lo = ma1;
              ca.push_back(snap_clebsch(x, 2 * ma1 - x, y, m2, J, M));
            }
            it.ma1lo = (int16_t)lo;
            it.na = (int16_t)ca.size();
            lo = -1;
            for (int mb1 = 0; mb1 <= x; ++mb1) {
              int m2 = Mp - (2 * mb1 - x);
              if (std::abs(m2) > y) continue;
              if (lo < 0) lo = mb1;
              cb.push_back(snap_clebsch(x, 2 * mb1 - x, y, m2, J, Mp));
            }
            it.mb1lo = (int16_t)lo;
            it.nb = (int16_t)cb.size();
            it.cga = (int32_t)pool.size();
            pool.insert(pool.end(), ca.begin(), ca.end());
            it.cgb = (int32_t)pool.size();
            pool.insert(pool.end(), cb.begin(), cb.end());
            it.w = half_weight(J, ma, mb);
            it.coefY = cy;
            it.bidx = (int16_t)bidx;
            it.coefE = bidx >= 0 ? beta[bidx + 1] * it.w : 0.0;
            int target = S->hoff[J] + mb * (J + 1) + ma;
            per_target[target].push_back(it);
          }
      }
  // cost-balanced units: ~4 units per thread of a YI CTA
  std::vector<SnapItem> items;
  std::vector<SnapUnit> units;
  std::vector<int32_t> useg(S->nhalf + 1, 0);
  double total = 0.0;
  for (auto& v : per_target)
    for (auto& it : v) total += (double)it.na * it.nb + 2.0;
  double unit_cost = total / (4.0 * YI_THREADS);
  double yflops = 0.0;
  for (int t = 0; t < S->nhalf; ++t) {
    useg[t] = (int32_t)units.size();
    auto& v = per_target[t];
    int start = (int)items.size();
    double acc = 0.0;
    int u0 = start;
    for (size_t k = 0; k < v.size(); ++k) {
      items.push_back(v[k]);
      double c = (double)v[k].na * v[k].nb + 2.0;
      yflops += 10.0 * v[k].na * v[k].nb + 4.0 * v[k].nb + 10.0;
      acc += c;
      if (acc >= unit_cost) {
        units.push_back({t, u0, (int32_t)items.size()});
        u0 = (int)items.size();
        acc = 0.0;
      }
    }
    if ((int)items.size() > u0 || units.empty() || useg[t] == (int32_t)units.size())
      units.push_back({t, u0, (int32_t)items.size()});
  }
  useg[S->nhalf] = (int32_t)units.size();
  // items of each target are contiguous in `items`
  std::vector<int32_t> tseg(S->nhalf + 1, 0);
  {
    int pos = 0;
    for (int t = 0; t < S->nhalf; ++t) {
      tseg[t] = pos;
      pos += (int)per_target[t].size();
    }
    tseg[S->nhalf] = pos;
  }
  // targets -> warps of k_snap_yi by longest-processing-time greedy on cost
  const int nwarps = YI_WARPS;
  std::vector<std::pair<double, int>> tc;
  for (int t = 0; t < S->nhalf; ++t) {
    double c = 0.0;
    for (auto& it : per_target[t]) c += (double)it.na * it.nb + 2.0 * it.nb + 4.0;
    tc.push_back({c, t});
  }
  std::sort(tc.begin(), tc.end(), [](auto& a, auto& b) { return a.first > b.first; });
  std::vector<std::vector<int32_t>> wt(nwarps);
  std::vector<double> wl(nwarps, 0.0);
  for (auto& c : tc) {
    int w = (int)(std::min_element(wl.begin(), wl.end()) - wl.begin());
    wt[w].push_back(c.second);
    wl[w] += c.first;
  }
  std::vector<int32_t> wtarget, wseg(nwarps + 1, 0);
  for (int w = 0; w < nwarps; ++w) {
    std::sort(wt[w].begin(), wt[w].end());
    wseg[w] = (int32_t)wtarget.size();
    wtarget.insert(wtarget.end(), wt[w].begin(), wt[w].end());
  }
  wseg[nwarps] = (int32_t)wtarget.size();
  S->nitems = (int)items.size();
  S->nunits = (int)units.size();
  // algorithmic flop counts (used for the roofline numerator)
  S->flops_yi_atom = yflops;
  S->flops_ui_pair = 0.0;
  S->flops_de_pair = 0.0;
  for (int J = 1; J <= tj; ++J) {
    int nel = (J + 1) * (J / 2 + 1);
    S->flops_ui_pair += nel * 24.0;   // 2 x (complex product + scaled accumulate) + fc accumulate
    S->flops_ui_pair_v += nel * 18.0; // V form (k_snap_ui_r4): 2 complex products + difference + fc accumulate
    S->flops_de_pair += nel * 160.0;  // U (20) + 3 dU (108) + 3 weighted contractions (~32)
  }
  S->flops_ui_pair += 40.0;
  S->flops_ui_pair_v += 40.0;
  S->flops_de_pair += 80.0;
  // reverse-mode pair kernel in the V form: forward V + F contraction (19/element),
  // adjoint (S_a, S_b, G update, direct Y term: 34/element), geometry + final (150)
  S->flops_de_pair_adj = 150.0;
  for (int J = 1; J <= tj; ++J) S->flops_de_pair_adj += (J + 1) * (J / 2 + 1) * 53.0;
  // register-tiled Z/Y: the middle row's upper half (zero weight) is skipped
  S->flops_yi_atom_reg = 0.0;
  for (int x = 0; x <= tj; ++x)
    for (int y = 0; y <= x; ++y)
      for (int J = x - y; J <= std::min(tj, x + y); J += 2) {
        const int sh = (x + y - J) / 2;
        for (int mb = 0; 2 * mb <= J; ++mb) {
          int nb = 0;
          for (int mb1 = 0; mb1 <= x; ++mb1) nb += (mb + sh - mb1 >= 0 && mb + sh - mb1 <= y);
          for (int ma = 0; ma <= J; ++ma) {
            if (2 * mb == J && 2 * ma > J) continue;
            int na = 0;
            for (int ma1 = 0; ma1 <= x; ++ma1) na += (ma + sh - ma1 >= 0 && ma + sh - ma1 <= y);
            S->flops_yi_atom_reg += 10.0 * na * nb + 4.0 * nb + 8.0;
          }
        }
      }
  cudaError_t e1 = cudaMalloc(&S->d_items, sizeof(SnapItem) * items.size());
  cudaError_t e2 = cudaMalloc(&S->d_units, sizeof(SnapUnit) * units.size());
  cudaError_t e3 = cudaMalloc(&S->d_useg, sizeof(int32_t) * useg.size());
  cudaError_t e4 = cudaMalloc(&S->d_cg, sizeof(double) * std::max<size_t>(pool.size(), 1));
  cudaError_t e5 = cudaMalloc(&S->d_tseg, sizeof(int32_t) * tseg.size());
  cudaError_t e6 = cudaMalloc(&S->d_wtarget, sizeof(int32_t) * wtarget.size());
  cudaError_t e7 = cudaMalloc(&S->d_wseg, sizeof(int32_t) * wseg.size());
  if (e1 || e2 || e3 || e4 || e5 || e6 || e7) {
    delete S;
    return fail(PL_ECUDA, "cudaMalloc SNAP index");
  }
  cudaMemcpy(S->d_items, items.data(), sizeof(SnapItem) * items.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(S->d_units, units.data(), sizeof(SnapUnit) * units.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(S->d_useg, useg.data(), sizeof(int32_t) * useg.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(S->d_cg, pool.data(), sizeof(double) * pool.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(S->d_tseg, tseg.data(), sizeof(int32_t) * tseg.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(S->d_wtarget, wtarget.data(), sizeof(int32_t) * wtarget.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(S->d_wseg, wseg.data(), sizeof(int32_t) * wseg.size(), cudaMemcpyHostToDevice);
  double rp[SNAP_JMAX + 2][SNAP_JMAX + 2];
  for (int p = 0; p < SNAP_JMAX + 2; ++p)
    for (int q = 0; q < SNAP_JMAX + 2; ++q) rp[p][q] = q ? std::sqrt((double)p / (double)q) : 0.0;
  PL_CUDA(cudaMemcpyToSymbol(c_rootpq, rp, sizeof(rp)));
  int ho[SNAP_JMAX + 2], fo[SNAP_JMAX + 2];
  for (int J = 0, hh = 0, ff = 0; J < SNAP_JMAX + 2; ++J) {
    ho[J] = hh;
    fo[J] = ff;
    hh += (J + 1) * (J / 2 + 1);
    ff += (J + 1) * (J + 1);
  }
  PL_CUDA(cudaMemcpyToSymbol(c_hoff, ho, sizeof(ho)));
  PL_CUDA(cudaMemcpyToSymbol(c_foff, fo, sizeof(fo)));
  pot->snap = S;
  // one system: N atoms x ~26 pairs (perfect BCC at rcut 4.73) is only an
  // estimate for reporting; the bench counts real pairs per launch.
  pot->flops = 0.0;
  return PL_OK;
}

void snap_release(pl_pot* pot) {
  SnapIndex* S = pot->snap;
  if (!S) return;
  cudaFree(S->d_items);
  cudaFree(S->d_units);
  cudaFree(S->d_useg);
  cudaFree(S->d_cg);
  cudaFree(S->d_tseg);
  cudaFree(S->d_wtarget);
  cudaFree(S->d_wseg);
  cudaFree(S->d_yi5);
  delete S;
  pot->snap = nullptr;
}

static SnapDev snap_dev(const pl_pot* pot) {
  const SnapIndex* S = pot->snap;
  SnapDev D;
  D.tj = S->tj; D.nhalf = S->nhalf; D.nfull = S->nfull; D.nB = S->nB; D.nunits = S->nunits;
  for (int J = 0; J <= SNAP_JMAX + 1; ++J) {
    D.hoff[J] = J <= S->tj + 1 ? S->hoff[J] : 0;
    D.foff[J] = J <= S->tj + 1 ? S->foff[J] : 0;
  }
  D.items = S->d_items; D.units = S->d_units; D.useg = S->d_useg; D.cg = S->d_cg;
  D.tseg = S->d_tseg; D.wtarget = S->d_wtarget; D.wseg = S->d_wseg;
  D.yi5 = S->d_yi5;
  D.vs = S->yi_reg ? S->d_yi5 + 2 * 125 : nullptr;
  D.beta0 = S->beta0; D.rcut = pot->rcut; D.rfac0 = pot->rfac0; D.rmin0 = pot->rmin0;
  D.wself = pot->wself; D.switchflag = pot->switchflag;
  D.lists_exact = 1;
  D.kappa = pot->rfac0 * M_PI / (pot->rcut - pot->rmin0);
  D.pi_span = M_PI / (pot->rcut - pot->rmin0);
  D.half_pi_span = 0.5 * M_PI / (pot->rcut - pot->rmin0);
  return D;
}

// ------------------------------------------------------------------ device helpers
struct C2 {
  double re, im;
};
__device__ __forceinline__ C2 cmulc(C2 a, C2 b) {  // conj(a) * b
  return C2{a.re * b.re + a.im * b.im, a.re * b.im - a.im * b.re};
}
__device__ __forceinline__ C2 cmul(C2 a, C2 b) {
  return C2{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}

struct PairGeom {
  double u[3], r, fc, dfc;
  C2 a, b, da[3], db[3];
};

// d(a, b)/dr_k from the unit vector, sin/cos of the angle and 1/r
__device__ __forceinline__ void pair_deriv(double kappa, const double (&u)[3], double s, double c, double inv,
                                           C2 (&da)[3], C2 (&db)[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double dxk = (k == 0) - u[0] * u[k], dyk = (k == 1) - u[1] * u[k];
    double dzk = (k == 2) - u[2] * u[k];
    da[k] = C2{-s * kappa * u[k], -(c * kappa * u[k] * u[2] + s * dzk * inv)};
    db[k] = C2{c * kappa * u[k] * u[1] + s * dyk * inv, -(c * kappa * u[k] * u[0] + s * dxk * inv)};
  }
}

__device__ __forceinline__ void pair_geom(const SnapDev& D, double dx, double dy, double dz, PairGeom& g,
                                          bool with_deriv) {
  double r = sqrt(dx * dx + dy * dy + dz * dz);
  double inv = 1.0 / r;
  g.r = r;
  g.u[0] = dx * inv; g.u[1] = dy * inv; g.u[2] = dz * inv;
  const double kappa = D.kappa;
  double s, c;
  sincos(kappa * (r - D.rmin0), &s, &c);
  g.a = C2{c, -g.u[2] * s};
  g.b = C2{g.u[1] * s, -g.u[0] * s};
  if (D.switchflag) {
    double sa, ca;
    sincos(D.pi_span * (r - D.rmin0), &sa, &ca);
    g.fc = 0.5 * (ca + 1.0);
    g.dfc = -D.half_pi_span * sa;
  } else {
    g.fc = 1.0;
    g.dfc = 0.0;
  }
  if (with_deriv) pair_deriv(kappa, g.u, s, c, inv, g.da, g.db);
}

// element (ma, mb) of layer Jp = J-1 from its half-row buffer (row length J);
// rows beyond Jp/2 through the inversion symmetry.
__device__ __forceinline__ C2 prev_elem(const C2* buf, int J, int ma, int mb) {
  const int Jp = J - 1;
  if (2 * mb <= Jp) return buf[mb * J + ma];
  // mb = J/2 (J even): U[ma][mb] = (-1)^(ma+mb) conj(U[Jp-ma][Jp-mb])
  C2 v = buf[(Jp - mb) * J + (Jp - ma)];
  return ((ma + mb) & 1) ? C2{-v.re, v.im} : C2{v.re, -v.im};
}

// ------------------------------------------------------------------ kernel: Utot
__global__ void __launch_bounds__(UI_WARPS * 32)
k_snap_ui(SnapDev D, int64_t natoms, int N, Box box, const double* __restrict__ q,
          const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt, int maxn,
          C2* __restrict__ utot) {
  extern __shared__ double smem[];
  const int nh = D.nhalf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  C2* part = reinterpret_cast<C2*>(smem) + warp * nh;              // per-warp partial Utot
  const int layer_max = (D.tj + 1) * (D.tj / 2 + 1);
  C2* lay = reinterpret_cast<C2*>(smem) + UI_WARPS * nh + warp * 2 * layer_max;
  int64_t atom = blockIdx.x;
  int64_t b = atom / N;
  int i = (int)(atom - b * N);
  const double* qb = q + b * (int64_t)N * 3;
  for (int t = lane; t < nh; t += 32) part[t] = C2{0.0, 0.0};
  int n = cnt[atom];
  const int32_t* nb = nbr + atom * maxn;
  for (int s = warp; s < n; s += UI_WARPS) {
    double dx, dy, dz;
    pair_vec(qb, i, nb[s], box, dx, dy, dz);
    PairGeom g;
    pair_geom(D, dx, dy, dz, g, false);
    C2* prev = lay;
    C2* cur = lay + layer_max;
    if (lane == 0) {
      prev[0] = C2{1.0, 0.0};
      part[0].re += g.fc;
    }
    __syncwarp();
    for (int J = 1; J <= D.tj; ++J) {
      int nel = (J + 1) * (J / 2 + 1);
      for (int e = lane; e < nel; e += 32) {
        int mb = e / (J + 1), ma = e - mb * (J + 1);
        C2 v{0.0, 0.0};
        if (ma < J) {
          C2 p = prev_elem(prev, J, ma, mb);
          C2 t = cmulc(g.a, p);
          double A = c_rootpq[J - ma][J - mb];
          v.re += A * t.re;
          v.im += A * t.im;
        }
        if (ma > 0) {
          C2 p = prev_elem(prev, J, ma - 1, mb);
          C2 t = cmulc(g.b, p);
          double Bc = c_rootpq[ma][J - mb];
          v.re -= Bc * t.re;
          v.im -= Bc * t.im;
        }
        cur[e] = v;
        C2& acc = part[c_hoff[J] + e];
        acc.re += g.fc * v.re;
        acc.im += g.fc * v.im;
      }
      __syncwarp();
      C2* tmp = prev;
      prev = cur;
      cur = tmp;
    }
  }
  __syncthreads();
  // fixed-order combine of the warp partials + self term on the diagonal
  C2* out = utot + atom * nh;
  for (int t = threadIdx.x; t < nh; t += blockDim.x) {
    C2 s{0.0, 0.0};
#pragma unroll
    for (int w = 0; w < UI_WARPS; ++w) {
      C2 v = reinterpret_cast<C2*>(smem)[w * nh + t];
      s.re += v.re;
      s.im += v.im;
    }
    // decode (J, ma, mb) of t to add wself on ma == mb
    int J = 0;
    while (J < D.tj && t >= c_hoff[J + 1]) ++J;
    int e = t - c_hoff[J];
    int mb = e / (J + 1), ma = e - mb * (J + 1);
    if (ma == mb) s.re += D.wself;
    out[t] = s;
  }
}

// ------------------------------------------------------------------ kernel: Y, E_i
// lanes = atoms: the 32 lanes of a warp walk the same Z items for 32 atoms,
// so control flow and CG loads are warp-uniform and the [element][atom]
// shared-memory layout is bank-conflict free.  Warps own disjoint sets of Y
// targets (host LPT schedule), so every Y element is summed by one lane in a
// fixed item order (deterministic, no atomics).
__device__ __forceinline__ C2 half_get(const C2* Us, int x, int ma, int mb, int lane) {
  // Utot^x[ma][mb] from half-row storage [nhalf][YI_ATOMS]
  if (2 * mb <= x) return Us[(c_hoff[x] + mb * (x + 1) + ma) * YI_ATOMS + lane];
  C2 v = Us[(c_hoff[x] + (x - mb) * (x + 1) + (x - ma)) * YI_ATOMS + lane];
  return ((ma + mb) & 1) ? C2{-v.re, v.im} : C2{v.re, -v.im};
}

__global__ void __launch_bounds__(YI_THREADS)
k_snap_yi(SnapDev D, int64_t natoms, const C2* __restrict__ utot, C2* __restrict__ ylist,
          double* __restrict__ eatom) {
  extern __shared__ double smem[];
  C2* Us = reinterpret_cast<C2*>(smem);                                // [nhalf][32]
  double* epart = reinterpret_cast<double*>(Us + D.nhalf * YI_ATOMS);  // [warps][32]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t a0 = (int64_t)blockIdx.x * YI_ATOMS;
  const int na_blk = (int)min((int64_t)YI_ATOMS, natoms - a0);
  // stage Utot of 32 atoms, transposed to [element][atom]
  for (int t = threadIdx.x; t < D.nhalf * YI_ATOMS; t += blockDim.x) {
    int at = t / D.nhalf, e = t - at * D.nhalf;
    Us[e * YI_ATOMS + at] = at < na_blk ? utot[(a0 + at) * D.nhalf + e] : C2{0.0, 0.0};
  }
  __syncthreads();
  double esum = 0.0;
  const int64_t atom = a0 + lane;
  for (int wt = D.wseg[warp]; wt < D.wseg[warp + 1]; ++wt) {
    const int target = D.wtarget[wt];
    C2 ysum{0.0, 0.0};
    for (int k = D.tseg[target]; k < D.tseg[target + 1]; ++k) {
      const SnapItem it = D.items[k];
      const double* ca = D.cg + it.cga;
      const double* cb = D.cg + it.cgb;
      const int x = it.x, y = it.y, J = it.J, sh = (x + y - J) / 2;
      C2 z{0.0, 0.0};
      for (int jb = 0; jb < it.nb; ++jb) {
        const int mb1 = it.mb1lo + jb, mb2 = it.mb - mb1 + sh;
        C2 sacc{0.0, 0.0};
        for (int ja = 0; ja < it.na; ++ja) {
          const int ma1 = it.ma1lo + ja, ma2 = it.ma - ma1 + sh;
          C2 t = cmul(half_get(Us, x, ma1, mb1, lane), half_get(Us, y, ma2, mb2, lane));
          const double c = ca[ja];
          sacc.re += c * t.re;
          sacc.im += c * t.im;
        }
        const double c = cb[jb];
        z.re += c * sacc.re;
        z.im += c * sacc.im;
      }
      ysum.re += it.coefY * z.re;
      ysum.im += it.coefY * z.im;
      if (it.bidx >= 0) {
        C2 uJ = Us[(c_hoff[J] + it.mb * (J + 1) + it.ma) * YI_ATOMS + lane];
        esum += it.coefE * (uJ.re * z.re + uJ.im * z.im);  // Re(conj(U) z)
      }
    }
    if (lane < na_blk) ylist[atom * D.nhalf + target] = ysum;
  }
  epart[warp * YI_ATOMS + lane] = esum;
  __syncthreads();
  if (warp == 0 && lane < na_blk) {
    double e = D.beta0;
    for (int w = 0; w < YI_WARPS; ++w) e += epart[w * YI_ATOMS + lane];
    eatom[atom] = e;
  }
}
// per-atom bispectrum (debug / parity path; per item, deterministic)
__global__ void k_snap_bispectrum(SnapDev D, const C2* __restrict__ utot, double* __restrict__ bout,
                                  int nitems) {
  extern __shared__ double smem[];
  C2* U = reinterpret_cast<C2*>(smem);
  int64_t atom = blockIdx.x;
  const C2* ut = utot + atom * D.nhalf;
  for (int J = 0; J <= D.tj; ++J) {
    int sz = (J + 1) * (J + 1);
    for (int t = threadIdx.x; t < sz; t += blockDim.x) {
      int mb = t / (J + 1), ma = t - mb * (J + 1);
      C2 v;
      if (2 * mb <= J) {
        v = ut[c_hoff[J] + mb * (J + 1) + ma];
      } else {
        C2 w = ut[c_hoff[J] + (J - mb) * (J + 1) + (J - ma)];
        v = ((ma + mb) & 1) ? C2{-w.re, w.im} : C2{w.re, -w.im};
      }
      U[c_foff[J] + t] = v;
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < D.nB; b += blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < nitems; ++k) {
      const SnapItem it = D.items[k];
      if (it.bidx != b) continue;
      const double* ca = D.cg + it.cga;
      const double* cb = D.cg + it.cgb;
      const int x = it.x, y = it.y, J = it.J, sh = (x + y - J) / 2;
      C2 z{0.0, 0.0};
      for (int jb = 0; jb < it.nb; ++jb) {
        int mb1 = it.mb1lo + jb, mb2 = it.mb - mb1 + sh;
        C2 s{0.0, 0.0};
        for (int ja = 0; ja < it.na; ++ja) {
          int ma1 = it.ma1lo + ja, ma2 = it.ma - ma1 + sh;
          C2 t = cmul(U[c_foff[x] + mb1 * (x + 1) + ma1], U[c_foff[y] + mb2 * (y + 1) + ma2]);
          s.re += ca[ja] * t.re;
          s.im += ca[ja] * t.im;
        }
        z.re += cb[jb] * s.re;
        z.im += cb[jb] * s.im;
      }
      C2 uJ = U[c_foff[J] + it.mb * (J + 1) + it.ma];
      acc += it.w * (uJ.re * z.re + uJ.im * z.im);
    }
    bout[atom * D.nB + b] = acc;
  }
}

// ------------------------------------------------------------------ kernel: dE_i/dr_ik
__global__ void __launch_bounds__(DE_WARPS * 32)
k_snap_deidrj(SnapDev D, int64_t natoms, int N, Box box, const double* __restrict__ q,
              const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt, int maxn,
              const C2* __restrict__ ylist, double* __restrict__ dedr) {
  extern __shared__ double smem[];
  const int nh = D.nhalf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  C2* Y = reinterpret_cast<C2*>(smem);
  const int layer_max = (D.tj + 1) * (D.tj / 2 + 1);
  // per warp: 2 layers x (U, dU0, dU1, dU2)
  C2* lay = Y + nh + warp * 2 * 4 * layer_max;
  int64_t atom = blockIdx.x;
  int64_t b = atom / N;
  int i = (int)(atom - b * N);
  const double* qb = q + b * (int64_t)N * 3;
  for (int t = threadIdx.x; t < nh; t += blockDim.x) Y[t] = ylist[atom * nh + t];
  __syncthreads();
  int n = cnt[atom];
  const int32_t* nb = nbr + atom * maxn;
  for (int s = warp; s < n; s += DE_WARPS) {
    double dx, dy, dz;
    pair_vec(qb, i, nb[s], box, dx, dy, dz);
    PairGeom g;
    pair_geom(D, dx, dy, dz, g, true);
    C2* prev = lay;
    C2* cur = lay + 4 * layer_max;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    if (lane == 0) {
      prev[0] = C2{1.0, 0.0};
      prev[layer_max] = prev[2 * layer_max] = prev[3 * layer_max] = C2{0.0, 0.0};
      // J = 0: U = 1, dU = 0, weight 1
      double y0 = Y[0].re;
      acc0 = g.dfc * g.u[0] * y0;
      acc1 = g.dfc * g.u[1] * y0;
      acc2 = g.dfc * g.u[2] * y0;
    }
    __syncwarp();
    for (int J = 1; J <= D.tj; ++J) {
      int nel = (J + 1) * (J / 2 + 1);
      for (int e = lane; e < nel; e += 32) {
        int mb = e / (J + 1), ma = e - mb * (J + 1);
        C2 v{0.0, 0.0}, dv0{0.0, 0.0}, dv1{0.0, 0.0}, dv2{0.0, 0.0};
        if (ma < J) {
          double A = c_rootpq[J - ma][J - mb];
          C2 p = prev_elem(prev, J, ma, mb);
          C2 p0 = prev_elem(prev + layer_max, J, ma, mb);
          C2 p1 = prev_elem(prev + 2 * layer_max, J, ma, mb);
          C2 p2 = prev_elem(prev + 3 * layer_max, J, ma, mb);
          C2 t = cmulc(g.a, p);
          v.re += A * t.re; v.im += A * t.im;
          C2 t0 = cmulc(g.da[0], p), s0 = cmulc(g.a, p0);
          C2 t1 = cmulc(g.da[1], p), s1 = cmulc(g.a, p1);
          C2 t2 = cmulc(g.da[2], p), s2 = cmulc(g.a, p2);
          dv0.re += A * (t0.re + s0.re); dv0.im += A * (t0.im + s0.im);
          dv1.re += A * (t1.re + s1.re); dv1.im += A * (t1.im + s1.im);
          dv2.re += A * (t2.re + s2.re); dv2.im += A * (t2.im + s2.im);
        }
        if (ma > 0) {
          double Bc = c_rootpq[ma][J - mb];
          C2 p = prev_elem(prev, J, ma - 1, mb);
          C2 p0 = prev_elem(prev + layer_max, J, ma - 1, mb);
          C2 p1 = prev_elem(prev + 2 * layer_max, J, ma - 1, mb);
          C2 p2 = prev_elem(prev + 3 * layer_max, J, ma - 1, mb);
          C2 t = cmulc(g.b, p);
          v.re -= Bc * t.re; v.im -= Bc * t.im;
          C2 t0 = cmulc(g.db[0], p), s0 = cmulc(g.b, p0);
          C2 t1 = cmulc(g.db[1], p), s1 = cmulc(g.b, p1);
          C2 t2 = cmulc(g.db[2], p), s2 = cmulc(g.b, p2);
          dv0.re -= Bc * (t0.re + s0.re); dv0.im -= Bc * (t0.im + s0.im);
          dv1.re -= Bc * (t1.re + s1.re); dv1.im -= Bc * (t1.im + s1.im);
          dv2.re -= Bc * (t2.re + s2.re); dv2.im -= Bc * (t2.im + s2.im);
        }
        cur[e] = v;
        cur[layer_max + e] = dv0;
        cur[2 * layer_max + e] = dv1;
        cur[3 * layer_max + e] = dv2;
        // weight of a half-row element in the full-matrix sum
        double w = (2 * mb < J || 2 * ma < J) ? 2.0 : (2 * ma == J ? 1.0 : 0.0);
        C2 y = Y[c_hoff[J] + e];
        double yu = v.re * y.re + v.im * y.im;
        acc0 += w * (g.fc * (dv0.re * y.re + dv0.im * y.im) + g.dfc * g.u[0] * yu);
        acc1 += w * (g.fc * (dv1.re * y.re + dv1.im * y.im) + g.dfc * g.u[1] * yu);
        acc2 += w * (g.fc * (dv2.re * y.re + dv2.im * y.im) + g.dfc * g.u[2] * yu);
      }
      __syncwarp();
      C2* tmp = prev;
      prev = cur;
      cur = tmp;
    }
    // fixed-order warp reduction
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      acc0 += __shfl_down_sync(0xffffffffu, acc0, off);
      acc1 += __shfl_down_sync(0xffffffffu, acc1, off);
      acc2 += __shfl_down_sync(0xffffffffu, acc2, off);
    }
    if (lane == 0) {
      double* o = dedr + (atom * maxn + s) * 3;
      o[0] = acc0;
      o[1] = acc1;
      o[2] = acc2;
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ register-resident recursion
// One lane owns one half row mb of U^J (and of dU^J/dr_k) for one neighbour
// pair; R = TJ/2 + 1 lanes per pair, P = 32/R pairs per warp.  Layer J is
// built from layer J-1 IN PLACE, descending ma, fully unrolled (J, ma are
// compile-time), so U lives in registers.  At even J the new middle row
// mb = J/2 is born from row J/2 - 1 of layer J-1 (held by the next lane down)
// through U[x][J/2] = (-1)^(x+J/2) conj(U[J-1-x][J/2-1]), one shuffle per element.
template <int TJ>
struct RowGeom {
  C2 a, b;     // Cayley-Klein parameters
  C2 da, db;   // d/dr_k of a, b (current Cartesian component)
};

__device__ __forceinline__ C2 shfl_up_c2(C2 v, int delta) {
  return C2{__shfl_up_sync(0xffffffffu, v.re, delta), __shfl_up_sync(0xffffffffu, v.im, delta)};
}

// Coefficient-free recursion.  With N(J, x) = sqrt(x! (J - x)!) and
//   U^J[ma][mb] = (N(J, ma) / N(J, mb)) V^J[ma][mb],
// the sqrt((J-ma)/(J-mb)) and sqrt(ma/(J-mb)) factors of the U recursion cancel:
//   V^J[ma][mb] = conj(a) V^{J-1}[ma][mb] - conj(b) V^{J-1}[ma-1][mb],
// and V keeps the inversion symmetry of U (the scale is invariant under
// (ma, mb) -> (J - ma, J - mb)).  The twojmax-8 kernels propagate V (8 FP64
// instructions per element instead of 12, no coefficient loads) and fold the
// scale S^J[ma][mb] = N(J, ma) / N(J, mb) into what they produce or consume once
// per atom: U_tot = S (.) sum_k fc_k V_k (k_snap_ui_r4), and the force sweep
// reads S (.) Y (written by the Y kernel), because Re<U, Y> = Re<V, S (.) Y>.
__device__ __forceinline__ C2 vstep(const C2& a, const C2& b, const C2& u, const C2& v, bool has_u, bool has_v) {
  // conj(a) u - conj(b) v
  C2 r{0.0, 0.0};
  if (has_u && has_v) {
    r.re = fma(a.re, u.re, fma(a.im, u.im, fma(-b.re, v.re, -b.im * v.im)));
    r.im = fma(a.re, u.im, fma(-a.im, u.re, fma(-b.re, v.im, b.im * v.re)));
  } else if (has_u) {
    r.re = fma(a.re, u.re, a.im * u.im);
    r.im = fma(a.re, u.im, -a.im * u.re);
  } else if (has_v) {
    r.re = fma(-b.re, v.re, -b.im * v.im);
    r.im = fma(-b.re, v.im, b.im * v.re);
  }
  return r;
}

// advance row mb of V from layer J-1 to layer J (in place, descending ma); at
// even J the middle row mb = J/2 is born from row J/2-1 of layer J-1 (lane - 1)
template <int TJ, int J>
__device__ __forceinline__ void row_born(C2 (&u)[TJ + 1], int mb) {
  if (J % 2 == 0 && J < TJ) {
#pragma unroll
    for (int i = 0; i < J; ++i) {
      C2 v = shfl_up_c2(u[i], 1);
      if (2 * mb == J) {
        const int x = J - 1 - i;  // destination index in row J/2 of layer J-1
        const bool neg = ((x + J / 2) & 1) != 0;
        u[x] = neg ? C2{-v.re, v.im} : C2{v.re, -v.im};
      }
    }
  }
}

template <int TJ, int J>
__device__ __forceinline__ void row_step(C2 (&u)[TJ + 1], const RowGeom<TJ>& g, int mb) {
  // (the callers run 4 lanes per pair, mb <= 3 = TJ/2 - 1: no lane is born at J = TJ, the
  // row-3 lane builds row TJ/2 itself, so the layer-TJ shuffles would be dead work)
  if (J % 2 == 0 && J < TJ) {
    // lane mb = J/2 receives row J/2-1 of layer J-1 from lane-1 (all lanes shuffle)
#pragma unroll
    for (int i = 0; i < J; ++i) {
      C2 v = shfl_up_c2(u[i], 1);
      if (2 * mb == J) {
        const int x = J - 1 - i;  // destination index in row J/2 of layer J-1
        const bool neg = ((x + J / 2) & 1) != 0;
        u[x] = neg ? C2{-v.re, v.im} : C2{v.re, -v.im};
      }
    }
  }
  if (2 * mb > J) return;
#pragma unroll
  for (int ma = J; ma >= 0; --ma) u[ma] = vstep(g.a, g.b, u[ma], u[ma > 0 ? ma - 1 : 0], ma < J, ma > 0);
}

// ------------------------------------------------------------------ reverse-mode dE/dr
// dE_i/dr_ik = dfc u_k F + fc Re(da_k S_a + db_k S_b), with F = sum w Re<U, Y> and
// the complex sensitivities S_a = dF/da, S_b = dF/db from ONE backward sweep of
// the adjoint through the U recursion
//   G^{J-1}[x] = w Y^{J-1}[x] + A(J,x) a G^J[x] - B(J,x+1) b G^J[x+1]
//   S_a += A(J,ma) conj(U^{J-1}[ma]) G^J[ma],  S_b -= B(J,ma) conj(U^{J-1}[ma-1]) G^J[ma]
// The forward rows are kept in shared memory ([slot][lane]); the middle row
// born at even J from row J/2-1 by symmetry passes its adjoint back the same
// way (G_{mb-1}[J-1-x] += (-1)^(x+mb) conj(G_mb[x])).  ~3x fewer FP64
// operations than propagating the three dU/dr_k.
// layer J of row mb from layer J-1 in place (V recursion), no born-row handling
template <int TJ, int J>
__device__ __forceinline__ void row_update(C2 (&u)[TJ + 1], const RowGeom<TJ>& g) {
#pragma unroll
  for (int ma = J; ma >= 0; --ma) u[ma] = vstep(g.a, g.b, u[ma], u[ma > 0 ? ma - 1 : 0], ma < J, ma > 0);
}

template <int TJ, int J>
__device__ __forceinline__ void row_update_active(C2 (&u)[TJ + 1], const RowGeom<TJ>& g, int mb) {
  if (2 * mb > J) return;
  row_update<TJ, J>(u, g);
}

// U_tot with 4 lanes per pair (twojmax 8; see k_snap_deidrj_adj4): lanes own
// rows 0..3, the row-3 lane also builds row 4 of layer 8 from its own row 3 of
// layer 7.  Each lane accumulates its rows over its pairs in registers; one
// store per element into its pair slot, then a fixed-order sum over 8 slots.
constexpr int UI4_WARPS = 4;

// Row 4 of layer 8 is born from row 3 of layer 7, which the row-3 lane parks in
// shared memory (sv: [8][pair slot], its own 8 slots) while its u registers
// advance row 3 to layer 8; the same registers then carry row 4 (no second row
// array: 18 fewer live doubles, no spills).
template <int J>
__device__ __forceinline__ void ui4_layers(C2 (&u)[9], const RowGeom<8>& g, int mb, bool on, double fc,
                                           C2 (&acc)[45], C2* row4, C2* sv) {
  if constexpr (J > 0) {
    ui4_layers<J - 1>(u, g, mb, on, fc, acc, row4, sv);
    if constexpr (J == 8) {
      if (mb == 3)
#pragma unroll
        for (int i = 0; i < J; ++i) sv[i * 8] = u[i];
    }
    row_step<8, J>(u, g, mb);
    if (on && 2 * mb <= J) {
#pragma unroll
      for (int ma = 0; ma <= J; ++ma) {
        C2& a = acc[J * (J + 1) / 2 + ma];
        a.re = fma(fc, u[ma].re, a.re);
        a.im = fma(fc, u[ma].im, a.im);
      }
    }
    if constexpr (J == 8) {
      if (mb == 3) {
#pragma unroll
        for (int i = 0; i < J; ++i) {
          const int x = J - 1 - i;
          const C2 v = sv[i * 8];
          u[x] = ((x + J / 2) & 1) ? C2{-v.re, v.im} : C2{v.re, -v.im};
        }
        u[J] = C2{0.0, 0.0};
      }
      row_update<8, 8>(u, g);
      if (on && mb == 3) {  // row 4 accumulates in the lane's own slot (shared memory)
#pragma unroll
        for (int ma = 0; ma <= 8; ++ma) {
          row4[ma].re = fma(fc, u[ma].re, row4[ma].re);
          row4[ma].im = fma(fc, u[ma].im, row4[ma].im);
        }
      }
    }
  }
}

__global__ void __launch_bounds__(UI4_WARPS * 32)
k_snap_ui_r4(SnapDev D, int64_t natoms, int N, Box box, const double* __restrict__ q,
             const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt, int maxn, C2* __restrict__ utot) {
  griddep_wait();
  constexpr int TJ = 8, R = 4, P = 8;
  extern __shared__ double smem[];
  const int nh = D.nhalf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ps = nh + 2;  // padded pair-slot stride
  C2* part = reinterpret_cast<C2*>(smem) + warp * P * ps;
  // per-pair (a, b, fc) of the whole list, one lane per pair (instead of the 4 row
  // lanes of a slot recomputing it every round)
  double* geo = reinterpret_cast<double*>(reinterpret_cast<C2*>(smem) + UI4_WARPS * P * ps) + warp * SNAP_MAXN * 5;
  C2* sv = reinterpret_cast<C2*>(reinterpret_cast<double*>(reinterpret_cast<C2*>(smem) + UI4_WARPS * P * ps) +
                                 UI4_WARPS * SNAP_MAXN * 5) +
           warp * 8 * P + lane / 4;  // row-3 lanes: layer 7 parked for the row-4 birth
  const int64_t atom = (int64_t)blockIdx.x * UI4_WARPS + warp;
  if (atom >= natoms) return;
  const int64_t b = atom / N;
  const int i = (int)(atom - b * N);
  const double* qb = q + b * (int64_t)N * 3;
  const int p = lane / R, mb = lane - p * R;
  const int32_t* nb = nbr + atom * maxn;
  const int nl = cnt[atom];
  const int k_first = nb[lane];  // with the count, not after it (maxn >= 32; entries past the count are not used)
  C2 acc[45];
#pragma unroll
  for (int k = 0; k < 45; ++k) acc[k] = C2{0.0, 0.0};
  C2* row4 = part + p * ps + c_hoff[TJ] + 4 * (TJ + 1);
  if (mb == 3)
#pragma unroll
    for (int k = 0; k <= TJ; ++k) row4[k] = C2{0.0, 0.0};
  // exact pairs (r < rc) compacted in list order (a Verlet-skin list also holds
  // pairs beyond rc): the slots are those of an exact list, bit for bit
  int n = 0;
  const double rc2 = D.rcut * D.rcut;
  for (int j0 = 0; j0 < nl; j0 += 32) {
    const int j = j0 + lane;
    double dx = 0.0, dy = 0.0, dz = 0.0;
    bool keep = false;
    if (j < nl) {
      pair_vec(qb, i, j0 == 0 ? k_first : nb[j], box, dx, dy, dz);
      keep = D.lists_exact || r2_exact(dx, dy, dz) < rc2;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      PairGeom pg;
      pair_geom(D, dx, dy, dz, pg, false);
      PL_DASSERT(n + __popc(bal & ((1u << lane) - 1u)) < SNAP_MAXN);
      double* o = geo + 5 * (n + __popc(bal & ((1u << lane) - 1u)));
      o[0] = pg.a.re; o[1] = pg.a.im; o[2] = pg.b.re; o[3] = pg.b.im; o[4] = pg.fc;
    }
    n += __popc(bal);
  }
  __syncwarp();
  for (int s0 = 0; s0 < n; s0 += P) {
    const int s = s0 + p;
    const bool valid = s < n;
    RowGeom<TJ> g;
    double fc = 0.0;
    if (valid) {
      const double* o = geo + 5 * s;
      g.a = C2{o[0], o[1]};
      g.b = C2{o[2], o[3]};
      fc = o[4];
    } else {
      g.a = C2{1.0, 0.0};
      g.b = C2{0.0, 0.0};
    }
    C2 u[TJ + 1];
#pragma unroll
    for (int k = 0; k <= TJ; ++k) u[k] = C2{0.0, 0.0};
    u[0] = C2{mb == 0 ? 1.0 : 0.0, 0.0};
    if (valid && mb == 0) acc[0].re += fc;  // J = 0
    ui4_layers<TJ>(u, g, mb, valid, fc, acc, row4, sv);
  }
  {  // each lane owns its (pair slot, rows): plain stores (every element of every slot is written)
    C2* mypart = part + p * ps;
#pragma unroll
    for (int J = 0; J <= TJ; ++J)
      if (2 * mb <= J)
#pragma unroll
        for (int ma = 0; ma <= J; ++ma) mypart[c_hoff[J] + mb * (J + 1) + ma] = acc[J * (J + 1) / 2 + ma];
  }
  __syncwarp();
  C2* out = utot + atom * nh;
  for (int t = lane; t < nh; t += 32) {
    C2 a{0.0, 0.0};
#pragma unroll
    for (int pp = 0; pp < P; ++pp) {
      a.re += part[pp * ps + t].re;
      a.im += part[pp * ps + t].im;
    }
    int J, base;
    half_layer8(t, J, base);
    const int e = t - base;
    const int mbb = e / (J + 1), maa = e - mbb * (J + 1);
    const double sc = __ldg(D.vs + t);  // U = S (.) V (1 on the diagonal)
    a = C2{a.re * sc, a.im * sc};
    if (maa == mbb) a.re += D.wself;
    out[t] = a;
  }
}

// ------------------------------------------------------------------ reverse-mode dE/dr, 4 lanes per pair
// twojmax 8: lanes own half rows 0..3 of a pair (8 pairs per warp instead of 6);
// row 4 exists only in layer 8, where it is born from row 3 of layer 7, so the
// row-3 lane carries it (forward step, direct term, adjoint, and the adjoint of
// the virtual row flowing back to row 3 stay inside that lane).  Balances the
// lanes (rows 0..4 carry 45, 42, 35, 24, 9 elements; the row-3 lane now 33) and
// stores only layers 0..7 (the backward never reads layer 8): 18.4 KB per warp.
__device__ __forceinline__ double half_w(int J, int mb, int ma) {
  return (2 * mb < J || 2 * ma < J) ? 2.0 : (2 * ma == J ? 1.0 : 0.0);
}

// Y sources of the adjoint sweep: one atom's Y half rows (shared memory), or
// the pair form Y_i + Y_k^dagger (see k_snap_deidrj_pair)
struct YSmem {
  const C2* y;
  __device__ __forceinline__ C2 operator()(int J, int row, int x) const { return y[c_hoff[J] + row * (J + 1) + x]; }
};
struct YPair {
  const C2* y;   // Y_i, shared memory
  const C2* yt;  // Y_k^dagger, global
  __device__ __forceinline__ C2 operator()(int J, int row, int x) const {
    // yt is column-interleaved: [J][x][row], so the 4 row lanes of a pair read 64 contiguous bytes
    const double2 t = __ldg(reinterpret_cast<const double2*>(yt) + c_hoff[J] + x * (J / 2 + 1) + row);
    const C2 a = y[c_hoff[J] + row * (J + 1) + x];
    return C2{a.re + t.x, a.im + t.y};
  }
};

// Y_k^dagger staged in shared memory (k_snap_deidrj_tm): same layout as global
// Y_i rows of layer 7 are padded to 9 elements (ypad7): 8 complex = 32 words put the 4
// row lanes of a pair on the same banks (a 4-way conflict on every layer-7 read)
__device__ __forceinline__ int ypad7(int e) {  // shift of half element e in the padded copy
  constexpr int H7 = hoff8(7);
  return e < H7 ? 0 : (e < H7 + 32 ? (e - H7) >> 3 : 4);
}
struct YPairS {
  const C2* y;   // Y_i, shared memory, layer-7 rows padded (ypad7)
  const C2* yt;  // Y_k^dagger, shared memory (staged by a bulk copy per pair)
  __device__ __forceinline__ C2 operator()(int J, int row, int x) const {
    const C2 t = yt[c_hoff[J] + x * (J / 2 + 1) + row];
    const C2 a = y[c_hoff[J] + (J == 7 ? row * 9 : row * (J + 1)) + (J == 8 ? 4 : 0) + x];
    return C2{a.re + t.re, a.im + t.im};
  }
};

// forward-row history of the adjoint sweep: [slot][lane] in shared memory, or
// the lane's own row of tensor memory (k_snap_deidrj_tm: TMEM holds it, freeing
// the shared memory that stages Y_k^dagger).  tcgen05.ld/st are warp-collective
// (.sync.aligned), so the TMEM policy stores and loads on every lane.
struct HistSmem {
  static constexpr bool kTmem = false;
  C2* h;
  int lane;
  template <int J>
  __device__ __forceinline__ void put(const C2 (&u)[9], bool active) const {
    if (active)
#pragma unroll
      for (int ma = 0; ma <= J; ++ma) h[(J * (J + 1) / 2 + ma) * 32 + lane] = u[ma];
  }
  __device__ __forceinline__ C2 at(int slot, int dlane) const { return h[slot * 32 + lane + dlane]; }
  __device__ __forceinline__ void sync() const {}
};

// A complex as two .x2 stores: a double already sits in an aligned register pair, so
// no operand moves (the .x4 form needs 4 consecutive registers and cost ~150 MOVs per
// round; the kernel is bound by instruction fetch, so every instruction counts).
__device__ __forceinline__ void tm_st(uint32_t addr, const C2& v) {
#ifndef PL_TM_ST4
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(__double2loint(v.re)),
               "r"(__double2hiint(v.re))
               : "memory");
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(addr + 2u), "r"(__double2loint(v.im)),
               "r"(__double2hiint(v.im))
               : "memory");
#else
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr),
               "r"(__double2loint(v.re)), "r"(__double2hiint(v.re)), "r"(__double2loint(v.im)),
               "r"(__double2hiint(v.im))
               : "memory");
#endif
}
// issue one load (no wait): the registers are valid only after tm_ld_wait + tm_ld_tie
struct TmRaw {
  uint32_t a, b, c, d;
};
__device__ __forceinline__ TmRaw tm_ld_issue(uint32_t addr) {
  TmRaw r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.a), "=r"(r.b), "=r"(r.c), "=r"(r.d)
               : "r"(addr)
               : "memory");
  return r;
}
__device__ __forceinline__ void tm_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// orders every use of the loaded registers after the wait (volatile statements keep
// their order; no instruction is emitted)
__device__ __forceinline__ C2 tm_ld_tie(TmRaw r) {
  asm volatile("" : "+r"(r.a), "+r"(r.b), "+r"(r.c), "+r"(r.d)::"memory");
  return C2{__hiloint2double((int)r.b, (int)r.a), __hiloint2double((int)r.d, (int)r.c)};
}

struct HistTmem {
  static constexpr bool kTmem = true;
  uint32_t taddr;  // TMEM address of this warp's 32 lanes, column 0 (4 columns per slot)
  template <int J>
  __device__ __forceinline__ void put(const C2 (&u)[9], bool) const {
#pragma unroll
    for (int ma = 0; ma <= J; ++ma) tm_st(taddr + 4u * (J * (J + 1) / 2 + ma), u[ma]);
  }
  // the lane's row of layer J - 1 (J elements): all loads in flight, one wait
  template <int J>
  __device__ __forceinline__ void row(C2 (&L)[9]) const {
    TmRaw r[J];
#pragma unroll
    for (int x = 0; x < J; ++x) r[x] = tm_ld_issue(taddr + 4u * ((J - 1) * J / 2 + x));
    tm_ld_wait();
#pragma unroll
    for (int x = 0; x < J; ++x) L[x] = tm_ld_tie(r[x]);
  }
  __device__ __forceinline__ void sync() const { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
};

struct AdjR4 {
  static constexpr int TJ = 8;
  // forward: layer J from J-1 (in place), store rows of layers <= 7, accumulate F
  template <int J, class YS, bool LAZY = false, class H = HistSmem>
  __device__ __forceinline__ static void fwd(C2 (&u)[TJ + 1], C2 (&u4)[TJ + 1], const RowGeom<TJ>& g, int mb,
                                             const YS& Y, const H& hist, double& F) {
    if constexpr (J > 0) {
      fwd<J - 1, YS, LAZY, H>(u, u4, g, mb, Y, hist, F);
      if constexpr (J == TJ) {
        // virtual row 4 of layer 7 = born image of this lane's row 3 of layer 7
#pragma unroll
        for (int i = 0; i < J; ++i) {
          const int x = J - 1 - i;
          const C2 v = u[i];
          u4[x] = ((x + J / 2) & 1) ? C2{-v.re, v.im} : C2{v.re, -v.im};
        }
        u4[J] = C2{0.0, 0.0};
      }
      // rows 1..3 are born at J = 2, 4, 6 from the lane below.  The history of layer J-1
      // is stored after the born lane received its (virtual) row of layer J-1, so with the
      // history in tensor memory (every lane stores and loads its own row) the adjoint
      // sweep finds the born row's upstream values in its own slots: no second shuffle
      if constexpr (H::kTmem) {
        row_born<TJ, J>(u, mb);
        hist.template put<J - 1>(u, true);
        row_update_active<TJ, J>(u, g, mb);
      } else {
        hist.template put<J - 1>(u, 2 * mb <= J - 1);
        row_step<TJ, J>(u, g, mb);
      }
      if constexpr (J == TJ) row_update<TJ, TJ>(u4, g);
    }
    if (2 * mb <= J) {
#pragma unroll
      for (int ma = 0; ma <= J; ++ma) {
        if constexpr (!LAZY) {
          const C2 y = Y(J, mb, ma);
          F += half_w(J, mb, ma) * (u[ma].re * y.re + u[ma].im * y.im);
        }
      }
    }
    if constexpr (J == TJ && !LAZY) {
      if (mb == TJ / 2 - 1) {
#pragma unroll
        for (int ma = 0; ma <= J; ++ma) {
          const C2 y = Y(J, TJ / 2, ma);
          F += half_w(J, TJ / 2, ma) * (u4[ma].re * y.re + u4[ma].im * y.im);
        }
      }
    }
  }

  // Sa/Sb of one row at layer J, then its adjoint to layer J-1 (in place), for
  // the V recursion V^J[ma] = conj(a) V^{J-1}[ma] - conj(b) V^{J-1}[ma-1]:
  //   S_a += conj(V^{J-1}[ma]) G^J[ma],  S_b -= conj(V^{J-1}[ma-1]) G^J[ma],
  //   G^{J-1}[x] (+)= a G^J[x] - b G^J[x+1]
  template <int J>
  __device__ __forceinline__ static void row_adj(C2 (&G)[TJ + 1], const C2 (&up)[TJ + 1], const RowGeom<TJ>& g,
                                                 C2& Sa, C2& Sb) {
#pragma unroll
    for (int ma = 0; ma <= J; ++ma) {
      if (ma < J) {  // Sa += conj(up) G
        Sa.re = fma(up[ma].re, G[ma].re, fma(up[ma].im, G[ma].im, Sa.re));
        Sa.im = fma(up[ma].re, G[ma].im, fma(-up[ma].im, G[ma].re, Sa.im));
      }
      if (ma > 0) {  // Sb -= conj(up) G
        Sb.re = fma(-up[ma - 1].re, G[ma].re, fma(-up[ma - 1].im, G[ma].im, Sb.re));
        Sb.im = fma(-up[ma - 1].re, G[ma].im, fma(up[ma - 1].im, G[ma].re, Sb.im));
      }
    }
#pragma unroll
    for (int x = 0; x < J; ++x) {  // a G[x] - b G[x+1]
      const C2 p = G[x], q = G[x + 1];
      G[x] = C2{fma(g.a.re, p.re, fma(-g.a.im, p.im, fma(-g.b.re, q.re, g.b.im * q.im))),
                fma(g.a.re, p.im, fma(g.a.im, p.re, fma(-g.b.re, q.im, -g.b.im * q.re)))};
    }
    G[J] = C2{0.0, 0.0};
  }

  // LAZY: F accumulates here from the history rows re-read for the adjoint and
  // the Y elements loaded for G (each Y element read once)
  template <int J, class YS, bool LAZY = false, class H = HistSmem>
  __device__ __forceinline__ static void bwd(C2 (&G)[TJ + 1], C2 (&G4)[TJ + 1], const RowGeom<TJ>& g, int mb,
                                             const YS& Y, const H& hist, C2& Sa, C2& Sb, double& F) {
    if constexpr (J > 0) {

      const bool active = 2 * mb <= J;
      const bool born = (J % 2 == 0) && (J < TJ) && (2 * mb == J);  // rows 1..3: virtual in layer J-1
      C2 up[TJ + 1];
      if constexpr (H::kTmem) {
        // every lane loads its own row of layer J-1 (born rows stored their image of the
        // lane below in the forward pass)
        hist.template row<J>(up);
        if (active) row_adj<J>(G, up, g, Sa, Sb);
      } else if (active) {
#pragma unroll
        for (int x = 0; x < J; ++x) {
          if (!born) {
            up[x] = hist.at((J - 1) * J / 2 + x, 0);
          } else {
            const C2 v = hist.at((J - 1) * J / 2 + (J - 1 - x), -1);
            up[x] = ((x + J / 2) & 1) ? C2{-v.re, v.im} : C2{v.re, -v.im};  // born: mb = J/2
          }
        }
        row_adj<J>(G, up, g, Sa, Sb);
      }
      if constexpr (J == TJ) {
        // row 4 (row-3 lane): its layer-7 image comes from this lane's own row 3
        if (mb == TJ / 2 - 1) {
          C2 up4[TJ + 1];
#pragma unroll
          for (int x = 0; x < J; ++x) {
            C2 v;
            if constexpr (H::kTmem)
              v = up[J - 1 - x];  // this lane's own layer-7 row (not born at J = 8)
            else
              v = hist.at((J - 1) * J / 2 + (J - 1 - x), 0);
            up4[x] = ((x + TJ / 2) & 1) ? C2{-v.re, v.im} : C2{v.re, -v.im};
          }
          row_adj<J>(G4, up4, g, Sa, Sb);
          // adjoint of the virtual row 4 of layer 7 flows to row 3
#pragma unroll
          for (int x = 0; x < J; ++x) {
            const C2 v = G4[x];
            const int xs = J - 1 - x;
            const bool neg = ((x + TJ / 2) & 1) != 0;
            G[xs].re += neg ? -v.re : v.re;
            G[xs].im += neg ? v.im : -v.im;
          }
        }
      } else if constexpr (J % 2 == 0) {
        // rows 1..3 born at J: their adjoint flows to the lane below (same pair)
#pragma unroll
        for (int x = 0; x < J; ++x) {
          const C2 v = C2{__shfl_down_sync(0xffffffffu, G[x].re, 1), __shfl_down_sync(0xffffffffu, G[x].im, 1)};
          if (2 * (mb + 1) == J) {
            const int xs = J - 1 - x;
            constexpr int MBB = J / 2;  // = mb + 1 on the receiving lane: compile-time parity
            const bool neg = ((x + MBB) & 1) != 0;
            G[xs].re += neg ? -v.re : v.re;
            G[xs].im += neg ? v.im : -v.im;
          }
        }
        if (born) {
#pragma unroll
          for (int x = 0; x <= J; ++x) G[x] = C2{0.0, 0.0};
        }
      }
      if (2 * mb <= J - 1) {
#pragma unroll
        for (int x = 0; x < J; ++x) {
          const double w = half_w(J - 1, mb, x);
          const C2 y = Y(J - 1, mb, x);
          if constexpr (LAZY) F += w * (up[x].re * y.re + up[x].im * y.im);
          G[x].re += w * y.re;
          G[x].im += w * y.im;
        }
      }
      bwd<J - 1, YS, LAZY, H>(G, G4, g, mb, Y, hist, Sa, Sb, F);
    }
  }
};

constexpr int ADJ4_SLOTS = 36;  // layers 0..7
// ------------------------------------------------------------------ pair-symmetric reverse-mode dE/dr
// U(-r) = U(r)^dagger (the Cayley-Klein parameters of -r are (conj a, -b), the
// inverse SU(2) element), and the adjoint sweep is linear in Y.  So for the
// unordered pair {i, k} (i < k, r = r_ik) one sweep with Y_i + Y_k^dagger gives
//   h_ik = dE_i/dr_ik - dE_k/dr_ki,
// the whole pair's contribution (grad_i -= h_ik, grad_k += h_ik): half the
// forward/adjoint work of k_snap_deidrj_adj4, same arithmetic per sweep.

// element (r, c) of the full layer-J Y matrix from the stored half rows
// (middle row valid for c <= J/2 after the box kernel's fold)
__device__ __forceinline__ C2 y_full(const C2* y, int J, int base, int r, int c) {  // base: offset of layer J
  if (2 * r > J || (2 * r == J && 2 * c > J)) {
    const C2 v = y[base + (J - r) * (J + 1) + (J - c)];
    return ((r + c) & 1) ? C2{-v.re, v.im} : C2{v.re, -v.im};  // (-1)^(r+c) conj
  }
  return y[base + r * (J + 1) + c];
}

// Y^dagger, half rows stored column-interleaved: yt[J][ma][mb] = conj(Y[J][ma][mb])
// for mb <= J/2 (element (mb, ma) of the Y^dagger half rows).  In the V form
// (see vstep) y holds S (.) Y and yt must hold S (.) Y^dagger:
//   S[ma][mb] conj(Y[ma][mb]) = S[ma][mb]^2 conj((S (.) Y)[ma][mb])   (S[mb][ma] = 1 / S[ma][mb])
__global__ void k_snap_ytrans(int64_t natoms, int nh, const double* __restrict__ vs2, const C2* __restrict__ y,
                              C2* __restrict__ yt) {
  griddep_wait();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= natoms * nh) return;
  const int64_t atom = t / nh;
  const int h = (int)(t - atom * nh);
  int J, base;
  half_layer8(h, J, base);  // the pair form runs at twojmax 8 only
  const int e = h - base;
  const int mb = e / (J + 1), ma = e - mb * (J + 1);
  const C2 v = y_full(y + atom * nh, J, base, ma, mb);
  const double f = __ldg(vs2 + h);
  yt[atom * nh + base + ma * (J / 2 + 1) + mb] = C2{f * v.re, -(f * v.im)};
}

// owner of the unordered pair {i, k}: i when (i + k even and k > i) or (i + k odd
// and k < i).  Antisymmetric, so every pair has one owner; on the BCC lattices
// every atom owns 10-17 of its 26 neighbours (k > i alone gives 0-26, and the
// slowest warp of a small batch waits for 7 rounds instead of 4).
__host__ __device__ __forceinline__ bool pair_owned(int i, int k) { return ((i + k) & 1) ? (k < i) : (k > i); }

constexpr int PAIR_WARPS = 4;  // 2 CTAs of 4 warps per SM (shared memory), neighbouring atoms share an SM
constexpr int PAIR_GEO = 12;   // doubles of geometry per pair (k_snap_deidrj_pair)

// APW atoms per warp; atom i owns its neighbours k > i (a suffix of its sorted
// list), the owned lists of the warp's atoms are concatenated into rounds of 8
// pair slots.  h_ik goes to dedr[i, s] (slots k < i are not written).  Y_i is
// staged in shared memory, Y_k^dagger read through L1/L2; F is accumulated in
// the backward sweep (AdjR4 LAZY) so every Y element is read once; Y^dagger is
// column-interleaved so the 4 row lanes of a pair read 64 contiguous bytes.
// Used for batches under 4 waves of runs (k_snap_deidrj_run otherwise).  At the
// larger config (1025 atoms x 64) this form took 1.30 ms against 1.78 ms for
// adj4 (0.6x its instructions); the global Y_k^dagger loads (long-scoreboard
// stalls) hold the issue rate near 30 %.  Staging Y_k^dagger in shared memory
// (cp.async during the forward pass, Y_i + Y_k^dagger per slot, or through the
// dead history slots) cost occupancy or barriers and measured slower.
template <int APW, int NWB>
__global__ void __launch_bounds__(NWB * 32)
k_snap_deidrj_pair(SnapDev D, int64_t natoms, int N, Box box, const double* __restrict__ q,
                   const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt, int maxn,
                   const C2* __restrict__ ylist, const C2* __restrict__ ytlist, double* __restrict__ dedr) {
  griddep_wait();
  constexpr int TJ = 8, R = 4, P = 8;
  extern __shared__ double smem[];
  const int nh = D.nhalf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  C2* Yw = reinterpret_cast<C2*>(smem) + warp * APW * nh;
  C2* hist = reinterpret_cast<C2*>(smem) + NWB * APW * nh + warp * ADJ4_SLOTS * 32;
  // geometry of 32 consecutive pairs (4 rounds), one lane per pair:
  // a, b, fc, dfc, u[3], sin, cos, 1/r and the partner atom
  double* gb = reinterpret_cast<double*>(reinterpret_cast<C2*>(smem) + NWB * (APW * nh + ADJ4_SLOTS * 32)) +
               warp * 32 * PAIR_GEO;
  int64_t* gk = reinterpret_cast<int64_t*>(reinterpret_cast<double*>(reinterpret_cast<C2*>(smem) +
                                                                     NWB * (APW * nh + ADJ4_SLOTS * 32)) +
                                           NWB * 32 * PAIR_GEO) + warp * 32;
  // list slots of the owned neighbours of the warp's atoms, [APW][SNAP_MAXN]
  int32_t* oslot = reinterpret_cast<int32_t*>(gk + (NWB - warp) * 32) + warp * APW * SNAP_MAXN;
  const int64_t atom0 = ((int64_t)blockIdx.x * NWB + warp) * APW;
  int nat[APW];
  int total = 0;
#pragma unroll
  for (int k = 0; k < APW; ++k) {
    const int64_t a = atom0 + k;
    nat[k] = 0;
    if (a < natoms) {
      const int i = (int)(a % N);
      const int c = cnt[a];
      int m = 0;
      for (int t0 = 0; t0 < c; t0 += 32) {  // compaction of the owned slots, list order
        const int kk = t0 + lane < c ? nbr[a * maxn + t0 + lane] : 0;
        const bool own = t0 + lane < c && pair_owned(i, kk) &&
                         (D.lists_exact || pair_exact(q + (a / N) * (int64_t)N * 3, i, kk, box, D.rcut * D.rcut));
        const unsigned bal = __ballot_sync(0xffffffffu, own);
        if (own) oslot[k * SNAP_MAXN + m + __popc(bal & ((1u << lane) - 1u))] = t0 + lane;
        m += __popc(bal);
      }
      nat[k] = m;
    }
    total += nat[k];
  }
  __syncwarp();
  {  // the warp's Y rows are one contiguous range: all loads in flight before the stores
    constexpr int NL = (APW * 155 + 31) / 32;  // twojmax 8: nh = 155
    const int nel = (int)min((int64_t)APW, natoms - atom0) * nh;
    C2 tmp[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j)
      if (lane + 32 * j < nel) tmp[j] = ylist[atom0 * nh + lane + 32 * j];
#pragma unroll
    for (int j = 0; j < NL; ++j)
      if (lane + 32 * j < nel) Yw[lane + 32 * j] = tmp[j];
  }
  __syncthreads();
  if (atom0 >= natoms) return;
  const int p = lane / R, mb = lane - p * R;
  for (int s0 = 0; s0 < total; s0 += P) {
    if ((s0 & 31) == 0) {  // geometry of pairs s0 .. s0 + 31
      __syncwarp();
      const int t = s0 + lane;
      int kt = t, wt = 0;
#pragma unroll
      for (int a = 0; a + 1 < APW; ++a)
        if (wt == a && kt >= nat[a]) {
          kt -= nat[a];
          wt = a + 1;
        }
      double* o = gb + lane * PAIR_GEO;
      if (t < total) {
        const int64_t at = atom0 + wt;
        const int64_t bt = at / N;
        const int kk = nbr[at * maxn + oslot[wt * SNAP_MAXN + kt]];
        // the partner's Y^dagger (2.5 KB) towards L2 ahead of the rounds that read it
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ytlist + (bt * N + kk) * nh),
                     "r"((unsigned)(nh * sizeof(C2)))
                     : "memory");
        double dx, dy, dz;
        pair_vec(q + bt * (int64_t)N * 3, (int)(at - bt * N), kk, box, dx, dy, dz);
        const double r = sqrt(dx * dx + dy * dy + dz * dz);
        const double inv = 1.0 / r;
        const double u0 = dx * inv, u1 = dy * inv, u2 = dz * inv;
        double sn, cs;
        sincos(D.kappa * (r - D.rmin0), &sn, &cs);
        double fc = 1.0, dfc = 0.0;
        if (D.switchflag) {
          double sa, ca;
          sincos(D.pi_span * (r - D.rmin0), &sa, &ca);
          fc = 0.5 * (ca + 1.0);
          dfc = -D.half_pi_span * sa;
        }
        o[0] = cs; o[1] = -u2 * sn; o[2] = u1 * sn; o[3] = -u0 * sn;  // a, b
        o[4] = fc; o[5] = dfc; o[6] = u0; o[7] = u1; o[8] = u2; o[9] = sn; o[10] = cs; o[11] = inv;
        gk[lane] = bt * N + kk;
      } else {
        o[0] = 1.0; o[1] = 0.0; o[2] = 0.0; o[3] = 0.0;
        gk[lane] = -1;
      }
      __syncwarp();
    }
    int k = s0 + p, w = 0;
#pragma unroll
    for (int a = 0; a + 1 < APW; ++a)
      if (w == a && k >= nat[a]) {
        k -= nat[a];
        w = a + 1;
      }
    const bool valid = s0 + p < total;
    const int64_t atom = atom0 + w;
    const int s = oslot[w * SNAP_MAXN + k];
    const double* go = gb + ((s0 & 31) + p) * PAIR_GEO;
    const int64_t katom = valid ? gk[(s0 & 31) + p] : atom;  // invalid slots: own Y^dagger (weight 0)
    const YPair Y{Yw + w * nh, ytlist + katom * nh};
    RowGeom<TJ> g{C2{go[0], go[1]}, C2{go[2], go[3]}, C2{0.0, 0.0}, C2{0.0, 0.0}};
    C2 u[TJ + 1], u4[TJ + 1];
#pragma unroll
    for (int e = 0; e <= TJ; ++e) u[e] = u4[e] = C2{0.0, 0.0};
    u[0] = C2{mb == 0 ? 1.0 : 0.0, 0.0};
    double F = 0.0;
    AdjR4::fwd<TJ, YPair, true>(u, u4, g, mb, Y, HistSmem{hist, lane}, F);
    __syncwarp();
    C2 G[TJ + 1], G4[TJ + 1];
    {
#pragma unroll
      for (int x = 0; x <= TJ; ++x) {
        G[x] = Y(TJ, mb, x);
        G4[x] = (mb == TJ / 2 - 1) ? Y(TJ, TJ / 2, x) : C2{0.0, 0.0};
      }
    }
#pragma unroll
    for (int x = 0; x <= TJ; ++x) {  // layer-8 terms of F (row mb; row 4 on the row-3 lane)
      const double w8 = half_w(TJ, mb, x), w4 = half_w(TJ, TJ / 2, x);
      if (2 * mb <= TJ) F += w8 * (u[x].re * G[x].re + u[x].im * G[x].im);
      if (mb == TJ / 2 - 1) F += w4 * (u4[x].re * G4[x].re + u4[x].im * G4[x].im);
      G[x] = C2{w8 * G[x].re, w8 * G[x].im};
      G4[x] = C2{w4 * G4[x].re, w4 * G4[x].im};
    }
    C2 Sa{0.0, 0.0}, Sb{0.0, 0.0};
    AdjR4::bwd<TJ, YPair, true>(G, G4, g, mb, Y, HistSmem{hist, lane}, Sa, Sb, F);
    __syncwarp();
#pragma unroll
    for (int r = 1; r < R; ++r) {
      const double f = __shfl_down_sync(0xffffffffu, F, r);
      const double ar = __shfl_down_sync(0xffffffffu, Sa.re, r), ai = __shfl_down_sync(0xffffffffu, Sa.im, r);
      const double br = __shfl_down_sync(0xffffffffu, Sb.re, r), bi = __shfl_down_sync(0xffffffffu, Sb.im, r);
      if (mb == 0) {
        F += f;
        Sa.re += ar; Sa.im += ai;
        Sb.re += br; Sb.im += bi;
      }
    }
    if (valid && mb == 0) {
      const double uu[3] = {go[6], go[7], go[8]};
      C2 da[3], db[3];
      pair_deriv(D.kappa, uu, go[9], go[10], go[11], da, db);
      const double fc = go[4], dfc = go[5];
      double* o = dedr + (atom * maxn + s) * 3;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double re = da[c].re * Sa.re - da[c].im * Sa.im + db[c].re * Sb.re - db[c].im * Sb.im;
        o[c] = dfc * uu[c] * F + fc * re;
      }
    }
  }
}

// Pair form, one warp walking a run of CH consecutive atoms: the owned lists of
// the run are concatenated, a round of 8 slots spans at most 2 atoms (a round
// that would reach a third atom stops short), and Y_i of the live atoms sit in a
// 2-slot ring (slot = local atom parity) refilled by cp.async as soon as an
// atom's last pair is done, behind the next round's forward pass (which reads
// no Y).  Slot fill ~98 % instead of 85 % for 2-atom warps.
template <int CH, int NWB>
__global__ void __launch_bounds__(NWB * 32)
k_snap_deidrj_run(SnapDev D, int64_t natoms, int N, Box box, const double* __restrict__ q,
                  const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt, int maxn,
                  const C2* __restrict__ ylist, const C2* __restrict__ ytlist, double* __restrict__ dedr) {
  griddep_wait();
  constexpr int TJ = 8, R = 4, P = 8;
  extern __shared__ double smem[];
  const int nh = D.nhalf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  C2* base = reinterpret_cast<C2*>(smem);
  C2* Yw = base + warp * 2 * nh;  // ring [2][nh]
  C2* hist = base + NWB * 2 * nh + warp * ADJ4_SLOTS * 32;
  double* gb0 = reinterpret_cast<double*>(base + NWB * (2 * nh + ADJ4_SLOTS * 32));
  double* gb = gb0 + warp * 32 * PAIR_GEO;
  int64_t* gk = reinterpret_cast<int64_t*>(gb0 + NWB * 32 * PAIR_GEO) + warp * 32;
  int16_t* oslot = reinterpret_cast<int16_t*>(reinterpret_cast<int64_t*>(gb0 + NWB * 32 * PAIR_GEO) + NWB * 32) +
                   warp * CH * SNAP_MAXN;
  int32_t* cum = reinterpret_cast<int32_t*>(reinterpret_cast<int16_t*>(
                     reinterpret_cast<int64_t*>(gb0 + NWB * 32 * PAIR_GEO) + NWB * 32) + NWB * CH * SNAP_MAXN) +
                 warp * (CH + 2);
  const int64_t a0 = ((int64_t)blockIdx.x * NWB + warp) * CH;
  const int nrun = (int)max((int64_t)0, min((int64_t)CH, natoms - a0));
  int tot = 0;
  for (int c = 0; c < CH; ++c) {
    if (lane == 0) cum[c] = tot;
    const int base_c = tot;
    if (c < nrun) {
      const int64_t a = a0 + c;
      const int i = (int)(a % N);
      const int n = cnt[a];
      for (int t0 = 0; t0 < n; t0 += 32) {
        const int kk = t0 + lane < n ? nbr[a * maxn + t0 + lane] : 0;
        const bool own = t0 + lane < n && pair_owned(i, kk) &&
                         (D.lists_exact || pair_exact(q + (a / N) * (int64_t)N * 3, i, kk, box, D.rcut * D.rcut));
        const unsigned bal = __ballot_sync(0xffffffffu, own);
        PL_DASSERT(!own || (tot - base_c) + __popc(bal & ((1u << lane) - 1u)) < SNAP_MAXN);
        if (own) oslot[c * SNAP_MAXN + (tot - base_c) + __popc(bal & ((1u << lane) - 1u))] = (int16_t)(t0 + lane);
        tot += __popc(bal);
      }
    }
  }
  if (lane == 0) {
    cum[CH] = tot;
    cum[CH + 1] = tot;
  }
  {  // Y of local atoms 0 and 1 (one contiguous range): loads in flight before the stores
    constexpr int NL = (2 * 155 + 31) / 32;
    const int nel = min(2, nrun) * nh;
    C2 tmp[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j)
      if (lane + 32 * j < nel) tmp[j] = ylist[a0 * nh + lane + 32 * j];
#pragma unroll
    for (int j = 0; j < NL; ++j)
      if (lane + 32 * j < nel) Yw[lane + 32 * j] = tmp[j];
  }
  __syncthreads();
  if (nrun == 0) return;
  const int p = lane / R, mb = lane - p * R;
  int pos = 0, ca = 0, gbase = -64, next_load = 2;
  while (pos < tot) {
    while (cum[ca + 1] <= pos) ++ca;  // first atom of the round (skips atoms without owned pairs)
    const int end = min(min(pos + P, tot), cum[ca + 2]);
    // ring refill: every finished atom hands its slot to the atom two ahead (atoms
    // already finished themselves are skipped, so a slot gets one copy at a time);
    // the copies land behind this round's forward pass
    while (next_load < nrun + 2 && cum[next_load - 1] <= pos) {
      if (next_load < nrun && cum[next_load + 1] > pos) {
        const C2* src = ylist + (a0 + next_load) * nh;
        C2* dst = Yw + (next_load & 1) * nh;
        for (int e = lane; e < nh; e += 32) {
          const unsigned d = (unsigned)__cvta_generic_to_shared(dst + e);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + e) : "memory");
        }
      }
      ++next_load;
    }
    if (pos + P > gbase + 32) {  // geometry of list positions pos .. pos + 31
      __syncwarp();
      gbase = pos;
      const int t = gbase + lane;
      double* o = gb + lane * PAIR_GEO;
      if (t < tot) {
        int ct = ca;
        while (cum[ct + 1] <= t) ++ct;
        const int64_t at = a0 + ct;
        const int64_t bt = at / N;
        const int kk = nbr[at * maxn + oslot[ct * SNAP_MAXN + (t - cum[ct])]];
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ytlist + (bt * N + kk) * nh),
                     "r"((unsigned)(nh * sizeof(C2)))
                     : "memory");
        double dx, dy, dz;
        pair_vec(q + bt * (int64_t)N * 3, (int)(at - bt * N), kk, box, dx, dy, dz);
        const double r = sqrt(dx * dx + dy * dy + dz * dz);
        const double inv = 1.0 / r;
        const double u0 = dx * inv, u1 = dy * inv, u2 = dz * inv;
        double sn, cs;
        sincos(D.kappa * (r - D.rmin0), &sn, &cs);
        double fc = 1.0, dfc = 0.0;
        if (D.switchflag) {
          double sa, ca2;
          sincos(D.pi_span * (r - D.rmin0), &sa, &ca2);
          fc = 0.5 * (ca2 + 1.0);
          dfc = -D.half_pi_span * sa;
        }
        o[0] = cs; o[1] = -u2 * sn; o[2] = u1 * sn; o[3] = -u0 * sn;  // a, b
        o[4] = fc; o[5] = dfc; o[6] = u0; o[7] = u1; o[8] = u2; o[9] = sn; o[10] = cs; o[11] = inv;
        gk[lane] = bt * N + kk;
      } else {
        o[0] = 1.0; o[1] = 0.0; o[2] = 0.0; o[3] = 0.0;
        gk[lane] = -1;
      }
      __syncwarp();
    }
    const int pp = pos + p;
    const bool valid = pp < end;
    const int c = (valid && pp >= cum[ca + 1]) ? ca + 1 : ca;
    const int64_t atom = a0 + c;
    PL_DASSERT(!valid || (c < CH && pp - cum[c] < SNAP_MAXN));
    const int s = valid ? oslot[c * SNAP_MAXN + (pp - cum[c])] : 0;
    const double* go = gb + (valid ? pp - gbase : 0) * PAIR_GEO;
    const int64_t katom = valid ? gk[pp - gbase] : atom;  // invalid slots: own Y^dagger (weight 0)
    const YPair Y{Yw + (c & 1) * nh, ytlist + katom * nh};
    RowGeom<TJ> g{valid ? C2{go[0], go[1]} : C2{1.0, 0.0}, valid ? C2{go[2], go[3]} : C2{0.0, 0.0}, C2{0.0, 0.0},
                  C2{0.0, 0.0}};
    C2 u[TJ + 1], u4[TJ + 1];
#pragma unroll
    for (int e = 0; e <= TJ; ++e) u[e] = u4[e] = C2{0.0, 0.0};
    u[0] = C2{mb == 0 ? 1.0 : 0.0, 0.0};
    double F = 0.0;
    AdjR4::fwd<TJ, YPair, true>(u, u4, g, mb, Y, HistSmem{hist, lane}, F);
    asm volatile("cp.async.wait_all;\n" ::: "memory");  // ring refills issued after the last round
    __syncwarp();
    C2 G[TJ + 1], G4[TJ + 1];
#pragma unroll
    for (int x = 0; x <= TJ; ++x) {
      G[x] = Y(TJ, mb, x);
      G4[x] = (mb == TJ / 2 - 1) ? Y(TJ, TJ / 2, x) : C2{0.0, 0.0};
    }
#pragma unroll
    for (int x = 0; x <= TJ; ++x) {  // layer-8 terms of F (row mb; row 4 on the row-3 lane)
      const double w8 = half_w(TJ, mb, x), w4 = half_w(TJ, TJ / 2, x);
      if (2 * mb <= TJ) F += w8 * (u[x].re * G[x].re + u[x].im * G[x].im);
      if (mb == TJ / 2 - 1) F += w4 * (u4[x].re * G4[x].re + u4[x].im * G4[x].im);
      G[x] = C2{w8 * G[x].re, w8 * G[x].im};
      G4[x] = C2{w4 * G4[x].re, w4 * G4[x].im};
    }
    C2 Sa{0.0, 0.0}, Sb{0.0, 0.0};
    AdjR4::bwd<TJ, YPair, true>(G, G4, g, mb, Y, HistSmem{hist, lane}, Sa, Sb, F);
    __syncwarp();
#pragma unroll
    for (int r = 1; r < R; ++r) {
      const double f = __shfl_down_sync(0xffffffffu, F, r);
      const double ar = __shfl_down_sync(0xffffffffu, Sa.re, r), ai = __shfl_down_sync(0xffffffffu, Sa.im, r);
      const double br = __shfl_down_sync(0xffffffffu, Sb.re, r), bi = __shfl_down_sync(0xffffffffu, Sb.im, r);
      if (mb == 0) {
        F += f;
        Sa.re += ar; Sa.im += ai;
        Sb.re += br; Sb.im += bi;
      }
    }
    if (valid && mb == 0) {
      const double uu[3] = {go[6], go[7], go[8]};
      C2 da[3], db[3];
      pair_deriv(D.kappa, uu, go[9], go[10], go[11], da, db);
      const double fc = go[4], dfc = go[5];
      double* o = dedr + (atom * maxn + s) * 3;
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) {
        const double re = da[cc].re * Sa.re - da[cc].im * Sa.im + db[cc].re * Sb.re - db[cc].im * Sb.im;
        o[cc] = dfc * uu[cc] * F + fc * re;
      }
    }
    pos = end;
  }
}

// k_snap_deidrj_tm: the run kernel with the forward-row history in tensor
// memory (each warp its 32 TMEM lanes, 36 slots x 4 columns) and the round's
// Y_k^dagger staged in the shared memory that frees: one bulk copy (TMA engine)
// per pair, issued when the round starts and landing behind its forward pass
// (which reads no Y), so the adjoint sweep reads both Y terms from shared memory
// instead of stalling on L2.  Same arithmetic as k_snap_deidrj_run (bitwise).
// Pair form, one warp walking a run of CH consecutive atoms: the owned lists of
// the run are concatenated, a round of 8 slots spans at most 2 atoms (a round
// that would reach a third atom stops short), and Y_i of the live atoms sit in a
// 2-slot ring (slot = local atom parity) refilled by cp.async as soon as an
// atom's last pair is done, behind the next round's forward pass (which reads
// no Y).  Slot fill ~98 % instead of 85 % for 2-atom warps.
template <int CH, int NWB>
__global__ void __launch_bounds__(NWB * 32)
k_snap_deidrj_tm(SnapDev D, int64_t natoms, int N, Box box, const double* __restrict__ q,
                  const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt, int maxn,
                  const C2* __restrict__ ylist, const C2* __restrict__ ytlist, double* __restrict__ dedr) {
  griddep_wait();
  constexpr int TJ = 8, R = 4, P = 8;
  extern __shared__ double smem[];
  const int nh = D.nhalf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int GB = 16;  // pairs per geometry batch (2 rounds; shared memory budget)
  C2* base = reinterpret_cast<C2*>(smem);
  const int nhp = nh + 4;           // Y_i slot with the layer-7 rows padded (ypad7)
  C2* Yw = base + warp * 2 * nhp;  // ring [2][nhp]
  // Y_k^dagger of the round's pairs [P][nh + 1]: the slot stride of 156 complex = 624
  // words = 16 mod 32 puts the 64-byte reads of the two pairs of a quarter warp on
  // disjoint bank halves (155: 12 mod 32, they overlap)
  const int sts = nh + 1;
  C2* stg = base + NWB * 2 * nhp + warp * P * sts;
  double* gb0 = reinterpret_cast<double*>(base + NWB * (2 * nhp + P * (nh + 1)));
  double* gb = gb0 + warp * GB * PAIR_GEO;
  int64_t* gk = reinterpret_cast<int64_t*>(gb0 + NWB * GB * PAIR_GEO) + warp * GB;
  int16_t* oslot = reinterpret_cast<int16_t*>(reinterpret_cast<int64_t*>(gb0 + NWB * GB * PAIR_GEO) + NWB * GB) +
                   warp * CH * SNAP_MAXN;
  int32_t* cum = reinterpret_cast<int32_t*>(reinterpret_cast<int16_t*>(
                     reinterpret_cast<int64_t*>(gb0 + NWB * GB * PAIR_GEO) + NWB * GB) + NWB * CH * SNAP_MAXN) +
                 warp * (CH + 2);
  __shared__ __align__(8) uint64_t s_mbar[NWB];
  __shared__ uint32_t s_tmem;
  // tensor memory: 256 columns per 4 warps (2 CTAs of 4 warps per SM, or one of 8), warp w
  // uses the lanes of its sub-partition (w % 4) and the column half w / 4
  constexpr unsigned TCOLS = NWB > 4 ? 512u : 256u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&s_tmem)), "n"(TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  const unsigned mbar = (unsigned)__cvta_generic_to_shared(&s_mbar[warp]);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // broadcast from lane 0: the compiler then knows the address is warp-uniform and keeps
  // it in a uniform register (otherwise one R2UR per tcgen05.ld/st, ~100 per round)
  const HistTmem hist{__shfl_sync(0xffffffffu, s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 256u * (uint32_t)(warp >> 2), 0)};
  unsigned phase = 0;
  const int64_t a0 = ((int64_t)blockIdx.x * NWB + warp) * CH;
  const int nrun = (int)max((int64_t)0, min((int64_t)CH, natoms - a0));
  int tot = 0;
  // the run's counts, list entries and exact-pair tests are loaded up front, all in
  // flight together (three dependent global loads per atom, one atom after the other,
  // were ~3 % of the kernel's samples); the lists hold SNAP_MAXN = 2 x 32 entries
  const int cn_l = lane < nrun ? cnt[a0 + lane] : 0;
  int kk_r[CH][2];
  bool own_r[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
      kk_r[c][hf] = (c < nrun && maxn == SNAP_MAXN) ? nbr[(a0 + c) * maxn + 32 * hf + lane] : 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int n = __shfl_sync(0xffffffffu, cn_l, c);
    const int64_t a = a0 + c;
    const int i = (int)(a % N);
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      const int kk = kk_r[c][hf];
      own_r[c][hf] = maxn == SNAP_MAXN && c < nrun && 32 * hf + lane < n && pair_owned(i, kk) &&
                     (D.lists_exact || pair_exact(q + (a / N) * (int64_t)N * 3, i, kk, box, D.rcut * D.rcut));
    }
  }
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    if (lane == 0) cum[c] = tot;
    const int base_c = tot;
    if (c < nrun) {
      const int64_t a = a0 + c;
      const int i = (int)(a % N);
      const int n = __shfl_sync(0xffffffffu, cn_l, c);
#pragma unroll 1
      for (int t0 = 0; t0 < n; t0 += 32) {
        bool own;
        if (maxn == SNAP_MAXN) {
          own = t0 == 0 ? own_r[c][0] : own_r[c][1];
        } else {
          const int kk = t0 + lane < n ? nbr[a * maxn + t0 + lane] : 0;
          own = t0 + lane < n && pair_owned(i, kk) &&
                (D.lists_exact || pair_exact(q + (a / N) * (int64_t)N * 3, i, kk, box, D.rcut * D.rcut));
        }
        const unsigned bal = __ballot_sync(0xffffffffu, own);
        PL_DASSERT(!own || (tot - base_c) + __popc(bal & ((1u << lane) - 1u)) < SNAP_MAXN);
        if (own) oslot[c * SNAP_MAXN + (tot - base_c) + __popc(bal & ((1u << lane) - 1u))] = (int16_t)(t0 + lane);
        tot += __popc(bal);
      }
    }
  }
  if (lane == 0) {
    cum[CH] = tot;
    cum[CH + 1] = tot;
  }
  {  // Y of local atoms 0 and 1 (one contiguous range): loads in flight before the stores
    constexpr int NL = (2 * 155 + 31) / 32;
    const int nel = min(2, nrun) * nh;
    C2 tmp[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j)
      if (lane + 32 * j < nel) tmp[j] = ylist[a0 * nh + lane + 32 * j];
#pragma unroll
    for (int j = 0; j < NL; ++j)
      if (lane + 32 * j < nel) {
        const int g = lane + 32 * j, w = g >= nh ? 1 : 0, e = g - w * nh;
        Yw[w * nhp + e + ypad7(e)] = tmp[j];
      }
  }
  __syncthreads();
  const int p = lane / R, mb = lane - p * R;
  int pos = 0, ca = 0, gbase = -64, next_load = 2;
  while (nrun > 0 && pos < tot) {
    while (cum[ca + 1] <= pos) ++ca;  // first atom of the round (skips atoms without owned pairs)
    const int end = min(min(pos + P, tot), cum[ca + 2]);
    // ring refill: every finished atom hands its slot to the atom two ahead (atoms
    // already finished themselves are skipped, so a slot gets one copy at a time);
    // the copies land behind this round's forward pass
    while (next_load < nrun + 2 && cum[next_load - 1] <= pos) {
      if (next_load < nrun && cum[next_load + 1] > pos) {
        const C2* src = ylist + (a0 + next_load) * nh;
        C2* dst = Yw + (next_load & 1) * nhp;
        for (int e = lane; e < nh; e += 32) {
          const unsigned d = (unsigned)__cvta_generic_to_shared(dst + e + ypad7(e));
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + e) : "memory");
        }
      }
      ++next_load;
    }
    if (pos + P > gbase + GB) {  // geometry of list positions pos .. pos + GB - 1
      __syncwarp();
      gbase = pos;
      const int t = gbase + lane;
      double* o = gb + (lane < GB ? lane : 0) * PAIR_GEO;
      if (lane < GB && t < tot) {
        int ct = ca;
        while (cum[ct + 1] <= t) ++ct;
        const int64_t at = a0 + ct;
        const int64_t bt = at / N;
        const int kk = nbr[at * maxn + oslot[ct * SNAP_MAXN + (t - cum[ct])]];
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ytlist + (bt * N + kk) * nh),
                     "r"((unsigned)(nh * sizeof(C2)))
                     : "memory");
        double dx, dy, dz;
        pair_vec(q + bt * (int64_t)N * 3, (int)(at - bt * N), kk, box, dx, dy, dz);
        const double r = sqrt(dx * dx + dy * dy + dz * dz);
        const double inv = 1.0 / r;
        const double u0 = dx * inv, u1 = dy * inv, u2 = dz * inv;
        double sn, cs;
        sincos(D.kappa * (r - D.rmin0), &sn, &cs);
        double fc = 1.0, dfc = 0.0;
        if (D.switchflag) {
          double sa, ca2;
          sincos(D.pi_span * (r - D.rmin0), &sa, &ca2);
          fc = 0.5 * (ca2 + 1.0);
          dfc = -D.half_pi_span * sa;
        }
        o[0] = cs; o[1] = -u2 * sn; o[2] = u1 * sn; o[3] = -u0 * sn;  // a, b
        o[4] = fc; o[5] = dfc; o[6] = u0; o[7] = u1; o[8] = u2; o[9] = sn; o[10] = cs; o[11] = inv;
        gk[lane] = bt * N + kk;
      } else if (lane < GB) {
        o[0] = 1.0; o[1] = 0.0; o[2] = 0.0; o[3] = 0.0;
        gk[lane] = -1;
      }
      __syncwarp();
    }
    // stage the round's Y_k^dagger: one bulk copy per valid pair, completing on the
    // warp's mbarrier; it lands while the forward pass (no Y) runs
    {
      const int nv = end - pos;
      // the previous round's reads of the staging buffer (generic proxy) are done
      // (consumed by its sweep); order them before the bulk writes (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar),
                     "r"((unsigned)(nv * nh * sizeof(C2)))
                     : "memory");
      __syncwarp();
      PL_DASSERT(nv >= 1 && nv <= P && pos + nv - 1 - gbase < GB);
      if (lane < nv)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                (unsigned)__cvta_generic_to_shared(stg + lane * sts)),
            "l"(ytlist + gk[pos + lane - gbase] * nh), "r"((unsigned)(nh * sizeof(C2))), "r"(mbar)
            : "memory");
    }
    const int pp = pos + p;
    const bool valid = pp < end;
    const int c = (valid && pp >= cum[ca + 1]) ? ca + 1 : ca;
    const int64_t atom = a0 + c;
    PL_DASSERT(!valid || (c < CH && pp - cum[c] < SNAP_MAXN));
    const int s = valid ? oslot[c * SNAP_MAXN + (pp - cum[c])] : 0;
    const double* go = gb + (valid ? pp - gbase : 0) * PAIR_GEO;
    const int64_t katom = valid ? gk[pp - gbase] : atom;  // invalid slots: own Y^dagger (weight 0)
    (void)katom;
    const YPairS Y{Yw + (c & 1) * nhp, stg + p * sts};  // invalid slots read stale but finite data (weight 0)
    RowGeom<TJ> g{valid ? C2{go[0], go[1]} : C2{1.0, 0.0}, valid ? C2{go[2], go[3]} : C2{0.0, 0.0}, C2{0.0, 0.0},
                  C2{0.0, 0.0}};
    C2 u[TJ + 1], u4[TJ + 1];
#pragma unroll
    for (int e = 0; e <= TJ; ++e) u[e] = u4[e] = C2{0.0, 0.0};
    u[0] = C2{mb == 0 ? 1.0 : 0.0, 0.0};
    double F = 0.0;
    AdjR4::fwd<TJ, YPairS, true>(u, u4, g, mb, Y, hist, F);
    asm volatile("cp.async.wait_all;\n" ::: "memory");  // ring refills issued after the last round
    asm volatile(
        "{\n .reg .pred q;\n WT: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n @!q bra WT;\n}" ::"r"(mbar),
        "r"(phase)
        : "memory");
    phase ^= 1u;
    hist.sync();  // history stores complete before the sweep reads them
    __syncwarp();
    C2 G[TJ + 1], G4[TJ + 1];
#pragma unroll
    for (int x = 0; x <= TJ; ++x) {
      G[x] = Y(TJ, mb, x);
      G4[x] = (mb == TJ / 2 - 1) ? Y(TJ, TJ / 2, x) : C2{0.0, 0.0};
    }
#pragma unroll
    for (int x = 0; x <= TJ; ++x) {  // layer-8 terms of F (row mb; row 4 on the row-3 lane)
      const double w8 = half_w(TJ, mb, x), w4 = half_w(TJ, TJ / 2, x);
      if (2 * mb <= TJ) F += w8 * (u[x].re * G[x].re + u[x].im * G[x].im);
      if (mb == TJ / 2 - 1) F += w4 * (u4[x].re * G4[x].re + u4[x].im * G4[x].im);
      G[x] = C2{w8 * G[x].re, w8 * G[x].im};
      G4[x] = C2{w4 * G4[x].re, w4 * G4[x].im};
    }
    C2 Sa{0.0, 0.0}, Sb{0.0, 0.0};
    AdjR4::bwd<TJ, YPairS, true>(G, G4, g, mb, Y, hist, Sa, Sb, F);
    __syncwarp();
#pragma unroll
    for (int r = 1; r < R; ++r) {
      const double f = __shfl_down_sync(0xffffffffu, F, r);
      const double ar = __shfl_down_sync(0xffffffffu, Sa.re, r), ai = __shfl_down_sync(0xffffffffu, Sa.im, r);
      const double br = __shfl_down_sync(0xffffffffu, Sb.re, r), bi = __shfl_down_sync(0xffffffffu, Sb.im, r);
      if (mb == 0) {
        F += f;
        Sa.re += ar; Sa.im += ai;
        Sb.re += br; Sb.im += bi;
      }
    }
    if (valid && mb == 0) {
      const double uu[3] = {go[6], go[7], go[8]};
      C2 da[3], db[3];
      pair_deriv(D.kappa, uu, go[9], go[10], go[11], da, db);
      const double fc = go[4], dfc = go[5];
      double* o = dedr + (atom * maxn + s) * 3;
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) {
        const double re = da[cc].re * Sa.re - da[cc].im * Sa.im + db[cc].re * Sb.re - db[cc].im * Sb.im;
        o[cc] = dfc * uu[cc] * F + fc * re;
      }
    }
    pos = end;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "n"(TCOLS) : "memory");
}

// gather of the pair form, one warp per atom (lanes over neighbour slots, the
// reverse-slot searches in parallel, fixed-order shuffle tree):
// grad_i = -sum_{owned} h_ik + sum_{owned by k} h_ki; the owner books the pair virial
__global__ void __launch_bounds__(128)
k_snap_gather_pair_w(int64_t natoms, int N, Box box, const double* __restrict__ q,
                     const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt, int maxn,
                     const double* __restrict__ dedr, double* __restrict__ grad, double* __restrict__ vatom,
                     double rc2, int lists_exact) {
  griddep_wait();
  __shared__ int16_t s_slot[4][SNAP_MAXN];  // list slots of the exact pairs, in list order
  const int64_t atom = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, wib = (threadIdx.x >> 5) & 3;
  if (atom >= natoms) return;
  const int64_t b = atom / N;
  const int a = (int)(atom - b * N);
  const int nl = cnt[atom];
  const int32_t* nb = nbr + atom * maxn;
  const double* qb = q + b * (int64_t)N * 3;
  // exact pairs (r < rc) compacted in list order: the e-th one is handled by lane
  // e % 32 as in an exact list, whatever skin pairs the list also holds
  int n = 0;
  for (int s0 = 0; s0 < nl; s0 += 32) {
    const int s = s0 + lane;
    const bool keep = s < nl && (lists_exact || pair_exact(qb, a, nb[s], box, rc2));
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      PL_DASSERT(n + __popc(bal & ((1u << lane) - 1u)) < SNAP_MAXN);
      s_slot[wib][n + __popc(bal & ((1u << lane) - 1u))] = (int16_t)s;
    }
    n += __popc(bal);
  }
  __syncwarp();
  double v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // g[3], vir[6]
  for (int e = lane; e < n; e += 32) {
    const int s = s_slot[wib][e];
    const int k = nb[s];
    if (pair_owned(a, k)) {
      const double* h = dedr + (atom * maxn + s) * 3;
      v[0] -= h[0];
      v[1] -= h[1];
      v[2] -= h[2];
      if (vatom) {
        double dx, dy, dz;
        pair_vec(qb, a, k, box, dx, dy, dz);
        v[3] -= h[0] * dx;
        v[4] -= h[1] * dy;
        v[5] -= h[2] * dz;
        v[6] -= 0.5 * (h[0] * dy + h[1] * dx);
        v[7] -= 0.5 * (h[0] * dz + h[2] * dx);
        v[8] -= 0.5 * (h[1] * dz + h[2] * dy);
      }
    } else {
      const int64_t katom = b * N + k;
      const int32_t* kl = nbr + katom * maxn;
      int lo = 0, hi = cnt[katom] - 1, sk = -1;
      while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        const int val = kl[mid];
        if (val == a) { sk = mid; break; }
        if (val < a) lo = mid + 1; else hi = mid - 1;
      }
      if (sk >= 0) {
        const double* h = dedr + (katom * maxn + sk) * 3;
        v[0] += h[0];
        v[1] += h[1];
        v[2] += h[2];
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 9; ++c)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[c] += __shfl_xor_sync(0xffffffffu, v[c], o);
  if (lane == 0) {
    if (grad) {
      grad[3 * atom] = v[0];
      grad[3 * atom + 1] = v[1];
      grad[3 * atom + 2] = v[2];
    }
    if (vatom)
      for (int c = 0; c < 6; ++c) vatom[6 * atom + c] = v[3 + c];
  }
}

// ------------------------------------------------------------------ kernel: gather
__global__ void k_snap_gather(int64_t natoms, int N, Box box, const double* __restrict__ q,
                              const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt,
                              int maxn, const double* __restrict__ dedr, double* __restrict__ grad,
                              double* __restrict__ vatom) {
  int64_t atom = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (atom >= natoms) return;
  int64_t b = atom / N;
  int a = (int)(atom - b * N);
  int n = cnt[atom];
  const int32_t* nb = nbr + atom * maxn;
  double gx = 0.0, gy = 0.0, gz = 0.0;
  double v[6] = {0, 0, 0, 0, 0, 0};
  const double* qb = q + b * (int64_t)N * 3;
  for (int s = 0; s < n; ++s) {
    int k = nb[s];
    int64_t katom = b * N + k;
    const int32_t* kl = nbr + katom * maxn;
    int lo = 0, hi = cnt[katom] - 1, sk = -1;
    while (lo <= hi) {  // lists are sorted ascending
      int mid = (lo + hi) >> 1;
      int val = kl[mid];
      if (val == a) { sk = mid; break; }
      if (val < a) lo = mid + 1; else hi = mid - 1;
    }
    const double* ga = dedr + (atom * maxn + s) * 3;
    gx -= ga[0];
    gy -= ga[1];
    gz -= ga[2];
    if (sk >= 0) {
      const double* gk = dedr + (katom * maxn + sk) * 3;
      gx += gk[0];
      gy += gk[1];
      gz += gk[2];
    }
    if (vatom) {
      double dx, dy, dz;
      pair_vec(qb, a, k, box, dx, dy, dz);
      v[0] -= ga[0] * dx;
      v[1] -= ga[1] * dy;
      v[2] -= ga[2] * dz;
      v[3] -= 0.5 * (ga[0] * dy + ga[1] * dx);
      v[4] -= 0.5 * (ga[0] * dz + ga[2] * dx);
      v[5] -= 0.5 * (ga[1] * dz + ga[2] * dy);
    }
  }
  if (grad) {
    grad[3 * atom] = gx;
    grad[3 * atom + 1] = gy;
    grad[3 * atom + 2] = gz;
  }
  if (vatom)
    for (int c = 0; c < 6; ++c) vatom[6 * atom + c] = v[c];
}

__global__ void k_sys_sum(int64_t B, int N, int width, const double* __restrict__ per_atom,
                          double* __restrict__ out) {
  griddep_wait();
  __shared__ double sh[256];
  int64_t b = blockIdx.x;
  for (int c = 0; c < width; ++c) {
    double s = 0.0;
    for (int i = threadIdx.x; i < N; i += blockDim.x) s += per_atom[(b * N + i) * width + c];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[b * width + c] = sh[0];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ host driver
struct SnapBuffers {
  C2* utot;
  C2* y;
  C2* yt;     // Y^dagger (pair form only)
  bool pair;  // dedr holds h_ik on owned slots (k_snap_deidrj_pair) instead of dE_i/dr_ik
  bool lists_exact = true;  // no Verlet-skin pairs in the lists
  double* eatom;
  double* dedr;
  double* vatom;
};

static size_t ui_smem(const SnapDev& D) {
  int layer_max = (D.tj + 1) * (D.tj / 2 + 1);
  return sizeof(C2) * (UI_WARPS * D.nhalf + UI_WARPS * 2 * layer_max);
}
static size_t yi_smem(const SnapDev& D) {
  return sizeof(C2) * D.nhalf * YI_ATOMS + sizeof(double) * YI_WARPS * YI_ATOMS;
}
static size_t de_smem(const SnapDev& D) {
  int layer_max = (D.tj + 1) * (D.tj / 2 + 1);
  return sizeof(C2) * (D.nhalf + DE_WARPS * 2 * 4 * layer_max);
}

// Kernel selection.  twojmax = 8 (the BASELINE potential) runs the specialised
// kernels: k_snap_ui_r4, the box-form Y kernel (snap_yi8.cu) and the
// pair-symmetric force kernels.  Every other twojmax runs the general kernels
// k_snap_ui / k_snap_yi / k_snap_deidrj, which PL_SNAP_GENERIC=1 also forces at
// twojmax = 8 so the two families can be checked against each other.
// PL_SNAP_PAIR_RUN = 0 / 2 forces 2-atom warps / 8-atom runs of the pair kernel
// at every batch size (both give bitwise-identical forces; tests).
static bool snap_generic_forced() {
  static const bool g = [] {
    const char* e = getenv("PL_SNAP_GENERIC");
    return e && e[0] == '1';
  }();
  return g;
}

static int snap_stages(pl_pot* pot, int64_t B, const double* q, SnapBuffers& buf, NeighList& nl) {
  pl_ctx* ctx = pot->ctx;
  SnapIndex* S = pot->snap;
  SnapDev D = snap_dev(pot);
  int N = pot->n_atoms;
  int64_t na = B * N;
  if (na > 0x7fffffff) return fail(PL_EARG, "too many atoms in one batch");
  // Verlet skin inside a window propagation (twojmax-8 kernels only: they compact
  // the exact pairs): lists to rcut + skin, rebuilt on the device when an atom
  // moved more than skin/2 (no host synchronisation); forced at every window start
  // (systems of >= 512 atoms, the cell-list builds; a brute-force build of a small
  // system costs less than the check)
  const bool skin = pot->skin_on && pot->skin > 0.0 && S->tj == 8 && S->yi_reg && !snap_generic_forced() &&
                    N >= 512;
  D.lists_exact = skin ? 0 : 1;
  buf.lists_exact = !skin;
  const int* go = nullptr;
  double* qref = nullptr;
  if (skin) {
    PL_TRY(pot->work[4].reserve(sizeof(double) * 3 * na + 64));
    qref = (double*)pot->work[4].ptr;
    int* flag = (int*)(qref + 3 * na);
    if (pot->skin_force || pot->skin_B != B) {
      PL_CUDA(cudaMemcpyAsync(qref, q, sizeof(double) * 3 * na, cudaMemcpyDeviceToDevice, ctx->stream));
      pot->skin_force = false;
      pot->skin_B = B;
    } else {
      PL_TRY(skin_check(pot, na, q, qref, flag));
      go = flag;
    }
  }
  PL_TRY(build_neighbours(pot, B, q, pot->rcut + (skin ? pot->skin : 0.0), SNAP_MAXN, &nl, go));
  if (go) PL_TRY(skin_ref(pot, na, q, qref, go));
  // + 25 x na doubles: per-row energies of the split Y kernel (small batches)
  // + na x nhalf C2: Y^dagger of the pair-symmetric force kernel
  size_t bytes = sizeof(C2) * 3 * na * S->nhalf + sizeof(double) * na * (1 + 3 * SNAP_MAXN + 6 + 25);
  PL_TRY(pot->work[2].reserve(bytes));
  buf.utot = (C2*)pot->work[2].ptr;
  buf.y = buf.utot + na * S->nhalf;
  buf.eatom = (double*)(buf.y + na * S->nhalf);
  buf.dedr = buf.eatom + na;
  buf.vatom = buf.dedr + na * 3 * SNAP_MAXN;
  double* erow = buf.vatom + na * 6;
  buf.yt = reinterpret_cast<C2*>(erow + na * 25);
  buf.pair = false;
  Box box = make_box(pot->box);
  static std::atomic<uint64_t> attr_devs{0};
  if (first_on_device(attr_devs)) {
    cudaFuncSetAttribute(k_snap_ui, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_yi, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_deidrj, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_bispectrum, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_deidrj_pair<2, PAIR_WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_deidrj_run<8, PAIR_WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_deidrj_tm<8, PAIR_WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_deidrj_tm<2, PAIR_WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_deidrj_tm<8, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
    cudaFuncSetAttribute(k_snap_ui_r4, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  const bool special = S->tj == 8 && S->yi_reg && !snap_generic_forced();
  prof_mark(ctx->stream, ST_UI, true);
  if (special) {
    const size_t sm4 = sizeof(C2) * UI4_WARPS * 8 * (D.nhalf + 2) + sizeof(double) * UI4_WARPS * SNAP_MAXN * 5 +
                       sizeof(C2) * UI4_WARPS * 8 * 8;
    PL_CUDA(launch_pdl(k_snap_ui_r4, dim3((unsigned)((na + UI4_WARPS - 1) / UI4_WARPS)), dim3(UI4_WARPS * 32), sm4,
                       ctx->stream, D, na, N, box, q, nl.nbr, nl.cnt, nl.maxn, buf.utot));
  } else {
    k_snap_ui<<<(unsigned)na, UI_WARPS * 32, ui_smem(D), ctx->stream>>>(D, na, N, box, q, nl.nbr, nl.cnt, nl.maxn,
                                                                       buf.utot);
  }
  PL_CHECK_LAUNCH();
  prof_mark(ctx->stream, ST_UI, false);
  prof_mark(ctx->stream, ST_YI, true);
  bool yt_done = false;  // the unsplit Y kernel also writes S (.) Y^dagger
  if (special) {
    PL_CUDA(snap_box_launch(ctx->stream, na, D.beta0, D.yi5, D.vs, buf.utot, buf.y, buf.eatom, erow, buf.yt, &yt_done));
  } else {
    k_snap_yi<<<(unsigned)((na + YI_ATOMS - 1) / YI_ATOMS), YI_THREADS, yi_smem(D), ctx->stream>>>(D, na, buf.utot,
                                                                                                 buf.y, buf.eatom);
  }
  PL_CHECK_LAUNCH();
  prof_mark(ctx->stream, ST_YI, false);
  prof_mark(ctx->stream, ST_DE, true);
  if (special) {
    const int64_t nel = na * D.nhalf;
    if (!yt_done) {
      PL_CUDA(launch_pdl(k_snap_ytrans, dim3((unsigned)((nel + 255) / 256)), dim3(256), 0, ctx->stream, na, D.nhalf,
                         D.vs + D.nhalf, buf.y, buf.yt));
      PL_CHECK_LAUNCH();
    }
    static const int prun = [] {
      const char* e = getenv("PL_SNAP_PAIR_RUN");
      return e ? atoi(e) : 1;  // 0: 2-atom warps only, 2: runs at every size (tests)
    }();
    constexpr int RUN = 8;
    static const bool tmem = [] {  // history in tensor memory + staged Y_k^dagger (PL_SNAP_TMEM=0: k_snap_deidrj_run)
      const char* e = getenv("PL_SNAP_TMEM");
      return !(e && e[0] == '0');
    }();
    // runs (8 atoms per warp, one 8-warp CTA per SM) when their waves are well filled: a
    // wave of run CTAs takes ~0.117 ms whatever its fill, the 2-atom form ~0.0148 ms per
    // 1000 atoms (measured, 8,200-65,600 atoms), so runs win at a fill >= 0.84
    // (8,200 atoms: 0.122 -> 0.117 ms; 16,001: 0.229 -> 0.218; 19,350: three waves at 0.68 lose)
    bool big = prun == 2;
    if (prun == 1) {
      const int64_t ctas = (na + 8 * RUN - 1) / (8 * RUN), waves = (ctas + 147) / 148;
      big = (double)na >= 0.84 * (double)(waves * 148 * 8 * RUN);
    }
    auto tm_smem = [&](int ch, int nwb = PAIR_WARPS) {
      constexpr int GB = 16;
      return sizeof(C2) * nwb * (2 * (D.nhalf + 4) + 8 * (D.nhalf + 1)) + (sizeof(double) * PAIR_GEO + sizeof(int64_t)) * nwb * GB +
             sizeof(int16_t) * nwb * ch * SNAP_MAXN + sizeof(int32_t) * nwb * (ch + 2);
    };
    // large batches: one CTA of 8 warps per SM instead of two of 4.  The round's code
    // (~75 KB) exceeds the SM's 32 KB instruction cache and the kernel is bound by
    // instruction fetches from the GPC-level cache (ncu: gcc instruction requests 91 % of
    // peak); 8 warps launched together walk the code closer to each other and share more
    // of the fetched lines: 0.912 -> 0.868 ms at the larger config.  (A barrier per round,
    // full lockstep, costs more than it saves: 0.94 ms.)  PL_SNAP_TM8=0: 4-warp CTAs.
    static const bool tm8 = [] {
      const char* e = getenv("PL_SNAP_TM8");
      return !(e && e[0] == '0');
    }();
    if (tmem && big && tm8) {
      constexpr int NWB8 = 8;
      const unsigned grid = (unsigned)((na + NWB8 * RUN - 1) / (NWB8 * RUN));
      PL_CUDA(launch_pdl(k_snap_deidrj_tm<RUN, NWB8>, dim3(grid), dim3(NWB8 * 32), tm_smem(RUN, NWB8), ctx->stream, D,
                         na, N, box, q, nl.nbr, nl.cnt, nl.maxn, buf.y, buf.yt, buf.dedr));
    } else if (tmem && big) {
      const unsigned grid = (unsigned)((na + PAIR_WARPS * RUN - 1) / (PAIR_WARPS * RUN));
      PL_CUDA(launch_pdl(k_snap_deidrj_tm<RUN, PAIR_WARPS>, dim3(grid), dim3(PAIR_WARPS * 32), tm_smem(RUN),
                         ctx->stream, D, na, N, box, q, nl.nbr, nl.cnt, nl.maxn, buf.y, buf.yt, buf.dedr));
    } else if (tmem) {  // small batches: 2-atom warps (the pair kernel's rounds) with the TMEM history
      const unsigned grid = (unsigned)((na + PAIR_WARPS * 2 - 1) / (PAIR_WARPS * 2));
      PL_CUDA(launch_pdl(k_snap_deidrj_tm<2, PAIR_WARPS>, dim3(grid), dim3(PAIR_WARPS * 32), tm_smem(2), ctx->stream,
                         D, na, N, box, q, nl.nbr, nl.cnt, nl.maxn, buf.y, buf.yt, buf.dedr));
    } else if (big) {  // PL_SNAP_TMEM=0: the run kernel with the history in shared memory
      const size_t sm = sizeof(C2) * PAIR_WARPS * (2 * D.nhalf + ADJ4_SLOTS * 32) +
                        (sizeof(double) * PAIR_GEO + sizeof(int64_t)) * PAIR_WARPS * 32 +
                        sizeof(int16_t) * PAIR_WARPS * RUN * SNAP_MAXN + sizeof(int32_t) * PAIR_WARPS * (RUN + 2);
      const unsigned grid = (unsigned)((na + PAIR_WARPS * RUN - 1) / (PAIR_WARPS * RUN));
      PL_CUDA(launch_pdl(k_snap_deidrj_run<RUN, PAIR_WARPS>, dim3(grid), dim3(PAIR_WARPS * 32), sm, ctx->stream, D,
                         na, N, box, q, nl.nbr, nl.cnt, nl.maxn, buf.y, buf.yt, buf.dedr));
    } else {
      const size_t sm = sizeof(C2) * PAIR_WARPS * (2 * D.nhalf + ADJ4_SLOTS * 32) +
                        (sizeof(double) * PAIR_GEO + sizeof(int64_t)) * PAIR_WARPS * 32 +
                        sizeof(int32_t) * PAIR_WARPS * 2 * SNAP_MAXN;
      const unsigned grid = (unsigned)((na + PAIR_WARPS * 2 - 1) / (PAIR_WARPS * 2));
      PL_CUDA(launch_pdl(k_snap_deidrj_pair<2, PAIR_WARPS>, dim3(grid), dim3(PAIR_WARPS * 32), sm, ctx->stream, D,
                         na, N, box, q, nl.nbr, nl.cnt, nl.maxn, buf.y, buf.yt, buf.dedr));
    }
    buf.pair = true;
  } else {
    k_snap_deidrj<<<(unsigned)na, DE_WARPS * 32, de_smem(D), ctx->stream>>>(D, na, N, box, q, nl.nbr, nl.cnt,
                                                                           nl.maxn, buf.y, buf.dedr);
  }
  PL_CHECK_LAUNCH();
  prof_mark(ctx->stream, ST_DE, false);
  return PL_OK;
}

int compute_snap(pl_pot* pot, int64_t B, const double* q, double* energy, double* grad, double* virial) {
  pl_ctx* ctx = pot->ctx;
  int N = pot->n_atoms;
  int64_t na = B * N;
  SnapBuffers buf;
  NeighList nl;
  PL_TRY(snap_stages(pot, B, q, buf, nl));
  Box box = make_box(pot->box);
  prof_mark(ctx->stream, ST_GATHER, true);
  if (buf.pair)
    PL_CUDA(launch_pdl(k_snap_gather_pair_w, dim3((unsigned)((na * 32 + 127) / 128)), dim3(128), 0, ctx->stream, na,
                       N, box, q, nl.nbr, nl.cnt, nl.maxn, buf.dedr, grad, virial ? buf.vatom : nullptr,
                       pot->rcut * pot->rcut, buf.lists_exact ? 1 : 0));
  else
    k_snap_gather<<<(unsigned)((na + 127) / 128), 128, 0, ctx->stream>>>(
        na, N, box, q, nl.nbr, nl.cnt, nl.maxn, buf.dedr, grad, virial ? buf.vatom : nullptr);
  PL_CHECK_LAUNCH();
  if (energy) {
    PL_CUDA(launch_pdl(k_sys_sum, dim3((unsigned)B), dim3(256), 0, ctx->stream, B, N, 1, buf.eatom, energy));
    PL_CHECK_LAUNCH();
  }
  if (virial) {
    PL_CUDA(launch_pdl(k_sys_sum, dim3((unsigned)B), dim3(256), 0, ctx->stream, B, N, 6, buf.vatom, virial));
    PL_CHECK_LAUNCH();
  }
  prof_mark(ctx->stream, ST_GATHER, false);
  return PL_OK;
}

int snap_bispectrum(pl_pot* pot, int64_t B, const double* q, double* out) {
  SnapBuffers buf;
  NeighList nl;
  PL_TRY(snap_stages(pot, B, q, buf, nl));
  SnapDev D = snap_dev(pot);
  size_t smem = sizeof(C2) * D.nfull;
  k_snap_bispectrum<<<(unsigned)(B * pot->n_atoms), 128, smem, pot->ctx->stream>>>(D, buf.utot, out,
                                                                                  pot->snap->nitems);
  PL_CHECK_LAUNCH();
  return neigh_check(pot);
}

double snap_flops(const pl_pot* pot, double pairs, double atoms) {
  const SnapIndex* S = pot->snap;
  return pairs * (S->flops_ui_pair + S->flops_de_pair) + atoms * S->flops_yi_atom;
}

}  // namespace pl

extern "C" int pl_snap_bispectrum(pl_ctx* ctx, pl_pot* pot, int64_t B, const double* d_q, double* d_out) {
  if (!ctx || !pot || !d_q || !d_out) return pl::fail(PL_EARG, "NULL argument");
  if (pot->kind != POT_SNAP) return pl::fail(PL_EARG, "not a SNAP potential");
  return pl::snap_bispectrum(pot, B, d_q, d_out);
}

extern "C" int pl_snap_info(pl_pot* pot, int32_t* h_counts, double* h_flops) {
  // h_counts: {nhalf, nfull, nB, nitems, nunits}; h_flops: {ui/pair, yi/atom, deidrj/pair}
  if (!pot || pot->kind != POT_SNAP || !h_counts || !h_flops) return pl::fail(PL_EARG, "bad argument");
  const pl::SnapIndex* S = pot->snap;
  h_counts[0] = S->nhalf; h_counts[1] = S->nfull; h_counts[2] = S->nB; h_counts[3] = S->nitems;
  h_counts[4] = S->nunits;
  // FLOPs of the kernel variants that compute_snap actually launches
  const bool special = S->tj == 8 && S->yi_reg && !pl::snap_generic_forced();
  h_flops[0] = special ? S->flops_ui_pair_v : S->flops_ui_pair;
  h_flops[1] = special ? S->flops_yi_atom_reg : S->flops_yi_atom;
  // pair form: one sweep (+ the Y_i + Y_k^dagger adds, one read of every half element) per
  // unordered pair, quoted per ordered pair like the other stages
  h_flops[2] = special ? 0.5 * (S->flops_de_pair_adj + 2.0 * S->nhalf) : S->flops_de_pair;
  return PL_OK;
}
