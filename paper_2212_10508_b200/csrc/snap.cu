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
constexpr int YI3_WARPS = 16;                // k_snap_yi_full: 512 threads, one CTA per SM

struct SnapItem {      // one half-row element of one Z^{xy}_J
  int16_t x, y, J, ma, mb;
  int16_t ma1lo, na, mb1lo, nb;
  int16_t bidx;        // canonical B index or -1
  int32_t cga, cgb;    // offsets into the CG pool (na, nb values)
  int32_t cgblk;       // offset of the (x,y,J) block [(J+1) x (x+1)] in c_cgt (dense table)
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
  double flops_de_pair_adj = 0, flops_yi_atom_reg = 0;
  bool cgt_fits = false;
  bool yi_reg = false;  // k_snap_yi_reg usable (twojmax = 8, CG table in constant memory)
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
  const double* cg;
  double beta0, rcut, rfac0, rmin0, wself;
  double kappa, pi_span, half_pi_span;  // rfac0*pi/(rcut-rmin0), pi/(rcut-rmin0), 0.5*pi/(rcut-rmin0)
  int switchflag;
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
// dense Clebsch-Gordan blocks C(x m1, y m2 | J M) as [M-row][m1] per (x, y, J),
// x >= y, read with warp-uniform addresses by k_snap_yi (36.7 KB at twojmax 8)
constexpr int CGT_MAX = 5000;  // doubles (40 KB; twojmax = 8 needs 4698)
__constant__ double c_cgt[CGT_MAX];

namespace yi5 {
constexpr int TJ = 8;
constexpr int foff(int J) { return J * (J + 1) * (2 * J + 1) / 6; }
constexpr int hoff(int J) {
  int h = 0;
  for (int j = 0; j < J; ++j) h += (j + 1) * (j / 2 + 1);
  return h;
}
constexpr int cgoff(int X, int Y, int J) {  // offset of block (X, Y, J) in c_cgt
  int o = 0;
  for (int x = 0; x <= TJ; ++x)
    for (int y = 0; y <= x; ++y)
      for (int j = x - y; j <= (TJ < x + y ? TJ : x + y); j += 2) {
        if (x == X && y == Y && j == J) return o;
        o += (j + 1) * (x + 1);
      }
  return -1;
}
constexpr int ntriples() {
  int n = 0;
  for (int x = 0; x <= TJ; ++x)
    for (int y = 0; y <= x; ++y)
      for (int j = x - y; j <= (TJ < x + y ? TJ : x + y); j += 2) ++n;
  return n;
}
constexpr int NT = ntriples();
}  // namespace yi5

constexpr int YI5_WARPS = 8;
__constant__ int c_yi5_code[130];     // triple id -> X*100 + Y*10 + J
__constant__ int c_yi5_jstart[yi5::TJ + 2];  // triples of row-layer J: [jstart[J], jstart[J+1]) in tlist
__constant__ int c_yi5_tlist[130];    // triple ids sorted by J
__constant__ int c_yi5_gseg[YI5_WARPS + 1];  // groups of warp w
__constant__ int c_yi5_groups[32];    // (J << 8) | mb
__constant__ int c_yi5_cgoff[130];    // triple id -> offset of its block in c_cgt
constexpr int YI6_WARPS = 16;
__constant__ int c_yi6_gseg[YI6_WARPS + 1];
__constant__ int c_yi6_groups[32];
// box-form Z/Y kernel (snap_yi8.cu, own constant bank)
cudaError_t snap_box_setup(const double* box, int nbox, const int* off, const int* code, const int* iseg,
                           const int* items, int nitems, const int* rowsplit);
int snap_box_variants(int* nw, int* ns);
cudaError_t snap_box_launch(int nw, cudaStream_t st, int64_t natoms, double beta0, const double* coef,
                            const void* utot, void* ylist, double* eatom, double* erow_g);

// ------------------------------------------------------------------ host setup
static double fact(int n) {
  double f = 1.0;
  for (int i = 2; i <= n; ++i) f *= (double)i;
  return f;
}

// Condon-Shortley <j1 m1 j2 m2 | J M> (Racah formula), arguments are 2j / 2m
static double clebsch(int j1, int m1, int j2, int m2, int J, int M) {
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
  // dense CG blocks per (x, y, J)
  std::map<std::tuple<int, int, int>, int> cgblk;
  std::vector<double> cgt;
  for (int x = 0; x <= tj; ++x)
    for (int y = 0; y <= x; ++y)
      for (int J = x - y; J <= std::min(tj, x + y); J += 2) {
        cgblk[{x, y, J}] = (int)cgt.size();
        for (int ma = 0; ma <= J; ++ma)
          for (int m1 = 0; m1 <= x; ++m1) {
            int M = 2 * ma - J, mm1 = 2 * m1 - x, m2 = M - mm1;
            cgt.push_back(std::abs(m2) <= y ? clebsch(x, mm1, y, m2, J, M) : 0.0);
          }
      }
  // the constant table's layout depends on twojmax: the first SNAP potential of
  // the process owns it; potentials with another twojmax use the global CG pool
  static int g_cgt_tj = -1;
  S->cgt_fits = cgt.size() <= (size_t)CGT_MAX && (g_cgt_tj < 0 || g_cgt_tj == tj);
  if (S->cgt_fits && g_cgt_tj < 0) {
    PL_CUDA(cudaMemcpyToSymbol(c_cgt, cgt.data(), sizeof(double) * cgt.size()));
    g_cgt_tj = tj;
  }
  // register-tiled Y (k_snap_yi_reg, twojmax = 8): per-triple coefficients, rows by J,
  // LPT schedule of the (J, mb) rows over the CTA's warps
  S->yi_reg = false;
  if (tj == 8 && S->cgt_fits) {
    std::vector<double> cy, be;
    std::vector<int> code;
    std::vector<std::vector<int>> byJ(tj + 1);
    std::vector<double> rowcost(64, 0.0);
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
    std::vector<int> tlist, jstart(tj + 2, 0);
    for (int J = 0; J <= tj; ++J) {
      jstart[J] = (int)tlist.size();
      tlist.insert(tlist.end(), byJ[J].begin(), byJ[J].end());
    }
    jstart[tj + 1] = (int)tlist.size();
    // row costs: sum over the row's triples of nb * (J+1) * (X+1)
    std::vector<std::pair<double, int>> rows;
    for (int J = 0; J <= tj; ++J)
      for (int mb = 0; 2 * mb <= J; ++mb) {
        double c = 0.0;
        for (int tid : byJ[J]) {
          int x = code[tid] / 100, y = (code[tid] / 10) % 10, sh = (x + y - J) / 2;
          int nb = 0;
          for (int mb1 = 0; mb1 <= x; ++mb1) nb += (mb + sh - mb1 >= 0 && mb + sh - mb1 <= y);
          c += (double)nb * (J + 1) * (x + 1) + 20.0;
        }
        rows.push_back({c, (J << 8) | mb});
      }
    std::sort(rows.begin(), rows.end(), [](auto& a, auto& b) { return a.first > b.first; });
    // rows -> NW warps: LPT, then deterministic local search (single moves and
    // pairwise swaps) that lowers the makespan, ties broken by the sum of
    // squared loads.  For 25 rows on 12 warps LPT reaches ~83 % balance, the
    // search ~96 % (cost model).
    auto lpt = [&](int NW, std::vector<int>& groups, std::vector<int>& gseg) {
      const int nr = (int)rows.size();
      std::vector<int> asg(nr);
      std::vector<double> wl(NW, 0.0);
      for (int i = 0; i < nr; ++i) {
        int w = (int)(std::min_element(wl.begin(), wl.end()) - wl.begin());
        asg[i] = w;
        wl[w] += rows[i].first;
      }
      auto score = [&](const std::vector<double>& l) {
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
        for (int i = 0; i < nr; ++i)
          for (int w = 0; w < NW; ++w) {
            if (w == asg[i]) continue;
            std::vector<double> nl(wl);
            nl[asg[i]] -= rows[i].first;
            nl[w] += rows[i].first;
            auto sc = score(nl);
            if (sc < cur) {
              wl = nl;
              asg[i] = w;
              cur = sc;
              improved = true;
            }
          }
        for (int i = 0; i < nr; ++i)
          for (int j = i + 1; j < nr; ++j) {
            const int a = asg[i], b = asg[j];
            if (a == b) continue;
            std::vector<double> nl(wl);
            nl[a] += rows[j].first - rows[i].first;
            nl[b] += rows[i].first - rows[j].first;
            auto sc = score(nl);
            if (sc < cur) {
              wl = nl;
              std::swap(asg[i], asg[j]);
              cur = sc;
              improved = true;
            }
          }
      }
      std::vector<std::vector<int>> wr(NW);
      for (int i = 0; i < nr; ++i) wr[asg[i]].push_back(rows[i].second);
      gseg.assign(NW + 1, 0);
      groups.clear();
      for (int w = 0; w < NW; ++w) {
        gseg[w] = (int)groups.size();
        groups.insert(groups.end(), wr[w].begin(), wr[w].end());
      }
      gseg[NW] = (int)groups.size();
    };
    std::vector<int> groups, gseg, groups16, gseg16;
    lpt(8, groups, gseg);
    lpt(YI6_WARPS, groups16, gseg16);
    {  // box kernel (snap_yi8.cu): every (X+1)(Y+1) product of each admissible mb1
      auto rows6 = rows;
      rows.clear();
      for (int J = 0; J <= tj; ++J)
        for (int mb = 0; 2 * mb <= J; ++mb) {
          double c = 0.0;
          for (int tid : byJ[J]) {
            int x = code[tid] / 100, y = (code[tid] / 10) % 10, sh = (x + y - J) / 2;
            const int mb1_hi = 2 * mb == J ? x / 2 : (x == y ? (mb + sh) / 2 : x);  // symmetry halvings
            for (int mb1 = 0; mb1 <= mb1_hi; ++mb1)
              if (mb + sh - mb1 >= 0 && mb + sh - mb1 <= y) c += 7.0 * (x + 1) * (y + 1) + 2.0 * (x + y + 2) + 12.0;
            c += 60.0;
          }
          rows.push_back({c, (J << 8) | mb});
        }
      std::sort(rows.begin(), rows.end(), [](auto& a, auto& b) { return a.first > b.first; });
      // rows -> NW*S virtual warps (LPT; virtual warp w runs on CTA w / NW of the
      // block), then each warp's (row, triple) items in ascending X
      auto row_index = [](int J, int mb) {
        int r = 0;
        for (int j = 0; j < J; ++j) r += j / 2 + 1;
        return r + mb;
      };
      auto itemize = [&](int NW, int NS, std::vector<int>& iseg, std::vector<int>& items,
                         std::vector<int>& rowsplit) {
        std::vector<int> g, sg;
        const int NV = NW * NS;
        lpt(NV, g, sg);
        iseg.assign(26, 0);
        rowsplit.assign(25, 0);
        items.clear();
        for (int w = 0; w < NV; ++w) {
          iseg[w] = (int)items.size();
          std::vector<std::pair<int, int>> mine;  // (sort key, item)
          for (int gi = sg[w]; gi < sg[w + 1]; ++gi) {
            const int J = g[gi] >> 8, mb = g[gi] & 0xff;
            rowsplit[row_index(J, mb)] = w / NW;
            for (int tid : byJ[J]) {
              const int x = code[tid] / 100, y = (code[tid] / 10) % 10;
              mine.push_back({x * 10000 + y * 100 + J * 10 + mb, (tid << 16) | (J << 8) | mb});
            }
          }
          std::sort(mine.begin(), mine.end());
          for (auto& m : mine) items.push_back(m.second);
        }
        for (int w = NV; w < 26; ++w) iseg[w] = (int)items.size();
      };
      int box_nw[8], box_ns[8];
      const int box_nv = snap_box_variants(box_nw, box_ns);
      std::vector<int> iseg_all(box_nv * 26, 0), items_all, rowsplit_all(box_nv * 25, 0);
      for (int v = 0; v < box_nv; ++v) {
        std::vector<int> is, it, rs;
        itemize(box_nw[v], box_ns[v], is, it, rs);
        std::copy(is.begin(), is.end(), iseg_all.begin() + v * 26);
        std::copy(rs.begin(), rs.end(), rowsplit_all.begin() + v * 25);
        items_all.insert(items_all.end(), it.begin(), it.end());
      }
      const int n_items = (int)items_all.size() / box_nv;
      rows = rows6;
      static bool box_done = false;
      if (!box_done) {
        std::vector<double> box;
        std::vector<int> boff;
        for (int c : code) {
          const int x = c / 100, y = (c / 10) % 10, J = c % 10, sh = (x + y - J) / 2;
          boff.push_back((int)box.size());
          for (int b = 0; b <= y; ++b)
            for (int a = 0; a <= x; ++a) {
              const int ma = a + b - sh;
              box.push_back(ma >= 0 && ma <= J ? clebsch(x, 2 * a - x, y, 2 * b - y, J, 2 * ma - J) : 0.0);
            }
        }
        if ((int)code.size() != yi5::NT) return fail(PL_EARG, "SNAP box tables: unexpected triple count");
        PL_CUDA(snap_box_setup(box.data(), (int)box.size(), boff.data(), code.data(), iseg_all.data(),
                               items_all.data(), n_items, rowsplit_all.data()));
        box_done = true;
      }
    }
    PL_CUDA(cudaMemcpyToSymbol(c_yi6_gseg, gseg16.data(), sizeof(int) * gseg16.size()));
    PL_CUDA(cudaMemcpyToSymbol(c_yi6_groups, groups16.data(), sizeof(int) * groups16.size()));
    std::vector<double> cb2(cy);
    cb2.insert(cb2.end(), be.begin(), be.end());
    PL_CUDA(cudaMalloc(&S->d_yi5, sizeof(double) * cb2.size()));
    PL_CUDA(cudaMemcpy(S->d_yi5, cb2.data(), sizeof(double) * cb2.size(), cudaMemcpyHostToDevice));
    PL_CUDA(cudaMemcpyToSymbol(c_yi5_code, code.data(), sizeof(int) * code.size()));
    {
      std::vector<int> offs;
      for (int c : code) offs.push_back(cgblk[{c / 100, (c / 10) % 10, c % 10}]);
      PL_CUDA(cudaMemcpyToSymbol(c_yi5_cgoff, offs.data(), sizeof(int) * offs.size()));
    }
    PL_CUDA(cudaMemcpyToSymbol(c_yi5_tlist, tlist.data(), sizeof(int) * tlist.size()));
    PL_CUDA(cudaMemcpyToSymbol(c_yi5_jstart, jstart.data(), sizeof(int) * jstart.size()));
    PL_CUDA(cudaMemcpyToSymbol(c_yi5_gseg, gseg.data(), sizeof(int) * gseg.size()));
    PL_CUDA(cudaMemcpyToSymbol(c_yi5_groups, groups.data(), sizeof(int) * groups.size()));
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
              ca.push_back(clebsch(x, 2 * ma1 - x, y, m2, J, M));
            }
            it.ma1lo = (int16_t)lo;
            it.na = (int16_t)ca.size();
            lo = -1;
            for (int mb1 = 0; mb1 <= x; ++mb1) {
              int m2 = Mp - (2 * mb1 - x);
              if (std::abs(m2) > y) continue;
              if (lo < 0) lo = mb1;
              cb.push_back(clebsch(x, 2 * mb1 - x, y, m2, J, Mp));
            }
            it.mb1lo = (int16_t)lo;
            it.nb = (int16_t)cb.size();
            it.cga = (int32_t)pool.size();
            pool.insert(pool.end(), ca.begin(), ca.end());
            it.cgb = (int32_t)pool.size();
            pool.insert(pool.end(), cb.begin(), cb.end());
            it.w = half_weight(J, ma, mb);
            it.cgblk = cgblk[{x, y, J}];
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
  // (the CG table must be known to fit constant memory to pick the kernel)
  size_t cg_doubles = 0;
  for (int x = 0; x <= tj; ++x)
    for (int y = 0; y <= x; ++y)
      for (int J = x - y; J <= std::min(tj, x + y); J += 2) cg_doubles += (size_t)(J + 1) * (x + 1);
  const int nwarps = S->cgt_fits ? YI3_WARPS : YI_WARPS;
  (void)cg_doubles;
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
    S->flops_de_pair += nel * 160.0;  // U (20) + 3 dU (108) + 3 weighted contractions (~32)
  }
  S->flops_ui_pair += 40.0;
  S->flops_de_pair += 80.0;
  // reverse-mode pair kernel: forward U + F contraction (25/element), adjoint
  // (S_a, S_b, G update, direct Y term: 42/element), geometry + final (150)
  S->flops_de_pair_adj = 150.0;
  for (int J = 1; J <= tj; ++J) S->flops_de_pair_adj += (J + 1) * (J / 2 + 1) * 67.0;
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
  D.beta0 = S->beta0; D.rcut = pot->rcut; D.rfac0 = pot->rfac0; D.rmin0 = pot->rmin0;
  D.wself = pot->wself; D.switchflag = pot->switchflag;
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

// v3: full matrices in shared memory ([285][32 atoms], no symmetry branch in
// the inner loop), CG from constant memory, strided inner walk.
__global__ void __launch_bounds__(YI3_WARPS * 32)
k_snap_yi_full(SnapDev D, int64_t natoms, const C2* __restrict__ utot, C2* __restrict__ ylist,
               double* __restrict__ eatom) {
  extern __shared__ double smem[];
  C2* Uf = reinterpret_cast<C2*>(smem);                                // [nfull][32]
  double* epart = reinterpret_cast<double*>(Uf + D.nfull * YI_ATOMS);  // [warps][32]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t a0 = (int64_t)blockIdx.x * YI_ATOMS;
  const int na_blk = (int)min((int64_t)YI_ATOMS, natoms - a0);
  // stage: half rows -> full matrices, transposed to [element][atom]
  for (int t = threadIdx.x; t < D.nfull * YI_ATOMS; t += blockDim.x) {
    const int at = t & (YI_ATOMS - 1), f = t >> 5;
    int J = 0;
    while (J < D.tj && f >= c_foff[J + 1]) ++J;
    const int e = f - c_foff[J], mb = e / (J + 1), ma = e - mb * (J + 1);
    C2 v{0.0, 0.0};
    if (at < na_blk) {
      if (2 * mb <= J) {
        v = utot[(a0 + at) * D.nhalf + c_hoff[J] + mb * (J + 1) + ma];
      } else {
        C2 w = utot[(a0 + at) * D.nhalf + c_hoff[J] + (J - mb) * (J + 1) + (J - ma)];
        v = ((ma + mb) & 1) ? C2{-w.re, w.im} : C2{w.re, -w.im};
      }
    }
    Uf[f * YI_ATOMS + at] = v;
  }
  __syncthreads();
  double esum = 0.0;
  const int64_t atom = a0 + lane;
  for (int wt = D.wseg[warp]; wt < D.wseg[warp + 1]; ++wt) {
    const int target = D.wtarget[wt];
    C2 ysum{0.0, 0.0};
    for (int k = D.tseg[target]; k < D.tseg[target + 1]; ++k) {
      const SnapItem it = D.items[k];
      const int x = it.x, y = it.y, J = it.J, sh = (x + y - J) / 2;
      const double* cga = c_cgt + it.cgblk + it.ma * (x + 1) + it.ma1lo;
      const double* cgb = c_cgt + it.cgblk + it.mb * (x + 1) + it.mb1lo;
      C2 z{0.0, 0.0};
      for (int jb = 0; jb < it.nb; ++jb) {
        const int mb1 = it.mb1lo + jb, mb2 = it.mb - mb1 + sh;
        // U^x[ma1][mb1] walks +1 in ma1, U^y[ma2][mb2] walks -1 (ma2 = ma - ma1 + sh)
        const C2* px = Uf + (c_foff[x] + mb1 * (x + 1) + it.ma1lo) * YI_ATOMS + lane;
        const C2* py = Uf + (c_foff[y] + mb2 * (y + 1) + (it.ma - it.ma1lo + sh)) * YI_ATOMS + lane;
        // two independent accumulator chains (ILP); fixed pairing => deterministic
        double s0r = 0.0, s0i = 0.0, s1r = 0.0, s1i = 0.0;
        int ja = 0;
        for (; ja + 1 < it.na; ja += 2) {
          const C2 ux0 = px[ja * YI_ATOMS], ux1 = px[(ja + 1) * YI_ATOMS];
          const C2 uy0 = py[-ja * YI_ATOMS], uy1 = py[-(ja + 1) * YI_ATOMS];
          const double c0 = cga[ja], c1 = cga[ja + 1];
          s0r += c0 * (ux0.re * uy0.re - ux0.im * uy0.im);
          s0i += c0 * (ux0.re * uy0.im + ux0.im * uy0.re);
          s1r += c1 * (ux1.re * uy1.re - ux1.im * uy1.im);
          s1i += c1 * (ux1.re * uy1.im + ux1.im * uy1.re);
        }
        if (ja < it.na) {
          const C2 ux0 = px[ja * YI_ATOMS], uy0 = py[-ja * YI_ATOMS];
          const double c0 = cga[ja];
          s0r += c0 * (ux0.re * uy0.re - ux0.im * uy0.im);
          s0i += c0 * (ux0.re * uy0.im + ux0.im * uy0.re);
        }
        const C2 sacc{s0r + s1r, s0i + s1i};
        const double c = cgb[jb];
        z.re += c * sacc.re;
        z.im += c * sacc.im;
      }
      ysum.re += it.coefY * z.re;
      ysum.im += it.coefY * z.im;
      if (it.bidx >= 0) {
        const C2 uJ = Uf[(c_foff[J] + it.mb * (J + 1) + it.ma) * YI_ATOMS + lane];
        esum += it.coefE * (uJ.re * z.re + uJ.im * z.im);  // Re(conj(U) z)
      }
    }
    if (lane < na_blk) ylist[atom * D.nhalf + target] = ysum;
  }
  epart[warp * YI_ATOMS + lane] = esum;
  __syncthreads();
  if (warp == 0 && lane < na_blk) {
    double e = D.beta0;
    for (int w = 0; w < YI3_WARPS; ++w) e += epart[w * YI_ATOMS + lane];
    eatom[atom] = e;
  }
}

// v4: half rows in shared memory ([155][32 atoms] = 79 KB -> 2 CTAs per SM).
// A column mb1 > x/2 of U^x is read through U[ma][mb] = (-1)^(ma+mb)
// conj(U[x-ma][x-mb]): per jb the two columns are direct or mirrored (warp-
// uniform), the conjugations select one of four compiled inner loops, and the
// alternating signs fold into the even/odd accumulator chains.
template <bool CX, bool CY>
__device__ __forceinline__ void yi_inner(const C2* px, int sx, const C2* py, int sy, const double* cga, int na,
                                         double& e_re, double& e_im, double& o_re, double& o_im) {
  // px/py: first element, sx/sy: element stride (+-YI_ATOMS); conj applied when CX/CY
  int ja = 0;
  for (; ja + 1 < na; ja += 2) {
    const C2 ux0 = px[ja * sx], ux1 = px[(ja + 1) * sx];
    const C2 uy0 = py[ja * sy], uy1 = py[(ja + 1) * sy];
    const double c0 = cga[ja], c1 = cga[ja + 1];
    const double x0i = CX ? -ux0.im : ux0.im, x1i = CX ? -ux1.im : ux1.im;
    const double y0i = CY ? -uy0.im : uy0.im, y1i = CY ? -uy1.im : uy1.im;
    e_re += c0 * (ux0.re * uy0.re - x0i * y0i);
    e_im += c0 * (ux0.re * y0i + x0i * uy0.re);
    o_re += c1 * (ux1.re * uy1.re - x1i * y1i);
    o_im += c1 * (ux1.re * y1i + x1i * uy1.re);
  }
  if (ja < na) {
    const C2 ux0 = px[ja * sx], uy0 = py[ja * sy];
    const double c0 = cga[ja];
    const double x0i = CX ? -ux0.im : ux0.im, y0i = CY ? -uy0.im : uy0.im;
    e_re += c0 * (ux0.re * uy0.re - x0i * y0i);
    e_im += c0 * (ux0.re * y0i + x0i * uy0.re);
  }
}

__global__ void __launch_bounds__(YI3_WARPS * 32, 2)
k_snap_yi_half(SnapDev D, int64_t natoms, const C2* __restrict__ utot, C2* __restrict__ ylist,
               double* __restrict__ eatom) {
  extern __shared__ double smem[];
  C2* Us = reinterpret_cast<C2*>(smem);                                // [nhalf][32]
  double* epart = reinterpret_cast<double*>(Us + D.nhalf * YI_ATOMS);  // [warps][32]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t a0 = (int64_t)blockIdx.x * YI_ATOMS;
  const int na_blk = (int)min((int64_t)YI_ATOMS, natoms - a0);
  for (int t = threadIdx.x; t < D.nhalf * YI_ATOMS; t += blockDim.x) {
    const int at = t / D.nhalf, e = t - at * D.nhalf;
    Us[e * YI_ATOMS + at] = at < na_blk ? utot[(a0 + at) * D.nhalf + e] : C2{0.0, 0.0};
  }
  __syncthreads();
  double esum = 0.0;
  const int64_t atom = a0 + lane;
  const C2* Ul = Us + lane;
  for (int wt = D.wseg[warp]; wt < D.wseg[warp + 1]; ++wt) {
    const int target = D.wtarget[wt];
    C2 ysum{0.0, 0.0};
    for (int k = D.tseg[target]; k < D.tseg[target + 1]; ++k) {
      const SnapItem it = D.items[k];
      const int x = it.x, y = it.y, J = it.J, sh = (x + y - J) / 2;
      const double* cga = c_cgt + it.cgblk + it.ma * (x + 1) + it.ma1lo;
      const double* cgb = c_cgt + it.cgblk + it.mb * (x + 1) + it.mb1lo;
      const int ma2s = it.ma - it.ma1lo + sh;  // ma2 of ja = 0 (then -1 per ja)
      C2 z{0.0, 0.0};
      for (int jb = 0; jb < it.nb; ++jb) {
        const int mb1 = it.mb1lo + jb, mb2 = it.mb - mb1 + sh;
        const bool mx = 2 * mb1 > x, my = 2 * mb2 > y;
        // first element addresses and strides ([element][atom] layout)
        const C2* px;
        int sx;
        int sgx = 1;
        if (!mx) {
          px = Ul + (c_hoff[x] + mb1 * (x + 1) + it.ma1lo) * YI_ATOMS;
          sx = YI_ATOMS;
        } else {
          px = Ul + (c_hoff[x] + (x - mb1) * (x + 1) + (x - it.ma1lo)) * YI_ATOMS;
          sx = -YI_ATOMS;
          sgx = ((it.ma1lo + mb1) & 1) ? -1 : 1;
        }
        const C2* py;
        int sy;
        int sgy = 1;
        if (!my) {
          py = Ul + (c_hoff[y] + mb2 * (y + 1) + ma2s) * YI_ATOMS;
          sy = -YI_ATOMS;
        } else {
          py = Ul + (c_hoff[y] + (y - mb2) * (y + 1) + (y - ma2s)) * YI_ATOMS;
          sy = YI_ATOMS;
          sgy = ((ma2s + mb2) & 1) ? -1 : 1;
        }
        double e_re = 0.0, e_im = 0.0, o_re = 0.0, o_im = 0.0;
        switch ((mx ? 2 : 0) | (my ? 1 : 0)) {
          case 0: yi_inner<false, false>(px, sx, py, sy, cga, it.na, e_re, e_im, o_re, o_im); break;
          case 1: yi_inner<false, true>(px, sx, py, sy, cga, it.na, e_re, e_im, o_re, o_im); break;
          case 2: yi_inner<true, false>(px, sx, py, sy, cga, it.na, e_re, e_im, o_re, o_im); break;
          default: yi_inner<true, true>(px, sx, py, sy, cga, it.na, e_re, e_im, o_re, o_im); break;
        }
        // signs: mirrored columns alternate with ja (x: +1 per step, y: -1 per step)
        const int s0 = sgx * sgy;
        const int s1 = s0 * (mx ? -1 : 1) * (my ? -1 : 1);
        const double sr = s0 > 0 ? e_re : -e_re, si = s0 > 0 ? e_im : -e_im;
        const double tr = s1 > 0 ? o_re : -o_re, ti = s1 > 0 ? o_im : -o_im;
        const double c = cgb[jb];
        z.re += c * (sr + tr);
        z.im += c * (si + ti);
      }
      ysum.re += it.coefY * z.re;
      ysum.im += it.coefY * z.im;
      if (it.bidx >= 0) {
        const C2 uJ = Ul[(c_hoff[J] + it.mb * (J + 1) + it.ma) * YI_ATOMS];
        esum += it.coefE * (uJ.re * z.re + uJ.im * z.im);  // Re(conj(U) z)
      }
    }
    if (lane < na_blk) ylist[atom * D.nhalf + target] = ysum;
  }
  epart[warp * YI_ATOMS + lane] = esum;
  __syncthreads();
  if (warp == 0 && lane < na_blk) {
    double e = D.beta0;
    for (int w = 0; w < YI3_WARPS; ++w) e += epart[w * YI_ATOMS + lane];
    eatom[atom] = e;
  }
}

// v5: register-tiled Z/Y for twojmax = 8.  Work = whole Y rows (J, mb) per warp
// (LPT schedule).  For every contributing (X, Y) pair one instantiation of
// yi_xyj<X,Y,J> loads the U^X column mb1 and the U^Y column mb2 into registers
// once per mb1 and produces all J+1 outputs of the row; all ma / ma1 indices
// are compile-time, CG coefficients are constant-bank operands at compile-time
// offsets (c_cgt layout = host enumeration, reproduced by constexpr below).



template <int X, int Y, int J>
__device__ __forceinline__ void yi_xyj(const C2* __restrict__ Ul, int mb, double cy, double be,
                                       C2 (&yacc)[yi5::TJ + 1], double& esum) {
  constexpr int SH = (X + Y - J) / 2;
  constexpr int OFF = yi5::cgoff(X, Y, J);
  constexpr int FX = yi5::foff(X), FY = yi5::foff(Y);
  C2 z[J + 1];
#pragma unroll
  for (int m = 0; m <= J; ++m) z[m] = C2{0.0, 0.0};
  const bool mid = (2 * mb == J);
  const int lo = max(0, mb + SH - Y), hi = min(X, mb + SH);
  for (int mb1 = lo; mb1 <= hi; ++mb1) {
    const int mb2 = mb + SH - mb1;
    C2 ux[X + 1], uy[Y + 1];
    const C2* px = Ul + (FX + mb1 * (X + 1)) * YI_ATOMS;
    const C2* py = Ul + (FY + mb2 * (Y + 1)) * YI_ATOMS;
#pragma unroll
    for (int a = 0; a <= X; ++a) ux[a] = px[a * YI_ATOMS];
#pragma unroll
    for (int a = 0; a <= Y; ++a) uy[a] = py[a * YI_ATOMS];
    const double cb = c_cgt[OFF + mb * (X + 1) + mb1];
#pragma unroll
    for (int ma = 0; ma <= J; ++ma) {
      if (mid && 2 * ma > J) continue;  // zero weight on the middle row's upper half
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int ma1 = 0; ma1 <= X; ++ma1) {
        const int ma2 = ma + SH - ma1;
        if (ma2 < 0 || ma2 > Y) continue;  // folded after unrolling
        const double c = c_cgt[OFF + ma * (X + 1) + ma1];
        sr += c * (ux[ma1].re * uy[ma2].re - ux[ma1].im * uy[ma2].im);
        si += c * (ux[ma1].re * uy[ma2].im + ux[ma1].im * uy[ma2].re);
      }
      z[ma].re += cb * sr;
      z[ma].im += cb * si;
    }
  }
  const C2* pj = Ul + (yi5::foff(J) + mb * (J + 1)) * YI_ATOMS;
#pragma unroll
  for (int ma = 0; ma <= J; ++ma) {
    yacc[ma].re += cy * z[ma].re;
    yacc[ma].im += cy * z[ma].im;
    if (be != 0.0) {
      const double w = (2 * mb < J || 2 * ma < J) ? 2.0 : (2 * ma == J ? 1.0 : 0.0);
      const C2 u = pj[ma * YI_ATOMS];
      esum += be * w * (u.re * z[ma].re + u.im * z[ma].im);
    }
  }
}

// flat switch (faster than the recursive compare chain): generated per triple id
#define YI5_CASES(F) \
  F(0,0,0) F(1,0,1) F(1,1,0) F(1,1,2) F(2,0,2) F(2,1,1) F(2,1,3) F(2,2,0) F(2,2,2) F(2,2,4) \
  F(3,0,3) F(3,1,2) F(3,1,4) F(3,2,1) F(3,2,3) F(3,2,5) F(3,3,0) F(3,3,2) F(3,3,4) F(3,3,6) \
  F(4,0,4) F(4,1,3) F(4,1,5) F(4,2,2) F(4,2,4) F(4,2,6) F(4,3,1) F(4,3,3) F(4,3,5) F(4,3,7) \
  F(4,4,0) F(4,4,2) F(4,4,4) F(4,4,6) F(4,4,8) F(5,0,5) F(5,1,4) F(5,1,6) F(5,2,3) F(5,2,5) \
  F(5,2,7) F(5,3,2) F(5,3,4) F(5,3,6) F(5,3,8) F(5,4,1) F(5,4,3) F(5,4,5) F(5,4,7) F(5,5,0) \
  F(5,5,2) F(5,5,4) F(5,5,6) F(5,5,8) F(6,0,6) F(6,1,5) F(6,1,7) F(6,2,4) F(6,2,6) F(6,2,8) \
  F(6,3,3) F(6,3,5) F(6,3,7) F(6,4,2) F(6,4,4) F(6,4,6) F(6,4,8) F(6,5,1) F(6,5,3) F(6,5,5) \
  F(6,5,7) F(6,6,0) F(6,6,2) F(6,6,4) F(6,6,6) F(6,6,8) F(7,0,7) F(7,1,6) F(7,1,8) F(7,2,5) \
  F(7,2,7) F(7,3,4) F(7,3,6) F(7,3,8) F(7,4,3) F(7,4,5) F(7,4,7) F(7,5,2) F(7,5,4) F(7,5,6) \
  F(7,5,8) F(7,6,1) F(7,6,3) F(7,6,5) F(7,6,7) F(7,7,0) F(7,7,2) F(7,7,4) F(7,7,6) F(7,7,8) \
  F(8,0,8) F(8,1,7) F(8,2,6) F(8,2,8) F(8,3,5) F(8,3,7) F(8,4,4) F(8,4,6) F(8,4,8) F(8,5,3) \
  F(8,5,5) F(8,5,7) F(8,6,2) F(8,6,4) F(8,6,6) F(8,6,8) F(8,7,1) F(8,7,3) F(8,7,5) F(8,7,7) \
  F(8,8,0) F(8,8,2) F(8,8,4) F(8,8,6) F(8,8,8)

__device__ __forceinline__ void yi5_call(int code, double cy, double be, const C2* Ul, int mb,
                                         C2 (&yacc)[yi5::TJ + 1], double& esum) {
  // code = X*100 + Y*10 + J
  switch (code) {
#define YI5_CASE(X, Y, J) \
  case X * 100 + Y * 10 + J: yi_xyj<X, Y, J>(Ul, mb, cy, be, yacc, esum); break;
    YI5_CASES(YI5_CASE)
#undef YI5_CASE
    default: break;
  }
}



__global__ void __launch_bounds__(YI5_WARPS * 32, 1)
k_snap_yi_reg(SnapDev D, int64_t natoms, const C2* __restrict__ utot, C2* __restrict__ ylist,
              double* __restrict__ eatom) {
  extern __shared__ double smem[];
  C2* Uf = reinterpret_cast<C2*>(smem);                                // [nfull][32]
  double* epart = reinterpret_cast<double*>(Uf + D.nfull * YI_ATOMS);  // [warps][32]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t a0 = (int64_t)blockIdx.x * YI_ATOMS;
  const int na_blk = (int)min((int64_t)YI_ATOMS, natoms - a0);
  for (int t = threadIdx.x; t < D.nfull * YI_ATOMS; t += blockDim.x) {
    const int at = t & (YI_ATOMS - 1), f = t >> 5;
    int J = 0;
    while (J < D.tj && f >= c_foff[J + 1]) ++J;
    const int e = f - c_foff[J], mb = e / (J + 1), ma = e - mb * (J + 1);
    C2 v{0.0, 0.0};
    if (at < na_blk) {
      if (2 * mb <= J) {
        v = utot[(a0 + at) * D.nhalf + c_hoff[J] + mb * (J + 1) + ma];
      } else {
        C2 w = utot[(a0 + at) * D.nhalf + c_hoff[J] + (J - mb) * (J + 1) + (J - ma)];
        v = ((ma + mb) & 1) ? C2{-w.re, w.im} : C2{w.re, -w.im};
      }
    }
    Uf[f * YI_ATOMS + at] = v;
  }
  __syncthreads();
  const C2* Ul = Uf + lane;
  const int64_t atom = a0 + lane;
  double esum = 0.0;
  for (int gi = c_yi5_gseg[warp]; gi < c_yi5_gseg[warp + 1]; ++gi) {
    const int J = c_yi5_groups[gi] >> 8, mb = c_yi5_groups[gi] & 0xff;
    C2 yacc[yi5::TJ + 1];
#pragma unroll
    for (int m = 0; m <= yi5::TJ; ++m) yacc[m] = C2{0.0, 0.0};
    for (int k = c_yi5_jstart[J]; k < c_yi5_jstart[J + 1]; ++k) {
      const int tid = c_yi5_tlist[k];
      yi5_call(c_yi5_code[tid], D.yi5[tid], D.yi5[yi5::NT + tid], Ul, mb, yacc, esum);
    }
    if (lane < na_blk) {
      C2* yo = ylist + atom * D.nhalf + c_hoff[J] + mb * (J + 1);
#pragma unroll
      for (int m = 0; m <= yi5::TJ; ++m)
        if (m <= J) yo[m] = yacc[m];
    }
  }
  epart[warp * YI_ATOMS + lane] = esum;
  __syncthreads();
  if (warp == 0 && lane < na_blk) {
    double e = D.beta0;
    for (int w = 0; w < YI5_WARPS; ++w) e += epart[w * YI_ATOMS + lane];
    eatom[atom] = e;
  }
}

// v6: small code.  Row work (J, mb) per warp as in v5, but one instantiation per X
// only: the U^X column sits in registers (compile-time ma1), U^Y is read from
// shared memory (one load per product), the z row accumulates in a per-lane
// shared strip, CG rows come from constant memory with warp-uniform offsets.
template <int X>
__device__ __forceinline__ void yi6_xyj(const C2* __restrict__ Ul, int Y, int J, int mb, int off, double cy,
                                        double be, C2* __restrict__ zs, C2 (&yacc)[yi5::TJ + 1], double& esum) {
  const int SH = (X + Y - J) / 2;
  const bool mid = (2 * mb == J);
  const int jtop = mid ? J / 2 : J;  // middle row: upper half has zero weight
  for (int ma = 0; ma <= jtop; ++ma) zs[ma * 32] = C2{0.0, 0.0};
  const int lo = max(0, mb + SH - Y), hi = min(X, mb + SH);
  const int FX = c_foff[X], FY = c_foff[Y];
  for (int mb1 = lo; mb1 <= hi; ++mb1) {
    const int mb2 = mb + SH - mb1;
    C2 ux[X + 1];
    const C2* px = Ul + (FX + mb1 * (X + 1)) * YI_ATOMS;
#pragma unroll
    for (int a = 0; a <= X; ++a) ux[a] = px[a * YI_ATOMS];
    const C2* py = Ul + (FY + mb2 * (Y + 1)) * YI_ATOMS;
    const double cb = c_cgt[off + mb * (X + 1) + mb1];
    for (int ma = 0; ma <= jtop; ++ma) {
      const double* cga = c_cgt + off + ma * (X + 1);
      const int base2 = ma + SH;  // ma2 = base2 - ma1
      // two accumulator pairs (even / odd ma1): shorter dependent FMA chains
      double sr0 = 0.0, si0 = 0.0, sr1 = 0.0, si1 = 0.0;
#pragma unroll
      for (int ma1 = 0; ma1 <= X; ++ma1) {
        const int ma2 = base2 - ma1;
        if (ma2 >= 0 && ma2 <= Y) {
          const C2 uy = py[ma2 * YI_ATOMS];
          const double c = cga[ma1];
          const double tr = ux[ma1].re * uy.re - ux[ma1].im * uy.im;
          const double ti = ux[ma1].re * uy.im + ux[ma1].im * uy.re;
          if (ma1 & 1) {
            sr1 += c * tr;
            si1 += c * ti;
          } else {
            sr0 += c * tr;
            si0 += c * ti;
          }
        }
      }
      C2 zz = zs[ma * 32];
      zz.re += cb * (sr0 + sr1);
      zz.im += cb * (si0 + si1);
      zs[ma * 32] = zz;
    }
  }
  const C2* pj = Ul + (c_foff[J] + mb * (J + 1)) * YI_ATOMS;
#pragma unroll
  for (int ma = 0; ma <= yi5::TJ; ++ma) {
    if (ma > jtop) break;
    const C2 z = zs[ma * 32];
    yacc[ma].re += cy * z.re;
    yacc[ma].im += cy * z.im;
    if (be != 0.0) {
      const double w = (2 * mb < J || 2 * ma < J) ? 2.0 : (2 * ma == J ? 1.0 : 0.0);
      const C2 u = pj[ma * YI_ATOMS];
      esum += be * w * (u.re * z.re + u.im * z.im);
    }
  }
}

template <int Y>
__device__ __forceinline__ void yi7_xyj(const C2* __restrict__ Ul, int X, int J, int mb, int off, double cy,
                                        double be, C2* __restrict__ zs, C2 (&yacc)[yi5::TJ + 1], double& esum) {
  const int SH = (X + Y - J) / 2;
  const bool mid = (2 * mb == J);
  const int jtop = mid ? J / 2 : J;  // middle row: upper half has zero weight
  for (int ma = 0; ma <= jtop; ++ma) zs[ma * 32] = C2{0.0, 0.0};
  const int lo = max(0, mb + SH - Y), hi = min(X, mb + SH);
  const int FX = c_foff[X], FY = c_foff[Y];
  for (int mb1 = lo; mb1 <= hi; ++mb1) {
    const int mb2 = mb + SH - mb1;
    C2 uy[Y + 1];
    const C2* py = Ul + (FY + mb2 * (Y + 1)) * YI_ATOMS;
#pragma unroll
    for (int a = 0; a <= Y; ++a) uy[a] = py[a * YI_ATOMS];
    const C2* px = Ul + (FX + mb1 * (X + 1)) * YI_ATOMS;
    const double cb = c_cgt[off + mb * (X + 1) + mb1];
    for (int ma = 0; ma <= jtop; ++ma) {
      const double* cga = c_cgt + off + ma * (X + 1);
      const int base1 = ma + SH;  // ma1 = base1 - ma2
      double sr0 = 0.0, si0 = 0.0, sr1 = 0.0, si1 = 0.0;
#pragma unroll
      for (int ma2 = 0; ma2 <= Y; ++ma2) {
        const int ma1 = base1 - ma2;
        if (ma1 >= 0 && ma1 <= X) {
          const C2 ux = px[ma1 * YI_ATOMS];
          const double c = cga[ma1];
          const double tr = ux.re * uy[ma2].re - ux.im * uy[ma2].im;
          const double ti = ux.re * uy[ma2].im + ux.im * uy[ma2].re;
          if (ma2 & 1) {
            sr1 += c * tr;
            si1 += c * ti;
          } else {
            sr0 += c * tr;
            si0 += c * ti;
          }
        }
      }
      C2 zz = zs[ma * 32];
      zz.re += cb * (sr0 + sr1);
      zz.im += cb * (si0 + si1);
      zs[ma * 32] = zz;
    }
  }
  const C2* pj = Ul + (c_foff[J] + mb * (J + 1)) * YI_ATOMS;
#pragma unroll
  for (int ma = 0; ma <= yi5::TJ; ++ma) {
    if (ma > jtop) break;
    const C2 z = zs[ma * 32];
    yacc[ma].re += cy * z.re;
    yacc[ma].im += cy * z.im;
    if (be != 0.0) {
      const double w = (2 * mb < J || 2 * ma < J) ? 2.0 : (2 * ma == J ? 1.0 : 0.0);
      const C2 u = pj[ma * YI_ATOMS];
      esum += be * w * (u.re * z.re + u.im * z.im);
    }
  }
}

__global__ void __launch_bounds__(YI6_WARPS * 32)
k_snap_yi_six(SnapDev D, int64_t natoms, const C2* __restrict__ utot, C2* __restrict__ ylist,
              double* __restrict__ eatom) {
  extern __shared__ double smem[];
  C2* Uf = reinterpret_cast<C2*>(smem);                                // [nfull][32]
  C2* zsm = Uf + D.nfull * YI_ATOMS;                                   // [warps][9][32]
  double* epart = reinterpret_cast<double*>(zsm + YI6_WARPS * (yi5::TJ + 1) * YI_ATOMS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t a0 = (int64_t)blockIdx.x * YI_ATOMS;
  const int na_blk = (int)min((int64_t)YI_ATOMS, natoms - a0);
  for (int t = threadIdx.x; t < D.nfull * YI_ATOMS; t += blockDim.x) {
    const int at = t & (YI_ATOMS - 1), f = t >> 5;
    int J = 0;
    while (J < D.tj && f >= c_foff[J + 1]) ++J;
    const int e = f - c_foff[J], mb = e / (J + 1), ma = e - mb * (J + 1);
    C2 v{0.0, 0.0};
    if (at < na_blk) {
      if (2 * mb <= J) {
        v = utot[(a0 + at) * D.nhalf + c_hoff[J] + mb * (J + 1) + ma];
      } else {
        C2 w = utot[(a0 + at) * D.nhalf + c_hoff[J] + (J - mb) * (J + 1) + (J - ma)];
        v = ((ma + mb) & 1) ? C2{-w.re, w.im} : C2{w.re, -w.im};
      }
    }
    Uf[f * YI_ATOMS + at] = v;
  }
  __syncthreads();
  const C2* Ul = Uf + lane;
  C2* zs = zsm + warp * (yi5::TJ + 1) * YI_ATOMS + lane;
  const int64_t atom = a0 + lane;
  double esum = 0.0;
  for (int gi = c_yi6_gseg[warp]; gi < c_yi6_gseg[warp + 1]; ++gi) {
    const int J = c_yi6_groups[gi] >> 8, mb = c_yi6_groups[gi] & 0xff;
    C2 yacc[yi5::TJ + 1];
#pragma unroll
    for (int m = 0; m <= yi5::TJ; ++m) yacc[m] = C2{0.0, 0.0};
    for (int k = c_yi5_jstart[J]; k < c_yi5_jstart[J + 1]; ++k) {
      const int tid = c_yi5_tlist[k];
      const int code = c_yi5_code[tid];
      const int X = code / 100, Y = (code / 10) % 10;
      const int off = c_yi5_cgoff[tid];
      const double cy = D.yi5[tid], be = D.yi5[yi5::NT + tid];
      switch (X) {
        case 0: yi6_xyj<0>(Ul, Y, J, mb, off, cy, be, zs, yacc, esum); break;
        case 1: yi6_xyj<1>(Ul, Y, J, mb, off, cy, be, zs, yacc, esum); break;
        case 2: yi6_xyj<2>(Ul, Y, J, mb, off, cy, be, zs, yacc, esum); break;
        case 3: yi6_xyj<3>(Ul, Y, J, mb, off, cy, be, zs, yacc, esum); break;
        case 4: yi6_xyj<4>(Ul, Y, J, mb, off, cy, be, zs, yacc, esum); break;
        case 5: yi6_xyj<5>(Ul, Y, J, mb, off, cy, be, zs, yacc, esum); break;
        case 6: yi6_xyj<6>(Ul, Y, J, mb, off, cy, be, zs, yacc, esum); break;
        case 7: yi6_xyj<7>(Ul, Y, J, mb, off, cy, be, zs, yacc, esum); break;
        default: yi6_xyj<8>(Ul, Y, J, mb, off, cy, be, zs, yacc, esum); break;
      }
    }
    if (lane < na_blk) {
      C2* yo = ylist + atom * D.nhalf + c_hoff[J] + mb * (J + 1);
#pragma unroll
      for (int m = 0; m <= yi5::TJ; ++m)
        if (m <= J) yo[m] = yacc[m];
    }
  }
  epart[warp * YI_ATOMS + lane] = esum;
  __syncthreads();
  if (warp == 0 && lane < na_blk) {
    double e = D.beta0;
    for (int w = 0; w < YI6_WARPS; ++w) e += epart[w * YI_ATOMS + lane];
    eatom[atom] = e;
  }
}

__global__ void __launch_bounds__(YI6_WARPS * 32)
k_snap_yi_seven(SnapDev D, int64_t natoms, const C2* __restrict__ utot, C2* __restrict__ ylist,
              double* __restrict__ eatom) {
  extern __shared__ double smem[];
  C2* Uf = reinterpret_cast<C2*>(smem);                                // [nfull][32]
  C2* zsm = Uf + D.nfull * YI_ATOMS;                                   // [warps][9][32]
  double* epart = reinterpret_cast<double*>(zsm + YI6_WARPS * (yi5::TJ + 1) * YI_ATOMS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t a0 = (int64_t)blockIdx.x * YI_ATOMS;
  const int na_blk = (int)min((int64_t)YI_ATOMS, natoms - a0);
  for (int t = threadIdx.x; t < D.nfull * YI_ATOMS; t += blockDim.x) {
    const int at = t & (YI_ATOMS - 1), f = t >> 5;
    int J = 0;
    while (J < D.tj && f >= c_foff[J + 1]) ++J;
    const int e = f - c_foff[J], mb = e / (J + 1), ma = e - mb * (J + 1);
    C2 v{0.0, 0.0};
    if (at < na_blk) {
      if (2 * mb <= J) {
        v = utot[(a0 + at) * D.nhalf + c_hoff[J] + mb * (J + 1) + ma];
      } else {
        C2 w = utot[(a0 + at) * D.nhalf + c_hoff[J] + (J - mb) * (J + 1) + (J - ma)];
        v = ((ma + mb) & 1) ? C2{-w.re, w.im} : C2{w.re, -w.im};
      }
    }
    Uf[f * YI_ATOMS + at] = v;
  }
  __syncthreads();
  const C2* Ul = Uf + lane;
  C2* zs = zsm + warp * (yi5::TJ + 1) * YI_ATOMS + lane;
  const int64_t atom = a0 + lane;
  double esum = 0.0;
  for (int gi = c_yi6_gseg[warp]; gi < c_yi6_gseg[warp + 1]; ++gi) {
    const int J = c_yi6_groups[gi] >> 8, mb = c_yi6_groups[gi] & 0xff;
    C2 yacc[yi5::TJ + 1];
#pragma unroll
    for (int m = 0; m <= yi5::TJ; ++m) yacc[m] = C2{0.0, 0.0};
    for (int k = c_yi5_jstart[J]; k < c_yi5_jstart[J + 1]; ++k) {
      const int tid = c_yi5_tlist[k];
      const int code = c_yi5_code[tid];
      const int X = code / 100, Y = (code / 10) % 10;
      const int off = c_yi5_cgoff[tid];
      const double cy = D.yi5[tid], be = D.yi5[yi5::NT + tid];
      switch (Y) {
        case 0: yi7_xyj<0>(Ul, X, J, mb, off, cy, be, zs, yacc, esum); break;
        case 1: yi7_xyj<1>(Ul, X, J, mb, off, cy, be, zs, yacc, esum); break;
        case 2: yi7_xyj<2>(Ul, X, J, mb, off, cy, be, zs, yacc, esum); break;
        case 3: yi7_xyj<3>(Ul, X, J, mb, off, cy, be, zs, yacc, esum); break;
        case 4: yi7_xyj<4>(Ul, X, J, mb, off, cy, be, zs, yacc, esum); break;
        case 5: yi7_xyj<5>(Ul, X, J, mb, off, cy, be, zs, yacc, esum); break;
        case 6: yi7_xyj<6>(Ul, X, J, mb, off, cy, be, zs, yacc, esum); break;
        case 7: yi7_xyj<7>(Ul, X, J, mb, off, cy, be, zs, yacc, esum); break;
        default: yi7_xyj<8>(Ul, X, J, mb, off, cy, be, zs, yacc, esum); break;
      }
    }
    if (lane < na_blk) {
      C2* yo = ylist + atom * D.nhalf + c_hoff[J] + mb * (J + 1);
#pragma unroll
      for (int m = 0; m <= yi5::TJ; ++m)
        if (m <= J) yo[m] = yacc[m];
    }
  }
  epart[warp * YI_ATOMS + lane] = esum;
  __syncthreads();
  if (warp == 0 && lane < na_blk) {
    double e = D.beta0;
    for (int w = 0; w < YI6_WARPS; ++w) e += epart[w * YI_ATOMS + lane];
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

// advance row mb of (u, du) from layer J-1 to layer J (WITH_D: also du)
template <int TJ, int J, bool WITH_D>
__device__ __forceinline__ void row_step(C2 (&u)[TJ + 1], C2 (&du)[TJ + 1], const RowGeom<TJ>& g, int mb,
                                         const double (*rp)[SNAP_JMAX + 2]) {
  if (J % 2 == 0) {
    // lane mb = J/2 receives row J/2-1 of layer J-1 from lane-1 (all lanes shuffle)
#pragma unroll
    for (int i = 0; i < J; ++i) {
      C2 v = shfl_up_c2(u[i], 1);
      C2 dv = WITH_D ? shfl_up_c2(du[i], 1) : C2{0.0, 0.0};
      if (2 * mb == J) {
        const int x = J - 1 - i;  // destination index in row J/2 of layer J-1
        const bool neg = ((x + J / 2) & 1) != 0;
        u[x] = neg ? C2{-v.re, v.im} : C2{v.re, -v.im};
        if (WITH_D) du[x] = neg ? C2{-dv.re, dv.im} : C2{dv.re, -dv.im};
      }
    }
  }
  if (2 * mb > J) return;
#pragma unroll
  for (int ma = J; ma >= 0; --ma) {
    C2 nu{0.0, 0.0}, nd{0.0, 0.0};
    if (ma < J) {
      const double A = rp[J - ma][J - mb];
      C2 t = cmulc(g.a, u[ma]);
      nu.re += A * t.re;
      nu.im += A * t.im;
      if (WITH_D) {
        C2 t1 = cmulc(g.da, u[ma]), t2 = cmulc(g.a, du[ma]);
        nd.re += A * (t1.re + t2.re);
        nd.im += A * (t1.im + t2.im);
      }
    }
    if (ma > 0) {
      const double Bc = rp[ma][J - mb];
      C2 t = cmulc(g.b, u[ma - 1]);
      nu.re -= Bc * t.re;
      nu.im -= Bc * t.im;
      if (WITH_D) {
        C2 t1 = cmulc(g.db, u[ma - 1]), t2 = cmulc(g.b, du[ma - 1]);
        nd.re -= Bc * (t1.re + t2.re);
        nd.im -= Bc * (t1.im + t2.im);
      }
    }
    u[ma] = nu;
    if (WITH_D) du[ma] = nd;
  }
}

// contraction of layer J's row with Y (full-matrix weights) for one component
template <int TJ, int J>
__device__ __forceinline__ double row_contract(const C2 (&u)[TJ + 1], const C2 (&du)[TJ + 1], const C2* Y,
                                               int mb, double fc, double dfc_uk) {
  if (2 * mb > J) return 0.0;
  double acc = 0.0;
  const C2* yr = Y + c_hoff[J] + mb * (J + 1);
#pragma unroll
  for (int ma = 0; ma <= J; ++ma) {
    const double w = (2 * mb < J || 2 * ma < J) ? 2.0 : (2 * ma == J ? 1.0 : 0.0);
    const C2 y = yr[ma];
    acc += w * (fc * (du[ma].re * y.re + du[ma].im * y.im) + dfc_uk * (u[ma].re * y.re + u[ma].im * y.im));
  }
  return acc;
}

template <int TJ, int J>
struct Layers {
  __device__ __forceinline__ static void de(C2 (&u)[TJ + 1], C2 (&du)[TJ + 1], const RowGeom<TJ>& g, int mb,
                                            const double (*rp)[SNAP_JMAX + 2], const C2* Y, double fc,
                                            double dfc_uk, double& acc) {
    Layers<TJ, J - 1>::de(u, du, g, mb, rp, Y, fc, dfc_uk, acc);
    row_step<TJ, J, true>(u, du, g, mb, rp);
    acc += row_contract<TJ, J>(u, du, Y, mb, fc, dfc_uk);
  }
  __device__ __forceinline__ static void ui(C2 (&u)[TJ + 1], C2 (&du)[TJ + 1], const RowGeom<TJ>& g, int mb,
                                            const double (*rp)[SNAP_JMAX + 2], C2* part, double fc) {
    Layers<TJ, J - 1>::ui(u, du, g, mb, rp, part, fc);
    row_step<TJ, J, false>(u, du, g, mb, rp);
    if (part && 2 * mb <= J) {
      C2* pr = part + c_hoff[J] + mb * (J + 1);
#pragma unroll
      for (int ma = 0; ma <= J; ++ma) {
        pr[ma].re = fma(fc, u[ma].re, pr[ma].re);
        pr[ma].im = fma(fc, u[ma].im, pr[ma].im);
      }
    }
  }
  // same recursion, the lane's row accumulated in registers over its pairs
  // (acc[J(J+1)/2 + ma]); one shared-memory write per element at the end
  __device__ __forceinline__ static void ui_reg(C2 (&u)[TJ + 1], C2 (&du)[TJ + 1], const RowGeom<TJ>& g, int mb,
                                                const double (*rp)[SNAP_JMAX + 2], bool on, double fc,
                                                C2 (&acc)[(TJ + 1) * (TJ + 2) / 2]) {
    Layers<TJ, J - 1>::ui_reg(u, du, g, mb, rp, on, fc, acc);
    row_step<TJ, J, false>(u, du, g, mb, rp);
    if (on && 2 * mb <= J) {
#pragma unroll
      for (int ma = 0; ma <= J; ++ma) {
        C2& a = acc[J * (J + 1) / 2 + ma];
        a.re = fma(fc, u[ma].re, a.re);
        a.im = fma(fc, u[ma].im, a.im);
      }
    }
  }
};
template <int TJ>
struct Layers<TJ, 0> {
  __device__ __forceinline__ static void de(C2 (&)[TJ + 1], C2 (&)[TJ + 1], const RowGeom<TJ>&, int,
                                            const double (*)[SNAP_JMAX + 2], const C2*, double, double, double&) {}
  __device__ __forceinline__ static void ui(C2 (&)[TJ + 1], C2 (&)[TJ + 1], const RowGeom<TJ>&, int,
                                            const double (*)[SNAP_JMAX + 2], C2*, double) {}
  __device__ __forceinline__ static void ui_reg(C2 (&)[TJ + 1], C2 (&)[TJ + 1], const RowGeom<TJ>&, int,
                                                const double (*)[SNAP_JMAX + 2], bool, double,
                                                C2 (&)[(TJ + 1) * (TJ + 2) / 2]) {}
};

constexpr int RR_WARPS = 4;  // warps per CTA of the register-resident kernels (one atom per warp)

// sqrt(p/q) table into shared memory, computed in place (correctly rounded
// divide and sqrt: the host table's values bit for bit) instead of 100
// lane-divergent constant-bank reads that serialise per warp
__device__ __forceinline__ void stage_rootpq(double (*rp)[SNAP_JMAX + 2]) {
  for (int t = threadIdx.x; t < (SNAP_JMAX + 2) * (SNAP_JMAX + 2); t += blockDim.x) {
    const int p = t / (SNAP_JMAX + 2), q = t % (SNAP_JMAX + 2);
    rp[p][q] = q ? __dsqrt_rn(__ddiv_rn((double)p, (double)q)) : 0.0;
  }
}

template <int TJ, bool REG>
__global__ void __launch_bounds__(RR_WARPS * 32)
k_snap_ui_rr(SnapDev D, int64_t natoms, int N, Box box, const double* __restrict__ q,
             const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt, int maxn,
             C2* __restrict__ utot) {
  constexpr int R = TJ / 2 + 1, P = 32 / R;
  extern __shared__ double smem[];
  double (*rp)[SNAP_JMAX + 2] = reinterpret_cast<double (*)[SNAP_JMAX + 2]>(smem);
  const int nh = D.nhalf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // pair-slot stride nh + 2 (= 5 mod 8 complex at twojmax 8): the 8 lanes of a
  // 128-bit shared-memory phase hit distinct bank groups in the top layer
  const int ps = nh + 2;
  C2* part = reinterpret_cast<C2*>(smem + (SNAP_JMAX + 2) * (SNAP_JMAX + 2)) + warp * P * ps;
  stage_rootpq(rp);
  const int64_t atom = (int64_t)blockIdx.x * RR_WARPS + warp;
  for (int t = lane; t < P * ps; t += 32) part[t] = C2{0.0, 0.0};
  __syncthreads();
  if (atom >= natoms) return;
  const int64_t b = atom / N;
  const int i = (int)(atom - b * N);
  const double* qb = q + b * (int64_t)N * 3;
  const int p = lane / R, mb = lane - p * R;
  const bool lane_ok = lane < P * R;
  const int n = cnt[atom];
  const int32_t* nb = nbr + atom * maxn;
  C2 acc[(TJ + 1) * (TJ + 2) / 2];
  if (REG) {
#pragma unroll
    for (int k = 0; k < (TJ + 1) * (TJ + 2) / 2; ++k) acc[k] = C2{0.0, 0.0};
  }
  for (int s0 = 0; s0 < n; s0 += P) {
    const int s = s0 + p;
    const bool valid = lane_ok && s < n;
    RowGeom<TJ> g;
    double fc = 0.0;
    if (valid) {
      double dx, dy, dz;
      pair_vec(qb, i, nb[s], box, dx, dy, dz);
      PairGeom pg;
      pair_geom(D, dx, dy, dz, pg, false);
      g.a = pg.a;
      g.b = pg.b;
      fc = pg.fc;
    } else {
      g.a = C2{1.0, 0.0};
      g.b = C2{0.0, 0.0};
    }
    C2 u[TJ + 1], du[TJ + 1];
#pragma unroll
    for (int k = 0; k <= TJ; ++k) u[k] = du[k] = C2{0.0, 0.0};
    u[0] = C2{mb == 0 ? 1.0 : 0.0, 0.0};
    if (REG) {
      if (valid && mb == 0) acc[0].re += fc;  // J = 0
      Layers<TJ, TJ>::ui_reg(u, du, g, mb, rp, valid, fc, acc);
    } else {
      C2* mypart = part + p * ps;
      if (valid && mb == 0) mypart[0].re += fc;  // J = 0
      // every lane runs the recursion (shuffles need the full warp); only valid
      // lanes accumulate, each into its own pair slot
      Layers<TJ, TJ>::ui(u, du, g, mb, rp, valid ? mypart : nullptr, fc);
    }
  }
  if (REG && lane_ok) {  // each lane owns its (pair slot, row): plain stores
    C2* mypart = part + p * ps;
#pragma unroll
    for (int J = 0; J <= TJ; ++J)
      if (2 * mb <= J)
#pragma unroll
        for (int ma = 0; ma <= J; ++ma) mypart[c_hoff[J] + mb * (J + 1) + ma] = acc[J * (J + 1) / 2 + ma];
  }
  __syncwarp();
  // fixed-order sum over the P pair slots + self term
  C2* out = utot + atom * nh;
  for (int t = lane; t < nh; t += 32) {
    C2 acc{0.0, 0.0};
#pragma unroll
    for (int pp = 0; pp < P; ++pp) {
      acc.re += part[pp * ps + t].re;
      acc.im += part[pp * ps + t].im;
    }
    int J = 0;
    while (J < TJ && t >= c_hoff[J + 1]) ++J;
    const int e = t - c_hoff[J];
    const int mbb = e / (J + 1), maa = e - mbb * (J + 1);
    if (maa == mbb) acc.re += D.wself;
    out[t] = acc;
  }
}

template <int TJ>
__global__ void __launch_bounds__(RR_WARPS * 32)
k_snap_deidrj_rr(SnapDev D, int64_t natoms, int N, Box box, const double* __restrict__ q,
                 const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt, int maxn,
                 const C2* __restrict__ ylist, double* __restrict__ dedr) {
  constexpr int R = TJ / 2 + 1, P = 32 / R;
  extern __shared__ double smem[];
  double (*rp)[SNAP_JMAX + 2] = reinterpret_cast<double (*)[SNAP_JMAX + 2]>(smem);
  const int nh = D.nhalf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  C2* Y = reinterpret_cast<C2*>(smem + (SNAP_JMAX + 2) * (SNAP_JMAX + 2)) + warp * nh;
  stage_rootpq(rp);
  const int64_t atom = (int64_t)blockIdx.x * RR_WARPS + warp;
  if (atom < natoms)
    for (int t = lane; t < nh; t += 32) Y[t] = ylist[atom * nh + t];
  __syncthreads();
  if (atom >= natoms) return;
  const int64_t b = atom / N;
  const int i = (int)(atom - b * N);
  const double* qb = q + b * (int64_t)N * 3;
  const int p = lane / R, mb = lane - p * R;
  const bool lane_ok = lane < P * R;
  const int n = cnt[atom];
  const int32_t* nb = nbr + atom * maxn;
  const double y0 = Y[0].re;
  for (int s0 = 0; s0 < n; s0 += P) {
    const int s = s0 + p;
    const bool valid = lane_ok && s < n;
    PairGeom pg;
    if (valid) {
      double dx, dy, dz;
      pair_vec(qb, i, nb[s], box, dx, dy, dz);
      pair_geom(D, dx, dy, dz, pg, true);
    } else {
      pair_geom(D, 1.0, 0.0, 0.0, pg, true);
      pg.fc = 0.0;
      pg.dfc = 0.0;
    }
    double res0 = 0.0, res1 = 0.0, res2 = 0.0;
#pragma unroll 1
    for (int k = 0; k < 3; ++k) {
      RowGeom<TJ> g{pg.a, pg.b, pg.da[k], pg.db[k]};
      C2 u[TJ + 1], du[TJ + 1];
#pragma unroll
      for (int e = 0; e <= TJ; ++e) u[e] = du[e] = C2{0.0, 0.0};
      u[0] = C2{mb == 0 ? 1.0 : 0.0, 0.0};
      const double dfc_uk = pg.dfc * pg.u[k];
      double acc = (mb == 0) ? dfc_uk * y0 : 0.0;  // J = 0: U = 1, dU = 0, weight 1
      Layers<TJ, TJ>::de(u, du, g, mb, rp, Y, pg.fc, dfc_uk, acc);
      // fixed-order sum over the R row lanes of this pair
#pragma unroll
      for (int r = 1; r < R; ++r) {
        double v = __shfl_down_sync(0xffffffffu, acc, r);
        if (mb == 0) acc += v;  // acc(mb=0) + acc(1) + ... in row order
      }
      if (k == 0) res0 = acc; else if (k == 1) res1 = acc; else res2 = acc;
    }
    if (valid && mb == 0) {
      double* o = dedr + (atom * maxn + s) * 3;
      o[0] = res0;
      o[1] = res1;
      o[2] = res2;
    }
  }
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
constexpr int ADJ_WARPS = 2;

// Forward-row history layouts: HL = 0 [slot (J, x)][lane] (23 KB per warp);
// HL = 1 [half index (J, row, x)][pair slot] (155 x 7 complex, 17.4 KB per warp:
// only the rows that exist are stored; slot 6 is the scratch of the two lanes
// without a pair), which leaves room for more warps per SM.
constexpr int ADJ_P = 7;  // pair slots per warp (32 / 5 rows = 6, + 1)

template <int HL, int J>
__device__ __forceinline__ int hpos(int x, int row, int mb, int lane, int p) {
  if constexpr (HL == 0) {
    return (J * (J + 1) / 2 + x) * 32 + lane + (row - mb);  // row mb - 1 is the lane below
  } else {
    return (yi5::hoff(J) + row * (J + 1) + x) * ADJ_P + p;
  }
}

template <int TJ, int HL>
struct AdjLayers {
  // forward: layer J from J-1 (in place), store the row, accumulate F
  template <int J>
  __device__ __forceinline__ static void fwd(C2 (&u)[TJ + 1], const RowGeom<TJ>& g, int mb,
                                             const double (*rp)[SNAP_JMAX + 2], const C2* Y, C2* hist,
                                             int lane, int p, double& F) {
    if constexpr (J > 0) {
      fwd<J - 1>(u, g, mb, rp, Y, hist, lane, p, F);
      C2 du[TJ + 1];
      row_step<TJ, J, false>(u, du, g, mb, rp);
    }
    if (2 * mb <= J) {
      const C2* yr = Y + c_hoff[J] + mb * (J + 1);
#pragma unroll
      for (int ma = 0; ma <= J; ++ma) {
        hist[hpos<HL, J>(ma, mb, mb, lane, p)] = u[ma];
        const double w = (2 * mb < J || 2 * ma < J) ? 2.0 : (2 * ma == J ? 1.0 : 0.0);
        F += w * (u[ma].re * yr[ma].re + u[ma].im * yr[ma].im);
      }
    }
  }

  // backward from layer J to J-1 (G holds the adjoint of layer J on entry)
  template <int J>
  __device__ __forceinline__ static void bwd(C2 (&G)[TJ + 1], const RowGeom<TJ>& g, int mb,
                                             const double (*rp)[SNAP_JMAX + 2], const C2* Y, const C2* hist,
                                             int lane, int p, C2& Sa, C2& Sb) {
    if constexpr (J > 0) {
      const bool active = 2 * mb <= J;
      const bool born = (J % 2 == 0) && (2 * mb == J);  // row mb of layer J-1 is virtual
      // U^{J-1} row mb (stored, or the symmetric image of row mb-1 of the same pair)
      C2 up[TJ + 1];
      if (active) {
#pragma unroll
        for (int x = 0; x < J; ++x) {
          if (!born) {
            up[x] = hist[hpos<HL, J - 1>(x, mb, mb, lane, p)];
          } else {
            const C2 v = hist[hpos<HL, J - 1>(J - 1 - x, mb - 1, mb, lane, p)];
            up[x] = ((x + mb) & 1) ? C2{-v.re, v.im} : C2{v.re, -v.im};
          }
        }
      }
      if (active) {
#pragma unroll
        for (int ma = 0; ma <= J; ++ma) {
          if (ma < J) {
            const double A = rp[J - ma][J - mb];
            const C2 t = cmulc(up[ma], G[ma]);  // conj(U') G
            Sa.re += A * t.re;
            Sa.im += A * t.im;
          }
          if (ma > 0) {
            const double Bc = rp[ma][J - mb];
            const C2 t = cmulc(up[ma - 1], G[ma]);
            Sb.re -= Bc * t.re;
            Sb.im -= Bc * t.im;
          }
        }
        // G^{J-1}[x] = A(J,x) a G[x] - B(J,x+1) b G[x+1]  (ascending x, in place)
#pragma unroll
        for (int x = 0; x < J; ++x) {
          const double A = rp[J - x][J - mb];
          const double Bc = rp[x + 1][J - mb];
          const C2 t1 = cmul(g.a, G[x]);
          const C2 t2 = cmul(g.b, G[x + 1]);
          G[x] = C2{A * t1.re - Bc * t2.re, A * t1.im - Bc * t2.im};
        }
        G[J] = C2{0.0, 0.0};
      }
      // adjoint of the virtual row flows to the lane below (row mb-1), all lanes shuffle
      if (J % 2 == 0) {
#pragma unroll
        for (int x = 0; x < J; ++x) {
          const C2 v = C2{__shfl_down_sync(0xffffffffu, G[x].re, 1), __shfl_down_sync(0xffffffffu, G[x].im, 1)};
          if (2 * (mb + 1) == J) {  // this lane is row J/2-1; the lane above was born at J
            const int xs = J - 1 - x;
            const bool neg = ((x + mb + 1) & 1) != 0;
            G[xs].re += neg ? -v.re : v.re;
            G[xs].im += neg ? v.im : -v.im;
          }
        }
        if (born) {
#pragma unroll
          for (int x = 0; x <= J; ++x) G[x] = C2{0.0, 0.0};
        }
      }
      // direct term of layer J-1 on stored rows
      if (2 * mb <= J - 1) {
        const C2* yr = Y + c_hoff[J - 1] + mb * J;
#pragma unroll
        for (int x = 0; x < J; ++x) {
          const double w = (2 * mb < J - 1 || 2 * x < J - 1) ? 2.0 : (2 * x == J - 1 ? 1.0 : 0.0);
          G[x].re += w * yr[x].re;
          G[x].im += w * yr[x].im;
        }
      }
      bwd<J - 1>(G, g, mb, rp, Y, hist, lane, p, Sa, Sb);
    }
  }
};

template <int TJ, int HL>
__global__ void __launch_bounds__(ADJ_WARPS * 32)
k_snap_deidrj_adj(SnapDev D, int64_t natoms, int N, Box box, const double* __restrict__ q,
                  const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt, int maxn,
                  const C2* __restrict__ ylist, double* __restrict__ dedr) {
  constexpr int R = TJ / 2 + 1, P = 32 / R;
  constexpr int HIST = HL == 0 ? (TJ + 1) * (TJ + 2) / 2 * 32 : yi5::hoff(TJ + 1) * ADJ_P;  // complex per warp
  extern __shared__ double smem[];
  double (*rp)[SNAP_JMAX + 2] = reinterpret_cast<double (*)[SNAP_JMAX + 2]>(smem);
  const int nh = D.nhalf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  C2* Y = reinterpret_cast<C2*>(smem + (SNAP_JMAX + 2) * (SNAP_JMAX + 2)) + warp * nh;
  C2* hist = reinterpret_cast<C2*>(smem + (SNAP_JMAX + 2) * (SNAP_JMAX + 2)) + ADJ_WARPS * nh + warp * HIST;
  stage_rootpq(rp);
  const int64_t atom = (int64_t)blockIdx.x * ADJ_WARPS + warp;
  if (atom < natoms)
    for (int t = lane; t < nh; t += 32) Y[t] = ylist[atom * nh + t];
  __syncthreads();
  if (atom >= natoms) return;
  const int64_t b = atom / N;
  const int i = (int)(atom - b * N);
  const double* qb = q + b * (int64_t)N * 3;
  const int p = lane / R, mb = lane - p * R;
  const int pc = p;  // lanes 30, 31 (no pair) write their own scratch slot 6
  const bool lane_ok = lane < P * R;
  const int n = cnt[atom];
  const int32_t* nb = nbr + atom * maxn;
  for (int s0 = 0; s0 < n; s0 += P) {
    const int s = s0 + p;
    const bool valid = lane_ok && s < n;
    PairGeom pg;
    if (valid) {
      double dx, dy, dz;
      pair_vec(qb, i, nb[s], box, dx, dy, dz);
      pair_geom(D, dx, dy, dz, pg, true);
    } else {
      pair_geom(D, 1.0, 0.0, 0.0, pg, true);
      pg.fc = 0.0;
      pg.dfc = 0.0;
    }
    RowGeom<TJ> g{pg.a, pg.b, C2{0.0, 0.0}, C2{0.0, 0.0}};
    C2 u[TJ + 1];
#pragma unroll
    for (int e = 0; e <= TJ; ++e) u[e] = C2{0.0, 0.0};
    u[0] = C2{mb == 0 ? 1.0 : 0.0, 0.0};
    double F = 0.0;
    AdjLayers<TJ, HL>::template fwd<TJ>(u, g, mb, rp, Y, hist, lane, pc, F);
    __syncwarp();
    // adjoint of the top layer: its direct term
    C2 G[TJ + 1];
#pragma unroll
    for (int e = 0; e <= TJ; ++e) G[e] = C2{0.0, 0.0};
    if (2 * mb <= TJ) {
      const C2* yr = Y + c_hoff[TJ] + mb * (TJ + 1);
#pragma unroll
      for (int x = 0; x <= TJ; ++x) {
        const double w = (2 * mb < TJ || 2 * x < TJ) ? 2.0 : (2 * x == TJ ? 1.0 : 0.0);
        G[x] = C2{w * yr[x].re, w * yr[x].im};
      }
    }
    C2 Sa{0.0, 0.0}, Sb{0.0, 0.0};
    AdjLayers<TJ, HL>::template bwd<TJ>(G, g, mb, rp, Y, hist, lane, pc, Sa, Sb);
    __syncwarp();
    // fixed-order sums over the R row lanes of the pair
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
      double* o = dedr + (atom * maxn + s) * 3;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double re = pg.da[k].re * Sa.re - pg.da[k].im * Sa.im + pg.db[k].re * Sb.re - pg.db[k].im * Sb.im;
        o[k] = pg.dfc * pg.u[k] * F + pg.fc * re;
      }
    }
  }
}

// layer J of row mb from layer J-1 in place, no born-row handling
template <int TJ, int J>
__device__ __forceinline__ void row_update(C2 (&u)[TJ + 1], const RowGeom<TJ>& g, int mb,
                                           const double (*rp)[SNAP_JMAX + 2]) {
#pragma unroll
  for (int ma = J; ma >= 0; --ma) {
    C2 nu{0.0, 0.0};
    if (ma < J) {
      const double A = rp[J - ma][J - mb];
      const C2 t = cmulc(g.a, u[ma]);
      nu.re += A * t.re;
      nu.im += A * t.im;
    }
    if (ma > 0) {
      const double Bc = rp[ma][J - mb];
      const C2 t = cmulc(g.b, u[ma - 1]);
      nu.re -= Bc * t.re;
      nu.im -= Bc * t.im;
    }
    u[ma] = nu;
  }
}

// U_tot with 4 lanes per pair (twojmax 8; see k_snap_deidrj_adj4): lanes own
// rows 0..3, the row-3 lane also builds row 4 of layer 8 from its own row 3 of
// layer 7.  Each lane accumulates its rows over its pairs in registers; one
// store per element into its pair slot, then a fixed-order sum over 8 slots.
constexpr int UI4_WARPS = 4;

template <int J>
__device__ __forceinline__ void ui4_layers(C2 (&u)[9], C2 (&u4)[9], const RowGeom<8>& g, int mb,
                                           const double (*rp)[SNAP_JMAX + 2], bool on, double fc,
                                           C2 (&acc)[45], C2* row4) {
  if constexpr (J > 0) {
    ui4_layers<J - 1>(u, u4, g, mb, rp, on, fc, acc, row4);
    if constexpr (J == 8) {
#pragma unroll
      for (int i = 0; i < J; ++i) {
        const int x = J - 1 - i;
        const C2 v = u[i];
        u4[x] = ((x + J / 2) & 1) ? C2{-v.re, v.im} : C2{v.re, -v.im};
      }
      u4[J] = C2{0.0, 0.0};
    }
    C2 du[9];
    row_step<8, J, false>(u, du, g, mb, rp);
    if (on && 2 * mb <= J) {
#pragma unroll
      for (int ma = 0; ma <= J; ++ma) {
        C2& a = acc[J * (J + 1) / 2 + ma];
        a.re = fma(fc, u[ma].re, a.re);
        a.im = fma(fc, u[ma].im, a.im);
      }
    }
    if constexpr (J == 8) {
      row_update<8, 8>(u4, g, 4, rp);
      if (on && mb == 3) {  // row 4 accumulates in the lane's own slot (shared memory)
#pragma unroll
        for (int ma = 0; ma <= 8; ++ma) {
          row4[ma].re = fma(fc, u4[ma].re, row4[ma].re);
          row4[ma].im = fma(fc, u4[ma].im, row4[ma].im);
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
  double (*rp)[SNAP_JMAX + 2] = reinterpret_cast<double (*)[SNAP_JMAX + 2]>(smem);
  const int nh = D.nhalf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ps = nh + 2;  // padded pair-slot stride
  C2* part = reinterpret_cast<C2*>(smem + (SNAP_JMAX + 2) * (SNAP_JMAX + 2)) + warp * P * ps;
  // per-pair (a, b, fc) of the whole list, one lane per pair (instead of the 4 row
  // lanes of a slot recomputing it every round)
  double* geo = reinterpret_cast<double*>(reinterpret_cast<C2*>(smem + (SNAP_JMAX + 2) * (SNAP_JMAX + 2)) +
                                          UI4_WARPS * P * ps) + warp * SNAP_MAXN * 5;
  stage_rootpq(rp);
  const int64_t atom = (int64_t)blockIdx.x * UI4_WARPS + warp;
  __syncthreads();
  if (atom >= natoms) return;
  const int64_t b = atom / N;
  const int i = (int)(atom - b * N);
  const double* qb = q + b * (int64_t)N * 3;
  const int p = lane / R, mb = lane - p * R;
  const int n = cnt[atom];
  const int32_t* nb = nbr + atom * maxn;
  C2 acc[45];
#pragma unroll
  for (int k = 0; k < 45; ++k) acc[k] = C2{0.0, 0.0};
  C2* row4 = part + p * ps + c_hoff[TJ] + 4 * (TJ + 1);
  if (mb == 3)
#pragma unroll
    for (int k = 0; k <= TJ; ++k) row4[k] = C2{0.0, 0.0};
  for (int j = lane; j < n; j += 32) {
    double dx, dy, dz;
    pair_vec(qb, i, nb[j], box, dx, dy, dz);
    PairGeom pg;
    pair_geom(D, dx, dy, dz, pg, false);
    double* o = geo + 5 * j;
    o[0] = pg.a.re; o[1] = pg.a.im; o[2] = pg.b.re; o[3] = pg.b.im; o[4] = pg.fc;
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
    C2 u[TJ + 1], u4[TJ + 1];
#pragma unroll
    for (int k = 0; k <= TJ; ++k) u[k] = u4[k] = C2{0.0, 0.0};
    u[0] = C2{mb == 0 ? 1.0 : 0.0, 0.0};
    if (valid && mb == 0) acc[0].re += fc;  // J = 0
    ui4_layers<TJ>(u, u4, g, mb, rp, valid, fc, acc, row4);
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

struct AdjR4 {
  static constexpr int TJ = 8;
  // forward: layer J from J-1 (in place), store rows of layers <= 7, accumulate F
  template <int J, class YS, bool LAZY = false>
  __device__ __forceinline__ static void fwd(C2 (&u)[TJ + 1], C2 (&u4)[TJ + 1], const RowGeom<TJ>& g, int mb,
                                             const double (*rp)[SNAP_JMAX + 2], const YS& Y, C2* hist, int lane,
                                             double& F) {
    if constexpr (J > 0) {
      fwd<J - 1, YS, LAZY>(u, u4, g, mb, rp, Y, hist, lane, F);
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
      C2 du[TJ + 1];
      row_step<TJ, J, false>(u, du, g, mb, rp);  // rows 1..3 are born at J = 2, 4, 6 from the lane below
      if constexpr (J == TJ) row_update<TJ, TJ>(u4, g, TJ / 2, rp);
    }
    if (2 * mb <= J) {
#pragma unroll
      for (int ma = 0; ma <= J; ++ma) {
        if constexpr (J < TJ) hist[(J * (J + 1) / 2 + ma) * 32 + lane] = u[ma];
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

  // Sa/Sb of one row at layer J, then its adjoint to layer J-1 (in place)
  template <int J>
  __device__ __forceinline__ static void row_adj(C2 (&G)[TJ + 1], const C2 (&up)[TJ + 1], const RowGeom<TJ>& g,
                                                 int mb, const double (*rp)[SNAP_JMAX + 2], C2& Sa, C2& Sb) {
#pragma unroll
    for (int ma = 0; ma <= J; ++ma) {
      if (ma < J) {
        const double A = rp[J - ma][J - mb];
        const C2 t = cmulc(up[ma], G[ma]);
        Sa.re += A * t.re;
        Sa.im += A * t.im;
      }
      if (ma > 0) {
        const double Bc = rp[ma][J - mb];
        const C2 t = cmulc(up[ma - 1], G[ma]);
        Sb.re -= Bc * t.re;
        Sb.im -= Bc * t.im;
      }
    }
#pragma unroll
    for (int x = 0; x < J; ++x) {
      const double A = rp[J - x][J - mb];
      const double Bc = rp[x + 1][J - mb];
      const C2 t1 = cmul(g.a, G[x]);
      const C2 t2 = cmul(g.b, G[x + 1]);
      G[x] = C2{A * t1.re - Bc * t2.re, A * t1.im - Bc * t2.im};
    }
    G[J] = C2{0.0, 0.0};
  }

  // LAZY: F accumulates here from the history rows re-read for the adjoint and
  // the Y elements loaded for G (each Y element read once)
  template <int J, class YS, bool LAZY = false>
  __device__ __forceinline__ static void bwd(C2 (&G)[TJ + 1], C2 (&G4)[TJ + 1], const RowGeom<TJ>& g, int mb,
                                             const double (*rp)[SNAP_JMAX + 2], const YS& Y, const C2* hist, int lane,
                                             C2& Sa, C2& Sb, double& F) {
    if constexpr (J > 0) {

      const bool active = 2 * mb <= J;
      const bool born = (J % 2 == 0) && (J < TJ) && (2 * mb == J);  // rows 1..3: virtual in layer J-1
      C2 up[TJ + 1];
      if (active) {
#pragma unroll
        for (int x = 0; x < J; ++x) {
          if (!born) {
            up[x] = hist[((J - 1) * J / 2 + x) * 32 + lane];
          } else {
            const C2 v = hist[((J - 1) * J / 2 + (J - 1 - x)) * 32 + lane - 1];
            up[x] = ((x + mb) & 1) ? C2{-v.re, v.im} : C2{v.re, -v.im};
          }
        }
        row_adj<J>(G, up, g, mb, rp, Sa, Sb);
      }
      if constexpr (J == TJ) {
        // row 4 (row-3 lane): its layer-7 image comes from this lane's own row 3
        if (mb == TJ / 2 - 1) {
          C2 up4[TJ + 1];
#pragma unroll
          for (int x = 0; x < J; ++x) {
            const C2 v = hist[((J - 1) * J / 2 + (J - 1 - x)) * 32 + lane];
            up4[x] = ((x + TJ / 2) & 1) ? C2{-v.re, v.im} : C2{v.re, -v.im};
          }
          row_adj<J>(G4, up4, g, TJ / 2, rp, Sa, Sb);
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
            const bool neg = ((x + mb + 1) & 1) != 0;
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
      bwd<J - 1, YS, LAZY>(G, G4, g, mb, rp, Y, hist, lane, Sa, Sb, F);
    }
  }
};

constexpr int ADJ4_WARPS = 2;
constexpr int ADJ4_SLOTS = 36;  // layers 0..7

// APW atoms per warp: their pair lists are concatenated so the 8 pair slots of
// a round stay filled across the atom boundary (26 pairs per atom fill 4
// rounds of 8 only to 81 %)
template <int APW>
__global__ void __launch_bounds__(ADJ4_WARPS * 32)
k_snap_deidrj_adj4(SnapDev D, int64_t natoms, int N, Box box, const double* __restrict__ q,
                   const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt, int maxn,
                   const C2* __restrict__ ylist, double* __restrict__ dedr) {
  constexpr int TJ = 8, R = 4, P = 8;
  extern __shared__ double smem[];
  double (*rp)[SNAP_JMAX + 2] = reinterpret_cast<double (*)[SNAP_JMAX + 2]>(smem);
  const int nh = D.nhalf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  C2* Yw = reinterpret_cast<C2*>(smem + (SNAP_JMAX + 2) * (SNAP_JMAX + 2)) + warp * APW * nh;
  C2* hist = reinterpret_cast<C2*>(smem + (SNAP_JMAX + 2) * (SNAP_JMAX + 2)) + ADJ4_WARPS * APW * nh +
             warp * ADJ4_SLOTS * 32;
  stage_rootpq(rp);
  const int64_t atom0 = ((int64_t)blockIdx.x * ADJ4_WARPS + warp) * APW;
  int nat[APW];
  int total = 0;
#pragma unroll
  for (int k = 0; k < APW; ++k) {
    const int64_t a = atom0 + k;
    nat[k] = a < natoms ? cnt[a] : 0;
    total += nat[k];
    if (a < natoms)
      for (int t = lane; t < nh; t += 32) Yw[k * nh + t] = ylist[a * nh + t];
  }
  __syncthreads();
  if (atom0 >= natoms) return;
  const int p = lane / R, mb = lane - p * R;
  for (int s0 = 0; s0 < total; s0 += P) {
    // pair slot -> (atom of the warp, neighbour slot)
    int k = s0 + p, w = 0;
#pragma unroll
    for (int a = 0; a + 1 < APW; ++a)
      if (w == a && k >= nat[a]) {
        k -= nat[a];
        w = a + 1;
      }
    const bool valid = s0 + p < total;
    const int64_t atom = atom0 + w;
    const int s = k;
    const C2* Y = Yw + w * nh;
    PairGeom pg;
    if (valid) {
      const int64_t b = atom / N;
      const int i = (int)(atom - b * N);
      double dx, dy, dz;
      pair_vec(q + b * (int64_t)N * 3, i, nbr[atom * maxn + s], box, dx, dy, dz);
      pair_geom(D, dx, dy, dz, pg, true);
    } else {
      pair_geom(D, 1.0, 0.0, 0.0, pg, true);
      pg.fc = 0.0;
      pg.dfc = 0.0;
    }
    RowGeom<TJ> g{pg.a, pg.b, C2{0.0, 0.0}, C2{0.0, 0.0}};
    C2 u[TJ + 1], u4[TJ + 1];
#pragma unroll
    for (int e = 0; e <= TJ; ++e) u[e] = u4[e] = C2{0.0, 0.0};
    u[0] = C2{mb == 0 ? 1.0 : 0.0, 0.0};
    double F = 0.0;
    AdjR4::fwd<TJ>(u, u4, g, mb, rp, YSmem{Y}, hist, lane, F);
    __syncwarp();
    C2 G[TJ + 1], G4[TJ + 1];
    {
      const C2* yr = Y + c_hoff[TJ] + mb * (TJ + 1);
      const C2* y4 = Y + c_hoff[TJ] + (TJ / 2) * (TJ + 1);
#pragma unroll
      for (int x = 0; x <= TJ; ++x) {
        const double w = half_w(TJ, mb, x), w4 = half_w(TJ, TJ / 2, x);
        G[x] = C2{w * yr[x].re, w * yr[x].im};
        G4[x] = C2{w4 * y4[x].re, w4 * y4[x].im};
      }
    }
    C2 Sa{0.0, 0.0}, Sb{0.0, 0.0};
    AdjR4::bwd<TJ>(G, G4, g, mb, rp, YSmem{Y}, hist, lane, Sa, Sb, F);
    __syncwarp();
    // fixed-order sums over the 4 row lanes of the pair
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
      double* o = dedr + (atom * maxn + s) * 3;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double re = pg.da[k].re * Sa.re - pg.da[k].im * Sa.im + pg.db[k].re * Sb.re - pg.db[k].im * Sb.im;
        o[k] = pg.dfc * pg.u[k] * F + pg.fc * re;
      }
    }
  }
}

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
// for mb <= J/2 (element (mb, ma) of the Y^dagger half rows)
__global__ void k_snap_ytrans(int64_t natoms, int nh, int tj, const C2* __restrict__ y, C2* __restrict__ yt) {
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
  yt[atom * nh + base + ma * (J / 2 + 1) + mb] = C2{v.re, -v.im};
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
  double (*rp)[SNAP_JMAX + 2] = reinterpret_cast<double (*)[SNAP_JMAX + 2]>(smem);
  const int nh = D.nhalf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  C2* Yw = reinterpret_cast<C2*>(smem + (SNAP_JMAX + 2) * (SNAP_JMAX + 2)) + warp * APW * nh;
  C2* hist = reinterpret_cast<C2*>(smem + (SNAP_JMAX + 2) * (SNAP_JMAX + 2)) + NWB * APW * nh +
             warp * ADJ4_SLOTS * 32;
  // geometry of 32 consecutive pairs (4 rounds), one lane per pair:
  // a, b, fc, dfc, u[3], sin, cos, 1/r and the partner atom
  double* gb = reinterpret_cast<double*>(reinterpret_cast<C2*>(smem + (SNAP_JMAX + 2) * (SNAP_JMAX + 2)) +
                                         NWB * (APW * nh + ADJ4_SLOTS * 32)) + warp * 32 * PAIR_GEO;
  int64_t* gk = reinterpret_cast<int64_t*>(reinterpret_cast<double*>(
                    reinterpret_cast<C2*>(smem + (SNAP_JMAX + 2) * (SNAP_JMAX + 2)) +
                    NWB * (APW * nh + ADJ4_SLOTS * 32)) + NWB * 32 * PAIR_GEO) + warp * 32;
  // list slots of the owned neighbours of the warp's atoms, [APW][SNAP_MAXN]
  int32_t* oslot = reinterpret_cast<int32_t*>(gk + (NWB - warp) * 32) + warp * APW * SNAP_MAXN;
  stage_rootpq(rp);
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
        const bool own = t0 + lane < c && pair_owned(i, nbr[a * maxn + t0 + lane]);
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
    AdjR4::fwd<TJ, YPair, true>(u, u4, g, mb, rp, Y, hist, lane, F);
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
    AdjR4::bwd<TJ, YPair, true>(G, G4, g, mb, rp, Y, hist, lane, Sa, Sb, F);
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
  double (*rp)[SNAP_JMAX + 2] = reinterpret_cast<double (*)[SNAP_JMAX + 2]>(smem);
  const int nh = D.nhalf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  C2* base = reinterpret_cast<C2*>(smem + (SNAP_JMAX + 2) * (SNAP_JMAX + 2));
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
  stage_rootpq(rp);
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
        const bool own = t0 + lane < n && pair_owned(i, nbr[a * maxn + t0 + lane]);
        const unsigned bal = __ballot_sync(0xffffffffu, own);
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
    AdjR4::fwd<TJ, YPair, true>(u, u4, g, mb, rp, Y, hist, lane, F);
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
    AdjR4::bwd<TJ, YPair, true>(G, G4, g, mb, rp, Y, hist, lane, Sa, Sb, F);
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

// gather of the pair form, one warp per atom (lanes over neighbour slots, the
// reverse-slot searches in parallel, fixed-order shuffle tree):
// grad_i = -sum_{owned} h_ik + sum_{owned by k} h_ki; the owner books the pair virial
__global__ void __launch_bounds__(128)
k_snap_gather_pair_w(int64_t natoms, int N, Box box, const double* __restrict__ q,
                     const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt, int maxn,
                     const double* __restrict__ dedr, double* __restrict__ grad, double* __restrict__ vatom) {
  griddep_wait();
  const int64_t atom = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (atom >= natoms) return;
  const int64_t b = atom / N;
  const int a = (int)(atom - b * N);
  const int n = cnt[atom];
  const int32_t* nb = nbr + atom * maxn;
  const double* qb = q + b * (int64_t)N * 3;
  double v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // g[3], vir[6]
  for (int s = lane; s < n; s += 32) {
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

static int snap_stages(pl_pot* pot, int64_t B, const double* q, SnapBuffers& buf, NeighList& nl) {
  pl_ctx* ctx = pot->ctx;
  SnapIndex* S = pot->snap;
  SnapDev D = snap_dev(pot);
  int N = pot->n_atoms;
  int64_t na = B * N;
  if (na > 0x7fffffff) return fail(PL_EARG, "too many atoms in one batch");
  PL_TRY(build_neighbours(pot, B, q, pot->rcut, SNAP_MAXN, &nl));
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
  size_t s1 = ui_smem(D), s2 = yi_smem(D), s3 = de_smem(D);
  static thread_local bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(k_snap_ui, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_yi, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_deidrj, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_bispectrum, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_ui_rr<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_ui_rr<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_yi_full, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_snap_yi_half, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    cudaFuncSetAttribute(k_snap_yi_reg, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_snap_yi_six, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
    cudaFuncSetAttribute(k_snap_yi_seven, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
    cudaFuncSetAttribute(k_snap_deidrj_rr<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_deidrj_adj<8, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_deidrj_adj<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_deidrj_adj4<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_deidrj_adj4<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_deidrj_pair<2, PAIR_WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_deidrj_run<8, PAIR_WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_snap_ui_r4, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_done = true;
  }
  // register-resident kernels are instantiated for twojmax = 8 (PL_SNAP_RR=0 selects the
  // shared-memory layer kernels, kept as the general-twojmax path and for A/B checks)
  static const bool rr_env = [] {
    const char* e = getenv("PL_SNAP_RR");
    return !(e && e[0] == '0');
  }();
  const bool rr = rr_env && (D.tj == 8);
  const size_t rp_bytes = sizeof(double) * (SNAP_JMAX + 2) * (SNAP_JMAX + 2);
  const unsigned rr_grid = (unsigned)((na + RR_WARPS - 1) / RR_WARPS);
  prof_mark(ctx->stream, ST_UI, true);
  if (rr) {
    size_t sm = rp_bytes + sizeof(C2) * RR_WARPS * (32 / 5) * (D.nhalf + 2);
    static const bool ui_reg = [] {
      const char* e = getenv("PL_SNAP_UI");
      return !(e && e[0] == '0');  // 0: accumulate through shared memory every pair
    }();
    static const bool ui4 = [] {
      const char* e = getenv("PL_SNAP_UI");
      return !(e && (e[0] == '0' || e[0] == '1'));  // 0/1: 5 lanes per pair (smem / register rows)
    }();
    if (ui4 && S->tj == 8) {
      const size_t sm4 = rp_bytes + sizeof(C2) * UI4_WARPS * 8 * (D.nhalf + 2) + sizeof(double) * UI4_WARPS * SNAP_MAXN * 5;
      PL_CUDA(launch_pdl(k_snap_ui_r4, dim3((unsigned)((na + UI4_WARPS - 1) / UI4_WARPS)), dim3(UI4_WARPS * 32), sm4,
                         ctx->stream, D, na, N, box, q, nl.nbr, nl.cnt, nl.maxn, buf.utot));
    } else if (ui_reg)
      k_snap_ui_rr<8, true><<<rr_grid, RR_WARPS * 32, sm, ctx->stream>>>(D, na, N, box, q, nl.nbr, nl.cnt,
                                                                          nl.maxn, buf.utot);
    else
      k_snap_ui_rr<8, false><<<rr_grid, RR_WARPS * 32, sm, ctx->stream>>>(D, na, N, box, q, nl.nbr, nl.cnt,
                                                                           nl.maxn, buf.utot);
  } else {
    k_snap_ui<<<(unsigned)na, UI_WARPS * 32, s1, ctx->stream>>>(D, na, N, box, q, nl.nbr, nl.cnt, nl.maxn,
                                                                 buf.utot);
  }
  PL_CHECK_LAUNCH();
  prof_mark(ctx->stream, ST_UI, false);
  prof_mark(ctx->stream, ST_YI, true);
  static const int yi_var = [] {
    const char* e = getenv("PL_SNAP_YI");
    return e ? atoi(e) : 8;
  }();
  static const int box_nw = [] {
    const char* e = getenv("PL_SNAP_BOXW");
    return e ? atoi(e) : 12;
  }();
  if (S->yi_reg && yi_var == 8) {
    PL_CUDA(snap_box_launch(box_nw, ctx->stream, na, D.beta0, D.yi5, buf.utot, buf.y, buf.eatom, erow));
  } else if (S->yi_reg && yi_var == 7) {
    size_t sm = sizeof(C2) * D.nfull * YI_ATOMS + sizeof(C2) * YI6_WARPS * 9 * YI_ATOMS +
                sizeof(double) * YI6_WARPS * YI_ATOMS;
    k_snap_yi_seven<<<(unsigned)((na + YI_ATOMS - 1) / YI_ATOMS), YI6_WARPS * 32, sm, ctx->stream>>>(
        D, na, buf.utot, buf.y, buf.eatom);
  } else if (S->yi_reg && yi_var == 6) {
    size_t sm = sizeof(C2) * D.nfull * YI_ATOMS + sizeof(C2) * YI6_WARPS * 9 * YI_ATOMS +
                sizeof(double) * YI6_WARPS * YI_ATOMS;
    k_snap_yi_six<<<(unsigned)((na + YI_ATOMS - 1) / YI_ATOMS), YI6_WARPS * 32, sm, ctx->stream>>>(
        D, na, buf.utot, buf.y, buf.eatom);
  } else if (S->yi_reg && yi_var >= 5) {
    size_t sm = sizeof(C2) * D.nfull * YI_ATOMS + sizeof(double) * YI5_WARPS * YI_ATOMS;
    k_snap_yi_reg<<<(unsigned)((na + YI_ATOMS - 1) / YI_ATOMS), YI5_WARPS * 32, sm, ctx->stream>>>(
        D, na, buf.utot, buf.y, buf.eatom);
  } else if (S->cgt_fits && yi_var == 4) {
    size_t sm = sizeof(C2) * D.nhalf * YI_ATOMS + sizeof(double) * YI3_WARPS * YI_ATOMS;
    k_snap_yi_half<<<(unsigned)((na + YI_ATOMS - 1) / YI_ATOMS), YI3_WARPS * 32, sm, ctx->stream>>>(
        D, na, buf.utot, buf.y, buf.eatom);
  } else if (S->cgt_fits) {
    size_t sm = sizeof(C2) * D.nfull * YI_ATOMS + sizeof(double) * YI3_WARPS * YI_ATOMS;
    k_snap_yi_full<<<(unsigned)((na + YI_ATOMS - 1) / YI_ATOMS), YI3_WARPS * 32, sm, ctx->stream>>>(
        D, na, buf.utot, buf.y, buf.eatom);
  } else {
    k_snap_yi<<<(unsigned)((na + YI_ATOMS - 1) / YI_ATOMS), YI_THREADS, s2, ctx->stream>>>(D, na, buf.utot,
                                                                                          buf.y, buf.eatom);
  }
  PL_CHECK_LAUNCH();
  prof_mark(ctx->stream, ST_YI, false);
  prof_mark(ctx->stream, ST_DE, true);
  static const bool adj_env = [] {
    const char* e = getenv("PL_SNAP_ADJ");
    return !(e && e[0] == '0');
  }();
  static const int adj_hl = [] {
    const char* e = getenv("PL_SNAP_ADJ");
    return (e && e[0] == '4') ? 1 : 0;  // 4: compact [half][pair] history (bitwise equal, measured slower)
  }();
  static const bool adj4 = [] {
    const char* e = getenv("PL_SNAP_ADJ");
    return !(e && (e[0] == '2' || e[0] == '4'));  // 2: 5 lanes per pair ([slot][lane] history)
  }();
  static const bool pair_env = [] {
    const char* e = getenv("PL_SNAP_PAIR");
    return !(e && e[0] == '0');  // 0: one adjoint sweep per ordered pair (k_snap_deidrj_adj4)
  }();
  if (rr && adj_env && adj4 && pair_env && S->tj == 8) {
    const int64_t nel = na * D.nhalf;
    PL_CUDA(launch_pdl(k_snap_ytrans, dim3((unsigned)((nel + 255) / 256)), dim3(256), 0, ctx->stream, na, D.nhalf,
                       D.tj, buf.y, buf.yt));
    PL_CHECK_LAUNCH();
    static const int prun = [] {
      const char* e = getenv("PL_SNAP_PAIR_RUN");
      return e ? atoi(e) : 1;  // 0: 2-atom warps only, 2: runs at every size (tests)
    }();
    constexpr int RUN = 8;
    if (prun == 2 || (prun == 1 && na >= (int64_t)RUN * PAIR_WARPS * 148 * 4)) {  // >= 4 waves of runs
      const size_t sm = rp_bytes + sizeof(C2) * PAIR_WARPS * (2 * D.nhalf + ADJ4_SLOTS * 32) +
                        (sizeof(double) * PAIR_GEO + sizeof(int64_t)) * PAIR_WARPS * 32 +
                        sizeof(int16_t) * PAIR_WARPS * RUN * SNAP_MAXN + sizeof(int32_t) * PAIR_WARPS * (RUN + 2);
      const unsigned grid = (unsigned)((na + PAIR_WARPS * RUN - 1) / (PAIR_WARPS * RUN));
      PL_CUDA(launch_pdl(k_snap_deidrj_run<RUN, PAIR_WARPS>, dim3(grid), dim3(PAIR_WARPS * 32), sm, ctx->stream, D,
                         na, N, box, q, nl.nbr, nl.cnt, nl.maxn, buf.y, buf.yt, buf.dedr));
    } else {
      const size_t sm = rp_bytes + sizeof(C2) * PAIR_WARPS * (2 * D.nhalf + ADJ4_SLOTS * 32) +
                        (sizeof(double) * PAIR_GEO + sizeof(int64_t)) * PAIR_WARPS * 32 +
                        sizeof(int32_t) * PAIR_WARPS * 2 * SNAP_MAXN;
      const unsigned grid = (unsigned)((na + PAIR_WARPS * 2 - 1) / (PAIR_WARPS * 2));
      PL_CUDA(launch_pdl(k_snap_deidrj_pair<2, PAIR_WARPS>, dim3(grid), dim3(PAIR_WARPS * 32), sm, ctx->stream, D,
                         na, N, box, q, nl.nbr, nl.cnt, nl.maxn, buf.y, buf.yt, buf.dedr));
    }
    buf.pair = true;
  } else if (rr && adj_env && adj4 && S->tj == 8) {
    static const int apw = [] {
      const char* e = getenv("PL_SNAP_ADJ_APW");
      return (e && e[0] == '1') ? 1 : 2;
    }();
    const size_t sm = rp_bytes + sizeof(C2) * ADJ4_WARPS * (apw * D.nhalf + ADJ4_SLOTS * 32);
    const unsigned grid = (unsigned)((na + ADJ4_WARPS * apw - 1) / (ADJ4_WARPS * apw));
    if (apw == 2)
      k_snap_deidrj_adj4<2><<<grid, ADJ4_WARPS * 32, sm, ctx->stream>>>(D, na, N, box, q, nl.nbr, nl.cnt, nl.maxn,
                                                                        buf.y, buf.dedr);
    else
      k_snap_deidrj_adj4<1><<<grid, ADJ4_WARPS * 32, sm, ctx->stream>>>(D, na, N, box, q, nl.nbr, nl.cnt, nl.maxn,
                                                                        buf.y, buf.dedr);
  } else if (rr && adj_env && adj_hl == 1) {
    size_t sm = rp_bytes + sizeof(C2) * ADJ_WARPS * (D.nhalf + yi5::hoff(9) * ADJ_P);
    k_snap_deidrj_adj<8, 1><<<(unsigned)((na + ADJ_WARPS - 1) / ADJ_WARPS), ADJ_WARPS * 32, sm, ctx->stream>>>(
        D, na, N, box, q, nl.nbr, nl.cnt, nl.maxn, buf.y, buf.dedr);
  } else if (rr && adj_env) {
    size_t sm = rp_bytes + sizeof(C2) * ADJ_WARPS * (D.nhalf + 45 * 32);
    k_snap_deidrj_adj<8, 0><<<(unsigned)((na + ADJ_WARPS - 1) / ADJ_WARPS), ADJ_WARPS * 32, sm, ctx->stream>>>(
        D, na, N, box, q, nl.nbr, nl.cnt, nl.maxn, buf.y, buf.dedr);
  } else if (rr) {
    size_t sm = rp_bytes + sizeof(C2) * RR_WARPS * D.nhalf;
    k_snap_deidrj_rr<8><<<rr_grid, RR_WARPS * 32, sm, ctx->stream>>>(D, na, N, box, q, nl.nbr, nl.cnt,
                                                                      nl.maxn, buf.y, buf.dedr);
  } else {
    k_snap_deidrj<<<(unsigned)na, DE_WARPS * 32, s3, ctx->stream>>>(D, na, N, box, q, nl.nbr, nl.cnt,
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
                       N, box, q, nl.nbr, nl.cnt, nl.maxn, buf.dedr, grad, virial ? buf.vatom : nullptr));
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
  const char* ey = getenv("PL_SNAP_YI");
  const int yv = ey ? atoi(ey) : 8;
  const char* ea = getenv("PL_SNAP_ADJ");
  const char* er = getenv("PL_SNAP_RR");
  const bool rr = !(er && er[0] == '0') && S->tj == 8;
  const bool adj = rr && !(ea && ea[0] == '0');
  const char* ep = getenv("PL_SNAP_PAIR");
  const bool pair = adj && !(ea && (ea[0] == '2' || ea[0] == '4')) && !(ep && ep[0] == '0');
  h_flops[0] = S->flops_ui_pair;
  h_flops[1] = (S->yi_reg && yv >= 5) ? S->flops_yi_atom_reg : S->flops_yi_atom;
  // pair form: one sweep (+ the Y_i + Y_k^dagger adds, one read of every half element) per
  // unordered pair, quoted per ordered pair like the other stages
  h_flops[2] = pair ? 0.5 * (S->flops_de_pair_adj + 2.0 * S->nhalf) : adj ? S->flops_de_pair_adj : S->flops_de_pair;
  return PL_OK;
}
