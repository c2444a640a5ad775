// gmp_layout.h -- host-side tile ownership of the P x Q process grid (SURVEY 8(e),
// 8(f) NEXT-3).
//
// Ownership (PAPER.md:179 distributes "2D block-cyclic"):
//   A(i, l) on process (rowP[i], l mod Q),  B(l, j) on (l mod P, colQ[j]),
//   C(i, j) on (rowP[i], colQ[j]).
// Block-cyclic is rowP[i] = i mod P, colQ[j] = j mod Q.  The K dimension always
// stays block-cyclic, so the SUMMA roots of step l are column l mod Q (A) and
// row l mod P (B) whatever the row/column owners are, and the fold order of every
// C tile (SUMMA step, class, l) does not depend on them: C is bitwise the same for
// every grid and every ownership (R15, R30).
//
// Precision-aware balancing (NEXT-3; PaRSEC's dynamic scheduling
// absorbs "the imbalanced workload introduced by the adaptive tile-centric
// mixed-precision algorithm").  Owner-computes with static ownership cannot steal
// work, so the balance is made at plan time instead: the tile-GEMM cost of C tile
// (i, j) is w(i, j) = sum_l cost[max(codeA(i,l), codeB(l,j))] (the pair classes
// of its K loop), and gmp_balance chooses row and column owners minimising the
// largest per-rank cost (tile-GEMMs plus a per-owned-tile term for the HBM-bound
// stats / pack / finalize work).  Deterministic (fixed iteration order, no
// randomness, doubles summed in a fixed order), so every rank that calls it with
// the same global maps gets the same owners.
#pragma once

#include <algorithm>
#include <cstdint>
#include <vector>

#include "gmp_common.cuh"

namespace gmp {

struct Layout {
  std::vector<int32_t> rowP, colQ;   // owner process row of tile row i / column of tile column j
  std::vector<int64_t> rowL, colL;   // local tile index of tile row i inside its owner (increasing i)
};

// fills rowP/colQ (block-cyclic when the given arrays are null) and the local
// indices; returns false if an owner is outside [0, P) / [0, Q)
inline bool make_layout(int64_t mt, int64_t nt, int P, int Q, const int32_t* row_owner,
                        const int32_t* col_owner, Layout* L) {
  L->rowP.resize(mt); L->colQ.resize(nt); L->rowL.resize(mt); L->colL.resize(nt);
  for (int64_t i = 0; i < mt; ++i) {
    L->rowP[i] = row_owner ? row_owner[i] : (int32_t)(i % P);
    if (L->rowP[i] < 0 || L->rowP[i] >= P) return false;
  }
  for (int64_t j = 0; j < nt; ++j) {
    L->colQ[j] = col_owner ? col_owner[j] : (int32_t)(j % Q);
    if (L->colQ[j] < 0 || L->colQ[j] >= Q) return false;
  }
  std::vector<int64_t> cr(P, 0), cc(Q, 0);
  for (int64_t i = 0; i < mt; ++i) L->rowL[i] = cr[L->rowP[i]]++;
  for (int64_t j = 0; j < nt; ++j) L->colL[j] = cc[L->colQ[j]]++;
  return true;
}

// Per-rank cost model of the balancer, in the units of `cost` (relative times).
//   cost[c], c = 0..GMP_NCLASS-1: one tile-GEMM of pair class c; cost[GMP_NCLASS]: per owned A, B or
//   C tile (stats + pack + W init / finalize, HBM-bound).
struct BalanceModel {
  int64_t mt, nt, kt;
  int P, Q;
  std::vector<double> w;         // mt x nt tile-GEMM cost of each C tile
  double tile_cost;
  std::vector<int64_t> kq, kp;   // #l with l mod Q == q / l mod P == p

  BalanceModel(int64_t mt_, int64_t nt_, int64_t kt_, int P_, int Q_, const uint8_t* acode,
               const uint8_t* bcode, const double* cost)
      : mt(mt_), nt(nt_), kt(kt_), P(P_), Q(Q_), w(mt_ * nt_, 0.0), tile_cost(cost[GMP_NCLASS]), kq(Q_, 0), kp(P_, 0) {
    for (int64_t i = 0; i < mt; ++i)
      for (int64_t j = 0; j < nt; ++j) {
        double s = 0.0;
        for (int64_t l = 0; l < kt; ++l) s += cost[std::max(acode[i * kt + l], bcode[l * nt + j])];
        w[i * nt + j] = s;
      }
    for (int64_t l = 0; l < kt; ++l) { kq[l % Q]++; kp[l % P]++; }
  }

  // block sums Bk[p][q] = sum of w over owned C tiles, nr[p] / nc[q] tile rows / columns owned
  void blocks(const std::vector<int32_t>& rowP, const std::vector<int32_t>& colQ, std::vector<double>& Bk) const {
    Bk.assign((size_t)P * Q, 0.0);
    for (int64_t i = 0; i < mt; ++i)
      for (int64_t j = 0; j < nt; ++j) Bk[(size_t)rowP[i] * Q + colQ[j]] += w[i * nt + j];
  }
  // per-rank cost: tile-GEMMs + owned tiles x tile_cost
  double rank_cost(const std::vector<double>& Bk, const std::vector<int64_t>& nr, const std::vector<int64_t>& nc,
                   int p, int q) const {
    const double tiles = (double)(nr[p] * kq[q] + kp[p] * nc[q] + nr[p] * nc[q]);
    return Bk[(size_t)p * Q + q] + tile_cost * tiles;
  }
  // (max, sum of squares) of the per-rank costs: lexicographic objective
  void objective(const std::vector<double>& Bk, const std::vector<int64_t>& nr, const std::vector<int64_t>& nc,
                 double* mx, double* ss, double* sum) const {
    *mx = 0.0; *ss = 0.0; *sum = 0.0;
    for (int p = 0; p < P; ++p)
      for (int q = 0; q < Q; ++q) {
        const double c = rank_cost(Bk, nr, nc, p, q);
        *mx = std::max(*mx, c); *ss += c * c; *sum += c;
      }
  }
};

static inline bool obj_less(double mx1, double ss1, double mx2, double ss2) {
  const double eps = 1e-12 * (mx2 > 0 ? mx2 : 1.0);
  if (mx1 < mx2 - eps) return true;
  if (mx1 > mx2 + eps) return false;
  return ss1 < ss2 * (1.0 - 1e-12);
}

// One dimension's local search: with the other dimension's owners fixed, move a
// tile row (column) to another process row (column), or swap two, whenever the
// lexicographic (max, sum of squares) rank cost decreases.  Best-improvement per
// sweep; `rows` selects the dimension.
inline bool balance_pass(const BalanceModel& M, bool rows, std::vector<int32_t>& rowP, std::vector<int32_t>& colQ) {
  const int64_t n = rows ? M.mt : M.nt;
  const int nbin = rows ? M.P : M.Q, nother = rows ? M.Q : M.P;
  std::vector<int32_t>& own = rows ? rowP : colQ;
  // v[x][o]: cost of tile row (column) x inside other-dimension bin o
  std::vector<double> v((size_t)n * nother, 0.0);
  for (int64_t i = 0; i < M.mt; ++i)
    for (int64_t j = 0; j < M.nt; ++j) {
      const int64_t x = rows ? i : j;
      const int o = rows ? colQ[j] : rowP[i];
      v[(size_t)x * nother + o] += M.w[i * M.nt + j];
    }
  bool improved_any = false;
  for (int sweep = 0; sweep < 64; ++sweep) {
    std::vector<double> Bk;
    M.blocks(rowP, colQ, Bk);
    std::vector<int64_t> nr(M.P, 0), nc(M.Q, 0);
    for (int64_t i = 0; i < M.mt; ++i) nr[rowP[i]]++;
    for (int64_t j = 0; j < M.nt; ++j) nc[colQ[j]]++;
    double mx0, ss0, sum0;
    M.objective(Bk, nr, nc, &mx0, &ss0, &sum0);
    double best_mx = mx0, best_ss = ss0;
    int64_t bx = -1, by = -1;
    int bto = -1;
    auto eval = [&](int64_t x, int to, int64_t y) {
      // apply: x -> to (and y -> own[x] when y >= 0), evaluate, undo
      const int from = own[x];
      auto shift = [&](int64_t t, int a, int b) {   // tile row/column t from bin a to bin b
        for (int o = 0; o < nother; ++o) {
          const double d = v[(size_t)t * nother + o];
          const size_t ia = rows ? (size_t)a * M.Q + o : (size_t)o * M.Q + a;
          const size_t ib = rows ? (size_t)b * M.Q + o : (size_t)o * M.Q + b;
          Bk[ia] -= d; Bk[ib] += d;
        }
        (rows ? nr : nc)[a]--; (rows ? nr : nc)[b]++;
      };
      shift(x, from, to);
      if (y >= 0) shift(y, to, from);
      double mx, ss, sum;
      M.objective(Bk, nr, nc, &mx, &ss, &sum);
      if (y >= 0) shift(y, from, to);
      shift(x, to, from);
      if (obj_less(mx, ss, best_mx, best_ss)) { best_mx = mx; best_ss = ss; bx = x; bto = to; by = y; }
    };
    for (int64_t x = 0; x < n; ++x)
      for (int to = 0; to < nbin; ++to) {
        if (to == own[x]) continue;
        eval(x, to, -1);
        for (int64_t y = x + 1; y < n; ++y)
          if (own[y] == to) eval(x, to, y);
      }
    if (bx < 0) break;
    const int from = own[bx];
    own[bx] = bto;
    if (by >= 0) own[by] = from;
    improved_any = true;
  }
  return improved_any;
}

// imbalance = max rank cost / mean rank cost
inline double layout_imbalance(const BalanceModel& M, const std::vector<int32_t>& rowP,
                               const std::vector<int32_t>& colQ) {
  std::vector<double> Bk;
  M.blocks(rowP, colQ, Bk);
  std::vector<int64_t> nr(M.P, 0), nc(M.Q, 0);
  for (int64_t i = 0; i < M.mt; ++i) nr[rowP[i]]++;
  for (int64_t j = 0; j < M.nt; ++j) nc[colQ[j]]++;
  double mx, ss, sum;
  M.objective(Bk, nr, nc, &mx, &ss, &sum);
  return sum > 0 ? mx / (sum / (M.P * M.Q)) : 1.0;
}

// LPT start: tile rows (columns) by decreasing total cost, each to the currently
// lightest process row (column); ties to the lower index.
inline void lpt_start(const BalanceModel& M, std::vector<int32_t>& rowP, std::vector<int32_t>& colQ) {
  std::vector<double> rw(M.mt, 0.0), cw(M.nt, 0.0);
  for (int64_t i = 0; i < M.mt; ++i)
    for (int64_t j = 0; j < M.nt; ++j) { rw[i] += M.w[i * M.nt + j]; cw[j] += M.w[i * M.nt + j]; }
  auto assign = [](const std::vector<double>& wt, int nbin, std::vector<int32_t>& own) {
    std::vector<int64_t> idx(wt.size());
    for (size_t t = 0; t < idx.size(); ++t) idx[t] = (int64_t)t;
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t x, int64_t y) { return wt[x] > wt[y]; });
    std::vector<double> load(nbin, 0.0);
    own.assign(wt.size(), 0);
    for (int64_t x : idx) {
      int b = 0;
      for (int k = 1; k < nbin; ++k) if (load[k] < load[b]) b = k;
      own[x] = b;
      load[b] += wt[x];
    }
  };
  assign(rw, M.P, rowP);
  assign(cw, M.Q, colQ);
}

inline void local_search(const BalanceModel& M, std::vector<int32_t>& rowP, std::vector<int32_t>& colQ) {
  for (int round = 0; round < 16; ++round) {
    bool a = M.P > 1 && balance_pass(M, true, rowP, colQ);
    bool b = M.Q > 1 && balance_pass(M, false, rowP, colQ);
    if (!a && !b) break;
  }
}

// Alternating row / column local search from several starts -- block-cyclic, LPT and
// GMP_BALANCE_RESTARTS block-cyclic layouts with their tile rows / columns shuffled by a
// fixed-seed SplitMix64 (deterministic: every rank gets the same owners) -- the best result
// (lexicographic max, sum of squares) wins, ties to the earlier start.
constexpr int GMP_BALANCE_RESTARTS = 8;
inline void balance_layout(const BalanceModel& M, std::vector<int32_t>& rowP, std::vector<int32_t>& colQ) {
  rowP.resize(M.mt); colQ.resize(M.nt);
  for (int64_t i = 0; i < M.mt; ++i) rowP[i] = (int32_t)(i % M.P);
  for (int64_t j = 0; j < M.nt; ++j) colQ[j] = (int32_t)(j % M.Q);
  local_search(M, rowP, colQ);
  auto obj = [&](const std::vector<int32_t>& r, const std::vector<int32_t>& c, double* mx, double* ss) {
    std::vector<double> Bk;
    M.blocks(r, c, Bk);
    std::vector<int64_t> nr(M.P, 0), nc(M.Q, 0);
    for (int64_t i = 0; i < M.mt; ++i) nr[r[i]]++;
    for (int64_t j = 0; j < M.nt; ++j) nc[c[j]]++;
    double sum;
    M.objective(Bk, nr, nc, mx, ss, &sum);
  };
  double m1, s1;
  obj(rowP, colQ, &m1, &s1);
  auto consider = [&](std::vector<int32_t>& r2, std::vector<int32_t>& c2) {
    local_search(M, r2, c2);
    double m2, s2;
    obj(r2, c2, &m2, &s2);
    if (obj_less(m2, s2, m1, s1)) { rowP = r2; colQ = c2; m1 = m2; s1 = s2; }
  };
  std::vector<int32_t> r2, c2;
  lpt_start(M, r2, c2);
  consider(r2, c2);
  uint64_t st = 0x9E3779B97F4A7C15ull;
  auto next = [&]() {   // SplitMix64
    uint64_t z = (st += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  auto shuffled_cyclic = [&](int64_t n, int bins, std::vector<int32_t>& own) {
    own.resize(n);
    for (int64_t t = 0; t < n; ++t) own[t] = (int32_t)(t % bins);
    for (int64_t t = n - 1; t > 0; --t) std::swap(own[t], own[(int64_t)(next() % (uint64_t)(t + 1))]);
  };
  for (int k = 0; k < GMP_BALANCE_RESTARTS; ++k) {
    shuffled_cyclic(M.mt, M.P, r2);
    shuffled_cyclic(M.nt, M.Q, c2);
    consider(r2, c2);
  }
}

}  // namespace gmp
