// gmp_map.cuh -- S1 map-stats and S2 map-finalize kernels.
//
// S1: per tile of A, B (and C if beta != 0): S_ij = sum x^2 in the canonical
//     CNORM order (O4), maxabs_ij, finiteness.  One 256-thread CTA per
//     tile; lane t of the CTA owns slot pair (2t, 2t+1) of every 512-element
//     chunk, i.e. one 16-byte load per chunk, and keeps two fma chains; a warp
//     butterfly with __shfl_xor_sync, then the 8 warp partials are summed in
//     warp order.  HBM-bound: 8 B read per element.
// S2: one CTA computes the global norms (sequential sums, O5), the
//     A/B codes, stored scales and every shadow scale, then the C codes with the
//     R23 range guards.  Every floating-point op is an explicit _rn intrinsic so
//     nvcc cannot contract it.
#pragma once
#include "gmp_common.cuh"

namespace gmp {

struct StatsJob {          // one tile of a local matrix
  const double* base;      // top-left element of the tile
  int64_t ld;
  int32_t out;             // index into the global stats arrays
};

__global__ void __launch_bounds__(256) k_tile_stats(const StatsJob* __restrict__ jobs, int nb,
                                                    double* __restrict__ S,
                                                    double* __restrict__ maxabs,
                                                    uint8_t* __restrict__ finite) {
  const StatsJob j = jobs[blockIdx.x];
  const int t = threadIdx.x;
  const int64_t n = (int64_t)nb * nb;
  double a0 = 0.0, a1 = 0.0, mx = 0.0;
  bool fin = true;
  // canonical order: w = 0,1,2,...; loads are batched U at a time (U x 16 B in
  // flight per thread: one CTA per tile must keep enough bytes in flight when a
  // rank holds few tiles), the fma chain of each slot stays in increasing w.
  // Element q = 2t + 512 w sits at row q / nb, column q % nb; both advance by a
  // constant per w (dr rows + dc columns, one carry).
#ifndef GMP_STATS_U
#define GMP_STATS_U 16
#endif
  constexpr int U = GMP_STATS_U;
  const int dr = 512 / nb, dc = 512 % nb;
  int r = (2 * t) / nb, c = (2 * t) % nb;
  auto step = [&] {
    r += dr;
    c += dc;
    if (c >= nb) { c -= nb; ++r; }
  };
  const int64_t nw = n / 512;            // chain length per slot (nb^2 is a multiple of 512)
  int64_t w = 0;
  for (; w + U <= nw; w += U) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = __ldg(reinterpret_cast<const double2*>(j.base + (int64_t)r * j.ld + c));
      step();
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a0 = __fma_rn(v[u].x, v[u].x, a0);
      a1 = __fma_rn(v[u].y, v[u].y, a1);
      double m0 = fabs(v[u].x), m1 = fabs(v[u].y);
      fin = fin && isfinite(m0) && isfinite(m1);
      mx = fmax(mx, fmax(m0, m1));
    }
  }
  for (; w < nw; ++w) {
    double2 v = __ldg(reinterpret_cast<const double2*>(j.base + (int64_t)r * j.ld + c));
    step();
    a0 = __fma_rn(v.x, v.x, a0);
    a1 = __fma_rn(v.y, v.y, a1);
    double m0 = fabs(v.x), m1 = fabs(v.y);
    fin = fin && isfinite(m0) && isfinite(m1);
    mx = fmax(mx, fmax(m0, m1));
  }
  double s = __dadd_rn(a0, a1);
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
  for (int off = 16; off >= 1; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  int allfin = __all_sync(0xffffffffu, fin);
  __shared__ double ws[8], wm[8];
  __shared__ int wf[8];
  if ((t & 31) == 0) { ws[t >> 5] = s; wm[t >> 5] = mx; wf[t >> 5] = allfin; }
  __syncthreads();
  if (t == 0) {
    double S_ = ws[0], M_ = wm[0];
    int F_ = wf[0];
    for (int w = 1; w < 8; ++w) { S_ = __dadd_rn(S_, ws[w]); M_ = fmax(M_, wm[w]); F_ &= wf[w]; }
    S[j.out] = F_ ? S_ : __longlong_as_double(0x7ff8000000000000ll);
    maxabs[j.out] = M_;
    finite[j.out] = (uint8_t)F_;
  }
}

struct FinalizeArgs {
  int64_t mt, nt, kt;
  int nb;
  double tol, alpha, beta;
  uint32_t mask;          // class mask, bit 0 forced on
  int explicit_a, explicit_b, explicit_c;
  // inputs (global tile grids)
  const double *SA, *MA, *SB, *MB, *SC, *MC;
  const uint8_t *FA, *FB, *FC;
  const uint8_t *mapA, *mapB, *mapC;   // explicit maps (device) or null
  // outputs
  uint8_t *codeA, *codeB, *codeC;
  int16_t *scaleA5, *scaleB5;          // [tile][GMP_NCLASS], class-c scale for c >= code
  int16_t *scaleCin;                   // packed C_in scale (beta != 0)
  int* status;                         // 0 ok, 4 non-finite
};

__device__ __forceinline__ double delta_in(int k, int nb) {
  // delta_k = u_k + sqrt(nb) * u_acc,k (u_acc = u64 for FP64 else u32)
  double uacc = (k == 0) ? 0x1p-53 : 0x1p-24;
  return __dadd_rn(class_u(k), __dmul_rn(__dsqrt_rn((double)nb), uacc));
}

// class-c scales of a tile stored at `code` with stored scale e_code and maxabs:
// shadow scale = e_code + scale_exp(RN_code(maxabs 2^e_code), c)  (max of the
// decoded payload, by monotonicity of RN; O6)
__device__ void fill_scales5(double maxabs, int code, int e_code, int16_t* s5) {
  double pm = (code == 0) ? maxabs : round_to_class(ldexp_fast(maxabs, e_code), code);
  for (int c = 0; c < GMP_NCLASS; ++c)
    s5[c] = (c < code) ? 0 : (c == code) ? (int16_t)e_code : (int16_t)(e_code + scale_exp(pm, c));
}

__global__ void __launch_bounds__(1024) k_map_finalize(FinalizeArgs a) {
  __shared__ double sh_nrm[3];
  __shared__ int sh_bad;
  const int t = threadIdx.x, nthr = blockDim.x;
  const int64_t nA = a.mt * a.kt, nB = a.kt * a.nt, nC = a.mt * a.nt;
  const bool hasC = a.beta != 0.0;
  if (t == 0) {
    int bad = 0;
    double s = 0.0;
    for (int64_t i = 0; i < nA; ++i) { s = __dadd_rn(s, a.SA[i]); bad |= !a.FA[i]; }
    sh_nrm[0] = s;
    s = 0.0;
    for (int64_t i = 0; i < nB; ++i) { s = __dadd_rn(s, a.SB[i]); bad |= !a.FB[i]; }
    sh_nrm[1] = s;
    s = 0.0;
    if (hasC)
      for (int64_t i = 0; i < nC; ++i) { s = __dadd_rn(s, a.SC[i]); bad |= !a.FC[i]; }
    sh_nrm[2] = s;
    sh_bad = bad;
    *a.status = bad ? 4 : 0;
  }
  __syncthreads();
  if (sh_bad) return;
  const uint32_t mask = a.mask | 1u;
  const double eps = __dmul_rn(a.tol, 0.25);
  // ---- A and B tiles (O5) ----
  for (int64_t idx = t; idx < nA + nB; idx += nthr) {
    const bool isB = idx >= nA;
    const int64_t tt = isB ? idx - nA : idx;
    const double SX = sh_nrm[isB ? 1 : 0];
    const double ntiles = (double)(isB ? nB : nA);
    const double S = isB ? a.SB[tt] : a.SA[tt];
    const double M = isB ? a.MB[tt] : a.MA[tt];
    int chosen = 0;
    const int expl = isB ? a.explicit_b : a.explicit_a;
    if (expl) {
      chosen = (isB ? a.mapB : a.mapA)[tt];
      if (chosen >= GMP_NCLASS || !(mask & (1u << chosen))) chosen = 0;
    } else if (!isinf(SX)) {
      const double rhs = __ddiv_rn(__dmul_rn(eps, __dsqrt_rn(SX)), __dsqrt_rn(ntiles));
      for (int kk = GMP_NCLASS - 1; kk >= 1; --kk) {   // ladder MXFP4, E5M2, E4M3, BF16, FP16, FP32 (then FP64)
        if (!(mask & (1u << kk))) continue;
        if (M == 0.0) { chosen = kk; break; }
        const int e = scale_exp(M, kk);
        // underflow term: nb x half the subnormal quantum of the scaled grid; MXFP4: of the
        // block holding the tile max (every block scale is <= it; R31)
        const int qe = (kk == GMP_MX) ? mx_block_exp(ldexp_fast(M, e)) : 0;
        const double lhs = __dadd_rn(__dmul_rn(delta_in(kk, a.nb), __dsqrt_rn(S)),
                                     __dmul_rn((double)a.nb, ldexp_fast(class_eta(kk), qe - e - 1)));
        if (lhs <= rhs) { chosen = kk; break; }
      }
    }
    const int e = scale_exp(M, chosen);
    (isB ? a.codeB : a.codeA)[tt] = (uint8_t)chosen;
    fill_scales5(M, chosen, e, (isB ? a.scaleB5 : a.scaleA5) + tt * GMP_NCLASS);
  }
  __syncthreads();
  // ---- C tiles (O7) ----
  const double nrmA = __dsqrt_rn(sh_nrm[0]), nrmB = __dsqrt_rn(sh_nrm[1]), nrmC = __dsqrt_rn(sh_nrm[2]);
  const double aa = fabs(a.alpha), ab = fabs(a.beta);
  const double Nhat = __dadd_rn(__dmul_rn(__dmul_rn(aa, nrmA), nrmB), __dmul_rn(ab, nrmC));
  const double rhsC = __ddiv_rn(__dmul_rn(__dmul_rn(a.tol, 0.5), Nhat), __dsqrt_rn((double)nC));
  const double sqkt = __dsqrt_rn((double)a.kt);
  for (int64_t ct = t; ct < nC; ct += nthr) {
    const int64_t i = ct / a.nt, j = ct - (ct / a.nt) * a.nt;
    int chosen = 0;
    double RA = 0.0, QB = 0.0;
    for (int64_t l = 0; l < a.kt; ++l) RA = __dadd_rn(RA, a.SA[i * a.kt + l]);
    for (int64_t l = 0; l < a.kt; ++l) QB = __dadd_rn(QB, a.SB[l * a.nt + j]);
    RA = __dsqrt_rn(RA);
    QB = __dsqrt_rn(QB);
    const double sc = hasC ? a.SC[ct] : 0.0;
    const double nhat = __dadd_rn(__dmul_rn(__dmul_rn(aa, RA), QB), __dmul_rn(ab, __dsqrt_rn(sc)));
    if (a.explicit_c) {   // MXFP4 is an operand class only (R31): never a C class
      chosen = a.mapC[ct];
      if (chosen >= GMP_NCLASS || chosen == GMP_MX || !(mask & (1u << chosen))) chosen = 0;
    } else {
      for (int k = GMP_NCLASS - 1; k >= 1; --k) {
        if (!(mask & (1u << k)) || k == GMP_MX) continue;
        const double dC = __dadd_rn(__dadd_rn(class_u(k), __dmul_rn(sqkt, 0x1p-24)),
                                    __ddiv_rn(__dmul_rn((double)a.nb, class_eta(k)), class_omega(k)));
        if (__dmul_rn(dC, nhat) <= rhsC) { chosen = k; break; }
      }
    }
    {
      // R23: FP32 accumulator range guards -- explicit codes included (a binary32 W
      // cannot hold an output or a fold factor outside its range)
      if (chosen != 0) {
        bool ok = nhat <= 0x1p100;
        if (a.beta != 0.0) {
          const double bf = (double)__double2float_rn(a.beta);
          ok = ok && fabs(bf) >= 0x1p-126 && fabs(bf) <= 0x1p100;
        }
        for (int64_t l = 0; ok && l < a.kt; ++l) {
          const int ca = a.codeA[i * a.kt + l], cb = a.codeB[l * a.nt + j];
          const int c = ca > cb ? ca : cb;
          const int ea = a.scaleA5[(i * a.kt + l) * GMP_NCLASS + c], eb = a.scaleB5[(l * a.nt + j) * GMP_NCLASS + c];
          const double f = ldexp_fast(a.alpha, -(ea + eb));
          if (f != 0.0 && !(fabs(f) >= 0x1p-126 && fabs(f) <= 0x1p100)) ok = false;
        }
        if (!ok) chosen = 0;
      }
    }
    a.codeC[ct] = (uint8_t)chosen;
    a.scaleCin[ct] = (int16_t)(hasC ? scale_exp(a.MC[ct], chosen) : 0);
  }
}

}  // namespace gmp
