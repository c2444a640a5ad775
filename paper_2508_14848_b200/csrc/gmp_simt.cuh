// gmp_simt.cuh -- S6 grouped tile-GEMM for the FP64 (DFMA) and FP32 (FFMA)
// precision classes, with the per-l fold epilogue.
//
// One launch per (SUMMA step, class).  A work item is a 128x128 sub-tile of one
// local C tile plus the ordered list of l (pairs) of this step whose pair class
// max(code_A(i,l), code_B(l,j)) equals the launch's class (O8-O9).
// For each pair the CTA computes P = A_il B_lj over K = nb in the class's
// arithmetic -- per-thread SEQUENTIAL k, one fma per k, from +0 -- so P is
// bitwise the oracle's emulation (O8).  Then the fold
//     W = fma_W(RN_W(alpha 2^-(eA+eB)), RN_W(P), W)
// is applied to the W accumulator in global memory (read-modify-write per
// pair: 2 x 64 KB per 128x128 binary32 sub-tile against 2*128*128*nb flops).
//
// Both operands are K-major in the packed arena (A row-major, B transposed),
// so one loader serves both: 128 rows x BK k-values per slice, staged through
// registers into k-major shared memory (As[k][m]) for 128-bit LDS; 2-stage
// shared memory ring with register prefetch of the next slice.
// Classes 2..4 can also run here (payload decoded to binary32): that is the
// bring-up / cross-check path; the product path for them is gmp_tc.cuh.
#pragma once
#include "gmp_common.cuh"
#include "gmp_convert.cuh"

namespace gmp {

struct WorkItem {
  int32_t ctile;       // index into the CTileDesc array
  int32_t m0, n0;      // sub-tile origin inside the C tile
  int32_t pbeg, pcnt;  // range in the PairDesc list
  int32_t pad;
};

struct PairDesc {
  int64_t a_off, b_off;  // byte offsets of the class-c payloads (A row-major, B K-major)
  int32_t fexp;          // -(eA + eB): fold factor alpha * 2^fexp
  int32_t l;             // global reduction tile index (bookkeeping)
  int32_t a_slot, b_slot;  // slot indices in the class arena (TMA row = slot * nb)
};

template <int C> struct SimtCfg {
  using T = float;
  static constexpr int BK = 8, BN = 128;   // 128x128 CTA tile, 8x8 per thread
};
template <> struct SimtCfg<0> {
  using T = double;
  static constexpr int BK = 8, BN = 64;    // 128x64 CTA tile, 8x4 per thread (register budget)
};
template <int C> constexpr int simt_bn() { return SimtCfg<C>::BN; }
inline int simt_bn_rt(int c) { return c == 0 ? 64 : 128; }

// load 4 consecutive payload elements (class C) -> 4 compute values
template <int C, typename T>
__device__ __forceinline__ void ld4(const uint8_t* p, T* v) {
  if constexpr (C == 0) {
    double2 a = __ldg(reinterpret_cast<const double2*>(p));
    double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  } else if constexpr (C == 1) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  } else if constexpr (C == 2 || C == 3) {
    uint2 a = __ldg(reinterpret_cast<const uint2*>(p));
    uint16_t h[4] = {(uint16_t)(a.x & 0xFFFF), (uint16_t)(a.x >> 16), (uint16_t)(a.y & 0xFFFF),
                     (uint16_t)(a.y >> 16)};
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = (C == 2) ? f16_to_f32(h[i]) : bf16_to_f32(h[i]);
  } else {
    uint32_t a = __ldg(reinterpret_cast<const uint32_t*>(p));
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = e4m3_to_f32((uint8_t)(a >> (8 * i)));
  }
}

template <int C, typename T, int NE>
__device__ __forceinline__ void ldn(const uint8_t* p, T* v) {
  if constexpr (NE == 4) {
    ld4<C>(p, v);
  } else {
    static_assert(C == 0 && NE == 2, "2-element loads are used by the binary64 B loader only");
    double2 a = __ldg(reinterpret_cast<const double2*>(p));
    v[0] = a.x; v[1] = a.y;
  }
}

template <typename T>
__device__ __forceinline__ T fma_rn(T a, T b, T c) {
  if constexpr (sizeof(T) == 8) return __fma_rn(a, b, c);
  else return __fmaf_rn(a, b, c);
}

template <int C>
__global__ void __launch_bounds__(256, 1)
k_simt_class(const WorkItem* __restrict__ items, const PairDesc* __restrict__ pairs,
             const CTileDesc* __restrict__ ctiles, uint8_t* __restrict__ ws, int nb, double alpha) {
  using T = typename SimtCfg<C>::T;
  constexpr int BK = SimtCfg<C>::BK;
  constexpr int BM = 128, BN = SimtCfg<C>::BN, PAD = 4;
  constexpr int TN = BN / 16, HN = TN / 2;        // per-thread columns, per half
  constexpr int EB = class_bytes(C);
  constexpr int EA = BM * BK / 256, EBn = BN * BK / 256;  // loader elements per thread
  __shared__ __align__(16) T As[2][BK][BM + PAD];
  __shared__ __align__(16) T Bs[2][BK][BN + PAD];

  const WorkItem it = items[blockIdx.x];
  const CTileDesc ct = ctiles[it.ctile];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  // loader mapping: rows x BK k; thread -> row, first k of its EA (EBn) run
  const int lrA = tid / (BK / EA), lkA = (tid % (BK / EA)) * EA;
  const int lrB = tid / (BK / EBn), lkB = (tid % (BK / EBn)) * EBn;

  for (int pi = 0; pi < it.pcnt; ++pi) {
    const PairDesc pd = pairs[it.pbeg + pi];
    const uint8_t* Ag = ws + pd.a_off + ((int64_t)(it.m0 + lrA) * nb + lkA) * EB;
    const uint8_t* Bg = ws + pd.b_off + ((int64_t)(it.n0 + lrB) * nb + lkB) * EB;
    T acc[8][TN];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

    T ra[EA], rb[EBn];
    ldn<C, T, EA>(Ag, ra);
    ldn<C, T, EBn>(Bg, rb);
#pragma unroll
    for (int e = 0; e < EA; ++e) As[0][lkA + e][lrA] = ra[e];
#pragma unroll
    for (int e = 0; e < EBn; ++e) Bs[0][lkB + e][lrB] = rb[e];
    __syncthreads();
    const int nsl = nb / BK;
    for (int s = 0; s < nsl; ++s) {
      const int buf = s & 1;
      if (s + 1 < nsl) {
        ldn<C, T, EA>(Ag + (int64_t)(s + 1) * BK * EB, ra);
        ldn<C, T, EBn>(Bg + (int64_t)(s + 1) * BK * EB, rb);
      }
#pragma unroll
      for (int k = 0; k < BK; ++k) {
        T a[8], b[TN];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int e = 0; e < 4; ++e) a[h * 4 + e] = As[buf][k][h * 64 + ty * 4 + e];
#pragma unroll
          for (int e = 0; e < HN; ++e) b[h * HN + e] = Bs[buf][k][h * (BN / 2) + tx * HN + e];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fma_rn(a[i], b[j], acc[i][j]);
      }
      if (s + 1 < nsl) {
#pragma unroll
        for (int e = 0; e < EA; ++e) As[buf ^ 1][lkA + e][lrA] = ra[e];
#pragma unroll
        for (int e = 0; e < EBn; ++e) Bs[buf ^ 1][lkB + e][lrB] = rb[e];
      }
      __syncthreads();
    }
    // ---- fold (O9): W = fma_W(RN_W(alpha 2^fexp), RN_W(P), W) ----
    const double f64 = ldexp(alpha, pd.fexp);
    const float f32 = __double2float_rn(f64);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = it.m0 + (i >> 2) * 64 + ty * 4 + (i & 3);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t base = (int64_t)r * nb + it.n0 + h * (BN / 2) + tx * HN;
        if (ct.code == 0) {
          double* w = reinterpret_cast<double*>(ws + ct.w_off) + base;
#pragma unroll
          for (int e = 0; e < HN; e += 2) {
            double2 v = *reinterpret_cast<double2*>(w + e);
            v.x = __fma_rn(f64, (double)acc[i][h * HN + e], v.x);
            v.y = __fma_rn(f64, (double)acc[i][h * HN + e + 1], v.y);
            *reinterpret_cast<double2*>(w + e) = v;
          }
        } else {
          float* w = reinterpret_cast<float*>(ws + ct.w_off) + base;
#pragma unroll
          for (int e = 0; e < HN; e += 2) {
            float2 v = *reinterpret_cast<float2*>(w + e);
            v.x = __fmaf_rn(f32, to_f32(acc[i][h * HN + e]), v.x);
            v.y = __fmaf_rn(f32, to_f32(acc[i][h * HN + e + 1]), v.y);
            *reinterpret_cast<float2*>(w + e) = v;
          }
        }
      }
    }
  }
}

}  // namespace gmp
