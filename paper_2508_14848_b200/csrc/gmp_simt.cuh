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
#include <type_traits>

#include "gmp_common.cuh"
#include "gmp_convert.cuh"

namespace gmp {

struct WorkItem {
  int32_t ctile;       // index into the CTileDesc array
  int32_t m0, n0;      // sub-tile origin inside the C tile (filled by expand_item)
  int32_t pbeg, pcnt;  // range in the PairDesc list
  int32_t pad;
};

// The host lists one WorkItem per (C tile, pair list); a launch covers
// items x S sub-tiles (S = (nb/128) * (nb/bn)).  Flat index -> item + sub-tile,
// consecutive flat indices walk the n-blocks of one 128-row band (A panel reuse).
__device__ __forceinline__ WorkItem expand_item(const WorkItem* __restrict__ items, int64_t flat, int nb, int bn,
                                                const int32_t* __restrict__ order = nullptr) {
  const int nbn = nb / bn, S = (nb / 128) * nbn;
  if (order) flat = order[flat];   // host raster (C tile row bands, sub-columns)
  const int64_t idx = flat / S;
  const int sub = (int)(flat - idx * S);
  WorkItem w = items[idx];
  w.m0 = (sub / nbn) * 128;
  w.n0 = (sub - (sub / nbn) * nbn) * bn;
  return w;
}
__host__ __device__ inline int64_t subtiles_per_item(int nb, int bn) { return (int64_t)(nb / 128) * (nb / bn); }

struct PairDesc {
  int64_t a_off, b_off;  // byte offsets of the class-c payloads (A row-major, B K-major)
  int32_t fexp;          // -(eA + eB): fold factor alpha * 2^fexp
  int32_t l;             // global reduction tile index (bookkeeping)
  int32_t a_slot, b_slot;  // slot indices in the class arena (TMA row = slot * nb)
  int32_t cls;             // pair class (the merged FP16+BF16 launch selects the operand map and the MMA kind by it)
  int32_t pad;
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
    for (int i = 0; i < 4; ++i) v[i] = (C == 4) ? e4m3_to_f32((uint8_t)(a >> (8 * i))) : e5m2_to_f32((uint8_t)(a >> (8 * i)));
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

  const WorkItem it = expand_item(items, blockIdx.x, nb, BN);
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
    // MXFP4 (class 6): nibbles + block scales, element (row, k) through mx_value
    auto loadA = [&](int sl, T* r) {
      if constexpr (C == GMP_MX) {
#pragma unroll
        for (int e = 0; e < EA; ++e) r[e] = mx_value(ws + pd.a_off, nb, it.m0 + lrA, sl * BK + lkA + e);
      } else {
        ldn<C, T, EA>(Ag + (int64_t)sl * BK * EB, r);
      }
    };
    auto loadB = [&](int sl, T* r) {
      if constexpr (C == GMP_MX) {
#pragma unroll
        for (int e = 0; e < EBn; ++e) r[e] = mx_value(ws + pd.b_off, nb, it.n0 + lrB, sl * BK + lkB + e);
      } else {
        ldn<C, T, EBn>(Bg + (int64_t)sl * BK * EB, r);
      }
    };
    loadA(0, ra);
    loadB(0, rb);
#pragma unroll
    for (int e = 0; e < EA; ++e) As[0][lkA + e][lrA] = ra[e];
#pragma unroll
    for (int e = 0; e < EBn; ++e) Bs[0][lkB + e][lrB] = rb[e];
    __syncthreads();
    const int nsl = nb / BK;
    for (int s = 0; s < nsl; ++s) {
      const int buf = s & 1;
      if (s + 1 < nsl) {
        loadA(s + 1, ra);
        loadB(s + 1, rb);
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
          for (int j = 0; j < TN; ++j) {
            // O8: acc + RN32(a b); the product is exact for classes 2..5 (one fmaf), not
            // always for MXFP4 (block scales summing below 2^-149)
            if constexpr (C == GMP_MX) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i], b[j]));
            else acc[i][j] = fma_rn(a[i], b[j], acc[i][j]);
          }
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
    const double f64 = ldexp_fast(alpha, pd.fexp);
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


// ---------------------------------------------------------------------------
// cp.async helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// packed FFMA2: two independent IEEE fma.rn.f32 in one instruction, `a` broadcast
__device__ __forceinline__ float2 ffma2_bcast(float a, float2 b, float2 c) {
  unsigned long long ra, rb, rc;
  asm("mov.b64 %0, {%1, %1};" : "=l"(ra) : "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rc) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(rc) : "l"(ra), "l"(rb));
  float2 d;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rc));
  return d;
}

// ---------------------------------------------------------------------------
// FP32 / FP64 outer-product kernel over MN-major payloads (O6):
// A tiles column-major, B tiles row-major, so a K-slice of a 128-row sub-tile
// is BK contiguous rows of 128 elements -- copied verbatim by a STAGES-deep
// cp.async ring into k-major shared memory As[k][m], Bs[k][n].
//   float  (class 1): 128x128 sub-tile, 8x8 outputs per thread, packed FFMA2
//                     (Blackwell's FP32 pipe reaches 128 FMA/clk/SM only through
//                     it); a[i] is a broadcast scalar operand, every lane is one
//                     fmaf in increasing k -> bitwise the oracle's O8.
//   double (class 0): 128x64 sub-tile, 8x4 outputs per thread, DFMA; bitwise O8.
//                     Cross-check kernel (GMP_FLAG_SIMT_ONLY); the product FP64
//                     path is k_dmma.
// The (pair, slice) sequence of an item is one continuous pipeline.
// ---------------------------------------------------------------------------
template <typename T> struct MnCfg;
template <> struct MnCfg<float> { static constexpr int BN = 128, BK = 16, ST = 4; };
template <> struct MnCfg<double> { static constexpr int BN = 64, BK = 16, ST = 4; };
template <typename T> constexpr int mn_smem_bytes() {
  return MnCfg<T>::ST * MnCfg<T>::BK * (128 + MnCfg<T>::BN) * (int)sizeof(T);
}
inline int mn_bn(int c) { return c == 0 ? 64 : 128; }

template <typename T>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? 2 : 1)
k_mn(const WorkItem* __restrict__ items, const PairDesc* __restrict__ pairs,
     const CTileDesc* __restrict__ ctiles, uint8_t* __restrict__ ws, int nb, double alpha) {
  constexpr int BN = MnCfg<T>::BN, BK = MnCfg<T>::BK, ST = MnCfg<T>::ST;
  constexpr int ES = sizeof(T);
  constexpr int ACH = 128 * ES / 16, BCH = BN * ES / 16;  // 16-byte chunks per smem row
  constexpr int CHUNKS = BK * (ACH + BCH), CPT = CHUNKS / 256;
  constexpr int STAGE = BK * (128 + BN) * ES;            // bytes
  static_assert(CHUNKS % 256 == 0, "loader");
  extern __shared__ __align__(128) uint8_t sm[];
  const WorkItem it = expand_item(items, blockIdx.x, nb, BN);
  const CTileDesc ct = ctiles[it.ctile];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int nsl = nb / BK;
  const int total = it.pcnt * nsl;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(sm));

  // producer cursor over the (pair, slice) sequence: no divisions in the loop
  int ip = 0, is = 0, istage = 0;
  const uint8_t *Ag = nullptr, *Bg = nullptr;
  const int64_t slice_bytes = (int64_t)BK * nb * ES;
  auto issue = [&](int g) {
    if (g < total) {
      if (is == 0) {
        const PairDesc pd = pairs[it.pbeg + ip];
        Ag = ws + pd.a_off + (int64_t)it.m0 * ES;
        Bg = ws + pd.b_off + (int64_t)it.n0 * ES;
      }
      const uint32_t stg = sbase + (uint32_t)(istage * STAGE);
#pragma unroll
      for (int u = 0; u < CPT; ++u) {
        const int c = tid + u * 256;
        if (c < BK * ACH) {
          const int k = c / ACH, ch = c - k * ACH;
          cp_async16(stg + (k * 128) * ES + ch * 16, Ag + (int64_t)k * nb * ES + ch * 16);
        } else {
          const int c2 = c - BK * ACH, k = c2 / BCH, ch = c2 - k * BCH;
          cp_async16(stg + (BK * 128 + k * BN) * ES + ch * 16, Bg + (int64_t)k * nb * ES + ch * 16);
        }
      }
      Ag += slice_bytes;
      Bg += slice_bytes;
      if (++is == nsl) { is = 0; ++ip; }
      if (++istage == ST) istage = 0;
    }
    cp_async_commit();
  };

#pragma unroll
  for (int g = 0; g < ST - 1; ++g) issue(g);

  constexpr int NJ = (sizeof(T) == 4) ? 4 : 4;  // float: 4 float2 pairs; double: 4 scalars
  using Acc = typename std::conditional<sizeof(T) == 4, float2, double>::type;
  Acc acc[8][NJ];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      if constexpr (sizeof(T) == 4) acc[i][j] = make_float2(0.f, 0.f);
      else acc[i][j] = 0.0;
    }

  int cstage = 0, cslice = 0, cpair = 0;
  for (int g = 0; g < total; ++g) {
    cp_async_wait<ST - 2>();
    __syncthreads();
    issue(g + ST - 1);
    const T* As = reinterpret_cast<const T*>(sm + cstage * STAGE);
    if (++cstage == ST) cstage = 0;
    const T* Bs = As + BK * 128;
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      T a[8];
      if constexpr (sizeof(T) == 4) {
        const float4 a0 = *reinterpret_cast<const float4*>(As + k * 128 + ty * 4);
        const float4 a1 = *reinterpret_cast<const float4*>(As + k * 128 + 64 + ty * 4);
        a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w; a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
        const float4 b0 = *reinterpret_cast<const float4*>(Bs + k * BN + tx * 4);
        const float4 b1 = *reinterpret_cast<const float4*>(Bs + k * BN + 64 + tx * 4);
        const float2 b[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                             make_float2(b1.z, b1.w)};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = ffma2_bcast(a[i], b[j], acc[i][j]);
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double2 x0 = *reinterpret_cast<const double2*>(As + k * 128 + h * 64 + ty * 4);
          const double2 x1 = *reinterpret_cast<const double2*>(As + k * 128 + h * 64 + ty * 4 + 2);
          a[h * 4 + 0] = x0.x; a[h * 4 + 1] = x0.y; a[h * 4 + 2] = x1.x; a[h * 4 + 3] = x1.y;
        }
        const double2 b0 = *reinterpret_cast<const double2*>(Bs + k * BN + tx * 2);
        const double2 b1 = *reinterpret_cast<const double2*>(Bs + k * BN + 32 + tx * 2);
        const double b[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(a[i], b[j], acc[i][j]);
      }
    }
    if (++cslice == nsl) {
      cslice = 0;
      const int pi = cpair++;
      // ---- fold (O9): W = fma_W(RN_W(alpha 2^fexp), RN_W(P), W) ----
      const PairDesc pd = pairs[it.pbeg + pi];
      const double f64 = ldexp_fast(alpha, pd.fexp);
      const float f32 = __double2float_rn(f64);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = it.m0 + (i >> 2) * 64 + ty * 4 + (i & 3);
#pragma unroll
        for (int j = 0; j < NJ; j += (sizeof(T) == 4 ? 1 : 2)) {
          // float: pair j -> cols (j>>1)*64 + tx*4 + (j&1)*2 + {0,1}
          // double: scalars j, j+1 -> cols (j>>1)*32 + tx*2 + {0,1}
          const int col = (sizeof(T) == 4) ? (j >> 1) * 64 + tx * 4 + (j & 1) * 2 : (j >> 1) * 32 + tx * 2;
          const int64_t e = (int64_t)r * nb + it.n0 + col;
          double v0, v1;
          if constexpr (sizeof(T) == 4) { v0 = acc[i][j].x; v1 = acc[i][j].y; }
          else { v0 = acc[i][j]; v1 = acc[i][j + 1]; }
          if (ct.code == 0) {
            double2* w = reinterpret_cast<double2*>(reinterpret_cast<double*>(ws + ct.w_off) + e);
            double2 v = *w;
            v.x = __fma_rn(f64, v0, v.x);
            v.y = __fma_rn(f64, v1, v.y);
            *w = v;
          } else {
            float2* w = reinterpret_cast<float2*>(reinterpret_cast<float*>(ws + ct.w_off) + e);
            float2 v = *w;
            v.x = __fmaf_rn(f32, __double2float_rn(v0), v.x);
            v.y = __fmaf_rn(f32, __double2float_rn(v1), v.y);
            *w = v;
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          if constexpr (sizeof(T) == 4) acc[i][j] = make_float2(0.f, 0.f);
          else acc[i][j] = 0.0;
        }
    }
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// Product-path FP64-class kernel on the FP64 tensor pipe (DMMA, legacy
// mma.sync.m16n8k16.row.col.f64 -- tcgen05 has no FP64 kind).
// 128x64 sub-tile, 8 warps (4 x 2), warp tile 32x32 = 2 m16 x 4 n8 MMA tiles,
// binary64 accumulation in registers, 2 CTAs per SM; MN-major payloads, BK = 16 k-rows per
// stage through a 4-stage cp.async ring into As[k][m] / Bs[k][n] rows whose
// pitch is 32 B mod 128 B, so the 16-byte fragment loads (per 8-lane phase: 4 k-rows x
// 2 consecutive 16-byte chunks) fall in eight distinct 16-byte bank groups.
// The accumulation order inside a DMMA is the hardware's: the parity bound is
// the all-FP64 1e-13 relative Frobenius.
// ---------------------------------------------------------------------------
template <int WN, int BK_ = 16, int ST_ = 4, int WGN_ = 2> struct DmmaCfg {
  static constexpr int BK = BK_, ST = ST_;          // k-rows per stage (multiple of 16), ring depth
  static constexpr int WGN = WGN_;                  // warp columns: 4 (m) x WGN (n) warps, warp tile 32 x WN
  static constexpr int BN = WGN * WN;
  static constexpr int THREADS = 4 * WGN * 32;
  static constexpr int AP = 128 + 4, BP = BN + 4;   // row pitches in doubles (= 32 B mod 128 B)
  static constexpr int SMEM = ST * BK * (AP + BP) * 8 + 2 * ST * 8;   // stages + full/empty mbarriers
  static constexpr int MINB = (THREADS == 256 && WN == 32) ? 2 : 1;
};
// product: 128 x 64 sub-tiles, 8 warps of 32 x 32, 2 CTAs/SM.  Measured alternatives
// (profiles/dmma_peak_r01.md): 32 x 64 warp tiles at 1 CTA/SM 9 % slower; 128 x 128
// sub-tiles with 16 warps (WGN = 4) at 1 CTA/SM 8 % slower (one barrier for all warps).
#ifndef GMP_DMMA_WGN   // experiment builds override the shape (-DGMP_DMMA_WGN=4 -DGMP_DMMA_ST=6)
#define GMP_DMMA_WGN 2
#endif
#ifndef GMP_DMMA_ST
#define GMP_DMMA_ST 4
#endif
constexpr int DMMA_WN = 32, DMMA_WGN = GMP_DMMA_WGN, DMMA_ST = GMP_DMMA_ST;
using DmmaProduct = DmmaCfg<DMMA_WN, 16, DMMA_ST, DMMA_WGN>;
constexpr int DMMA_BN = DmmaProduct::BN;

__device__ __forceinline__ void dmma16816(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int WN, int BK_ = 16, int ST_ = 4, int WGN_ = 2>
__global__ void __launch_bounds__(DmmaCfg<WN, BK_, ST_, WGN_>::THREADS, DmmaCfg<WN, BK_, ST_, WGN_>::MINB)
k_dmma(const WorkItem* __restrict__ items, const PairDesc* __restrict__ pairs,
       const CTileDesc* __restrict__ ctiles, uint8_t* __restrict__ ws, int nb, double alpha) {
  using Cfg = DmmaCfg<WN, BK_, ST_, WGN_>;
  constexpr int BK = Cfg::BK, ST = Cfg::ST, AP = Cfg::AP, BP = Cfg::BP, BN = Cfg::BN, NJ = WN / 8;
  constexpr int NT = Cfg::THREADS, WGN = Cfg::WGN;
  constexpr int ACH = 64, BCH = BN / 2;             // 16-byte chunks per k-row (A: 128 doubles, B: BN)
  constexpr int CHUNKS = BK * (ACH + BCH), CPT = CHUNKS / NT;
  constexpr int STAGE = BK * (AP + BP) * 8;
  static_assert(CHUNKS % NT == 0, "loader");
  extern __shared__ __align__(128) uint8_t sm[];
  const WorkItem it = expand_item(items, blockIdx.x, nb, BN);
  const CTileDesc ct = ctiles[it.ctile];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp / WGN) * 32, wn = (warp % WGN) * WN;
  const int nsl = nb / BK;
  const int total = it.pcnt * nsl;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
#ifndef GMP_DMMA_SYNC
  // stage hand-off through mbarriers instead of a CTA barrier per stage: full[s] completes
  // when every thread's cp.async of the fill landed (noinc arrivals), empty[s] when all 8
  // warps read the stage; a thread refills a buffer only after its previous fill was read,
  // and issues that refill after computing its current stage, so warps run decoupled
  // (no lock-step barrier bubble in the DMMA pipe) with ST - 2 stages of load lead
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + ST * STAGE);
  uint64_t* empty = full + ST;
  if (tid == 0)
    for (int s2 = 0; s2 < ST; ++s2) {
      mbar_init(&full[s2], NT);
      mbar_init(&empty[s2], NT / 32);
    }
  __syncthreads();
  uint32_t iphase = 0;
#endif

  // producer cursor over the (pair, slice) sequence (no divisions in the loop)
  int ip = 0, is = 0, istage = 0;
  const uint8_t *Ag = nullptr, *Bg = nullptr;
  const int64_t slice_bytes = (int64_t)BK * nb * 8;
  auto issue = [&](int gi) {
    if (gi < total) {
#ifndef GMP_DMMA_SYNC
      if (gi >= ST) mbar_wait(&empty[istage], iphase ^ 1);   // previous fill of this buffer read by all warps
#endif
      if (is == 0) {
        const PairDesc pd = pairs[it.pbeg + ip];
        Ag = ws + pd.a_off + (int64_t)it.m0 * 8;
        Bg = ws + pd.b_off + (int64_t)it.n0 * 8;
      }
      const uint32_t stg = sbase + (uint32_t)(istage * STAGE);
#pragma unroll
      for (int u = 0; u < CPT; ++u) {
        const int c = tid + u * NT;
        if (c < BK * ACH) {
          const int k = c / ACH, ch = c - k * ACH;
          cp_async16(stg + k * AP * 8 + ch * 16, Ag + (int64_t)k * nb * 8 + ch * 16);
        } else {
          const int c2 = c - BK * ACH, k = c2 / BCH, ch = c2 - k * BCH;
          cp_async16(stg + BK * AP * 8 + k * BP * 8 + ch * 16, Bg + (int64_t)k * nb * 8 + ch * 16);
        }
      }
#ifndef GMP_DMMA_SYNC
      cp_async_mbar_arrive_noinc(&full[istage]);
#endif
      Ag += slice_bytes;
      Bg += slice_bytes;
      if (++is == nsl) { is = 0; ++ip; }
      if (++istage == ST) {
        istage = 0;
#ifndef GMP_DMMA_SYNC
        iphase ^= 1;
#endif
      }
    }
#ifdef GMP_DMMA_SYNC
    cp_async_commit();
#endif
  };

#pragma unroll
  for (int gi = 0; gi < ST - 1; ++gi) issue(gi);

  double acc[2][NJ][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

  int cstage = 0, cslice = 0, cpair = 0;
#ifndef GMP_DMMA_SYNC
  uint32_t cphase = 0;
#endif
  for (int gi = 0; gi < total; ++gi) {
#ifdef GMP_DMMA_SYNC
    cp_async_wait<ST - 2>();
    __syncthreads();
    issue(gi + ST - 1);
#else
    mbar_wait(&full[cstage], cphase);
#endif
    const double* As = reinterpret_cast<const double*>(sm + cstage * STAGE);
    const double* Bs = As + BK * AP;
    // fragment permutation (bitwise neutral: every output is the same k-ordered DMMA dot
    // product): MMA rows g / g+8 of an m16 tile are sub-tile rows 2g / 2g+1, MMA column g of
    // n8 tiles 2J / 2J+1 is column 16J + 2g / 16J + 2g + 1 -- each fragment pair is one
    // 16-byte LDS.128 (half the shared-load instructions of per-element loads)
#pragma unroll
    for (int kk = 0; kk < BK; kk += 16) {
      double a[2][8];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 x = *reinterpret_cast<const double2*>(As + (kk + t + 4 * q) * AP + wm + i * 16 + 2 * g);
          a[i][2 * q] = x.x;
          a[i][2 * q + 1] = x.y;
        }
#pragma unroll
      for (int J = 0; J < NJ / 2; ++J) {
        double b0[4], b1[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const double2 x = *reinterpret_cast<const double2*>(Bs + (kk + t + 4 * r) * BP + wn + J * 16 + 2 * g);
          b0[r] = x.x;
          b1[r] = x.y;
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          dmma16816(acc[i][2 * J], a[i], b0);
          dmma16816(acc[i][2 * J + 1], a[i], b1);
        }
      }
    }
#ifdef GMP_DMMA_SYNC
    if (++cstage == ST) cstage = 0;
#else
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[cstage]);
    if (++cstage == ST) { cstage = 0; cphase ^= 1; }
    issue(gi + ST - 1);
#endif
    if (++cslice == nsl) {
      cslice = 0;
      // ---- fold (O9, R25): consecutive pairs with the same fold
      // factor (every FP64-class pair: eA = eB = 0) keep accumulating in the
      // DMMA registers; W is read and written once per run of equal factors ----
      const PairDesc pd = pairs[it.pbeg + cpair++];
      if (cpair < it.pcnt && pairs[it.pbeg + cpair].fexp == pd.fexp) continue;
      const double f64 = ldexp_fast(alpha, pd.fexp);
      const float f32 = __double2float_rn(f64);
      // lane (g, t), half hv: sub-tile row wm + 16i + 2g + hv, columns wn + 16J + 4t + 0..3
      // = {acc[i][2J][2hv], acc[i][2J+1][2hv], acc[i][2J][2hv+1], acc[i][2J+1][2hv+1]}
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int J = 0; J < NJ / 2; ++J)
#pragma unroll
          for (int hv = 0; hv < 2; ++hv) {
            const int r = it.m0 + wm + i * 16 + 2 * g + hv;
            const int64_t e = (int64_t)r * nb + it.n0 + wn + J * 16 + 4 * t;
            double* p0 = acc[i][2 * J];
            double* p1 = acc[i][2 * J + 1];
            const double x0 = p0[2 * hv], x1 = p1[2 * hv], x2 = p0[2 * hv + 1], x3 = p1[2 * hv + 1];
            if (ct.code == 0) {
              double2* w = reinterpret_cast<double2*>(reinterpret_cast<double*>(ws + ct.w_off) + e);
              double2 v = w[0], u = w[1];
              v.x = __fma_rn(f64, x0, v.x);
              v.y = __fma_rn(f64, x1, v.y);
              u.x = __fma_rn(f64, x2, u.x);
              u.y = __fma_rn(f64, x3, u.y);
              w[0] = v;
              w[1] = u;
            } else {
              float4* w = reinterpret_cast<float4*>(reinterpret_cast<float*>(ws + ct.w_off) + e);
              float4 v = *w;
              v.x = __fmaf_rn(f32, __double2float_rn(x0), v.x);
              v.y = __fmaf_rn(f32, __double2float_rn(x1), v.y);
              v.z = __fmaf_rn(f32, __double2float_rn(x2), v.z);
              v.w = __fmaf_rn(f32, __double2float_rn(x3), v.w);
              *w = v;
            }
            p0[2 * hv] = p1[2 * hv] = p0[2 * hv + 1] = p1[2 * hv + 1] = 0.0;
          }
    }
  }
  cp_async_wait<0>();
}

}  // namespace gmp
