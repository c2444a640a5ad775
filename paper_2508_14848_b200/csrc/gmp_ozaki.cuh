// gmp_ozaki.cuh -- OPT-IN: the FP64 class on the INT8 tensor pipe (Ozaki-style
// error-free slicing + tcgen05.mma kind::i8), enabled with GMP_FLAG_FP64_INT8.
// The product FP64 path stays k_dmma (binary64 arithmetic, as north_star and the
// paper's FP64 class specify); this path reaches binary64-level NORMWISE accuracy
// (tested to the 1e-13 FP64 parity bound) but not DGEMM's componentwise bound.
// Measured on B200 (profiles/ozaki_r01.md): all-FP64 cfg2 61 TFLOP/s vs 32.6
// for DMMA; mixed cfg2 execute 70 ms vs 94 ms.
//
// Slicing (k_slice64, receiver-side from the stored binary64 payload): for each
// K-major operand row r (A: tile row, B: tile column) with e_r the frexp
// exponent of max_k |x(r,k)| (all |x| 2^-e_r < 1), the normalised value
// a = x 2^-e_r is cut into NS = 7 signed 8-bit digits by exact truncation:
//     t = a 2^7 ; q_i = trunc(t) in [-127, 127] ; a = t - q_i   (all exact in binary64)
// so x = 2^e_r (sum_i q_i 2^-7i + rho), |rho| < 2^-49.
// Product: P(r,c) = 2^(e_r + f_c) sum_{d=2..8} 2^-7d S_d(r,c),
//          S_d = sum_{i+j=d} Q^A_i Q^B_j^T   (exact int32: <= 7 * 127^2 * nb < 2^31)
// -- 28 int8 MMAs per K block (terms i + j <= NS + 1), the dropped terms and rho
// are below 2^-48 of |A||B| row/column scales: binary64-level normwise accuracy
// (parity bound 1e-13).  The seven diagonal accumulators
// live in TMEM (7 x 64 int32 columns); the epilogue combines them in binary64,
// smallest first, applies the two power-of-two row/column scales and folds into
// the register-resident W row segment (O9).
#pragma once
#include "gmp_tc.cuh"

namespace gmp {

constexpr int OZ_NS = 7;              // int8 digits per element
constexpr int OZ_BN = 64;             // N of the MMA tile (= OZ2_BN)
constexpr int OZ_THREADS = 320;       // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue
constexpr int OZ_EPI_WARPS = 8;       // 2 per TMEM lane quarter, 32 columns each

// ---------------------------------------------------------------------------
// slicing kernel: one job = one tile (MN-major binary64 payload -> NS K-major
// int8 digit planes + nb row exponents).  One CTA per 64 output rows.
// ---------------------------------------------------------------------------
struct SliceJob {
  int64_t src_off;   // binary64 payload (MN-major: element (r, k) at k*nb + r)
  int64_t dst_off;   // NS planes of nb x nb int8, K-major (element (r, k) at r*nb + k)
  int64_t exp_off;   // nb int16 row exponents
};

__global__ void __launch_bounds__(256) k_slice64(const SliceJob* __restrict__ jobs, uint8_t* ws, int nb) {
  __shared__ double sm[64][65];
  __shared__ int sexp[64];
  __shared__ double smax[4][64];
  const SliceJob j = jobs[blockIdx.y];
  const int r0 = blockIdx.x * 64;
  const double* src = reinterpret_cast<const double*>(ws + j.src_off);
  int8_t* dst = reinterpret_cast<int8_t*>(ws + j.dst_off);
  const int t = threadIdx.x, rr = t & 63, kq = t >> 6;   // 64 rows x 4 k-lanes
  // pass 1: row maxima over k (coalesced: 64 consecutive r per k)
  double m = 0.0;
  for (int k = kq; k < nb; k += 4) m = fmax(m, fabs(src[(int64_t)k * nb + r0 + rr]));
  smax[kq][rr] = m;
  __syncthreads();
  if (t < 64) {
    const double mx = fmax(fmax(smax[0][t], smax[1][t]), fmax(smax[2][t], smax[3][t]));
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);            // mx in [2^(e-1), 2^e)
    sexp[t] = e;
    reinterpret_cast<int16_t*>(ws + j.exp_off)[r0 + t] = (int16_t)e;
  }
  __syncthreads();
  const int64_t plane = (int64_t)nb * nb;
  // pass 2: 64 x 64 blocks, transpose through shared memory, digits per element
  for (int k0 = 0; k0 < nb; k0 += 64) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int unit = t + u * 256;
      const int kk = unit >> 6, r = unit & 63;
      sm[kk][r] = src[(int64_t)(k0 + kk) * nb + r0 + r];
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      // thread -> (row r, 4 consecutive k)
      const int unit = t + u * 256;
      const int r = unit >> 4, kk0 = (unit & 15) * 4;
      int8_t q[OZ_NS][4];
#pragma unroll
      for (int e4 = 0; e4 < 4; ++e4) {
        double a = ldexp_fast(sm[kk0 + e4][r], -sexp[r]);
#pragma unroll
        for (int i = 0; i < OZ_NS; ++i) {
          const double tt = a * 128.0;        // exact
          const double qi = trunc(tt);        // |qi| <= 127
          q[i][e4] = (int8_t)qi;
          a = tt - qi;                        // exact
        }
      }
#pragma unroll
      for (int i = 0; i < OZ_NS; ++i) {
        const uint32_t w = (uint32_t)(uint8_t)q[i][0] | ((uint32_t)(uint8_t)q[i][1] << 8) |
                           ((uint32_t)(uint8_t)q[i][2] << 16) | ((uint32_t)(uint8_t)q[i][3] << 24);
        *reinterpret_cast<uint32_t*>(dst + i * plane + (int64_t)(r0 + r) * nb + k0 + kk0) = w;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// INT8 tcgen05 kernel.  M = 128, N = 64, 64-byte K blocks (SWIZZLE_64B), all
// seven diagonal accumulators live in TMEM (7 x 64 int32 columns), one pass
// over K per pair (each digit plane is read once).  The epilogue keeps its W row
// segment in registers for the whole item and folds each pair's binary64
// product into it (O9).
// ---------------------------------------------------------------------------
constexpr int OZ2_BN = 64, OZ2_BK = 64, OZ2_STAGES = 2;
// (sdesc_k_sw64: K-major SWIZZLE_64B descriptor, gmp_tc.cuh)
// D = S32 (c_format 2), A/B signed int8 (format 1), K-major, N = 64, M = 128
constexpr uint32_t oz_idesc() {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ2_BN >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);
}
__device__ __forceinline__ void tc_mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_ld8_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __noinline__ double pow2_scale_slow(double x, int e) { return ldexp(x, e); }
__device__ __forceinline__ double pow2_scale(double x, int e) {
  return (e > -1000 && e < 1000) ? x * __longlong_as_double((long long)(1023 + e) << 52) : pow2_scale_slow(x, e);
}

constexpr int OZ2_PLANE_A = TC_BM * OZ2_BK, OZ2_PLANE_B = OZ2_BN * OZ2_BK;   // 8 KB each
constexpr int OZ2_STAGE = OZ_NS * (OZ2_PLANE_A + OZ2_PLANE_B);                 // 112 KB
constexpr int oz_smem_bytes() { return OZ2_STAGES * OZ2_STAGE + 1024 + 256; }

__global__ void __launch_bounds__(OZ_THREADS, 1)
k_tc_fp64(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
          const WorkItem* __restrict__ items, int64_t nitems, const PairDesc* __restrict__ pairs,
          const CTileDesc* __restrict__ ctiles, uint8_t* __restrict__ ws, int nb, double alpha,
          int64_t exp_off) {
  constexpr uint32_t TMEM_COLS = 512;
  constexpr uint32_t IDESC = oz_idesc();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OZ2_STAGES * OZ2_STAGE);
  uint64_t* empty = full + OZ2_STAGES;
  uint64_t* tfull = empty + OZ2_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int16_t* __restrict__ exps = reinterpret_cast<const int16_t*>(ws + exp_off);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < OZ2_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, OZ_EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int kblocks = nb / OZ2_BK;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        const WorkItem w = expand_item(items, it, nb, OZ2_BN);
        for (int pi = 0; pi < w.pcnt; ++pi) {
          const PairDesc pd = pairs[w.pbeg + pi];
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * OZ2_STAGE;
            mbar_expect_tx(&full[stage], (uint32_t)OZ2_STAGE);
            for (int p = 0; p < OZ_NS; ++p) {
              tma_load_2d(sa + p * OZ2_PLANE_A, &tmA, kb * OZ2_BK, (pd.a_slot * OZ_NS + p) * nb + w.m0, &full[stage]);
              tma_load_2d(sa + OZ_NS * OZ2_PLANE_A + p * OZ2_PLANE_B, &tmB, kb * OZ2_BK,
                          (pd.b_slot * OZ_NS + p) * nb + w.n0, &full[stage]);
            }
            if (++stage == OZ2_STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        const WorkItem w = expand_item(items, it, nb, OZ2_BN);
        for (int pi = 0; pi < w.pcnt; ++pi) {
          mbar_wait(tempty, acc_phase ^ 1);
          tc_fence_after();
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + stage * OZ2_STAGE);
            for (int d = OZ_NS + 1; d >= 2; --d) {           // smallest diagonal first
              const uint32_t d_tmem = tmem_base + (uint32_t)((d - 2) * OZ2_BN);
              for (int i = 1; i < d; ++i) {
                const int j = d - i;
                const uint64_t ad = sdesc_k_sw64(sa + (i - 1) * OZ2_PLANE_A);
                const uint64_t bd = sdesc_k_sw64(sa + OZ_NS * OZ2_PLANE_A + (j - 1) * OZ2_PLANE_B);
#pragma unroll
                for (int k = 0; k < OZ2_BK / 32; ++k)
                  tc_mma_i8(d_tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), IDESC,
                            (kb == 0 && i == 1 && k == 0) ? 0u : 1u);
              }
            }
            tc_commit(&empty[stage]);
            if (++stage == OZ2_STAGES) { stage = 0; phase ^= 1; }
          }
          tc_commit(tfull);
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // epilogue: 8 warps; warp w reads TMEM lanes 32*(w%4)..+31 (tile rows) and
    // column group (w-2)/4 (32 columns, four 8-column chunks).  The thread's W row
    // segment (32 binary64 or binary32 values) stays in registers for the whole
    // item: one W read and one W write per item instead of two per pair.
    const int quarter = warp & 3, cg = (warp - 2) >> 2;
    const int rloc = quarter * 32 + lane;
    uint32_t acc_phase = 0;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
      const WorkItem w = expand_item(items, it, nb, OZ2_BN);
      const CTileDesc ct = ctiles[w.ctile];
      const int64_t rowoff = (int64_t)(w.m0 + rloc) * nb + w.n0 + cg * 32;
      const bool w64 = ct.code == 0;
      double accd[32];
      if (w64) {
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          const double2 x = reinterpret_cast<const double2*>(reinterpret_cast<const double*>(ws + ct.w_off) + rowoff)[v];
          accd[2 * v] = x.x; accd[2 * v + 1] = x.y;
        }
      } else {
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const float4 x = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(ws + ct.w_off) + rowoff)[v];
          accd[4 * v] = x.x; accd[4 * v + 1] = x.y; accd[4 * v + 2] = x.z; accd[4 * v + 3] = x.w;
        }
      }
      for (int pi = 0; pi < w.pcnt; ++pi) {
        const PairDesc pd = pairs[w.pbeg + pi];
        const double f64 = ldexp_fast(alpha, pd.fexp);
        const float f32 = __double2float_rn(f64);
        const int er = exps[(int64_t)pd.a_slot * nb + w.m0 + rloc];
        const int16_t* fcol = exps + (int64_t)pd.b_slot * nb + w.n0 + cg * 32;
        mbar_wait(tfull, acc_phase);
        tc_fence_after();
        const uint32_t tq = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(cg * 32);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {                   // four 8-column chunks
          double p[8];
#pragma unroll
          for (int v = 0; v < 8; ++v) p[v] = 0.0;
#pragma unroll 1
          for (int d = OZ_NS + 1; d >= 2; --d) {           // smallest diagonal first
            uint32_t r[8];
            tmem_ld8_nowait(tq + (uint32_t)((d - 2) * OZ2_BN + ch * 8), r);
            tmem_wait_ld();
            const double sc = __longlong_as_double((long long)(1023 - 7 * d) << 52);   // 2^-7d
#pragma unroll
            for (int v = 0; v < 8; ++v) p[v] = __fma_rn((double)(int32_t)r[v], sc, p[v]);
          }
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            // P = p 2^(e_r + f_c): exact power-of-two scaling
            const double P = pow2_scale(p[v], er + fcol[ch * 8 + v]);
            if (w64) accd[ch * 8 + v] = __fma_rn(f64, P, accd[ch * 8 + v]);
            else accd[ch * 8 + v] = (double)__fmaf_rn(f32, __double2float_rn(P), (float)accd[ch * 8 + v]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
        acc_phase ^= 1;
      }
      if (w64) {
#pragma unroll
        for (int v = 0; v < 16; ++v)
          reinterpret_cast<double2*>(reinterpret_cast<double*>(ws + ct.w_off) + rowoff)[v] =
              make_double2(accd[2 * v], accd[2 * v + 1]);
      } else {
#pragma unroll
        for (int v = 0; v < 8; ++v)
          reinterpret_cast<float4*>(reinterpret_cast<float*>(ws + ct.w_off) + rowoff)[v] =
              make_float4((float)accd[4 * v], (float)accd[4 * v + 1], (float)accd[4 * v + 2], (float)accd[4 * v + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
}

// host: TMA maps over the digit arena (rows = slot * NS * nb + plane * nb + r)
struct OzTables {
  CUtensorMap mapA, mapB;
  bool ready = false;
};

inline gmp_status_t oz_prepare(OzTables& t, uint8_t* ws, int64_t arena_off, int64_t slots, int nb) {
  t.ready = false;
  if (slots == 0) return GMP_OK;
  PFN_encodeTiled enc = get_encode_tiled();
  if (!enc) return GMP_ERR_CUDA;
  cuuint64_t dims[2] = {(cuuint64_t)nb, (cuuint64_t)(slots * OZ_NS * nb)};
  cuuint64_t strides[1] = {(cuuint64_t)nb};
  cuuint32_t estr[2] = {1, 1};
  cuuint32_t boxA[2] = {(cuuint32_t)OZ2_BK, (cuuint32_t)TC_BM};
  cuuint32_t boxB[2] = {(cuuint32_t)OZ2_BK, (cuuint32_t)OZ2_BN};
  if (enc(&t.mapA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, ws + arena_off, dims, strides, boxA, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return GMP_ERR_CUDA;
  if (enc(&t.mapB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, ws + arena_off, dims, strides, boxB, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return GMP_ERR_CUDA;
  t.ready = true;
  return GMP_OK;
}

inline cudaError_t oz_launch(OzTables& t, const WorkItem* it, int64_t n, const PairDesc* pd, const CTileDesc* ct,
                             uint8_t* ws, int nb, double alpha, int64_t exp_off, cudaStream_t s) {
  if (!t.ready) return cudaErrorNotReady;
  {
    const cudaError_t e = ensure_max_smem(k_tc_fp64, oz_smem_bytes());
    if (e != cudaSuccess) return e;
  }
  // one CTA per (item, sub-tile), scheduled in flat order: the CTAs of one C
  // tile run together and walk its pair list in step (L2 reuse of the planes)
  const int grid = (int)n;
  k_tc_fp64<<<grid, OZ_THREADS, oz_smem_bytes(), s>>>(t.mapA, t.mapB, it, n, pd, ct, ws, nb, alpha, exp_off);
  return cudaGetLastError();
}

}  // namespace gmp
