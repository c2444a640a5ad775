// gmp_tc.cuh -- S6 grouped tile-GEMM for the FP16 / BF16 / E4M3 precision
// classes on the 5th-generation tensor cores.
//
// Persistent, warp-specialised kernel, one CTA per SM:
//   warp 0      TMA producer: 128x128B (A) and BNx128B (B) boxes, SWIZZLE_128B,
//               into a STAGES-deep shared-memory ring (mbarrier full/empty).
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (kind::f16 for FP16/BF16, kind::f8f6f4 for E4M3; M=128, N=BN,
//               K=32 bytes per instruction), FP32 accumulation in TMEM,
//               double-buffered accumulator (2 x BN columns) so the epilogue of
//               pair p overlaps the MMAs of pair p+1.
//   warps 2..9  epilogue: tcgen05.ld 32x32b, then the fold of DESIGN.md O9
//               W = fma_W(RN_W(alpha 2^-(eA+eB)), P, W); binary32 W rows stay in
//               registers for the whole item (one W read/write per item).
// A work item is a 128 x BN sub-tile of one C tile with its ordered pair list
// (l of the SUMMA step whose pair class is this launch's class); both operands
// are K-major payloads in the class arena (A row-major, B transposed), one
// 2-D TMA descriptor per arena: rows = slot*nb + r, cols = k.
// Tensor-core accumulation order differs from the oracle's sequential sum: the
// parity bound is 4 u32 sqrt(K); maps and bytes stay exact.
#pragma once
#include <cuda.h>

#include <vector>

#include "gmp_common.cuh"
#include "gmp_simt.cuh"

namespace gmp {

constexpr bool kTcAvailable = true;
constexpr int TC_BM = 128;
constexpr int TC_STAGES = 4;
constexpr int TC_THREADS = 320;   // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue
constexpr int TC_EPI_WARPS = 8;

__host__ __device__ constexpr int tc_bn(int nb) { return (nb % 256 == 0) ? 256 : 128; }

// ---------------------------------------------------------------------------
// PTX wrappers (sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// plain bulk copy global -> shared (16-byte aligned, size a multiple of 16)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}
// K-major operand, SWIZZLE_128B canonical layout: 8-row x 128-byte atoms,
// SBO = 1024 B between 8-row groups, LBO unused (1), version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc_k_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// K-major SWIZZLE_64B canonical layout: 8-row x 64-byte atoms, SBO = 512 B.
__device__ __forceinline__ uint64_t sdesc_k_sw64(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
// instruction descriptor: D = F32, A/B format, K-major both, N>>3, M>>4
template <int C, int BN>
__host__ __device__ constexpr uint32_t tc_idesc() {
  constexpr uint32_t ab = (C == 3 || C == 5) ? 1u : 0u;   // kind::f16: F16 0, BF16 1; kind::f8f6f4: E4M3 0, E5M2 1
  return (1u << 4) | (ab << 7) | (ab << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);
}
// MXFP4 (kind::mxf4.block_scale, E2M1 x E2M1, E8M0 scales per 32 K): block-scaled
// instruction descriptor -- a/b format E2M1 (1) at bits 7/10, N>>3 at 17, scale format
// E8M0 (bit 23), M>>4 at 24; the scale-factor ids (byte of the 32-bit TMEM column) are
// OR-ed in per instruction at bits 4-5 (B) and 29-30 (A)
template <int BN>
__host__ __device__ constexpr uint32_t mx_idesc() {
  return (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | (1u << 23) | ((uint32_t)(TC_BM >> 4) << 24);
}
__device__ __forceinline__ uint32_t mx_sf_id(uint32_t id) { return (id << 4) | (id << 29); }
__device__ __forceinline__ void tc_mma_mx(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate, uint32_t tsfa, uint32_t tsfb) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(tsfa), "r"(tsfb));
}
// scale factors smem -> TMEM: one 512-byte chunk (32 x 16 B, no swizzle, 8-row core
// matrices 128 B apart) into 4 TMEM columns, broadcast to the 4 lane quarters
__device__ __forceinline__ uint64_t sdesc_sf(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(512 >> 4) << 16) | ((uint64_t)(128 >> 4) << 32) |
         ((uint64_t)1 << 46);
}
__device__ __forceinline__ void tc_cp_sf(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sdesc));
}
template <int C>
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  if constexpr (C == 4 || C == 5) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  }
}
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Work distribution of a persistent launch.  Static (default): CTA b takes items b, b + grid, ...
// Dynamic (GMP_FLAG_DYN_SCHED): the TMA producer takes the next item from a global
// atomic counter when it is about to load it, so the CTAs stay on a narrow window of
// consecutive items (sub-tiles of ~1 C tile sharing the same operand tiles in L2) instead
// of drifting apart when items differ in length; it hands each index to the MMA warp and
// the epilogue warps through a small shared-memory ring (mbarrier full / empty).
constexpr int TC_RING = 4;
struct TcSched {
  int* counter = nullptr;          // device counter (zeroed before the launch); null: static
  int64_t* ring = nullptr;         // [TC_RING] item indices (shared memory)
  uint64_t* rfull = nullptr;       // [TC_RING]
  uint64_t* rempty = nullptr;      // [TC_RING], MMA warp + epilogue warps arrive
  int64_t nitems = 0;
  // producer: k-th item of this CTA (>= nitems: done)
  __device__ __forceinline__ int64_t produce(int k) const {
    int64_t it;
    if (counter) it = (int64_t)atomicAdd(counter, 1);
    else it = (int64_t)blockIdx.x + (int64_t)k * gridDim.x;
    if (ring) {
      const int r = k % TC_RING;
      mbar_wait(&rempty[r], ((k / TC_RING) & 1) ^ 1);
      ring[r] = it;
      mbar_arrive(&rfull[r]);
    }
    return it;
  }
  // consumers: k-th item; whole_warp = all 32 lanes call it (the epilogue warps: lane 0
  // releases the slot after the warp has read it), else a single thread (the MMA issuer)
  __device__ __forceinline__ int64_t consume(int k, int lane, bool whole_warp) const {
    if (!ring) return (int64_t)blockIdx.x + (int64_t)k * gridDim.x;
    const int r = k % TC_RING;
    mbar_wait(&rfull[r], (k / TC_RING) & 1);
    const int64_t it = *(volatile int64_t*)&ring[r];
    if (whole_warp) __syncwarp();
    if (lane == 0) mbar_arrive(&rempty[r]);
    return it;
  }
};

// Epilogue warps 2..9 of the 1-SM tcgen05 kernel (k_tc_class): per
// pair, read the FP32 product from TMEM and fold it into W (O9).
template <int BN>
__device__ __forceinline__ void tc_epilogue(const WorkItem* __restrict__ items, int64_t nitems,
                                            const PairDesc* __restrict__ pairs, const CTileDesc* __restrict__ ctiles,
                                            uint8_t* __restrict__ ws, int nb, double alpha, double beta,
                                            uint32_t tmem_base, uint64_t* tfull, uint64_t* tempty, int warp,
                                            int lane, const int32_t* __restrict__ order = nullptr,
                                            const TcSched sc = TcSched(),
                                            unsigned long long* __restrict__ maxbits = nullptr) {
  // epilogue: 8 warps; warp w reads TMEM lanes 32*(w%4)..+31 (= tile rows) and
  // half (w-2)/4 of the BN columns.  binary32 W: the W row segment lives in
  // registers for the whole item (one read + one write per item instead of
  // per pair); binary64 W: read-modify-write per pair.
  constexpr int HC = BN / 2;                  // columns per epilogue thread
  const int quarter = warp & 3, half = (warp - 2) >> 2;
  const int rloc = quarter * 32 + lane;
  int acc = 0;
  uint32_t acc_phase = 0;
  for (int k = 0;; ++k) {
    const int64_t it = sc.consume(k, lane, true);
    if (it >= nitems) break;
    const WorkItem w = expand_item(items, it, nb, BN, order);
    const CTileDesc ct = ctiles[w.ctile];
    const int64_t rowoff = (int64_t)(w.m0 + rloc) * nb + w.n0 + half * HC;
    if (ct.code != 0) {
      float* wrow = reinterpret_cast<float*>(ws + ct.w_off) + rowoff;
      float accr[HC];
      if (w.pad & 1) {   // first tile-GEMM launch of this C tile: W0 from C_in (O9)
#pragma unroll
        for (int v = 0; v < HC; ++v) accr[v] = w0_f32(ct, ws, rowoff + v, beta);
      } else {
#pragma unroll
        for (int v = 0; v < HC / 4; ++v) {
          float4 x = reinterpret_cast<const float4*>(wrow)[v];
          accr[4 * v] = x.x; accr[4 * v + 1] = x.y; accr[4 * v + 2] = x.z; accr[4 * v + 3] = x.w;
        }
      }
      for (int pi = 0; pi < w.pcnt; ++pi) {
        const PairDesc pd = pairs[w.pbeg + pi];
        const float f32 = __double2float_rn(ldexp_fast(alpha, pd.fexp));
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN + half * HC);
#pragma unroll
        for (int ch = 0; ch < HC / 16; ++ch) {
#ifdef GMP_EXP_NOEPI   // power experiments only (exp/ builds): no TMEM read, no fold
          if (f32 == 12345.0f) accr[ch] += 1.0f;
#else
          uint32_t r[16];
          tmem_ld16_nowait(tbase + ch * 16, r);
          tmem_wait_ld();
#pragma unroll
          for (int v = 0; v < 16; ++v) accr[ch * 16 + v] = __fmaf_rn(f32, __uint_as_float(r[v]), accr[ch * 16 + v]);
#endif
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
#pragma unroll
      for (int v = 0; v < HC / 4; ++v)
        reinterpret_cast<float4*>(wrow)[v] = make_float4(accr[4 * v], accr[4 * v + 1], accr[4 * v + 2], accr[4 * v + 3]);
      if (w.pad & 2) {   // last launch of this C tile: max|W| for the finalize scale (S7)
        float m = 0.f;
#pragma unroll
        for (int v = 0; v < HC; ++v) m = fmaxf(m, fabsf(accr[v]));
        for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
        if (lane == 0 && m > 0.f) atomicMax(maxbits + w.ctile, (unsigned long long)__double_as_longlong((double)m));
      }
    } else if constexpr (HC <= 64) {
      // binary64 W, BN <= 128: the W row segment lives in registers for the item
      double* wrow = reinterpret_cast<double*>(ws + ct.w_off) + rowoff;
      double accd[HC];
      if (w.pad & 1) {   // first tile-GEMM launch of this C tile: W0 from C_in (O9)
#pragma unroll
        for (int v = 0; v < HC; ++v) accd[v] = w0_f64(ct, ws, rowoff + v, beta);
      } else {
#pragma unroll
        for (int v = 0; v < HC / 2; ++v) {
          const double2 x = reinterpret_cast<const double2*>(wrow)[v];
          accd[2 * v] = x.x; accd[2 * v + 1] = x.y;
        }
      }
      for (int pi = 0; pi < w.pcnt; ++pi) {
        const PairDesc pd = pairs[w.pbeg + pi];
        const double f64 = ldexp_fast(alpha, pd.fexp);
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN + half * HC);
#pragma unroll
        for (int ch = 0; ch < HC / 16; ++ch) {
          uint32_t r[16];
          tmem_ld16_nowait(tbase + ch * 16, r);
          tmem_wait_ld();
#pragma unroll
          for (int v = 0; v < 16; ++v)
            accd[ch * 16 + v] = __fma_rn(f64, (double)__uint_as_float(r[v]), accd[ch * 16 + v]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
#pragma unroll
      for (int v = 0; v < HC / 2; ++v)
        reinterpret_cast<double2*>(wrow)[v] = make_double2(accd[2 * v], accd[2 * v + 1]);
    } else {
      // binary64 W with BN = 256: read-modify-write per pair (the host prefers
      // BN = 128 for launches that hold binary64 accumulators)
      double* wrow = reinterpret_cast<double*>(ws + ct.w_off) + rowoff;
      if (w.pad & 1) {   // first tile-GEMM launch of this C tile: W0 from C_in (O9)
#pragma unroll 1
        for (int v = 0; v < HC; ++v) wrow[v] = w0_f64(ct, ws, rowoff + v, beta);
      }
      for (int pi = 0; pi < w.pcnt; ++pi) {
        const PairDesc pd = pairs[w.pbeg + pi];
        const double f64 = ldexp_fast(alpha, pd.fexp);
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN + half * HC);
#pragma unroll 1
        for (int ch = 0; ch < HC / 16; ++ch) {
          uint32_t r[16];
          tmem_ld16_nowait(tbase + ch * 16, r);
          tmem_wait_ld();
          double2* wp = reinterpret_cast<double2*>(wrow + ch * 16);
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            double2 x = wp[v];
            x.x = __fma_rn(f64, (double)__uint_as_float(r[2 * v]), x.x);
            x.y = __fma_rn(f64, (double)__uint_as_float(r[2 * v + 1]), x.y);
            wp[v] = x;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
// C = 2, 3, 4, 5: FP16 / BF16 / E4M3 / E5M2 classes, NP = 1 operand part.
// C = TC_SPLIT: the FP32 class on the tensor pipe ("BF16x9"): each FP32 operand tile is
// split exactly into three BF16 parts x = x0 + x1 + x2 (k_split, receiver-side
// from the stored FP32 payload), NP = 3, and all nine part products -- each
// exact in the FP32 accumulator's inputs -- are accumulated per K block,
// smallest terms first; binary32 inputs, exact products, binary32 accumulation.
constexpr int TC_SPLIT = 9;    // template id of the FP32-class kernel, all nine part products (BF16x9, exact)
constexpr int TC_SPLIT6 = 10;  // the six part products x_i y_j with i + j <= 2 (BF16x6, the default; R32)
// BF16x6 at BN = 256 (binary32 W, nb % 256 == 0): 64-byte K blocks (SWIZZLE_64B), 3 stages of
// 3 x (8 + 16) KB -- 175 instead of 131 flop per staged byte, for a kernel the L2 -> SMEM feed limits
constexpr int TC_SPLIT6W = 11;
template <int C> constexpr bool tc_is_split() { return C == TC_SPLIT || C == TC_SPLIT6 || C == TC_SPLIT6W; }
template <int C> constexpr int tc_np() { return tc_is_split<C>() ? 3 : 1; }
template <int C> constexpr int tc_t0() { return (C == TC_SPLIT6 || C == TC_SPLIT6W) ? 3 : 0; }   // smallest first
template <int C> constexpr int tc_kbytes() { return C == TC_SPLIT6W ? 64 : 128; }   // bytes of K per stage row
// MXFP4: 4 stages of 34 KB (6 measured 13 % slower in the cfg4-mx4 step)
#ifndef GMP_MX_STAGES
#define GMP_MX_STAGES 4
#endif
template <int C> constexpr int tc_stages() {
  return C == TC_SPLIT6W ? 3 : tc_is_split<C>() ? 2 : C == GMP_MX ? GMP_MX_STAGES : TC_STAGES;
}
template <int C> constexpr int tc_map_index() { return tc_is_split<C>() ? GMP_AR_SPLIT : C; }

template <int C, int BN>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_tc_class(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
           const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2,
           const WorkItem* __restrict__ items, int64_t nitems, const PairDesc* __restrict__ pairs,
           const CTileDesc* __restrict__ ctiles, uint8_t* __restrict__ ws, int nb, double alpha, double beta,
           const int32_t* __restrict__ order, int* __restrict__ sched_counter,
           unsigned long long* __restrict__ maxbits) {
  constexpr int NP = tc_np<C>(), ST = tc_stages<C>();
  constexpr bool MX = (C == GMP_MX);       // MXFP4: 4-bit elements + scale-factor chunks per stage
  static_assert(!MX || BN == 128, "MXFP4 runs at BN = 128 (TMEM: 2 x 128 accumulator + scale columns)");
  constexpr int ESZ = (C == 4 || C == 5) ? 1 : 2;
  constexpr int KB = tc_kbytes<C>();       // bytes of K per staged row: 128 (SWIZZLE_128B) or 64 (SWIZZLE_64B)
  constexpr int BK = MX ? 256 : KB / ESZ;  // elements per K block
  constexpr int NMMA = KB / 32;            // 32-byte K per tcgen05.mma
  constexpr int A_BYTES = TC_BM * KB, B_BYTES = BN * KB;
  constexpr int SF_BYTES = MX ? 1024 : 0;  // per operand: 128 rows x 8 scales = 2 chunks of 512 B
  constexpr int STAGE_BYTES = NP * (A_BYTES + B_BYTES) + 2 * SF_BYTES;
  constexpr uint32_t TMEM_COLS = MX ? 512 : 2 * BN;
  constexpr uint32_t IDESC = MX ? mx_idesc<BN>() : tc_idesc<(tc_is_split<C>() || C == GMP_MX ? 3 : C), BN>();

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * STAGE_BYTES);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint64_t* rfull = tempty + 2;
  uint64_t* rempty = rfull + TC_RING;
  int64_t* ring = reinterpret_cast<int64_t*>(rempty + TC_RING);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + TC_RING);
  TcSched sc;
  sc.nitems = nitems;
  if (sched_counter) { sc.counter = sched_counter; sc.ring = ring; sc.rfull = rfull; sc.rempty = rempty; }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], TC_EPI_WARPS); }
    for (int s = 0; s < TC_RING; ++s) { mbar_init(&rfull[s], 1); mbar_init(&rempty[s], 1 + TC_EPI_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    if (C == 3) {   // merged 16-bit launch: FP16 pairs read the FP16 arena (tmA2 / tmB2)
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA2) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB2) : "memory");
    }
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
  const int kblocks = nb / BK;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kk = 0;; ++kk) {
        const int64_t it = sc.produce(kk);
        if (it >= nitems) break;
        const WorkItem w = expand_item(items, it, nb, BN, order);
        for (int pi = 0; pi < w.pcnt; ++pi) {
          const PairDesc pd = pairs[w.pbeg + pi];
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * STAGE_BYTES;
            mbar_expect_tx(&full[stage], STAGE_BYTES);
            if constexpr (MX) {
              // elements: 3-D maps (byte in row, row, slot); scales: the two 512-byte chunks
              // of this 128-row group and K block, contiguous in the slot (mx_sf_offset)
              tma_load_3d(sa, &tmA, kb * 128, w.m0, pd.a_slot, &full[stage]);
              tma_load_3d(sa + A_BYTES, &tmB, kb * 128, w.n0, pd.b_slot, &full[stage]);
              const int64_t sfa = mx_sf_offset(nb, w.m0, kb * 8), sfb = mx_sf_offset(nb, w.n0, kb * 8);
              bulk_load(sa + A_BYTES + B_BYTES, ws + pd.a_off + sfa, SF_BYTES, &full[stage]);
              bulk_load(sa + A_BYTES + B_BYTES + SF_BYTES, ws + pd.b_off + sfb, SF_BYTES, &full[stage]);
            } else {
              // C = 3 launches may carry FP16 pairs too (BF16 pairs first, then FP16, per item:
              // the fold order of DESIGN.md O9); same element size, the FP16 arena's maps
              const bool f16 = (C == 3) && pd.cls == 2;
              const CUtensorMap* ma = f16 ? &tmA2 : &tmA;
              const CUtensorMap* mb = f16 ? &tmB2 : &tmB;
#pragma unroll
              for (int p = 0; p < NP; ++p) {
                tma_load_2d(sa + p * A_BYTES, ma, kb * BK, (pd.a_slot * NP + p) * nb + w.m0, &full[stage]);
                tma_load_2d(sa + NP * A_BYTES + p * B_BYTES, mb, kb * BK, (pd.b_slot * NP + p) * nb + w.n0,
                            &full[stage]);
              }
            }
            if (++stage == ST) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int kk = 0;; ++kk) {
        const int64_t it = sc.consume(kk, 0, false);
        if (it >= nitems) break;
        const WorkItem w = expand_item(items, it, nb, BN, order);
        for (int pi = 0; pi < w.pcnt; ++pi) {
          const uint32_t idesc = (C == 3 && pairs[w.pbeg + pi].cls == 2) ? tc_idesc<2, BN>() : IDESC;
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
            if constexpr (MX) {
              // scales of this K block -> TMEM (in issue order with the MMAs: the previous
              // block's MMAs have read the same columns before these copies land), then
              // 4 MMAs of K = 64; MMA k reads chunk k/2 at byte 2 (k%2) of each column
              const uint32_t tsfa = tmem_base + 2 * BN, tsfb = tsfa + 8;
              const uint32_t ssf = sa + A_BYTES + B_BYTES;
#pragma unroll
              for (int c = 0; c < 2; ++c) {
                tc_cp_sf(tsfa + 4 * c, sdesc_sf(ssf + 512 * c));
                tc_cp_sf(tsfb + 4 * c, sdesc_sf(ssf + SF_BYTES + 512 * c));
              }
              const uint64_t ad = sdesc_k_sw128(sa), bd = sdesc_k_sw128(sa + A_BYTES);
#pragma unroll
              for (int k = 0; k < NMMA; ++k)
                tc_mma_mx(d_tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), IDESC | mx_sf_id(2 * (k & 1)),
                          (kb | k) != 0, tsfa + 4 * (k >> 1), tsfb + 4 * (k >> 1));
            } else {
            constexpr int t0 = tc_t0<C>();
#pragma unroll
            for (int t = t0; t < NP * NP; ++t) {
              // terms (i, j) by decreasing i + j: the smallest part products first
              constexpr int TI[9] = {2, 2, 1, 2, 1, 0, 1, 0, 0}, TJ[9] = {2, 1, 2, 0, 1, 2, 0, 1, 0};
              const int ti = (NP == 1) ? 0 : TI[t], tj = (NP == 1) ? 0 : TJ[t];
              const uint64_t ad = (KB == 64) ? sdesc_k_sw64(sa + ti * A_BYTES) : sdesc_k_sw128(sa + ti * A_BYTES);
              const uint64_t bd = (KB == 64) ? sdesc_k_sw64(sa + NP * A_BYTES + tj * B_BYTES)
                                             : sdesc_k_sw128(sa + NP * A_BYTES + tj * B_BYTES);
#pragma unroll
              for (int k = 0; k < NMMA; ++k)
                tc_mma<C>(d_tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc, (kb | (t - t0) | k) != 0);
            }
            }
            tc_commit(&empty[stage]);
            if (++stage == ST) { stage = 0; phase ^= 1; }
          }
          tc_commit(&tfull[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
    }
  } else {
    tc_epilogue<BN>(items, nitems, pairs, ctiles, ws, nb, alpha, beta, tmem_base, tfull, tempty, warp, lane, order,
                    sc, maxbits);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
}

template <int C, int BN>
constexpr int tc_smem_bytes() {
  return tc_stages<C>() * (tc_np<C>() * (TC_BM + BN) * tc_kbytes<C>() + (C == GMP_MX ? 2048 : 0)) + 1024 /*align*/ +
         512 /*barriers, scheduler ring*/;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct TcTables {
  int* counters = nullptr;   // device counters of the dynamic scheduler (one per launch of an execute)
  int ncounters = 0;
  CUtensorMap mapA[GMP_NARENA], mapB[GMP_NARENA];   // classes 2..5 and GMP_AR_SPLIT (FP32 BF16 parts);
                                                    // B box rows = tc_bn(nb)
  CUtensorMap mapB128[GMP_NARENA];                  // B box of 128 rows (launches with binary64 W)
  CUtensorMap splitA64, splitB64;                   // split arena, 64-byte x {128, 256}-row boxes (SW64)
  bool ready[GMP_NARENA] = {};
  int nb = 0;
  unsigned long long* maxbits = nullptr;   // per-C-tile max|W| bits of the current execute (items with pad bit 1)
};

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline PFN_encodeTiled get_encode_tiled() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}


// arena_off / arena_slots have GMP_NARENA entries; arena GMP_AR_SPLIT holds FP32
// splits (3 BF16 parts per slot)
inline gmp_status_t tc_prepare(TcTables& t, uint8_t* ws, const int64_t* arena_off, const int64_t* arena_slots, int nb) {
  t.nb = nb;
  for (int c = 2; c <= GMP_AR_SPLIT; ++c) {
    t.ready[c] = false;
    if (arena_slots[c] == 0) continue;
    PFN_encodeTiled enc = get_encode_tiled();
    if (!enc) return GMP_ERR_CUDA;
    const bool split = c == GMP_AR_SPLIT;
    if (c == GMP_MX) {
      // MXFP4 slots hold nb rows of nb/2 element bytes, then the scale bytes: 3-D map
      // (byte in row, row, slot), 128-byte x 128-row boxes
      cuuint64_t dims[3] = {(cuuint64_t)(nb / 2), (cuuint64_t)nb, (cuuint64_t)arena_slots[c]};
      cuuint64_t strides[2] = {(cuuint64_t)(nb / 2), (cuuint64_t)mx_slot_bytes(nb)};
      cuuint32_t box[3] = {128u, 128u, 1u};
      cuuint32_t estr[3] = {1, 1, 1};
      void* base = ws + arena_off[c];
      if (enc(&t.mapA[c], CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, base, dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return GMP_ERR_CUDA;
      t.mapB[c] = t.mapA[c];
      t.mapB128[c] = t.mapA[c];
      t.ready[c] = true;
      continue;
    }
    const int esz = (c == 4 || c == 5) ? 1 : 2;
    const int64_t rows = arena_slots[c] * (split ? 3 : 1) * nb;
    cuuint64_t dims[2] = {(cuuint64_t)nb, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)nb * esz};
    cuuint32_t estr[2] = {1, 1};
    const CUtensorMapDataType dt = (esz == 1) ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16;
    const int bn = split ? 128 : tc_bn(nb);
    cuuint32_t boxA[2] = {(cuuint32_t)(128 / esz), (cuuint32_t)TC_BM};
    cuuint32_t boxB[2] = {(cuuint32_t)(128 / esz), (cuuint32_t)bn};
    void* base = ws + arena_off[c];
    if (enc(&t.mapA[c], dt, 2, base, dims, strides, boxA, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return GMP_ERR_CUDA;
    if (enc(&t.mapB[c], dt, 2, base, dims, strides, boxB, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return GMP_ERR_CUDA;
    cuuint32_t boxB128[2] = {(cuuint32_t)(128 / esz), 128u};
    if (enc(&t.mapB128[c], dt, 2, base, dims, strides, boxB128, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return GMP_ERR_CUDA;
    if (split && nb % 256 == 0) {   // BF16x6 at BN = 256: 64-byte K boxes, SWIZZLE_64B
      cuuint32_t a64[2] = {32u, (cuuint32_t)TC_BM}, b64[2] = {32u, 256u};
      if (enc(&t.splitA64, dt, 2, base, dims, strides, a64, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
          enc(&t.splitB64, dt, 2, base, dims, strides, b64, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return GMP_ERR_CUDA;
    }
    t.ready[c] = true;
  }
  return GMP_OK;
}

template <int C, int BN>
inline gmp_status_t tc_launch_t(TcTables& t, const WorkItem* it, int64_t n, const PairDesc* pd, const CTileDesc* ct,
                                uint8_t* ws, int nb, double alpha, double beta, const int32_t* order, cudaStream_t s,
                                int* counter) {
  constexpr int smem = tc_smem_bytes<C, BN>();
  if (ensure_max_smem(k_tc_class<C, BN>, smem) != cudaSuccess) return GMP_ERR_CUDA;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(n, sms);
  // a merged 16-bit launch (C = 3) may hold FP16 pairs only: then the BF16 arena is empty
  const int mi = (C == 3 && !t.ready[3]) ? 2 : tc_map_index<C>();
  const int m2 = (C == 3 && t.ready[2]) ? 2 : mi;   // FP16 arena for merged 16-bit launches
  const CUtensorMap& ma = (C == TC_SPLIT6W) ? t.splitA64 : t.mapA[mi];
  const CUtensorMap& mb = (C == TC_SPLIT6W) ? t.splitB64 : (BN == 128 ? t.mapB128[mi] : t.mapB[mi]);
  k_tc_class<C, BN><<<grid, TC_THREADS, smem, s>>>(ma, mb, t.mapA[m2],
                                                    BN == 128 ? t.mapB128[m2] : t.mapB[m2], it, n, pd, ct,
                                                    ws, nb, alpha, beta, order, counter, t.maxbits);
  return cudaGetLastError() == cudaSuccess ? GMP_OK : GMP_ERR_CUDA;
}

// cls: 2..5 for the 16/8-bit classes, TC_SPLIT for the FP32 class on the tensor
// pipe; bn: 256 or 128 (128 when the launch folds into binary64 W)
// counter: device int of the dynamic scheduler, zeroed here on the stream; null = static
inline gmp_status_t tc_launch(TcTables& t, int cls, int bn, const WorkItem* it, int64_t n, const PairDesc* pd,
                              const CTileDesc* ct, uint8_t* ws, int nb, double alpha, double beta, const int32_t* order,
                              cudaStream_t s, int* counter = nullptr) {
  const bool split = cls == TC_SPLIT || cls == TC_SPLIT6 || cls == TC_SPLIT6W;
  const int mi = split ? GMP_AR_SPLIT : cls;
  const bool ok = t.ready[mi] || (cls == 3 && t.ready[2]);   // merged 16-bit launch with FP16 pairs only
  if (!((cls >= 2 && cls <= GMP_MX) || split) || !ok) return GMP_ERR_STATE;
  if (cls == TC_SPLIT6W && (bn != 256 || t.nb % 256)) return GMP_ERR_STATE;
  if (cls == GMP_MX && bn != 128) return GMP_ERR_STATE;
  if (counter && cudaMemsetAsync(counter, 0, sizeof(int), s) != cudaSuccess) return GMP_ERR_CUDA;
  const bool wide = bn == 256;
#define GMP_TCL(C_, BN_) tc_launch_t<C_, BN_>(t, it, n, pd, ct, ws, nb, alpha, beta, order, s, counter)
  switch (cls) {
    case GMP_MX: return GMP_TCL(GMP_MX, 128);
    case 2: return wide ? GMP_TCL(2, 256) : GMP_TCL(2, 128);
    case 3: return wide ? GMP_TCL(3, 256) : GMP_TCL(3, 128);
    case 4: return wide ? GMP_TCL(4, 256) : GMP_TCL(4, 128);
    case 5: return wide ? GMP_TCL(5, 256) : GMP_TCL(5, 128);
    case TC_SPLIT6: return GMP_TCL(TC_SPLIT6, 128);
    case TC_SPLIT6W: return GMP_TCL(TC_SPLIT6W, 256);
    default: return GMP_TCL(TC_SPLIT, 128);
  }
#undef GMP_TCL
}

inline void tc_release(TcTables&) {}

}  // namespace gmp
