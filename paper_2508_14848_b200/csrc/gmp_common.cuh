// gmp_common.cuh -- device-side number formats and exact helpers for the
// tile-centric mixed-precision GEMM (arxiv 2508.14848).  sm_100a only.
//
// Class codes: 0 FP64, 1 FP32, 2 FP16, 3 BF16, 4 E4M3 (OCP FN),
// 5 E5M2 (OCP), 6 MXFP4 (OCP MX: E2M1 elements, one E8M0 scale
// per 32 K-elements; NEXT-4, R31).  Ordered by unit roundoff: pair class = max.
// Every conversion from binary64 is ONE round-to-nearest-even (PAPER.md:148
// receiver-side conversion; R11): hardware cvt.rn for FP32/FP16/BF16,
// round-to-odd into binary32 followed by cvt.rn.satfinite for E4M3 / E5M2 (the
// per-tile scale keeps every value <= Omega', so satfinite never triggers).
// No code here is shared with oracle/ (which re-derives everything from the
// format definitions in plain C).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <mutex>
#include <utility>
#include <vector>

#define GMP_NCLASS 7
#define GMP_MX 6   // MXFP4 class (operands only: A/B tiles, never C)
// workspace arenas: one per class, then the FP32 BF16x3 splits and the FP64 int8 digits
#define GMP_AR_SPLIT (GMP_NCLASS)
#define GMP_AR_SLICE (GMP_NCLASS + 1)
#define GMP_NARENA (GMP_NCLASS + 2)
#define GMP_STEP_DEPTH 8  // SUMMA step depth D (R15): fold order is G-independent

namespace gmp {

__host__ __device__ constexpr int class_bytes(int c) {   // per element; MXFP4: see mx_slot_bytes
  return c == 0 ? 8 : c == 1 ? 4 : c >= 4 ? 1 : 2;
}

// MXFP4 slot (O6/R31): nb*nb/2 element bytes -- K-major payload row m (A: tile
// row, B: tile column), element k in byte m*nb/2 + k/2, low nibble for even k -- then
// nb*nb/32 E8M0 scale bytes (s + 127 of block k/32 of row m) in the tcgen05 scale-factor
// layout: per 128-row group g and per 4 blocks c a 512-byte chunk, byte
// (m%32)*16 + ((m%128)/32)*4 + blk%4 (the smem image tcgen05.cp 32x128b.warpx4 copies to
// TMEM; tools/microbench/mxf4_probe.cu).
__host__ __device__ inline int64_t mx_slot_bytes(int nb) { return (int64_t)nb * nb / 2 + (int64_t)nb * nb / 32; }
__host__ __device__ inline int64_t mx_sf_offset(int nb, int m, int blk) {
  const int g = m >> 7, mm = m & 127;
  return (int64_t)nb * nb / 2 + ((int64_t)g * (nb >> 7) + (blk >> 2)) * 512 + (mm & 31) * 16 + (mm >> 5) * 4 + (blk & 3);
}
// bytes of one nb x nb payload slot of class c
__host__ __device__ inline int64_t slot_bytes_of(int c, int nb) {
  return c == GMP_MX ? mx_slot_bytes(nb) : (int64_t)nb * nb * class_bytes(c);
}

// unit roundoff u_k, smallest subnormal eta_k, scale target Omega'_k (R10)
__host__ __device__ inline double class_u(int c) {
  return c == 0 ? 0x1p-53 : c == 1 ? 0x1p-24 : c == 2 ? 0x1p-11 : c == 3 ? 0x1p-8 : c == 4 ? 0x1p-4
       : c == 5 ? 0x1p-3 : 0x1p-2;
}
// MXFP4: eta is the E2M1 subnormal quantum in block units (0.5 x 2^s_b)
__host__ __device__ inline double class_eta(int c) {
  return c == 0 ? 0x1p-1074 : c == 1 ? 0x1p-149 : c == 2 ? 0x1p-24 : c == 3 ? 0x1p-133 : c == 4 ? 0x1p-9
       : c == 5 ? 0x1p-16 : 0.5;
}
__host__ __device__ inline double class_omega(int c) {   // MXFP4: the tile max is scaled to <= 1 too
  return c == 2 ? 65504.0 : c == 4 ? 448.0 : c == 5 ? 57344.0 : 1.0;
}

// ---- binary64 -> class bits, one RNE rounding --------------------------------
__device__ __forceinline__ uint32_t cvt_f32_rn(double x) {
  float f;
  asm("cvt.rn.f32.f64 %0, %1;" : "=f"(f) : "d"(x));
  return __float_as_uint(f);
}
__device__ __forceinline__ uint16_t cvt_f16_rn(double x) {
  uint16_t h;
  asm("cvt.rn.f16.f64 %0, %1;" : "=h"(h) : "d"(x));
  return h;
}
__device__ __forceinline__ uint16_t cvt_bf16_rn(double x) {
  uint16_t h;
  asm("cvt.rn.bf16.f64 %0, %1;" : "=h"(h) : "d"(x));
  return h;
}
// E4M3: round-to-odd into binary32 (24 bits >> 4+2), then RNE with saturation.
// RTO keeps the sticky information, so the second rounding is exact RNE.
__device__ __forceinline__ float rto_f32(double x) {
  float f;
  asm("cvt.rz.f32.f64 %0, %1;" : "=f"(f) : "d"(x));
  if ((double)f != x) f = __uint_as_float(__float_as_uint(f) | 1u);
  return f;
}
__device__ __forceinline__ uint16_t cvt_e4m3x2_rn(double lo, double hi) {
  uint16_t r;
  float flo = rto_f32(lo), fhi = rto_f32(hi);
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(fhi), "f"(flo));
  return r;
}
__device__ __forceinline__ uint8_t cvt_e4m3_rn(double x) {
  return (uint8_t)(cvt_e4m3x2_rn(x, 0.0) & 0xFF);
}
__device__ __forceinline__ uint16_t cvt_e5m2x2_rn(double lo, double hi) {
  uint16_t r;
  float flo = rto_f32(lo), fhi = rto_f32(hi);
  asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(fhi), "f"(flo));
  return r;
}
__device__ __forceinline__ uint8_t cvt_e5m2_rn(double x) {
  return (uint8_t)(cvt_e5m2x2_rn(x, 0.0) & 0xFF);
}

// MXFP4 block scale (R31): the smallest s >= -127 with amax <= 6 * 2^s (no element of the
// block saturates); amax = m 2^E (frexp), 6 = 0.75 * 2^3: s = E - 3 if m <= 0.75 else E - 2.
__host__ __device__ inline int mx_block_exp(double amax) {
  if (amax == 0.0) return -127;
  int E;
  const double m = frexp(amax, &E);
  const int s = (m <= 0.75) ? E - 3 : E - 2;
  return s < -127 ? -127 : s;
}
// two E2M1 codes (lo in bits 0-3) from binary64 values already divided by the block
// scale (|x| <= 6): round-to-odd into binary32, then RNE (exact: 24 >= 2 + 2 bits)
__device__ __forceinline__ uint32_t cvt_e2m1x2_rn(double lo, double hi) {
  uint16_t r;
  const float flo = rto_f32(lo), fhi = rto_f32(hi);
  asm("{.reg .b8 t; cvt.rn.satfinite.e2m1x2.f32 t, %1, %2; cvt.u16.u8 %0, t;}" : "=h"(r) : "f"(fhi), "f"(flo));
  return (uint32_t)r & 0xFFu;
}
__host__ __device__ inline float e2m1_value(uint32_t q) {
  const float v = (q & 7u) < 2u ? 0.5f * (float)(q & 7u)
                : (float)(((q & 1u) + 2u) << ((q & 7u) >> 1)) * 0.25f;
  return (q & 8u) ? -v : v;
}
// exact value (scaled units) of element (m, k) of an MXFP4 slot: E2M1(q) x 2^(s_b)
__device__ __forceinline__ float mx_value(const uint8_t* slot, int nb, int m, int k) {
  const uint32_t q = (slot[(int64_t)m * (nb >> 1) + (k >> 1)] >> (4 * (k & 1))) & 15u;
  const int s = (int)slot[mx_sf_offset(nb, m, k >> 5)] - 127;
  return (float)ldexp((double)e2m1_value(q), s);
}

// ---- class bits -> exact binary64 / binary32 ----------------------------------
__device__ __forceinline__ float f16_to_f32(uint16_t h) {
  float f;
  asm("{.reg .b16 t; mov.b16 t, %1; cvt.f32.f16 %0, t;}" : "=f"(f) : "h"(h));
  return f;
}
__device__ __forceinline__ float bf16_to_f32(uint16_t h) {
  return __uint_as_float(((uint32_t)h) << 16);
}
__device__ __forceinline__ float e4m3_to_f32(uint8_t b) {
  uint32_t h2;
  uint16_t in = b;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(in));
  return f16_to_f32((uint16_t)(h2 & 0xFFFF));
}
__device__ __forceinline__ float e5m2_to_f32(uint8_t b) {
  uint32_t h2;
  uint16_t in = b;
  asm("cvt.rn.f16x2.e5m2x2 %0, %1;" : "=r"(h2) : "h"(in));
  return f16_to_f32((uint16_t)(h2 & 0xFFFF));
}
// value of element i of a payload of class c, as binary32 (exact for c >= 1)
template <int C>
__device__ __forceinline__ float payload_f32(const void* p, int64_t i) {
  if constexpr (C == 1) return reinterpret_cast<const float*>(p)[i];
  if constexpr (C == 2) return f16_to_f32(reinterpret_cast<const uint16_t*>(p)[i]);
  if constexpr (C == 3) return bf16_to_f32(reinterpret_cast<const uint16_t*>(p)[i]);
  if constexpr (C == 4) return e4m3_to_f32(reinterpret_cast<const uint8_t*>(p)[i]);
  if constexpr (C == 5) return e5m2_to_f32(reinterpret_cast<const uint8_t*>(p)[i]);
  return 0.f;
}
__device__ __forceinline__ double payload_f64(const void* p, int64_t i, int c) {
  switch (c) {
    case 0: return reinterpret_cast<const double*>(p)[i];
    case 1: return (double)reinterpret_cast<const float*>(p)[i];
    case 2: return (double)f16_to_f32(reinterpret_cast<const uint16_t*>(p)[i]);
    case 3: return (double)bf16_to_f32(reinterpret_cast<const uint16_t*>(p)[i]);
    case 4: return (double)e4m3_to_f32(reinterpret_cast<const uint8_t*>(p)[i]);
    default: return (double)e5m2_to_f32(reinterpret_cast<const uint8_t*>(p)[i]);
  }
}
// store RN_c(x) as element i of a payload of class c
__device__ __forceinline__ void payload_store(void* p, int64_t i, int c, double x) {
  switch (c) {
    case 0: reinterpret_cast<double*>(p)[i] = x; break;
    case 1: reinterpret_cast<uint32_t*>(p)[i] = cvt_f32_rn(x); break;
    case 2: reinterpret_cast<uint16_t*>(p)[i] = cvt_f16_rn(x); break;
    case 3: reinterpret_cast<uint16_t*>(p)[i] = cvt_bf16_rn(x); break;
    case 4: reinterpret_cast<uint8_t*>(p)[i] = cvt_e4m3_rn(x); break;
    default: reinterpret_cast<uint8_t*>(p)[i] = cvt_e5m2_rn(x); break;
  }
}
// RN_c(x) as an exact binary64 value (used for the analytic shadow scale)
__device__ __forceinline__ double round_to_class(double x, int c) {
  switch (c) {
    case 0: return x;
    case 1: return (double)__uint_as_float(cvt_f32_rn(x));
    case 2: return (double)f16_to_f32(cvt_f16_rn(x));
    case 3: return (double)bf16_to_f32(cvt_bf16_rn(x));
    case 4: return (double)e4m3_to_f32(cvt_e4m3_rn(x));
    default: return (double)e5m2_to_f32(cvt_e5m2_rn(x));
  }
}

// x * 2^e with one rounding (exact unless the result under/overflows), as ldexp:
// when 2^e is a normal binary64 the product IS ldexp(x, e) (multiplication by a
// power of two rounds once, like scalbn), built from the exponent bits instead of
// the library's branchy loop (measured: the per-pair ldexp of the fold was a
// quarter of the stall samples of the FP16-class epilogue).
__device__ __forceinline__ double ldexp_fast(double x, int e) {
  if (e >= -1022 && e <= 1023) return __dmul_rn(x, __longlong_as_double((long long)(1023 + e) << 52));
  return ldexp(x, e);
}

// RN_32 of a binary64 tile-GEMM result (class 0 folded into a binary32 W)
__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(double x) { return __double2float_rn(x); }

// Per-tile power-of-two scale (R10): largest e with maxabs*2^e <= Omega'_c.
// Closed form through frexp: maxabs = m 2^E, Omega' = m_o 2^E_o:
//   e = E_o - E if m <= m_o else E_o - 1 - E.   maxabs == 0 or FP64 -> 0.
__device__ __forceinline__ int scale_exp(double maxabs, int c) {
  if (c == 0 || maxabs == 0.0) return 0;
  int E, Eo;
  double m = frexp(maxabs, &E);
  double mo = frexp(class_omega(c), &Eo);
  return (m <= mo) ? (Eo - E) : (Eo - 1 - E);
}

// Opt a kernel into `bytes` of dynamic shared memory once per (kernel, device):
// the attribute is per device, so a process driving several GPUs sets it on each.
template <class K>
inline cudaError_t ensure_max_smem(K kernel, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const void* key = reinterpret_cast<const void*>(kernel);
  std::lock_guard<std::mutex> lk(mu);
  for (const auto& d : done)
    if (d.first == key && d.second == dev) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.emplace_back(key, dev);
  return e;
}

// mbarrier wrappers (shared by the tcgen05 kernels and k_dmma)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
// cp.async completion as one arrival on an mbarrier (no pending-count increment)
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}

}  // namespace gmp
