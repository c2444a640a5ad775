// gmp_convert.cuh -- S3 convert-and-pack, S5 shadow convert, accumulator init,
// S7 C-finalize and the N1 synthetic generator.
//
// All of these are HBM-bound streaming kernels: 16-byte vector loads, one RNE
// rounding per element from binary64 (or from the decoded stored value for a
// shadow, PAPER.md:148 receiver-side conversion), power-of-two scaling with
// ldexp (exact).  Algorithmic bytes per element are listed in DESIGN.md.
#pragma once
#include "gmp_common.cuh"

namespace gmp {

// ---------------------------------------------------------------------------
// S3 convert-and-pack: one job = one tile, 64x64 sub-block per CTA.  The job's
// transpose flag follows the packed layout of DESIGN.md O6: FP64/FP32 operand
// tiles MN-major (A transposed), FP16/BF16/E4M3 K-major (B transposed), C tiles
// row-major.
// ---------------------------------------------------------------------------
struct PackJob {
  const double* src;  // top-left element of the binary64 tile
  int64_t ld;
  int64_t dst_off;    // byte offset of the payload in the workspace
  int16_t cls;
  int16_t scale;
  int16_t transpose;
  int16_t pad;
};

template <int C>
__device__ __forceinline__ void store8(uint8_t* dst, const double* v) {
  // 8 consecutive payload elements of class C from 8 binary64 values
  if constexpr (C == 0) {
    double2* d = reinterpret_cast<double2*>(dst);
    d[0] = make_double2(v[0], v[1]); d[1] = make_double2(v[2], v[3]);
    d[2] = make_double2(v[4], v[5]); d[3] = make_double2(v[6], v[7]);
  } else if constexpr (C == 1) {
    uint4* d = reinterpret_cast<uint4*>(dst);
    d[0] = make_uint4(cvt_f32_rn(v[0]), cvt_f32_rn(v[1]), cvt_f32_rn(v[2]), cvt_f32_rn(v[3]));
    d[1] = make_uint4(cvt_f32_rn(v[4]), cvt_f32_rn(v[5]), cvt_f32_rn(v[6]), cvt_f32_rn(v[7]));
  } else if constexpr (C == 2 || C == 3) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint16_t lo = (C == 2) ? cvt_f16_rn(v[2 * i]) : cvt_bf16_rn(v[2 * i]);
      uint16_t hi = (C == 2) ? cvt_f16_rn(v[2 * i + 1]) : cvt_bf16_rn(v[2 * i + 1]);
      w[i] = (uint32_t)lo | ((uint32_t)hi << 16);
    }
    *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
    uint32_t w[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      uint32_t lo = (C == 4) ? cvt_e4m3x2_rn(v[4 * i], v[4 * i + 1]) : cvt_e5m2x2_rn(v[4 * i], v[4 * i + 1]);
      uint32_t hi = (C == 4) ? cvt_e4m3x2_rn(v[4 * i + 2], v[4 * i + 3]) : cvt_e5m2x2_rn(v[4 * i + 2], v[4 * i + 3]);
      w[i] = lo | (hi << 16);
    }
    *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
  }
}

template <int C>
__device__ __forceinline__ void pack_block(const PackJob& j, uint8_t* ws, int nb, int r0, int c0) {
  const int t = threadIdx.x;
  constexpr int B = class_bytes(C);
  uint8_t* dst = ws + j.dst_off;
  if (!j.transpose) {
    // thread -> (row, 8-col group): 64 rows x 8 groups = 512 units, 2 per thread
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int unit = t + u * 256;
      int r = unit >> 3, g = unit & 7;
      const double2* s = reinterpret_cast<const double2*>(j.src + (int64_t)(r0 + r) * j.ld + c0 + g * 8);
      double v[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double2 x = __ldg(s + i);
        v[2 * i] = (C == 0) ? x.x : ldexp_fast(x.x, j.scale);
        v[2 * i + 1] = (C == 0) ? x.y : ldexp_fast(x.y, j.scale);
      }
      store8<C>(dst + ((int64_t)(r0 + r) * nb + c0 + g * 8) * B, v);
    }
  } else {
    // transposed (K-major) write, register transpose: warp w takes source rows 8w..8w+7,
    // lane l the column pair (2l, 2l+1) -- one coalesced 512-byte row per warp load -- and
    // writes 8 consecutive output elements of each of its two output rows (the next warp
    // fills the rest of the 32-byte sectors).  No shared memory, no barrier.
    const int w = t >> 5, c = 2 * (t & 31);
    double2 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      x[i] = __ldg(reinterpret_cast<const double2*>(j.src + (int64_t)(r0 + 8 * w + i) * j.ld + c0 + c));
    double v0[8], v1[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v0[i] = (C == 0) ? x[i].x : ldexp_fast(x[i].x, j.scale);
      v1[i] = (C == 0) ? x[i].y : ldexp_fast(x[i].y, j.scale);
    }
    store8<C>(dst + ((int64_t)(c0 + c) * nb + r0 + 8 * w) * B, v0);
    store8<C>(dst + ((int64_t)(c0 + c + 1) * nb + r0 + 8 * w) * B, v1);
  }
}

__global__ void __launch_bounds__(256) k_pack(const PackJob* __restrict__ jobs, uint8_t* ws, int nb) {
  const PackJob j = jobs[blockIdx.y];
  const int per = nb / 64;
  const int r0 = (blockIdx.x / per) * 64, c0 = (blockIdx.x % per) * 64;
  switch (j.cls) {
    case 0: pack_block<0>(j, ws, nb, r0, c0); break;
    case 1: pack_block<1>(j, ws, nb, r0, c0); break;
    case 2: pack_block<2>(j, ws, nb, r0, c0); break;
    case 3: pack_block<3>(j, ws, nb, r0, c0); break;
    case 4: pack_block<4>(j, ws, nb, r0, c0); break;
    default: pack_block<5>(j, ws, nb, r0, c0); break;
  }
}

// ---------------------------------------------------------------------------
// S5 shadow convert (receiver-side, from the STORED payload):
//   shadow = RN_to(decode_from(stored) * 2^d),  d = shadow scale - stored scale.
// k_shadow keeps the layout (8 elements per thread-iteration); k_shadow_t
// handles the MN-major -> K-major class changes.
// ---------------------------------------------------------------------------
struct ShadowJob {
  int64_t src_off, dst_off;  // byte offsets in the workspace (or panel buffers)
  int16_t from, to, d;
  int16_t transpose;         // 1: layout changes (MN-major FP64/FP32 -> K-major 16/8-bit)
};

template <int F, int T>
__device__ __forceinline__ void shadow_run(const ShadowJob& j, uint8_t* ws, int64_t n) {
  const uint8_t* src = ws + j.src_off;
  uint8_t* dst = ws + j.dst_off;
  for (int64_t e0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; e0 < n;
       e0 += (int64_t)gridDim.x * blockDim.x * 8) {
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = ldexp_fast(payload_f64(src, e0 + i, F), j.d);
    store8<T>(dst + e0 * class_bytes(T), v);
  }
}

__global__ void __launch_bounds__(256) k_shadow(const ShadowJob* __restrict__ jobs, uint8_t* ws, int64_t n) {
  const ShadowJob j = jobs[blockIdx.y];
  const int key = j.from * 8 + j.to;
  switch (key) {
#define GMP_SH(F, T) case F * 8 + T: shadow_run<F, T>(j, ws, n); break;
    GMP_SH(0, 1) GMP_SH(0, 2) GMP_SH(0, 3) GMP_SH(0, 4) GMP_SH(0, 5)
    GMP_SH(1, 2) GMP_SH(1, 3) GMP_SH(1, 4) GMP_SH(1, 5)
    GMP_SH(2, 3) GMP_SH(2, 4) GMP_SH(2, 5)
    GMP_SH(3, 4) GMP_SH(3, 5)
    GMP_SH(4, 5)
#undef GMP_SH
    default: break;
  }
}

// Transposing shadow (source MN-major class 0/1 -> target K-major class 2..5): per 64x64
// block, warp w takes source rows 8w..8w+7 and lane l the column pair (2l, 2l+1) (8- or
// 16-byte coalesced loads), decodes exactly, scales, rounds once into the target class and
// writes 8 consecutive elements of each of its two output rows (register transpose).
template <int F, int T>
__device__ __forceinline__ void shadow_t_block(const ShadowJob& j, uint8_t* ws, int nb, int r0, int c0) {
  static_assert(F == 0 || F == 1, "transposing shadows start from the MN-major binary64 / binary32 classes");
  const int t = threadIdx.x, w = t >> 5, c = 2 * (t & 31);
  const uint8_t* src = ws + j.src_off;
  uint8_t* dst = ws + j.dst_off;
  double v0[8], v1[8];
  if constexpr (F == 1) {
    float2 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      x[i] = __ldg(reinterpret_cast<const float2*>(src + ((int64_t)(r0 + 8 * w + i) * nb + c0 + c) * 4));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v0[i] = ldexp_fast((double)x[i].x, j.d);
      v1[i] = ldexp_fast((double)x[i].y, j.d);
    }
  } else {
    double2 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      x[i] = __ldg(reinterpret_cast<const double2*>(src + ((int64_t)(r0 + 8 * w + i) * nb + c0 + c) * 8));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v0[i] = ldexp_fast(x[i].x, j.d);
      v1[i] = ldexp_fast(x[i].y, j.d);
    }
  }
  store8<T>(dst + ((int64_t)(c0 + c) * nb + r0 + 8 * w) * class_bytes(T), v0);
  store8<T>(dst + ((int64_t)(c0 + c + 1) * nb + r0 + 8 * w) * class_bytes(T), v1);
}

__global__ void __launch_bounds__(256) k_shadow_t(const ShadowJob* __restrict__ jobs, uint8_t* ws, int nb) {
  const ShadowJob j = jobs[blockIdx.y];
  const int per = nb / 64;
  const int r0 = (blockIdx.x / per) * 64, c0 = (blockIdx.x % per) * 64;
  switch (j.from * 8 + j.to) {
#define GMP_ST(F, T) case F * 8 + T: shadow_t_block<F, T>(j, ws, nb, r0, c0); break;
    GMP_ST(0, 2) GMP_ST(0, 3) GMP_ST(0, 4) GMP_ST(0, 5) GMP_ST(1, 2) GMP_ST(1, 3) GMP_ST(1, 4) GMP_ST(1, 5)
#undef GMP_ST
    default: break;
  }
}

// ---------------------------------------------------------------------------
// MXFP4 encode (S3 pack of an MXFP4 tile and S5 shadows INTO MXFP4; O6, R31):
//   y = x 2^scale (pack: x = binary64 user element) or y = decode_from(stored) 2^d
//   (shadow, receiver-side from the stored payload); per block of 32 consecutive
//   K-elements of a K-major payload row: s_b = mx_block_exp(max |y|), q = RN_E2M1(y 2^-s_b).
//   transpose = 0: element (m, k) at src[m * ld + k]; 1: at src[k * ld + m].
// ---------------------------------------------------------------------------
struct MxJob {
  const uint8_t* src;   // pack: the binary64 tile, top-left (from = -1)
  int64_t src_off;      // shadow: byte offset of the stored payload in the workspace
  int64_t ld;           // elements
  int64_t dst_off;      // byte offset of the MXFP4 slot in the workspace
  int16_t from;         // -1: binary64 user matrix; else the stored class of the payload
  int16_t scale;        // pack: per-tile scale e; shadow: d
  int16_t transpose;
  int16_t pad;
};


// Warp-per-unit, no shared memory.  transpose = 0 (payload row = source row): a unit is one
// payload row x 128 K; lane l holds elements 4l..4l+3 (one 32-byte coalesced load per
// lane), the 8 lanes of a block reduce max|y| by shuffles, every lane writes its 2 bytes of
// nibbles and lane 8b the scale byte.  transpose = 1 (payload row = source column): a unit
// is 32 payload rows x 32 K; lane l owns payload row m0 + l, the warp reads 32 source rows of
// 32 consecutive elements (coalesced), each lane keeps its block in registers and writes
// 16 bytes of nibbles and its scale byte.
// Values are held as round-to-odd binary32 images of the exact binary64 y: RTO keeps every
// comparison with a binary32 threshold (the block-scale test amax <= 6 * 2^s, the binade of
// amax) and the final RNE onto the 2-bit E2M1 significand exact (>= 20 bits kept even for
// binary32-subnormal y), at half the registers of binary64.
constexpr int MX_UNITS_PER_WARP = 8;
__device__ __forceinline__ uint32_t mx_enc2f(float a, float b) {   // two scaled values -> one byte
  uint16_t r;
  asm("{.reg .b8 t; cvt.rn.satfinite.e2m1x2.f32 t, %1, %2; cvt.u16.u8 %0, t;}" : "=h"(r) : "f"(b), "f"(a));
  return (uint32_t)r & 0xFFu;
}
__device__ __forceinline__ uint32_t mx_enc4f(const float* v, float inv) {   // 4 values -> 2 bytes
  return mx_enc2f(v[0] * inv, v[1] * inv) | (mx_enc2f(v[2] * inv, v[3] * inv) << 8);
}
__device__ __forceinline__ float mx_inv_scale(int sb) { return __int_as_float((127 - sb) << 23); }   // 2^-sb, sb in [-127, 125]
__device__ __forceinline__ float mx_load(const MxJob& j, const uint8_t* base, int64_t idx) {
  const double x = j.from < 0 ? __ldg(reinterpret_cast<const double*>(base) + idx) : payload_f64(base, idx, j.from);
  return rto_f32(ldexp_fast(x, j.scale));
}
__global__ void __launch_bounds__(256, 4) k_mx(const MxJob* __restrict__ jobs, uint8_t* ws, int nb) {
  const MxJob j = jobs[blockIdx.y];
  const uint8_t* base = j.from < 0 ? j.src : ws + j.src_off;
  uint8_t* slot = ws + j.dst_off;
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * MX_UNITS_PER_WARP;
  if (!j.transpose) {
    const int per = nb / 128;   // units per payload row
    // four units per round: their loads are all in flight before any reduction
    for (int u0 = 0; u0 < MX_UNITS_PER_WARP; u0 += 4) {
      float v[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t unit = warp0 + u0 + q;
        const int m = (int)(unit / per), k0 = (int)(unit % per) * 128 + 4 * lane;
        if (unit >= (int64_t)nb * per) { v[q][0] = v[q][1] = v[q][2] = v[q][3] = 0.f; continue; }
        if (j.from < 0) {
          const double2* p = reinterpret_cast<const double2*>(reinterpret_cast<const double*>(base) + (int64_t)m * j.ld + k0);
          const double2 a = __ldg(p), b = __ldg(p + 1);
          v[q][0] = rto_f32(ldexp_fast(a.x, j.scale)); v[q][1] = rto_f32(ldexp_fast(a.y, j.scale));
          v[q][2] = rto_f32(ldexp_fast(b.x, j.scale)); v[q][3] = rto_f32(ldexp_fast(b.y, j.scale));
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) v[q][e] = mx_load(j, base, (int64_t)m * j.ld + k0 + e);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t unit = warp0 + u0 + q;
        if (unit >= (int64_t)nb * per) break;
        const int m = (int)(unit / per), k0 = (int)(unit % per) * 128 + 4 * lane;
        float amax = fmaxf(fmaxf(fabsf(v[q][0]), fabsf(v[q][1])), fmaxf(fabsf(v[q][2]), fabsf(v[q][3])));
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 2));
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 4));
        const int sb = mx_block_exp((double)amax);
        *reinterpret_cast<uint16_t*>(slot + (int64_t)m * (nb >> 1) + (k0 >> 1)) = (uint16_t)mx_enc4f(v[q], mx_inv_scale(sb));
        if ((lane & 7) == 0) slot[mx_sf_offset(nb, m, k0 >> 5)] = (uint8_t)(sb + 127);
      }
    }
  } else {
    const int per = nb / 32;    // units per 32-row band
    for (int u = 0; u < MX_UNITS_PER_WARP; ++u) {
      const int64_t unit = warp0 + u;
      if (unit >= (int64_t)per * per) break;
      const int m = (int)(unit / per) * 32 + lane, kb = (int)(unit % per);
      float v[32];
      float amax = 0.f;
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        v[e] = mx_load(j, base, (int64_t)(kb * 32 + e) * j.ld + m);
        amax = fmaxf(amax, fabsf(v[e]));
      }
      const int sb = mx_block_exp((double)amax);
      const float inv = mx_inv_scale(sb);
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = mx_enc4f(v + 8 * q, inv) | (mx_enc4f(v + 8 * q + 4, inv) << 16);
      *reinterpret_cast<uint4*>(slot + (int64_t)m * (nb >> 1) + kb * 16) = make_uint4(w[0], w[1], w[2], w[3]);
      slot[mx_sf_offset(nb, m, kb)] = (uint8_t)(sb + 127);
    }
  }
}

// ---------------------------------------------------------------------------
// FP32 class on the tensor pipe: exact 3-way BF16 split of an FP32 payload
// (MN-major) into three K-major BF16 parts, x = x0 + x1 + x2 with
// x0 = RN_bf16(x), x1 = RN_bf16(x - x0), x2 = x - x0 - x1 (both differences
// are exact in binary32, x2 has at most 8 significant bits).  Receiver-side:
// made from the stored (or shadow) FP32 payload.  64x64 blocks, transposed.
// ---------------------------------------------------------------------------
struct SplitJob {
  int64_t src_off;   // FP32 payload (MN-major)
  int64_t dst_off;   // 3 consecutive nb x nb BF16 parts (K-major)
};

__global__ void __launch_bounds__(256) k_split(const SplitJob* __restrict__ jobs, uint8_t* ws, int nb) {
  // 64x64 binary32 block, element (r, c) at r*64 + (c ^ 4*((r >> 3) & 7)):
  // row-wise writes and the transposed 8-row reads are both conflict-free
  __shared__ float sm[64 * 64];
  const SplitJob j = jobs[blockIdx.y];
  const int per = nb / 64;
  const int r0 = (blockIdx.x / per) * 64, c0 = (blockIdx.x % per) * 64;
  const float* src = reinterpret_cast<const float*>(ws + j.src_off);
  uint8_t* dst = ws + j.dst_off;
  const int64_t part = (int64_t)nb * nb * 2;   // bytes per BF16 part
  const int t = threadIdx.x;
  float4 x[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int unit = t + u * 256;              // 64 rows x 16 float4
    x[u] = *reinterpret_cast<const float4*>(src + (int64_t)(r0 + (unit >> 4)) * nb + c0 + 4 * (unit & 15));
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int unit = t + u * 256;
    const int r = unit >> 4, q = unit & 15;
    *reinterpret_cast<float4*>(sm + r * 64 + ((4 * q) ^ (((r >> 3) & 7) << 2))) = x[u];
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int unit = t + u * 256;
    const int oc = unit >> 3, g = unit & 7;    // output row oc (= source col), elements 8g..8g+7
    uint32_t w0[4], w1[4], w2[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = g * 8 + i;
      const float x = sm[r * 64 + (oc ^ (g << 2))];
      const uint16_t h0 = cvt_bf16_rn((double)x);
      const float r1 = __fsub_rn(x, bf16_to_f32(h0));
      const uint16_t h1 = cvt_bf16_rn((double)r1);
      const float r2 = __fsub_rn(r1, bf16_to_f32(h1));
      const uint16_t h2 = cvt_bf16_rn((double)r2);
      const int sh = (i & 1) * 16;
      if (sh == 0) { w0[i >> 1] = h0; w1[i >> 1] = h1; w2[i >> 1] = h2; }
      else { w0[i >> 1] |= (uint32_t)h0 << 16; w1[i >> 1] |= (uint32_t)h1 << 16; w2[i >> 1] |= (uint32_t)h2 << 16; }
    }
    const int64_t o = ((int64_t)(c0 + oc) * nb + r0 + g * 8) * 2;
    *reinterpret_cast<uint4*>(dst + o) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
    *reinterpret_cast<uint4*>(dst + part + o) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
    *reinterpret_cast<uint4*>(dst + 2 * part + o) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
  }
}

// ---------------------------------------------------------------------------
// accumulator init (O9):  W = beta == 0 ? 0 : RN_W(RN_W(beta) decode(C_in))
// ---------------------------------------------------------------------------
struct CTileDesc {
  int64_t w_off;       // byte offset of the W accumulator (nb*nb of binary64 or binary32)
  int64_t cin_off;     // byte offset of the packed C_in payload (beta != 0), -1 otherwise
  int64_t cout_off;    // byte offset of the packed C_out payload
  int64_t user_off;    // element offset of the tile's top-left in the user's C (local)
  int16_t code;        // class of the C tile (W = binary64 iff code == 0)
  int16_t cin_scale;
  int32_t pad;
};

// W0 of element e of a C tile (binary64 W for code 0, binary32 otherwise)
__device__ __forceinline__ double w0_f64(const CTileDesc& c, const uint8_t* ws, int64_t e, double beta) {
  return (beta == 0.0) ? 0.0 : __dmul_rn(beta, payload_f64(ws + c.cin_off, e, 0));
}
__device__ __forceinline__ float w0_f32(const CTileDesc& c, const uint8_t* ws, int64_t e, double beta) {
  if (beta == 0.0) return 0.f;
  const float bf = __double2float_rn(beta);
  return __double2float_rn(__dmul_rn((double)bf, ldexp_fast(payload_f64(ws + c.cin_off, e, c.code), -c.cin_scale)));
}

// W0 of the C tiles listed in idx (the tiles whose first tile-GEMM launch does not
// initialise W itself; WorkItem.pad bit 0 marks the items that do)
__global__ void __launch_bounds__(256) k_acc_init(const CTileDesc* __restrict__ ct, const int32_t* __restrict__ idx,
                                                  uint8_t* ws, int64_t n, double beta) {
  const CTileDesc c = ct[idx[blockIdx.y]];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (c.code == 0) reinterpret_cast<double*>(ws + c.w_off)[e] = w0_f64(c, ws, e, beta);
    else reinterpret_cast<float*>(ws + c.w_off)[e] = w0_f32(c, ws, e, beta);
  }
}

// ---------------------------------------------------------------------------
// S7 C-finalize: pass 1 maxabs(W) per tile (bit-pattern atomicMax on |x|),
// pass 2 encode into the C class with the scale of maxabs, decode to user C.
// ---------------------------------------------------------------------------
// (pass 1 runs over the tiles listed in idx: the ones whose last tile-GEMM launch does not
// emit max|W| itself, WorkItem.pad bit 1; maxbits is zeroed before the first launch)
__global__ void __launch_bounds__(256) k_c_maxabs(const CTileDesc* __restrict__ ct, const int32_t* __restrict__ idx,
                                                  const uint8_t* ws, int64_t n, unsigned long long* maxbits) {
  const int32_t k = idx[blockIdx.y];
  const CTileDesc c = ct[k];
  if (c.code == 0) return;                      // FP64 C tiles carry no scale
  float m = 0.f;
  for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; e < n;
       e += (int64_t)gridDim.x * blockDim.x * 4) {
    const float4 a = reinterpret_cast<const float4*>(ws + c.w_off)[e / 4];
    m = fmaxf(m, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
  }
  for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0 && m > 0.f)
    atomicMax(maxbits + k, (unsigned long long)__double_as_longlong((double)m));
}

// one CTA per FP_ROWS rows of a C tile, threads along the row (coalesced user C
// stores).  FP64 C tiles: the packed C_out IS the binary64 W (plan aliases
// cout_off = w_off), so only the user's C is written.
constexpr int FIN_ROWS = 4;
// 4 consecutive W values of a binary32-W tile -> packed class-C payload (one RN each) and
// the decoded binary64 user values; rounded values stay in registers (no payload read-back)
template <int C>
__device__ __forceinline__ void fin4(const float4 w, int e, uint8_t* pay, int64_t i, double* u) {
  const double y[4] = {ldexp_fast((double)w.x, e), ldexp_fast((double)w.y, e), ldexp_fast((double)w.z, e),
                       ldexp_fast((double)w.w, e)};
  double r[4];
  if constexpr (C == 1) {
    uint32_t b[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) { b[v] = cvt_f32_rn(y[v]); r[v] = (double)__uint_as_float(b[v]); }
    *reinterpret_cast<uint4*>(pay + i * 4) = make_uint4(b[0], b[1], b[2], b[3]);
  } else if constexpr (C == 2 || C == 3) {
    uint16_t h[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      h[v] = (C == 2) ? cvt_f16_rn(y[v]) : cvt_bf16_rn(y[v]);
      r[v] = (double)((C == 2) ? f16_to_f32(h[v]) : bf16_to_f32(h[v]));
    }
    *reinterpret_cast<uint2*>(pay + i * 2) =
        make_uint2((uint32_t)h[0] | ((uint32_t)h[1] << 16), (uint32_t)h[2] | ((uint32_t)h[3] << 16));
  } else {
    const uint32_t lo = (C == 4) ? cvt_e4m3x2_rn(y[0], y[1]) : cvt_e5m2x2_rn(y[0], y[1]);
    const uint32_t hi = (C == 4) ? cvt_e4m3x2_rn(y[2], y[3]) : cvt_e5m2x2_rn(y[2], y[3]);
    const uint32_t b = lo | (hi << 16);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const uint8_t q = (uint8_t)(b >> (8 * v));
      r[v] = (double)((C == 4) ? e4m3_to_f32(q) : e5m2_to_f32(q));
    }
    *reinterpret_cast<uint32_t*>(pay + i) = b;
  }
#pragma unroll
  for (int v = 0; v < 4; ++v) u[v] = ldexp_fast(r[v], -e);
}

template <int C>
__device__ __forceinline__ void fin_rows(const CTileDesc& c, uint8_t* ws, int e, double* cuser, int64_t ldc, int nb) {
  uint8_t* pay = ws + c.cout_off;
  for (int rr = 0; rr < FIN_ROWS; ++rr) {
    const int64_t r = (int64_t)blockIdx.x * FIN_ROWS + rr;
    double* urow = cuser + c.user_off + r * ldc;
    const float4* wrow = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(ws + c.w_off) + r * nb);
    for (int q = threadIdx.x; q < nb / 4; q += blockDim.x) {
      double u[4];
      fin4<C>(wrow[q], e, pay, r * nb + 4 * q, u);
      reinterpret_cast<double2*>(urow + 4 * q)[0] = make_double2(u[0], u[1]);
      reinterpret_cast<double2*>(urow + 4 * q)[1] = make_double2(u[2], u[3]);
    }
  }
}

__global__ void __launch_bounds__(256) k_c_finalize(const CTileDesc* __restrict__ ct, uint8_t* ws,
                                                    const unsigned long long* maxbits, int16_t* cscale,
                                                    double* cuser, int64_t ldc, int nb) {
  const CTileDesc c = ct[blockIdx.y];
  const double m = __longlong_as_double((long long)maxbits[blockIdx.y]);
  const int e = scale_exp(m, c.code);
  if (blockIdx.x == 0 && threadIdx.x == 0) cscale[blockIdx.y] = (int16_t)e;
  switch (c.code) {
    case 0:
      for (int rr = 0; rr < FIN_ROWS; ++rr) {
        const int64_t r = (int64_t)blockIdx.x * FIN_ROWS + rr;
        double* urow = cuser + c.user_off + r * ldc;
        const double2* wrow = reinterpret_cast<const double2*>(reinterpret_cast<const double*>(ws + c.w_off) + r * nb);
        for (int q = threadIdx.x; q < nb / 2; q += blockDim.x) reinterpret_cast<double2*>(urow)[q] = wrow[q];
      }
      break;
    case 1: fin_rows<1>(c, ws, e, cuser, ldc, nb); break;
    case 2: fin_rows<2>(c, ws, e, cuser, ldc, nb); break;
    case 3: fin_rows<3>(c, ws, e, cuser, ldc, nb); break;
    case 4: fin_rows<4>(c, ws, e, cuser, ldc, nb); break;
    default: fin_rows<5>(c, ws, e, cuser, ldc, nb); break;
  }
}

// ---------------------------------------------------------------------------
// N1 synthetic generator (benchmark input only):
// x(r,c) = v(r,c) 2^(s - e(r/nb, c/nb)); local tile (il, jl) of the output is the
// global tile (trow[il], tcol[jl]) (block-cyclic or the caller's ownership).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct SynthArgs {
  double* out;
  int64_t ld, lrows, lcols;        // local matrix (lrows x lcols)
  int64_t grows, gcols;            // global matrix
  int nb;
  const int32_t *trow, *tcol;      // global tile row / column of each local tile row / column
  uint64_t seed, tau;
  int mode, E, s;
};

__global__ void __launch_bounds__(256) k_synth(SynthArgs a) {
  const int64_t mtg = a.grows / a.nb, ntg = a.gcols / a.nb;
  const int64_t total = a.lrows * a.lcols;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lr = idx / a.lcols, lc = idx - (idx / a.lcols) * a.lcols;
    const int64_t ti = a.trow[lr / a.nb], tj = a.tcol[lc / a.nb];
    const int64_t gr = ti * a.nb + lr % a.nb, gc = tj * a.nb + lc % a.nb;
    const uint64_t u = mix64(a.seed + ((uint64_t)(gr * a.gcols + gc) + 1ull) * 0x9E3779B97F4A7C15ull);
    const double v = ((double)(u >> 11) * 0x1p-53) * 2.0 - 1.0;
    int e = 0;
    if (a.mode == 1) {
      int64_t den = mtg + ntg - 2;
      if (den < 1) den = 1;
      e = (int)(((ti + tj) * (int64_t)a.E) / den);
    } else if (a.mode == 2) {
      const uint64_t w = mix64(a.tau + ((uint64_t)(ti * ntg + tj) + 1ull) * 0x9E3779B97F4A7C15ull);
      e = (int)(w % (uint64_t)(a.E + 1));
    }
    a.out[lr * a.ld + lc] = ldexp_fast(v, a.s - e);
  }
}

}  // namespace gmp
