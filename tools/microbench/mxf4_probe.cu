// mxf4_probe.cu -- layout probe for tcgen05.mma kind::mxf4.block_scale.block32 (NEXT-4):
// one CTA computes D (128 x 128, FP32) = A (128 x 256 E2M1, K-major) x B^T (128 x 256 E2M1,
// K-major) with one E8M0 scale per 32 K-elements, and compares it with a host reference.
//   operands: SWIZZLE_128B K-major smem (rows of 128 B = 256 FP4, element 2i in the low
//             nibble of byte i), the same canonical layout the 8-bit kernels use;
//   scales:   per 128 rows x 4 scales a 512-byte chunk, byte (m % 32)*16 + (m / 32)*4 + s % 4,
//             copied to TMEM with tcgen05.cp.32x128b.warpx4 (4 columns per chunk); MMA t
//             (K = 64) reads chunk t/2 at byte offset 2*(t%2) (the a/b_sf_id fields).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mxf4_probe mxf4_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(2);                                                                      \
    }                                                                               \
  } while (0)

constexpr int M = 128, N = 128, K = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
// no swizzle, K-major: 8-row x 16-byte core matrices, SBO = 128 B between them
__device__ __forceinline__ uint64_t sdesc_none(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(512 >> 4) << 16) | ((uint64_t)(128 >> 4) << 32) |
         ((uint64_t)1 << 46);
}

__global__ void k_probe(const uint8_t* A, const uint8_t* B, const uint8_t* SFA, const uint8_t* SFB, float* D,
                        int sfmode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;               // 16 KB
  uint8_t* sB = smem + 16384;       // 16 KB
  uint8_t* sSFA = smem + 32768;     // 1 KB (2 chunks)
  uint8_t* sSFB = smem + 33792;     // 1 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x;
  // operands: row r, 16-byte chunk c stored at chunk c ^ (r & 7) (SWIZZLE_128B)
  for (int u = t; u < 128 * 8; u += blockDim.x) {
    const int r = u >> 3, c = u & 7;
    const uint4 va = *reinterpret_cast<const uint4*>(A + r * 128 + c * 16);
    const uint4 vb = *reinterpret_cast<const uint4*>(B + r * 128 + c * 16);
    *reinterpret_cast<uint4*>(sA + r * 128 + ((c ^ (r & 7)) * 16)) = va;
    *reinterpret_cast<uint4*>(sB + r * 128 + ((c ^ (r & 7)) * 16)) = vb;
  }
  // scales: SFA[m][s] (m < 128, s < 8) -> chunk s/4, byte (m%32)*16 + (m/32)*4 + s%4
  for (int u = t; u < 128 * 8; u += blockDim.x) {
    const int m = u >> 3, s = u & 7;
    const int off = (s >> 2) * 512 + (m & 31) * 16 + (m >> 5) * 4 + (s & 3);
    sSFA[off] = SFA[m * 8 + s];
    sSFB[off] = SFB[m * 8 + s];
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if ((t >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  const uint32_t t_acc = tm, t_sfa = tm + 128, t_sfb = tm + 136;
  if (t == 0) {
    for (int c = 0; c < 2; ++c) {
      asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(t_sfa + 4 * c),
                   "l"(sdesc_none(smem_u32(sSFA + 512 * c))));
      asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(t_sfb + 4 * c),
                   "l"(sdesc_none(smem_u32(sSFB + 512 * c))));
    }
    for (int k = 0; k < 4; ++k) {   // K = 64 per instruction = 32 bytes of the 128-byte row
      const uint64_t ad = sdesc_sw128(smem_u32(sA)) + (uint64_t)((k * 32) >> 4);
      const uint64_t bd = sdesc_sw128(smem_u32(sB)) + (uint64_t)((k * 32) >> 4);
      const uint32_t sfid = (uint32_t)(2 * (k & 1));
      uint32_t idesc = (sfid << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) |
                       ((uint32_t)(M >> 4) << 24) | (sfid << 29);
      uint32_t sa = t_sfa + 4 * (k >> 1), sb = t_sfb + 4 * (k >> 1);
      if (sfmode == 1) { sa |= sfid << 30; sb |= sfid << 30; }
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(t_acc),
          "l"(ad), "l"(bd), "r"(idesc), "r"(k > 0 ? 1u : 0u), "r"(sa), "r"(sb));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  {
    const uint32_t a = smem_u32(&bar);
    asm volatile(
        "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(a)
        : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int w = t >> 5, lane = t & 31;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(t_acc + ((uint32_t)(w * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int v = 0; v < 16; ++v) D[(w * 32 + lane) * N + c0 + v] = __uint_as_float(r[v]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

static double e2m1(int q) {
  static const double v[8] = {0, 0.5, 1, 1.5, 2, 3, 4, 6};
  return (q & 8 ? -1 : 1) * v[q & 7];
}

int main() {
  std::vector<uint8_t> A(M * K / 2), B(N * K / 2), SFA(M * 8), SFB(N * 8);
  uint64_t s = 12345;
  auto rnd = [&]() { s = s * 6364136223846793005ull + 1442695040888963407ull; return (uint32_t)(s >> 33); };
  for (auto& x : A) x = (uint8_t)rnd();
  for (auto& x : B) x = (uint8_t)rnd();
  for (auto& x : SFA) x = (uint8_t)(127 - 3 + rnd() % 7);
  for (auto& x : SFB) x = (uint8_t)(127 - 3 + rnd() % 7);
  std::vector<double> ref(M * N);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double acc = 0;
      for (int k = 0; k < K; ++k) {
        const int qa = (A[m * 128 + k / 2] >> (4 * (k & 1))) & 15;
        const int qb = (B[n * 128 + k / 2] >> (4 * (k & 1))) & 15;
        acc += e2m1(qa) * std::ldexp(1.0, SFA[m * 8 + k / 32] - 127) * e2m1(qb) *
               std::ldexp(1.0, SFB[n * 8 + k / 32] - 127);
      }
      ref[m * N + n] = acc;
    }
  uint8_t *dA, *dB, *dSA, *dSB;
  float* dD;
  CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dSA, SFA.size())); CK(cudaMalloc(&dSB, SFB.size()));
  CK(cudaMalloc(&dD, M * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dSA, SFA.data(), SFA.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dSB, SFB.data(), SFB.size(), cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 36 * 1024));
  int rc = 0;
  for (int mode = 0; mode < 2; ++mode) {
    CK(cudaMemset(dD, 0, M * N * 4));
    k_probe<<<1, 128, 36 * 1024>>>(dA, dB, dSA, dSB, dD, mode);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> D(M * N);
    CK(cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost));
    double maxrel = 0, maxref = 0;
    int bad = 0;
    for (int i = 0; i < M * N; ++i) {
      maxref = std::fmax(maxref, std::fabs(ref[i]));
      const double e = std::fabs(D[i] - ref[i]);
      if (e > 1e-5 * (std::fabs(ref[i]) + 1)) ++bad;
      maxrel = std::fmax(maxrel, e);
    }
    printf("sf-address mode %d: mismatches %d / %d, max |D-ref| %.3e (max |ref| %.3e); D[0]=%g ref %g D[1]=%g ref %g\n",
           mode, bad, M * N, maxrel, maxref, D[0], ref[0], D[1], ref[1]);
    if (bad) rc = 1;
  }
  return rc;
}
