// Microbenchmark: do the FP64 tensor (DMMA, mma.sync.f64) path and the 5th-gen
// tensor cores (tcgen05.mma kind::f16) run concurrently on one SM?
// Kernel D: DMMA back to back from registers, 1 CTA of 8 warps per SM.
// Kernel T: one elected thread issues tcgen05.mma (BF16, M=128, N=256, K=16)
//           back to back on fixed shared-memory operands into TMEM, 1 CTA per SM.
// Runs D alone, T alone, then D and T on two streams with both resident on every
// SM; prints each kernel's TFLOP/s and the SM clock it saw.  If the two pipes are
// independent the concurrent wall time is ~max(tD, tT), otherwise ~tD + tT.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_tc_concurrent dmma_tc_concurrent.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__global__ void __launch_bounds__(256, 1) kD(double* out, int iters, long long* cyc, unsigned long long* tm) {
  if (threadIdx.x == 0) { unsigned sm; asm("mov.u32 %0, %smid;" : "=r"(sm)); tm[3 * blockIdx.x] = gtime(); tm[3 * blockIdx.x + 2] = sm; }
  double a[8], b[4], acc[8][4];
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
  for (int j = 0; j < 8; ++j)
    for (int v = 0; v < 4; ++v) acc[j][v] = 0.0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(acc[j], a, b);
  }
  const long long t1 = clock64();
  double s = 0.0;
  for (int j = 0; j < 8; ++j)
    for (int v = 0; v < 4; ++v) s += acc[j][v];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = t1 - t0;
  if (threadIdx.x == 0) tm[3 * blockIdx.x + 1] = gtime();
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {   // K-major SWIZZLE_128B
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
constexpr int TBN = 256;
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TBN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

__global__ void __launch_bounds__(128, 1) kT(float* out, int iters, long long* cyc, unsigned long long* tm) {
  if (threadIdx.x == 0) { unsigned sm; asm("mov.u32 %0, %smid;" : "=r"(sm)); tm[3 * blockIdx.x] = gtime(); tm[3 * blockIdx.x + 2] = sm; }
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;               // 128 rows x 128 B
  uint8_t* sB = base + 128 * 128;   // 256 rows x 128 B
  for (int i = threadIdx.x; i < (128 + TBN) * 128 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(base)[i] = 0x3C003C00u ^ (i & 0x00010001u);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint64_t ad = sdesc(smem_u32(sA)), bd = sdesc(smem_u32(sB));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {   // 4 x K=16 covers the 128-byte atom
        const uint32_t acc = (it | k) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad + 2 * k), "l"(bd + 2 * k), "r"(kIdesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  __syncwarp();
  {
    const uint32_t a = smem_u32(&bar);
    asm volatile(
        "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(a)
        : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  long long t1 = clock64();
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(v);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = t1 - t0;
  if (threadIdx.x == 0) tm[3 * blockIdx.x + 1] = gtime();
}

static void summarize(const char* name, unsigned long long* dtm, int n, unsigned long long t0) {
  unsigned long long h[3 * 1024];
  cudaMemcpy(h, dtm, sizeof(unsigned long long) * 3 * n, cudaMemcpyDeviceToHost);
  double smin = 1e30, smax = 0, emin = 1e30, emax = 0;
  for (int i = 0; i < n; ++i) {
    double st = (double)(h[3 * i] - t0) * 1e-6, en = (double)(h[3 * i + 1] - t0) * 1e-6;
    smin = st < smin ? st : smin; smax = st > smax ? st : smax;
    emin = en < emin ? en : emin; emax = en > emax ? en : emax;
  }
  int late = 0;
  for (int i = 0; i < n; ++i) late += ((double)(h[3 * i] - t0) * 1e-6 > smin + 1.0);
  printf("  {\"kernel\": \"%s\", \"start_ms\": [%.2f, %.2f], \"end_ms\": [%.2f, %.2f], \"ctas_started_late\": %d}\n",
         name, smin, smax, emin, emax, late);
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smemT = (128 + TBN) * 128 + 1024;
  cudaFuncSetAttribute(kT, cudaFuncAttributeMaxDynamicSharedMemorySize, smemT);
  double* outD;
  float* outT;
  long long *cD, *cT;
  cudaMalloc(&outD, (size_t)sms * 256 * 8);
  cudaMalloc(&outT, (size_t)sms * 128 * 4);
  cudaMalloc(&cD, 8);
  cudaMalloc(&cT, 8);
  unsigned long long *tmD, *tmT;
  cudaMalloc(&tmD, 8 * 3 * 1024);
  cudaMalloc(&tmT, 8 * 3 * 1024);
  const int itD = argc > 1 ? atoi(argv[1]) : 20000;
  const int itT = argc > 2 ? atoi(argv[2]) : 100000;
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, eD, eT;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&eD);
  cudaEventCreate(&eT);
  kD<<<sms, 256, 0, s1>>>(outD, 100, cD, tmD);
  kT<<<sms, 128, smemT, s1>>>(outT, 100, cT, tmT);
  cudaDeviceSynchronize();
  const double fD = 2.0 * 16 * 8 * 16 * 8.0 * itD * 8 * sms;
  const double fT = 2.0 * 128 * TBN * 16 * 4.0 * itT * sms;
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0, s1);
      cudaStreamWaitEvent(s2, e0, 0);
      if (mode == 3) kT<<<sms, 128, smemT, s2>>>(outT, itT, cT, tmT);
      if (mode != 1) kD<<<sms, 256, 0, s1>>>(outD, itD, cD, tmD);
      if (mode == 1 || mode == 2) kT<<<sms, 128, smemT, s2>>>(outT, itT, cT, tmT);
      cudaEventRecord(eD, s1);
      cudaEventRecord(eT, s2);
      cudaStreamWaitEvent(s1, eT, 0);
      cudaEventRecord(e1, s1);
      cudaEventSynchronize(e1);
      float ms = 0, msD = 0, msT = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaEventElapsedTime(&msD, e0, eD);
      cudaEventElapsedTime(&msT, e0, eT);
      long long cyd = 0, cyt = 0;
      cudaMemcpy(&cyd, cD, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(&cyt, cT, 8, cudaMemcpyDeviceToHost);
      const char* name = mode == 0 ? "dmma_alone" : mode == 1 ? "tc_alone" : mode == 2 ? "dmma_then_tc" : "tc_then_dmma";
      printf("{\"mode\": \"%s\", \"rep\": %d, \"wall_ms\": %.3f, \"dmma_ms\": %.3f, \"tc_ms\": %.3f, "
             "\"dmma_tflops\": %.2f, \"tc_tflops\": %.1f, \"dmma_cyc\": %lld, \"tc_cyc\": %lld}\n",
             name, rep, ms, mode != 1 ? msD : 0.0, mode != 0 ? msT : 0.0,
             mode != 1 ? fD / (msD * 1e-3) / 1e12 : 0.0, mode != 0 ? fT / (msT * 1e-3) / 1e12 : 0.0,
             mode != 1 ? cyd : 0LL, mode != 0 ? cyt : 0LL);
      if (rep == 2 && mode >= 1) {
        unsigned long long a, b;
        cudaMemcpy(&a, tmD, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(&b, tmT, 8, cudaMemcpyDeviceToHost);
        unsigned long long hD[3 * 1024], hT[3 * 1024], t0 = ~0ull;
        cudaMemcpy(hD, tmD, 8 * 3 * sms, cudaMemcpyDeviceToHost);
        cudaMemcpy(hT, tmT, 8 * 3 * sms, cudaMemcpyDeviceToHost);
        for (int i = 0; i < sms; ++i) { t0 = hD[3 * i] < t0 ? hD[3 * i] : t0; t0 = hT[3 * i] < t0 ? hT[3 * i] : t0; }
        summarize("dmma", tmD, sms, t0);
        summarize("tc", tmT, sms, t0);
        int shared = 0;
        for (int i = 0; i < sms; ++i)
          for (int j = 0; j < sms; ++j) shared += (hT[3 * i + 2] == hD[3 * j + 2]);
        int distinct = 0;
        for (int i = 0; i < sms; ++i) {
          bool seen = false;
          for (int j = 0; j < i; ++j) seen |= (hT[3 * j + 2] == hT[3 * i + 2]);
          distinct += !seen;
        }
        printf("  {\"tc_ctas_on_an_sm_with_a_dmma_cta\": %d, \"tc_distinct_sms\": %d}\n", shared, distinct);
      }
    }
  }
  int occD = 0, occT = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occD, kD, 256, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occT, kT, 128, smemT);
  cudaError_t err = cudaGetLastError();
  printf("{\"occ_dmma\": %d, \"occ_tc\": %d, \"err\": \"%s\"}\n", occD, occT, cudaGetErrorString(err));
  return 0;
}
