// Microbenchmark: the practical FP64 tensor (DMMA) peak on this GPU.
// Every warp issues mma.sync.m16n8k16.f64 back to back from registers into
// NACC independent accumulators (no memory traffic); grid = 148 SMs x CPS CTAs
// of 8 warps.  Prints TFLOP/s and the SM clock the run saw (clock64 / ns).
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

template <int NACC>
__global__ void __launch_bounds__(256) k(double* out, int iters, long long* cyc) {
  double a[8], b[4], acc[NACC][4];
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
  for (int j = 0; j < NACC; ++j)
    for (int v = 0; v < 4; ++v) acc[j][v] = 0.0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) dmma(acc[j], a, b);
  }
  const long long t1 = clock64();
  double s = 0.0;
  for (int j = 0; j < NACC; ++j)
    for (int v = 0; v < 4; ++v) s += acc[j][v];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = t1 - t0;
}

template <int NACC>
void run(int cps, int iters) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * cps;
  double* out;
  long long* cyc;
  cudaMalloc(&out, (size_t)grid * 256 * 8);
  cudaMalloc(&cyc, 8);
  k<NACC><<<grid, 256>>>(out, 10, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  long long c = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k<NACC><<<grid, 256>>>(out, iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) { best = ms; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); }
  }
  const double flops = 2.0 * 16 * 8 * 16 * (double)NACC * iters * 8 /*warps*/ * grid;
  printf("{\"nacc\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f, \"sm_mhz_est\": %.0f, "
         "\"fma_per_clk_per_sm\": %.1f}\n",
         NACC, cps, best, flops / (best * 1e-3) / 1e12, c / (best * 1e3),
         flops / 2 / sms / (double)c);
  cudaFree(out);
  cudaFree(cyc);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
}

int main() {
  run<4>(1, 4000);
  run<8>(1, 2000);
  run<8>(2, 2000);
  run<16>(1, 1000);
  run<8>(4, 1000);
  return 0;
}
