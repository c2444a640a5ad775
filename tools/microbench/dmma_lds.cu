// Microbenchmark: what costs the k_dmma mainloop its last ~12 %?  Same warp
// tile as k_dmma<32> (2 m16 x 4 n8 DMMAs per k-step, 8 warps, 2 CTAs/SM),
// operands from shared memory (no global traffic):
//   mode 0: fragments loaded once (registers only)        -> DMMA pipe bound
//   mode 1: 32 LDS.64 per k-step as in k_dmma               -> + LDS cost
//   mode 2: mode 1 + __syncthreads per k-step               -> + barrier cost
//   mode 3: 16 LDS.128 per k-step (permuted m/n labelling)  -> fewer LDS
//   mode 4: mode 3 + __syncthreads per k-step
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

constexpr int AP = 132, BP = 68, BK = 16, ST = 4;

template <int MODE>
__global__ void __launch_bounds__(256, 2) k(double* out, int iters) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  for (int i = tid; i < ST * BK * (AP + BP); i += 256) sm[i] = 1e-3 * (i & 255);
  __syncthreads();
  double acc[2][4][4];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 4; ++j)
      for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;
  double a[2][8], b[4][4];
  for (int i = 0; i < 2; ++i)
    for (int r = 0; r < 8; ++r) a[i][r] = sm[(t + 4 * (r >> 1)) * AP + wm + i * 16 + g + 8 * (r & 1)];
  for (int j = 0; j < 4; ++j)
    for (int r = 0; r < 4; ++r) b[j][r] = sm[BK * AP + (t + 4 * r) * BP + wn + j * 8 + g];
  int stage = 0;
  for (int it = 0; it < iters; ++it) {
    const double* As = sm + stage * BK * (AP + BP);
    const double* Bs = As + BK * AP;
    if (++stage == ST) stage = 0;
    if (MODE == 2 || MODE == 4) __syncthreads();
    if (MODE == 1 || MODE == 2) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int r = 0; r < 8; ++r) a[i][r] = As[(t + 4 * (r >> 1)) * AP + wm + i * 16 + g + 8 * (r & 1)];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) b[j][r] = Bs[(t + 4 * r) * BP + wn + j * 8 + g];
    } else if (MODE == 3 || MODE == 4) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 x = *reinterpret_cast<const double2*>(As + (t + 4 * q) * AP + wm + i * 16 + 2 * g);
          a[i][2 * q] = x.x;
          a[i][2 * q + 1] = x.y;
        }
#pragma unroll
      for (int jp = 0; jp < 2; ++jp)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const double2 x = *reinterpret_cast<const double2*>(Bs + (t + 4 * r) * BP + wn + jp * 16 + 2 * g);
          b[2 * jp][r] = x.x;
          b[2 * jp + 1][r] = x.y;
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) dmma(acc[i][j], a[i], b[j]);
  }
  double s = 0.0;
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 4; ++j)
      for (int v = 0; v < 4; ++v) s += acc[i][j][v];
  out[blockIdx.x * 256 + tid] = s;
}

template <int MODE>
void run(int iters) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 2 * 8;   // 8 waves of 2 CTAs/SM
  const int smem = ST * BK * (AP + BP) * 8;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  double* out;
  cudaMalloc(&out, (size_t)grid * 256 * 8);
  k<MODE><<<grid, 256, smem>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k<MODE><<<grid, 256, smem>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * 8 * grid;
  printf("{\"mode\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", MODE, best, flops / (best * 1e-3) / 1e12);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  cudaFree(out);
}

int main(int argc, char** argv) {
  if (argc > 1) {   // sustained: ~1 s per launch
    run<0>(60000);
    run<2>(60000);
    return 0;
  }
  run<0>(1000);
  run<1>(1000);
  run<2>(1000);
  run<3>(1000);
  run<4>(1000);
  return 0;
}
