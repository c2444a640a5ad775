// Microbenchmark: FP32 outer-product GEMM with FFMA2 and a cp.async ring over
// MN-major operands (A stored [k][m], B stored [k][n]).  C(128x128) per CTA,
// grid of independent CTAs, K = 4096.  Prints TFLOP/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) {
  unsigned long long ra, rb, rc;
  asm("mov.b64 %0, {%1, %1};" : "=l"(ra) : "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rc) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(rc) : "l"(ra), "l"(rb));
  float2 d;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rc));
  return d;
}
__device__ __forceinline__ void cp16(uint32_t s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}

template <int BK, int ST, int MINB>
__global__ void __launch_bounds__(256, MINB) k(const float* A, const float* B, float* C, int K, int ld) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int m0 = (blockIdx.x % 8) * 128, n0 = (blockIdx.x / 8 % 8) * 128;
  const float* Ab = A + m0;
  const float* Bb = B + n0;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
  constexpr int STAGE = 2 * BK * 128;  // floats
  const int nsl = K / BK;
  auto issue = [&](int s) {
    if (s < nsl) {
      const uint32_t st = sb + (uint32_t)((s % ST) * STAGE * 4);
#pragma unroll
      for (int u = 0; u < BK * 32 * 2 / 256; ++u) {
        int c = tid + u * 256;           // 16-byte chunks: BK rows x 32 chunks, A then B
        int op = c / (BK * 32), r = (c / 32) % BK, ch = c % 32;
        const float* src = (op == 0 ? Ab : Bb) + (size_t)(s * BK + r) * ld + ch * 4;
        cp16(st + (op * BK * 128 + r * 128 + ch * 4) * 4, src);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int s = 0; s < ST - 1; ++s) issue(s);
  float2 acc[8][4];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
  for (int s = 0; s < nsl; ++s) {
    asm volatile("cp.async.wait_group %0;" ::"n"(ST - 2) : "memory");
    __syncthreads();
    issue(s + ST - 1);
    const float* As = sm + (s % ST) * STAGE;
    const float* Bs = As + BK * 128;
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float4 a0 = *(const float4*)(As + k * 128 + ty * 4), a1 = *(const float4*)(As + k * 128 + 64 + ty * 4);
      float4 b0 = *(const float4*)(Bs + k * 128 + tx * 4), b1 = *(const float4*)(Bs + k * 128 + 64 + tx * 4);
      float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float2 b[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y), make_float2(b1.z, b1.w)};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = ffma2(a[i], b[j], acc[i][j]);
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += acc[i][j].x + acc[i][j].y;
  C[blockIdx.x * 256 + tid] = s;
}

template <int BK, int ST, int MINB>
void run(const float* A, const float* B, float* C, int K, int ld, int grid) {
  size_t smem = (size_t)ST * 2 * BK * 128 * 4;
  cudaFuncSetAttribute(k<BK, ST, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<BK, ST, MINB><<<grid, 256, smem>>>(A, B, C, K, ld);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<BK, ST, MINB><<<grid, 256, smem>>>(A, B, C, K, ld);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 5.0 * grid * 2.0 * 128 * 128 * K;
  printf("BK=%d ST=%d MINB=%d: %.1f TFLOP/s (%s)\n", BK, ST, MINB, fl / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int K = 4096, ld = 1024;
  float *A, *B, *C;
  cudaMalloc(&A, (size_t)K * ld * 4); cudaMalloc(&B, (size_t)K * ld * 4); cudaMalloc(&C, 1 << 24);
  cudaMemset(A, 0, (size_t)K * ld * 4); cudaMemset(B, 0, (size_t)K * ld * 4);
  const int grid = 148 * 8;
  run<16, 4, 1>(A, B, C, K, ld, grid);
  run<16, 4, 2>(A, B, C, K, ld, grid);
  run<32, 3, 1>(A, B, C, K, ld, grid);
  run<32, 4, 1>(A, B, C, K, ld, grid);
  run<8, 4, 2>(A, B, C, K, ld, grid);
  run<16, 3, 2>(A, B, C, K, ld, grid);
  return 0;
}
