// gmp_tcf.cuh -- S6 for all tensor-core classes of one SUMMA step in ONE launch
// (fold order DESIGN.md O9).
//
// k_tc_class runs one launch per (step, class): each launch reads and writes the
// whole W accumulator of every C tile it touches.  With binary64 W (FP64 C tiles,
// the cfg2 bench workload) a launch of short FP16 pairs spends more time moving W
// (128 KB in + 128 KB out per 128 x 128 sub-tile) than multiplying.  This kernel
// takes, per 128 x 128 C sub-tile, the step's pairs of EVERY tensor class in the
// fold order of O9 -- class 5, 4, 3, 2, then the FP32 class (BF16x9 split), l
// increasing inside a class -- so W is loaded once and stored once per step for
// all of them and the short classes run inside the long FP32 class's W-hidden
// pipeline.  The arithmetic per pair (operands, MMA kind, FP32 TMEM accumulation,
// fold) is exactly k_tc_class's, so C is bit-identical to the per-class launches.
//
// Opt-in (GMP_FLAG_TC_FUSED).  Measured on cfg2 (profiles/tc_fused_r01.md): the
// saved W traffic is real (1.8 GB less DRAM written per step) but the launch takes
// ~10 % more cycles than the two per-class launches it replaces -- the 16-bit
// pairs at 128 x 128 need ~118 B/clk/SM of operands (the full-chip L2 averages
// ~43 B/clk/SM), so W traffic is not what limits them, and inside the fused
// launch they also slow the FP32 class's pipeline (tensor pipe 72.6 % vs 88.3 %).
//
// Warp roles as k_tc_class (warp 0 TMA, warp 1 TMEM alloc + MMA issue, warps 2..9
// tc_epilogue).  Shared memory is a ring of 6 slots of one 128-byte K block of A
// (128 rows) and of B (128 rows), 32 KB each: an FP32-class K block takes 3 slots
// (its three BF16 parts), a 16-/8-bit-class K block takes 1, so the short classes
// get a 6-deep pipeline and the split class keeps its 2 K blocks in flight.
#pragma once
#include "gmp_tc.cuh"

namespace gmp {

constexpr int TCF_BN = 128;
constexpr int TCF_SLOTS = 6;
constexpr int TCF_SLOT_A = TC_BM * 128, TCF_SLOT_B = TCF_BN * 128, TCF_SLOT = TCF_SLOT_A + TCF_SLOT_B;

// operand maps per tensor class: index 0 = FP32 class (BF16x3 split arena), 1..4 = classes 2..5
struct TcfMaps {
  CUtensorMap a[5], b[5];
};
__host__ __device__ constexpr int tcf_index(int cls) { return cls == 1 ? 0 : cls - 1; }

// ring cursor: slot index and the parity of the current pass over the ring
struct TcfRing {
  int slot = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void advance() {
    if (++slot == TCF_SLOTS) { slot = 0; phase ^= 1; }
  }
  __device__ __forceinline__ int at(int p, uint32_t& ph) const {   // slot p ahead, with its parity
    const int s = slot + p;
    ph = phase ^ (s >= TCF_SLOTS ? 1u : 0u);
    return s >= TCF_SLOTS ? s - TCF_SLOTS : s;
  }
};

// T0: first FP32-split part product (3: BF16x6, the default; 0: BF16x9), as k_tc_class
template <int T0>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_tc_fused(const __grid_constant__ TcfMaps maps, const WorkItem* __restrict__ items, int64_t nitems,
           const PairDesc* __restrict__ pairs, const CTileDesc* __restrict__ ctiles, uint8_t* __restrict__ ws, int nb,
           double alpha, double beta) {
  constexpr int BN = TCF_BN, NMMA = 4;
  constexpr uint32_t TMEM_COLS = 2 * BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TCF_SLOTS * TCF_SLOT);
  uint64_t* empty = full + TCF_SLOTS;
  uint64_t* tfull = empty + TCF_SLOTS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < TCF_SLOTS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], TC_EPI_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
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

  if (warp == 0) {
    if (lane == 0) {
      TcfRing r;
      for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        const WorkItem w = expand_item(items, it, nb, BN);
        for (int pi = 0; pi < w.pcnt; ++pi) {
          const PairDesc pd = pairs[w.pbeg + pi];
          const int np = pd.cls == 1 ? 3 : 1;
          const int bk = pd.cls >= 4 ? 128 : 64;   // elements per 128-byte K block
          const CUtensorMap* ma = &maps.a[tcf_index(pd.cls)];
          const CUtensorMap* mb = &maps.b[tcf_index(pd.cls)];
          const int kblocks = nb / bk;
          for (int kb = 0; kb < kblocks; ++kb) {
            for (int p = 0; p < np; ++p) {
              mbar_wait(&empty[r.slot], r.phase ^ 1);
              uint8_t* sa = smem + r.slot * TCF_SLOT;
              mbar_expect_tx(&full[r.slot], TCF_SLOT);
              tma_load_2d(sa, ma, kb * bk, (pd.a_slot * np + p) * nb + w.m0, &full[r.slot]);
              tma_load_2d(sa + TCF_SLOT_A, mb, kb * bk, (pd.b_slot * np + p) * nb + w.n0, &full[r.slot]);
              r.advance();
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      TcfRing r;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        const WorkItem w = expand_item(items, it, nb, BN);
        for (int pi = 0; pi < w.pcnt; ++pi) {
          const int cls = pairs[w.pbeg + pi].cls;
          const int np = cls == 1 ? 3 : 1;
          const int kblocks = nb / (cls >= 4 ? 128 : 64);
          const uint32_t idesc = cls == 2 ? tc_idesc<2, BN>() : cls == 4 ? tc_idesc<4, BN>()
                               : cls == 5 ? tc_idesc<5, BN>() : tc_idesc<3, BN>();   // 1 (split) and 3: BF16
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
          for (int kb = 0; kb < kblocks; ++kb) {
            uint32_t sl[3];
            for (int p = 0; p < np; ++p) {
              uint32_t ph;
              const int s = r.at(p, ph);
              mbar_wait(&full[s], ph);
              sl[p] = smem_u32(smem + s * TCF_SLOT);
            }
            tc_fence_after();
            if (np == 3) {
#pragma unroll
              for (int t = T0; t < 9; ++t) {
                // terms (i, j) by decreasing i + j: the smallest part products first (as k_tc_class;
                // split_t0 = 3: BF16x6, 0: BF16x9)
                constexpr int TI[9] = {2, 2, 1, 2, 1, 0, 1, 0, 0}, TJ[9] = {2, 1, 2, 0, 1, 2, 0, 1, 0};
                const uint64_t ad = sdesc_k_sw128(sl[TI[t]]);
                const uint64_t bd = sdesc_k_sw128(sl[TJ[t]] + TCF_SLOT_A);
#pragma unroll
                for (int k = 0; k < NMMA; ++k)
                  tc_mma<3>(d_tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc,
                            (kb | (t - T0) | k) != 0);
              }
            } else {
              const uint64_t ad = sdesc_k_sw128(sl[0]);
              const uint64_t bd = sdesc_k_sw128(sl[0] + TCF_SLOT_A);
              if (cls >= 4) {
#pragma unroll
                for (int k = 0; k < NMMA; ++k)
                  tc_mma<4>(d_tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc, (kb | k) != 0);
              } else {
#pragma unroll
                for (int k = 0; k < NMMA; ++k)
                  tc_mma<2>(d_tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc, (kb | k) != 0);
              }
            }
            for (int p = 0; p < np; ++p) {
              tc_commit(&empty[r.slot]);
              r.advance();
            }
          }
          tc_commit(&tfull[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
    }
  } else {
    tc_epilogue<BN>(items, nitems, pairs, ctiles, ws, nb, alpha, beta, tmem_base, tfull, tempty, warp, lane);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
}

constexpr int tcf_smem_bytes() { return TCF_SLOTS * TCF_SLOT + 1024 /*align*/ + 256 /*barriers*/; }

// cls_present: bit c set when the launch holds class-c pairs (c = 1 means the split arena)
inline gmp_status_t tcf_launch(TcTables& t, unsigned cls_present, const WorkItem* it, int64_t n, const PairDesc* pd,
                               const CTileDesc* ct, uint8_t* ws, int nb, double alpha, double beta, cudaStream_t s,
                               int split_t0 = 3) {
  TcfMaps m;
  std::memset(&m, 0, sizeof m);
  for (int c = 1; c <= 5; ++c) {
    if (!(cls_present >> c & 1)) continue;
    const int ar = c == 1 ? GMP_AR_SPLIT : c;
    if (!t.ready[ar]) return GMP_ERR_STATE;
    m.a[tcf_index(c)] = t.mapA[ar];
    m.b[tcf_index(c)] = t.mapB128[ar];
  }
  constexpr int smem = tcf_smem_bytes();
  if (ensure_max_smem(k_tc_fused<0>, smem) != cudaSuccess || ensure_max_smem(k_tc_fused<3>, smem) != cudaSuccess)
    return GMP_ERR_CUDA;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(n, sms);
  if (split_t0) k_tc_fused<3><<<grid, TC_THREADS, smem, s>>>(m, it, n, pd, ct, ws, nb, alpha, beta);
  else k_tc_fused<0><<<grid, TC_THREADS, smem, s>>>(m, it, n, pd, ct, ws, nb, alpha, beta);
  return cudaGetLastError() == cudaSuccess ? GMP_OK : GMP_ERR_CUDA;
}

}  // namespace gmp
