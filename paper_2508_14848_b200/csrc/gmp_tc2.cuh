// gmp_tc2.cuh -- S6 grouped tile-GEMM for the FP16 / BF16 / E4M3 classes on a
// PAIR of SMs (tcgen05 cta_group::2), for launches whose C tiles accumulate in
// binary32 W and whose tiles are multiples of 256 (the nb = 2048 configs).
//
// A cluster of 2 CTAs computes a 256 x 256 sub-tile of one C tile per pair:
// CTA r holds rows 128r..128r+127 of the A operand and columns 128r..128r+127 of
// the (K-major) B operand in its shared memory; one tcgen05.mma.cta_group::2
// (M = 256, N = 256, issued by CTA 0) reads both CTAs' halves and writes rows
// 128r.. of the FP32 accumulator into CTA r's TMEM.  Per SM and per flop this
// halves the B bytes staged through shared memory and read from L2 compared with
// the 1-SM 128 x 256 kernel -- the 16-bit classes run at the board power cap on
// long runs, so bytes moved per flop set the clock (profiles/power_r01.md).
//
// Protocol (both CTAs run warp 0 = TMA, warp 1 = TMEM alloc (+ MMA on CTA 0),
// warps 2..9 = epilogue):
//   full[s]   CTA 0's barrier; CTA 0's producer arrives with expect_tx of BOTH
//             CTAs' bytes; both CTAs' cta_group::2 TMA loads complete_tx on it.
//   empty[s]  each CTA's own; the MMA commit multicasts to both.
//   tfull[a]  each CTA's own; the MMA commit multicasts to both epilogues.
//   tempty[a] CTA 0's; all 16 epilogue warps of the pair arrive (remote for CTA 1).
// The epilogue is the 1-SM kernel's binary32-W fold (O9): W rows live
// in registers for the whole item, one fma per pair per element.
#pragma once
#include "gmp_tc.cuh"

namespace gmp {

constexpr int TC2_BN = 256;          // N of the pair's MMA (= C sub-tile width)
constexpr int TC2_STAGES = 6;
constexpr uint32_t TC2_PEER_MASK = 0xFEFFFFFFu;   // shared::cluster address of the even CTA of the pair

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1, uint32_t bar0) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(bar0)
      : "memory");
}
// the same with an L2 cache-policy operand (createpolicy)
__device__ __forceinline__ void tma_load_2d_pair_hint(void* dst, const CUtensorMap* map, int c0, int c1,
                                                      uint32_t bar0, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(bar0), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tc2_commit_both(uint64_t* b) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(b)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cta0(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(b) & TC2_PEER_MASK) : "memory");
}
template <int C>
__device__ __forceinline__ void tc2_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  if constexpr (C == 4 || C == 5) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  }
}
// D = F32, A/B format, K-major, N = 256, M = 256 (the pair)
template <int C>
__host__ __device__ constexpr uint32_t tc2_idesc() {
  constexpr uint32_t ab = (C == 3 || C == 5) ? 1u : 0u;
  return (1u << 4) | (ab << 7) | (ab << 10) | ((uint32_t)(TC2_BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}
__host__ __device__ inline int64_t tc2_subtiles_per_item(int nb) { return (int64_t)(nb / 256) * (nb / 256); }

template <int C>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
k_tc2_class(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
            const WorkItem* __restrict__ items, int64_t nitems, const PairDesc* __restrict__ pairs,
            const CTileDesc* __restrict__ ctiles, uint8_t* __restrict__ ws, int nb, double alpha, double beta,
            const int32_t* __restrict__ order, uint32_t hints) {
  constexpr int ESZ = (C == 4 || C == 5) ? 1 : 2;
  constexpr int BK = 128 / ESZ;                  // elements per 128-byte K block
  constexpr int NMMA = 4;                        // 32-byte K per tcgen05.mma
  constexpr int A_BYTES = 128 * 128, B_BYTES = 128 * 128, STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr int ST = TC2_STAGES;
  constexpr uint32_t TMEM_COLS = 2 * TC2_BN;     // two accumulators of 256 columns
  constexpr uint32_t IDESC = tc2_idesc<C>();
  constexpr int HC = TC2_BN / 2;                 // columns per epilogue thread

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * STAGE_BYTES);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t rank = cluster_ctarank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 2 * TC_EPI_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();            // barriers of both CTAs initialised before any remote use
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int kblocks = nb / BK;
  const int64_t cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int nsub = nb / 256;

  // flat index -> (item, 256 x 256 sub-tile): the host's raster order when given
  // (C tile row bands, sub-columns), else item-major row by row
  auto item_at = [&](int64_t flat) {
    const int S = nsub * nsub;
    const int64_t v = order ? (int64_t)order[flat] : flat;
    const int64_t idx = v / S;
    const int sub = (int)(v - idx * S);
    WorkItem w = items[idx];
    w.m0 = (sub / nsub) * 256;
    w.n0 = (sub - (sub / nsub) * nsub) * 256;
    return w;
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full0 = smem_u32(full) & TC2_PEER_MASK;
      // the A panel of the running row band stays in L2 across its C tiles; B streams
      const uint64_t polA = l2_policy_evict_last(), polB = l2_policy_evict_first();
      for (int64_t it = cluster; it < nitems; it += nclusters) {
        const WorkItem w = item_at(it);
        for (int pi = 0; pi < w.pcnt; ++pi) {
          const PairDesc pd = pairs[w.pbeg + pi];
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * STAGE_BYTES;
            if (rank == 0) mbar_expect_tx(&full[stage], 2 * STAGE_BYTES);
            const uint32_t fb = full0 + (uint32_t)(stage * 8);
            if (hints & 1)
              tma_load_2d_pair_hint(sa, &tmA, kb * BK, pd.a_slot * nb + w.m0 + 128 * (int)rank, fb, polA);
            else
              tma_load_2d_pair(sa, &tmA, kb * BK, pd.a_slot * nb + w.m0 + 128 * (int)rank, fb);
            if (hints & 2)
              tma_load_2d_pair_hint(sa + A_BYTES, &tmB, kb * BK, pd.b_slot * nb + w.n0 + 128 * (int)rank, fb, polB);
            else
              tma_load_2d_pair(sa + A_BYTES, &tmB, kb * BK, pd.b_slot * nb + w.n0 + 128 * (int)rank, fb);
            if (++stage == ST) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int64_t it = cluster; it < nitems; it += nclusters) {
        const WorkItem w = item_at(it);
        for (int pi = 0; pi < w.pcnt; ++pi) {
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + (uint32_t)(acc * TC2_BN);
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
            const uint64_t ad = sdesc_k_sw128(sa), bd = sdesc_k_sw128(sa + A_BYTES);
#pragma unroll
            for (int k = 0; k < NMMA; ++k)
              tc2_mma<C>(d_tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), IDESC, (kb | k) != 0);
            tc2_commit_both(&empty[stage]);
            if (++stage == ST) { stage = 0; phase ^= 1; }
          }
          tc2_commit_both(&tfull[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
    }
  } else {
    // epilogue: CTA r owns rows 128r.. of the pair's 256 x 256 sub-tile; warp w
    // reads TMEM lanes 32*(w%4)..+31 and half (w-2)/4 of the 256 columns
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int rloc = 128 * (int)rank + quarter * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t it = cluster; it < nitems; it += nclusters) {
      const WorkItem w = item_at(it);
      const CTileDesc ct = ctiles[w.ctile];
      const int64_t rowoff = (int64_t)(w.m0 + rloc) * nb + w.n0 + half * HC;
      float* wrow = reinterpret_cast<float*>(ws + ct.w_off) + rowoff;
      float accr[HC];
      if (w.pad & 1) {   // first tile-GEMM launch of this C tile: W0 from C_in (O9)
#pragma unroll
        for (int v = 0; v < HC; ++v) accr[v] = w0_f32(ct, ws, rowoff + v, beta);
      } else {
#pragma unroll
        for (int v = 0; v < HC / 4; ++v) {
          const float4 x = reinterpret_cast<const float4*>(wrow)[v];
          accr[4 * v] = x.x; accr[4 * v + 1] = x.y; accr[4 * v + 2] = x.z; accr[4 * v + 3] = x.w;
        }
      }
      for (int pi = 0; pi < w.pcnt; ++pi) {
        const PairDesc pd = pairs[w.pbeg + pi];
        const float f32 = __double2float_rn(ldexp_fast(alpha, pd.fexp));
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * TC2_BN + half * HC);
#pragma unroll
        for (int ch = 0; ch < HC / 16; ++ch) {
          uint32_t r[16];
          tmem_ld16_nowait(tbase + ch * 16, r);
          tmem_wait_ld();
#pragma unroll
          for (int v = 0; v < 16; ++v) accr[ch * 16 + v] = __fmaf_rn(f32, __uint_as_float(r[v]), accr[ch * 16 + v]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cta0(&tempty[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
#pragma unroll
      for (int v = 0; v < HC / 4; ++v)
        reinterpret_cast<float4*>(wrow)[v] = make_float4(accr[4 * v], accr[4 * v + 1], accr[4 * v + 2], accr[4 * v + 3]);
    }
  }
  tc_fence_before();
  cluster_sync_all();            // no CTA leaves while its pair may still touch its smem / barriers
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
}


constexpr int tc2_smem_bytes() { return TC2_STAGES * (128 * 128 * 2) + 1024 /*align*/ + 256 /*barriers*/; }

// L2 cache hints of the pair kernel's TMA loads (bit 0: A evict_last, bit 1: B
// evict_first); GMP_TC2_HINTS overrides the default (A/B measurements)
inline uint32_t tc2_hints() {
  static const uint32_t h = [] {
    const char* e = getenv("GMP_TC2_HINTS");
    return (uint32_t)(e ? atoi(e) : 0);
  }();
  return h;
}

template <int C>
inline gmp_status_t tc2_launch_t(TcTables& t, const WorkItem* it, int64_t n, const PairDesc* pd, const CTileDesc* ct,
                                 uint8_t* ws, int nb, double alpha, double beta, const int32_t* order, cudaStream_t s) {
  constexpr int smem = tc2_smem_bytes();
  if (ensure_max_smem(k_tc2_class<C>, smem) != cudaSuccess) return GMP_ERR_CUDA;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t clusters = std::min<int64_t>(n, sms / 2);
  k_tc2_class<C><<<(unsigned)(2 * clusters), TC_THREADS, smem, s>>>(t.mapA[C], t.mapB128[C], it, n, pd, ct, ws, nb,
                                                                    alpha, beta, order, tc2_hints());
  return cudaGetLastError() == cudaSuccess ? GMP_OK : GMP_ERR_CUDA;
}

// cls: 2..5; n = items x tc2_subtiles_per_item(nb); order: raster (n entries) or NULL
inline gmp_status_t tc2_launch(TcTables& t, int cls, const WorkItem* it, int64_t n, const PairDesc* pd,
                               const CTileDesc* ct, uint8_t* ws, int nb, double alpha, double beta,
                               const int32_t* order, cudaStream_t s) {
  if (cls < 2 || cls > 5 || !t.ready[cls]) return GMP_ERR_STATE;
  switch (cls) {
    case 2: return tc2_launch_t<2>(t, it, n, pd, ct, ws, nb, alpha, beta, order, s);
    case 3: return tc2_launch_t<3>(t, it, n, pd, ct, ws, nb, alpha, beta, order, s);
    case 4: return tc2_launch_t<4>(t, it, n, pd, ct, ws, nb, alpha, beta, order, s);
    default: return tc2_launch_t<5>(t, it, n, pd, ct, ws, nb, alpha, beta, order, s);
  }
}

}  // namespace gmp
