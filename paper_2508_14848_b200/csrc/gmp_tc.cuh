// gmp_tc.cuh -- S6 grouped tile-GEMM for the FP16 / BF16 / E4M3 classes on the
// 5th-generation tensor cores (tcgen05.mma, TMEM accumulators, TMA-fed shared
// memory ring).  [bring-up stub: classes 2..4 run on gmp_simt.cuh until the
// tcgen05 kernel lands]
#pragma once
#include "gmp_common.cuh"
#include "gmp_simt.cuh"

namespace gmp {

constexpr bool kTcAvailable = false;

struct TcTables {
  int dummy = 0;
};

inline int64_t tc_items_per_tile(int64_t nb) { return (nb / 128) * (nb / 128); }

inline void tc_make_items(int64_t nb, int32_t ctile, int32_t pbeg, int32_t pcnt, std::vector<WorkItem>& its) {
  for (int64_t m0 = 0; m0 < nb; m0 += 128)
    for (int64_t n0 = 0; n0 < nb; n0 += 128)
      its.push_back(WorkItem{ctile, (int32_t)m0, (int32_t)n0, pbeg, pcnt, 0});
}

inline gmp_status_t tc_prepare(TcTables&, uint8_t*, const int64_t*, const int64_t*, int) { return GMP_OK; }

inline gmp_status_t tc_launch(TcTables&, int cls, const WorkItem* it, int64_t n, const PairDesc* pd,
                              const CTileDesc* ct, uint8_t* ws, int nb, double alpha, cudaStream_t s) {
  switch (cls) {
    case 2: k_simt_class<2><<<(unsigned)n, 256, 0, s>>>(it, pd, ct, ws, nb, alpha); break;
    case 3: k_simt_class<3><<<(unsigned)n, 256, 0, s>>>(it, pd, ct, ws, nb, alpha); break;
    default: k_simt_class<4><<<(unsigned)n, 256, 0, s>>>(it, pd, ct, ws, nb, alpha); break;
  }
  return cudaGetLastError() == cudaSuccess ? GMP_OK : GMP_ERR_CUDA;
}

inline void tc_release(TcTables&) {}

}  // namespace gmp
