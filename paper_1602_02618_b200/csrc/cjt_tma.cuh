// TMA tensor-map encoding through the driver entry point (no -lcuda link),
// shared by the kernels that move tiles with cp.async.bulk.tensor.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "cjt_internal.cuh"

namespace cjt {

inline PFN_cuTensorMapEncodeTiled_v12000 tmap_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// rank-R tiled map: dims innermost first, strides[R-1] in bytes for dims 1..R-1
inline int tmap_make(CUtensorMap* map, CUtensorMapDataType dt, int rank, const void* base, const cuuint64_t* dims,
                     const cuuint64_t* strides, const cuuint32_t* box, CUtensorMapSwizzle swz) {
  auto fn = tmap_encode_fn();
  if (!fn) return fail(CJT_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUresult r = fn(map, dt, (cuuint32_t)rank, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CJT_ECUDA, "cuTensorMapEncodeTiled failed");
  return CJT_OK;
}

}  // namespace cjt
