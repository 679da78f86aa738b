// Host-side encoding of the 3-D tensor maps the DMMA tile engine (dmma_engine.cuh) loads its
// A / B^T operands through: a complex matrix [rows][cols] with row stride ld (complex elements),
// replicated per energy point at a stride of estride complex elements, seen by the TMA unit as
// FLOAT64 {2*cols, rows, energies}, box {16 doubles = 8 complex, 64 rows, 1}, SWIZZLE_128B,
// zero fill outside the tensor.  cuTensorMapEncodeTiled is fetched through the runtime's driver
// entry point (no -lcuda link).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace findb200 {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// Returns false when the driver entry point is unavailable or the encoding is rejected.
inline bool encode_complex_tmap(CUtensorMap* out, const void* base, int64_t cols, int64_t rows, int64_t ld,
                                int64_t estride, int64_t energies = 0xffff) {
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn) return false;
  if (cols < 1) cols = 1;
  if (rows < 1) rows = 1;
  const cuuint64_t dims[3] = {(cuuint64_t)(2 * cols), (cuuint64_t)rows, (cuuint64_t)energies};
  const cuuint64_t strides[2] = {(cuuint64_t)(ld * 16), (cuuint64_t)(estride * 16)};
  const cuuint32_t box[3] = {16, 64, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace findb200
