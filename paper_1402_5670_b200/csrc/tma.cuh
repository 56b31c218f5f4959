// Tensor-map (TMA descriptor) construction for the bulk tensor copies. The
// driver entry point is fetched through the runtime (no libcuda link).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace slb {

static PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        SL_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) throw SlError(SL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    return enc;
}

// fp64 tensor of rank <= 4 (dims[0] fastest, strides in bytes for dims 1..),
// 128-byte swizzle (box[0] * 8 must be 128)
static CUtensorMap tma_map_f64(const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                               const cuuint32_t* box) {
    CUtensorMap m;
    const cuuint32_t es[4] = {1, 1, 1, 1};
    const CUresult r = tma_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, static_cast<cuuint32_t>(rank),
                                     const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw SlError(SL_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    return m;
}

}  // namespace slb
