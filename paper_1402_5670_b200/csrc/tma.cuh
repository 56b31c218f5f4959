// Tensor-map (TMA descriptor) construction and the bulk-tensor copy helpers.
// The driver entry point is fetched through the runtime (no libcuda link).
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

// fp64 tensor of rank <= 5 (dims[0] fastest, strides in bytes for dims 1..)
static CUtensorMap tma_map_f64(const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                               const cuuint32_t* box, CUtensorMapSwizzle swz) {
    CUtensorMap m;
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    const CUresult r = tma_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, static_cast<cuuint32_t>(rank),
                                     const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                     swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw SlError(SL_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    return m;
}

// 16-byte slot of byte offset `b` inside a buffer written / read by a TMA copy
// with 64-byte swizzle (bits [4,5] ^= bits [7,8]; the buffer is 1024-aligned)
__device__ __forceinline__ int sw64_slot(int b) { return (b ^ (((b >> 7) & 3) << 4)) >> 4; }
// ... with 128-byte swizzle (bits [4,6] ^= bits [7,9])
__device__ __forceinline__ int sw128_slot(int b) { return (b ^ (((b >> 7) & 7) << 4)) >> 4; }

// 5D bulk tensor store smem -> global (bulk async group of the calling thread)
__device__ __forceinline__ void tma_store_5d(const CUtensorMap* m, const void* smem, int c0, int c1, int c2, int c3,
                                             int c4) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(sa)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// 5D bulk tensor load global -> smem, completing `bytes` on the mbarrier `bar`
// (the issuing thread arms the barrier with the expected transaction count)
__device__ __forceinline__ void tma_load_5d(const CUtensorMap* m, void* smem, uint64_t* bar, unsigned bytes, int c0,
                                            int c1, int c2, int c3, int c4) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const unsigned ba = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];" ::"r"(sa),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(ba)
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    const unsigned ba = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(bytes) : "memory");
}
// 3D bulk tensor load (the barrier armed separately with the total bytes)
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* m, void* smem, uint64_t* bar, int c0, int c1, int c2) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const unsigned ba = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            sa),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(ba)
        : "memory");
}
// 3D bulk tensor store (no commit: the caller commits the group)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* m, const void* smem, int c0, int c1, int c2) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(sa)
                 : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    const unsigned ba = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ba), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, unsigned phase) {
    const unsigned ba = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(ba),
        "r"(phase)
        : "memory");
}

}  // namespace slb
