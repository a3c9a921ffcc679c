// TMA tensor-map copies and 128-byte-swizzled K-major operand descriptors for tcgen05 (sm_100a).
// Used by the calibration pass (attention.cu) and the skinny tensor-core GEMM (gemm_tc.cu).
#pragma once

#include <cuda.h>  // CUtensorMap (driver types only; the encoder comes via cudaGetDriverEntryPoint)
#include <cudaTypedefs.h>

#include "common.cuh"

namespace ap {

// UMMA shared-memory descriptor for a K-major operand in the canonical 128-byte-swizzled layout
// (8-row x 128-byte atoms, atom base 1024-aligned; the K offset inside an atom is added to the start
// address in 32-byte steps of 16 bf16).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;                      // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;            // SBO: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                      // descriptor version (Blackwell)
    d |= (uint64_t)2 << 61;                      // SWIZZLE_128B
    return d;
}

// as desc_sw128 with an explicit stride between 8-row core-matrix groups (bytes, multiple of 16)
__device__ __forceinline__ uint64_t desc_sw128_sbo(uint32_t saddr, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
        :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
           "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

static inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2-D bf16 tensor map over a row-major [rows][cols] matrix, boxes {64 columns, box_rows rows},
// 128-byte swizzle (the layout desc_sw128 describes).  Returns false if the encoder fails.
static inline bool make_tmap_bf16_sw128(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                                        uint32_t box_rows) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    const cuuint32_t box[2] = {64, box_rows}, estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 4-D bf16 view of a row-major [rows][cols] matrix (rows % 8 == 0, cols % 64 == 0) whose boxes
// {64, 8, slabs, groups} land in shared memory as [group][slab][8 rows][128 B], 128-byte swizzled:
// per slab the K-major SW128 operand layout with 8-row groups slabs x 1024 B apart (desc_sw128_sbo),
// and one copy covers every slab of a row group, so each row's slabs x 128 B are requested together.
static inline bool make_tmap_bf16_sw128_grouped(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                                                uint32_t slabs, uint32_t groups) {
    auto enc = tensor_map_encoder();
    if (!enc || rows % 8 || cols % 64) return false;
    const cuuint64_t dims[4] = {64, 8, (cuuint64_t)(cols / 64), (cuuint64_t)(rows / 8)};
    const cuuint64_t strides[3] = {(cuuint64_t)cols * 2, 128, (cuuint64_t)cols * 16};
    const cuuint32_t box[4] = {64, 8, slabs, groups}, estr[4] = {1, 1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace ap
