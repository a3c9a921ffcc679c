// Accumulator dependence of tcgen05.mma (M=128, K=16, fp16 -> fp32, SS): cycles per MMA when every MMA
// accumulates into the same TMEM columns (a dependent chain, as the forecaster's 9 MMAs per a1 row and
// output-row group) versus round-robin over ND disjoint accumulators (independent MMAs).
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a scripts/tc_micro3.cu -o tc_micro3
#include <cstdio>
#include "../paper_2502_04077_b200/csrc/common.cuh"

using namespace ap;

template <int N, int ND>
__global__ void dep_bench(long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    const int tid = threadIdx.x;
    for (int i = tid; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (tid < 32) tmem_alloc(&tslot, 512);
    if (tid == 0) mbar_init(&bar, 1);
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t = tslot;
    if (tid == 0) {
        const uint32_t idesc = idesc_f16_f32(128, N, 0);
        const uint64_t adesc = umma_desc(smem_u32(sm), 2048, 128), bdesc = umma_desc(smem_u32(sm + 32768), N * 16, 128);
        const long long t0 = clock64();
        for (int i = 0; i < iters; i += ND)
#pragma unroll
            for (int d = 0; d < ND; ++d) mma_f16(t + d * N, adesc, bdesc, idesc, 1);
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        out[0] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (tid < 32) tmem_dealloc(t, 512);
}

template <int N, int ND>
void run(int iters) {
    long long* d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(dep_bench<N, ND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    dep_bench<N, ND><<<1, 128, 64 * 1024>>>(d, iters);
    long long h = 0;
    const cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("N=%3d, %d accumulator(s) round-robin: %6.1f cycles/MMA  %s\n", N, ND, (double)h / iters, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    const int it = 4096;
    run<32, 1>(it);  run<32, 2>(it);  run<32, 4>(it);  run<32, 8>(it);
    run<64, 1>(it);  run<64, 2>(it);  run<64, 4>(it);
    run<96, 1>(it);  run<96, 2>(it);  run<96, 4>(it);
    return 0;
}
