// tcgen05 issue-pattern microbenchmark: cycles per MMA (M=128, K=16, fp16 -> fp32) when consecutive MMAs
// change (a) nothing, (b) the A / B / D addresses, (c) N, (d) the forecaster's real 63-MMA band pattern.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a scripts/tc_micro2.cu -o scripts/tc_micro2
#include <cstdio>
#include "../paper_2502_04077_b200/csrc/common.cuh"

using namespace ap;

__global__ void bench(long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    const int tid = threadIdx.x;
    for (int i = tid; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (tid < 32) tmem_alloc(&tslot, 512);
    if (tid == 0) mbar_init(&bar, 1);
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t = tslot;
    if (tid == 0) {
        const uint32_t a_addr = smem_u32(sm), b_addr = smem_u32(sm + 96 * 1024);
        const int PL = 9 * 130 * 16;  // a1 plane bytes as in the forecaster
        uint32_t ph = 0;
        for (int mode = 0; mode < 5; ++mode) {
            long long t0 = clock64();
            for (int i = 0; i < iters; ++i) {
                if (mode == 0) {  // identical MMAs, N = 64
                    mma_f16(t, umma_desc(a_addr, PL, 128), umma_desc(b_addr, 1536, 128), idesc_f16_f32(128, 64, 0), 1);
                } else if (mode == 1) {  // A walks 7 rows x 3 shifts, B 6 tiles, D 5 regions; N = 64
                    const int r = i % 7, dj = (i / 7) % 3, bt = i % 6, dd = i % 5;
                    mma_f16(t + dd * 32, umma_desc(a_addr + (r * 130 + dj) * 16, PL, 128),
                            umma_desc(b_addr + bt * 3072, 1536, 128), idesc_f16_f32(128, 64, 0), 1);
                } else if (mode == 2) {  // identical addresses, N cycles 32 / 64 / 96
                    const int n = 32 * (1 + i % 3);
                    mma_f16(t, umma_desc(a_addr, PL, 128), umma_desc(b_addr, 1536, 128), idesc_f16_f32(128, n, 0), 1);
                } else if (mode == 3) {  // identical, N = 96
                    mma_f16(t, umma_desc(a_addr, PL, 128), umma_desc(b_addr, 1536, 128), idesc_f16_f32(128, 96, 0), 1);
                } else {  // the band: 7 a1 rows feeding n = 2,2,1 | 1,2,3,2 outputs, x 3 dj x 3 hi/lo
                    static const int nn[7] = {2, 2, 1, 1, 2, 3, 2};
                    const int r = (i / 9) % 7, dj = (i / 3) % 3, v = i % 3;
                    mma_f16(t + (r < 3 ? 0 : 64) + 0, umma_desc(a_addr + (v == 2 ? 2 * PL : 0) + (r * 130 + dj) * 16, PL, 128),
                            umma_desc(b_addr + ((v == 1) * 3 + dj) * 3072, 1536, 128), idesc_f16_f32(128, 32 * nn[r], 0), 1);
                }
            }
            mma_commit(&bar);
            mbar_wait(&bar, ph);
            ph ^= 1;
            out[mode] = clock64() - t0;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tid < 32) tmem_dealloc(t, 512);
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    const int it = 63 * 64;
    bench<<<1, 128, 160 * 1024>>>(d, it);
    long long h[5];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const char* names[5] = {"identical N=64", "walking A/B/D N=64", "N cycling 32/64/96", "identical N=96",
                            "forecaster band pattern"};
    for (int m = 0; m < 5; ++m) printf("%-26s %.1f cycles/MMA\n", names[m], (double)h[m] / it);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
