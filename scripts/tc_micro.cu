// tcgen05 throughput microbenchmark: cycles per MMA (M=128, K=16, fp16, fp32 accumulate)
// for N in {32, 64, 96, 128, 192, 256}, A from TMEM (TS) or shared memory (SS), and
// cycles per tcgen05.cp 128x256b.  One CTA, back-to-back issue from one thread, clock64.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a scripts/tc_micro.cu -o tc_micro && ./tc_micro
#include <cstdio>
#include "../paper_2502_04077_b200/csrc/common.cuh"

using namespace ap;

// TS: 0 = SS, 1 = TS (A from TMEM), 2 = SS with the A collector (fill / lastuse pairs: A read once per 2 MMAs)
template <int N, int TS>
__global__ void mma_bench(long long* out, int iters) {
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
        const uint32_t a_addr = smem_u32(sm), b_addr = smem_u32(sm + 32768);
        const uint64_t adesc = umma_desc(a_addr, 2048, 128), bdesc = umma_desc(b_addr, N * 16, 128);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (TS == 1) mma_f16_ts(t + 256, t, bdesc, idesc, 1);
            else if (TS == 2 && (i & 1) == 0) mma_f16_afill(t + 256, adesc, bdesc, idesc, 1);
            else if (TS == 2) mma_f16_alast(t + 256, adesc, bdesc, idesc, 1);
            else mma_f16(t + 256, adesc, bdesc, idesc, 1);
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        out[0] = t1 - t0;
        // cp throughput
        t0 = clock64();
        for (int i = 0; i < iters; ++i) tmem_cp_128x256b(t + (i & 7) * 8, adesc);
        mma_commit(&bar);
        mbar_wait(&bar, 1);
        t1 = clock64();
        out[1] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (tid < 32) tmem_dealloc(t, 512);
}

template <int N, int TS>
void run(int iters) {
    long long* d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(mma_bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    mma_bench<N, TS><<<1, 128, 64 * 1024>>>(d, iters);
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    printf("N=%3d %s: %.1f cycles/MMA  (%.0f MAC/clk)   cp128x256b: %.1f cycles  %s\n", N, TS == 1 ? "TS" : TS == 2 ? "SS+collector" : "SS",
           (double)h[0] / iters, 128.0 * N * 16 * iters / h[0], (double)h[1] / iters, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    const int it = 4096;
    run<32, 1>(it);  run<32, 0>(it);  run<32, 2>(it);
    run<64, 1>(it);  run<64, 0>(it);  run<64, 2>(it);
    run<96, 1>(it);  run<96, 0>(it);  run<96, 2>(it);
    run<128, 1>(it); run<128, 0>(it); run<128, 2>(it);
    run<192, 1>(it); run<192, 0>(it); run<192, 2>(it);
    run<256, 1>(it); run<256, 0>(it); run<256, 2>(it);
    return 0;
}
