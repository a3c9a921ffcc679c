// CTA-pair tcgen05 microbenchmark: cycles per tcgen05.mma.cta_group::2 (M = 256 over two SMs, K = 16,
// fp16, fp32 accumulate, A and B from shared memory, B split N/2 per CTA) for N in {32, 64, 96, 128},
// against the single-CTA M = 128 form — does a pair MMA cost the same per instruction as a single one
// (the ~46-cycle small-N floor of scripts/tc_micro.cu), i.e. twice the pixels per instruction?
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a scripts/tc_pair_micro.cu -o tc_pair_micro
#include <cstdio>
#include "../paper_2502_04077_b200/csrc/common.cuh"

using namespace ap;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N, int PAIR>
__global__ void __cluster_dims__(2, 1, 1) pair_bench(long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    const uint32_t rank = cluster_rank();
    for (int i = tid; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (tid < 32) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                         :: "r"(smem_u32(&tslot)), "r"(512) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            tmem_alloc(&tslot, 512);
        }
    }
    if (tid == 0) mbar_init(&bar, 1);
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t t = tslot;
    const uint32_t a_addr = smem_u32(sm), b_addr = smem_u32(sm + 32768);
    if (PAIR) {
        if (rank == 0 && tid == 0) {
            const uint32_t idesc = idesc_f16_f32(256, N, 0);
            const uint64_t adesc = umma_desc(a_addr, 2048, 128), bdesc = umma_desc(b_addr, (N / 2) * 16, 128);
            const long long t0 = clock64();
            for (int i = 0; i < iters; ++i)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                    :: "r"(t + 256), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(1) : "memory");
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                         :: "r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
            mbar_wait(&bar, 0);
            out[0] = clock64() - t0;
        } else if (rank == 1 && tid == 0) {
            mbar_wait(&bar, 0);
        }
    } else if (rank == 0 && tid == 0) {
        const uint32_t idesc = idesc_f16_f32(128, N, 0);
        const uint64_t adesc = umma_desc(a_addr, 2048, 128), bdesc = umma_desc(b_addr, N * 16, 128);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) mma_f16(t + 256, adesc, bdesc, idesc, 1);
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        out[0] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (tid < 32) {
        if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(t), "r"(512) : "memory");
        else tmem_dealloc(t, 512);
    }
}

template <int N, int PAIR>
void run(int iters) {
    long long* d;
    cudaMalloc(&d, 16);
    cudaMemset(d, 0, 16);
    cudaFuncSetAttribute(pair_bench<N, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    pair_bench<N, PAIR><<<2, 128, 64 * 1024>>>(d, iters);
    const cudaError_t e = cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%s N=%3d: %6.1f cycles/MMA  (%.0f MAC/clk per SM)  %s\n", PAIR ? "pair M=256" : "single M=128", N,
           (double)h / iters, (double)128 * N * 16 * iters / h, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<32, 0>(4096);
    run<32, 1>(4096);
    run<64, 0>(4096);
    run<64, 1>(4096);
    run<96, 0>(4096);
    run<96, 1>(4096);
    run<128, 0>(4096);
    run<128, 1>(4096);
    return 0;
}
