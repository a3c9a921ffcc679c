// TMEM read / write throughput microbenchmark: cycles per tcgen05.ld (32x32b) for 4 / 8 / 16 warps
// (warp w reads lane quadrant w % 4), x16 pairs (the forecaster epilogue's pattern) and x32 loads,
// and per tcgen05.st x32.  One CTA, clock64 around the loop of each warp; bytes/clk over the CTA.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a scripts/tmem_micro.cu -o tmem_micro && ./tmem_micro
#include <cstdio>
#include "../paper_2502_04077_b200/csrc/common.cuh"

using namespace ap;

__device__ __forceinline__ void ld8(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void wait8(uint32_t (&r)[8]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7])
                 :: "memory");
}

// MODE 0: two x16 loads then wait (per 32 columns); 1: one x32 load then wait; 2: x32 load, no wait until
// the next (double-buffered); 3: tcgen05.st x32 (zero), wait::st every 5
template <int MODE>
__global__ void tmem_bench(long long* out, float* sink, int iters) {
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t base = tslot + ((uint32_t)((warp & 3) * 32) << 16);
    float acc = 0.f;
    uint32_t ra[16], rb[16], q0[32], q1[32];
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const uint32_t col = base + (uint32_t)((i * 32 + (warp >> 2) * 160) & 511);
        if (MODE == 0) {
            tmem_ld16_start(col, ra);
            tmem_ld16_start(col + 16, rb);
            tmem_ld_wait(ra);
            tmem_ld_wait(rb);
#pragma unroll
            for (int n = 0; n < 16; ++n) acc += __uint_as_float(ra[n]) + __uint_as_float(rb[n]);
        } else if (MODE == 1) {
            tmem_ld32_start(col, q0);
            tmem_ld_wait(q0);
#pragma unroll
            for (int n = 0; n < 32; ++n) acc += __uint_as_float(q0[n]);
        } else if (MODE == 2) {
            if (i & 1) {
                tmem_ld32_start(col, q1);
                tmem_ld_wait(q1);
#pragma unroll
                for (int n = 0; n < 32; ++n) acc += __uint_as_float(q1[n]);
            } else {
                tmem_ld32_start(col, q0);
                tmem_ld_wait(q0);
#pragma unroll
                for (int n = 0; n < 32; ++n) acc += __uint_as_float(q0[n]);
            }
        } else if (MODE == 4) {  // x16 pairs, next 32 columns in flight while these are consumed
            if (i == 0) { tmem_ld16_start(col, ra); tmem_ld16_start(col + 16, rb); }
            tmem_ld_wait(ra);
            tmem_ld_wait(rb);
            uint32_t ca[16], cb[16];
#pragma unroll
            for (int n = 0; n < 16; ++n) { ca[n] = ra[n]; cb[n] = rb[n]; }
            const uint32_t nx = base + (uint32_t)(((i + 1) * 32 + (warp >> 2) * 160) & 511);
            tmem_ld16_start(nx, ra);
            tmem_ld16_start(nx + 16, rb);
#pragma unroll
            for (int n = 0; n < 16; ++n) acc += __uint_as_float(ca[n]) * __uint_as_float(cb[n]) + acc * 0.5f;
        } else if (MODE == 5) {  // four x8 loads, one wait
            uint32_t e0[8], e1[8], e2[8], e3[8];
            ld8(col, e0); ld8(col + 8, e1); ld8(col + 16, e2); ld8(col + 24, e3);
            wait8(e0); wait8(e1); wait8(e2); wait8(e3);
#pragma unroll
            for (int n = 0; n < 8; ++n) acc += __uint_as_float(e0[n]) + __uint_as_float(e1[n]) + __uint_as_float(e2[n]) + __uint_as_float(e3[n]);
        } else if (MODE == 6) {  // 64 columns as four x16 loads, one wait (counted per 32 columns)
            if (i & 1) continue;
            uint32_t e2[16], e3[16];
            tmem_ld16_start(col, ra); tmem_ld16_start(col + 16, rb); tmem_ld16_start(col + 32, e2); tmem_ld16_start(col + 48, e3);
            tmem_ld_wait(ra); tmem_ld_wait(rb); tmem_ld_wait(e2); tmem_ld_wait(e3);
#pragma unroll
            for (int n = 0; n < 16; ++n) acc += __uint_as_float(ra[n]) + __uint_as_float(rb[n]) + __uint_as_float(e2[n]) + __uint_as_float(e3[n]);
        } else {
            tmem_zero32(col);
            if (i % 5 == 4) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    const long long t1 = clock64();
    if (MODE == 4) tmem_ld_wait(ra), tmem_ld_wait(rb);
    if ((tid & 31) == 0) out[warp] = t1 - t0;
    sink[tid] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tslot, 512);
}

template <int MODE>
void run(int warps, int iters) {
    long long* d;
    float* s;
    cudaMalloc(&d, 64 * 8);
    cudaMalloc(&s, 1024 * 4);
    tmem_bench<MODE><<<1, warps * 32>>>(d, s, iters);
    long long h[64];
    cudaMemcpy(h, d, warps * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
    const double bytes = (double)warps * 32 * 32 * 4 * iters;
    const char* name[] = {"ld x16 pair", "ld x32", "ld x32 alt regs", "st x32", "ld x16 pair dbuf+fma", "ld 4 x8", "ld 4 x16 (64c)"};
    printf("%-16s warps %2d: %7.1f cycles per 32-col op per warp, %6.1f B/clk per SM  %s\n", name[MODE], warps,
           (double)mx / iters, bytes / mx, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
    cudaFree(s);
}

int main() {
    for (int w : {4, 8, 16}) {
        run<0>(w, 4096);
        run<1>(w, 4096);
        run<2>(w, 4096);
        run<3>(w, 4096);
        run<4>(w, 4096);
        run<5>(w, 4096);
        run<6>(w, 4096);
    }
    return 0;
}
