// HBM read-streaming microbenchmark on one persistent CTA per SM: how the way bytes are moved
// into the SM (cp.async.bulk copies of S bytes with D in flight, issued by one thread or by
// several lanes; 16-byte LDG into registers) sets the achievable read bandwidth.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a scripts/stream_micro.cu -o /tmp/sm && /tmp/sm
#include <cstdio>
#include <vector>
#include "../paper_2502_04077_b200/csrc/common.cuh"

using namespace ap;

// mode 0: thread 0 issues one bulk copy of S bytes per ring slot; mode 1: lanes of warp 0 issue
// S/PIECE copies per slot.  The CTA waits each slot (all threads), then re-issues it.
__global__ void bulk_stream(const uint8_t* src, int64_t bytes_per_cta, int S, int D, int piece, unsigned long long* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[32];
    const int tid = threadIdx.x;
    const uint8_t* base = src + (int64_t)blockIdx.x * bytes_per_cta;
    const int n = (int)(bytes_per_cta / S);
    if (tid == 0)
        for (int i = 0; i < D; ++i) mbar_init(&bar[i], 1);
    __syncthreads();
    auto issue = [&](int j) {
        const int slot = j % D;
        if (piece >= S) {
            if (tid == 0) {
                mbar_arrive_tx(&bar[slot], S);
                bulk_g2s(sm + slot * S, base + (int64_t)j * S, S, &bar[slot]);
            }
        } else if (tid < 32) {
            if (tid == 0) mbar_arrive_tx(&bar[slot], S);
            __syncwarp();
            for (int p = tid; p < S / piece; p += 32)
                bulk_g2s(sm + slot * S + p * piece, base + (int64_t)j * S + p * piece, piece, &bar[slot]);
        }
    };
    for (int j = 0; j < D && j < n; ++j) issue(j);
    unsigned long long acc = 0;
    for (int j = 0; j < n; ++j) {
        mbar_wait_spin(&bar[j % D], (j / D) & 1);
        acc += sm[(j % D) * S + tid];
        __syncthreads();
        if (j + D < n) issue(j + D);
    }
    if (acc == 0x1234567) sink[0] = acc;
}

// 16-byte loads into registers, U independent loads per thread in flight
template <int U>
__global__ void ldg_stream(const uint4* src, int64_t vec_per_cta, unsigned long long* sink) {
    const uint4* base = src + (int64_t)blockIdx.x * vec_per_cta;
    uint32_t acc = 0;
    for (int64_t i = threadIdx.x; i < vec_per_cta; i += (int64_t)blockDim.x * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t k = i + (int64_t)u * blockDim.x;
            v[u] = k < vec_per_cta ? __ldcs(base + k) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc == 0x1234567) sink[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t per_cta = 8ll << 20;  // 8 MiB per SM -> ~1.2 GB total
    const int64_t total = per_cta * sms;
    uint8_t* buf;
    unsigned long long* sink;
    cudaMalloc(&buf, total);
    cudaMalloc(&sink, 8);
    cudaMemset(buf, 1, total);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    auto time_it = [&](auto&& launch) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        return total / (best * 1e-3) / 1e9;
    };
    for (int S : {4096, 8192, 16384, 32768, 65536}) {
        for (int D : {2, 3, 4, 6, 8, 12, 16}) {
            if ((int64_t)S * D > 192 * 1024) continue;
            for (int piece : {S, 4096, 1024}) {
                if (piece > S || (piece != S && piece == 4096 && S == 4096)) continue;
                for (int threads : {128, 512}) {
                    double gbs = time_it([&] {
                        bulk_stream<<<sms, threads, S * D>>>(buf, per_cta, S, D, piece, sink);
                    });
                    printf("bulk S=%6d D=%2d piece=%6d threads=%3d  %7.1f GB/s  (%s)\n", S, D, piece, threads, gbs,
                           cudaGetErrorString(cudaGetLastError()));
                }
            }
        }
    }
    for (int threads : {256, 512, 1024}) {
        double g2 = time_it([&] { ldg_stream<2><<<sms, threads>>>((const uint4*)buf, per_cta / 16, sink); });
        double g4 = time_it([&] { ldg_stream<4><<<sms, threads>>>((const uint4*)buf, per_cta / 16, sink); });
        double g8 = time_it([&] { ldg_stream<8><<<sms, threads>>>((const uint4*)buf, per_cta / 16, sink); });
        printf("ldg threads=%4d  U=2 %7.1f  U=4 %7.1f  U=8 %7.1f GB/s\n", threads, g2, g4, g8);
    }
    return 0;
}
