// Decode-engine GEMV (not a reference function: the reference has no model).  y[s] = W x[s] for
// the few sequences of a decode step, bf16 weights [N][K] row-major, fp32 accumulation — an
// HBM-streaming kernel: every weight byte is read exactly once per call with 16-byte loads, the
// NS activation rows sit in shared memory, each warp owns ROWS output rows and keeps ROWS x UNROLL
// independent 16-byte loads in flight per lane.
//
// Fused variants remove the neighbouring elementwise launches of a LLaMA layer:
//   * prologue RMSNORM: x = rmsnorm(x_in [+ residual]) * ln_w computed per CTA from the raw
//     activations (the 4096-float row is L2-resident); CTA 0 also writes the updated residual
//     stream to a separate buffer (every CTA still reads the old one);
//   * epilogue SILU: W = [gate; up] (2F rows): the warp that owns row i also owns row F + i and
//     writes act[i] = silu(gate_i) * up_i;
//   * epilogue ARGMAX: per-CTA best (value, lowest index) merged with a 64-bit atomicMax into
//     out_arg[s] (LM head + greedy sampling in one pass; `tokens` receives the index).
#include "common.cuh"

namespace ap {
namespace gemv {

constexpr int THREADS = 256, WARPS = THREADS / 32, UNROLL = 4, MAX_NS = 4;

enum Prologue { PRO_NONE = 0, PRO_RMSNORM = 1 };
enum Epilogue { EPI_STORE = 0, EPI_SILU = 1, EPI_ARGMAX = 2 };

struct Params {
    const __nv_bfloat16* W;  // [N][K]
    const __nv_bfloat16* x;  // [NS][K] activations (prologue input when RMSNORM)
    const __nv_bfloat16* residual;  // RMSNORM: h = x + residual when non-null
    __nv_bfloat16* residual_out;    // RMSNORM: h written here by CTA 0 (must not alias residual / x)
    const __nv_bfloat16* ln_w;
    float eps;
    __nv_bfloat16* y;        // STORE: [NS][N]; SILU: [NS][N/2]
    unsigned long long* arg; // ARGMAX: [NS] packed (orderable value << 32 | ~index)
    int64_t* tokens;         // ARGMAX: [NS] decoded indices (written by the last CTA)
    int32_t* counter;        // ARGMAX: CTA completion counter (self-resetting)
    int N, K, NS;
};

// 8 bf16 of a uint4 dotted with 8 floats
__device__ __forceinline__ float dot8(const uint4& w, const float* x) {
    const uint32_t v[4] = {w.x, w.y, w.z, w.w};
    float a = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        a = fmaf(__uint_as_float(v[i] << 16), x[2 * i], a);
        a = fmaf(__uint_as_float(v[i] & 0xffff0000u), x[2 * i + 1], a);
    }
    return a;
}

__device__ __forceinline__ uint32_t order_f32(float f) {  // monotone float -> u32
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

template <int ROWS, int NS, int PRO, int EPI>
__global__ void __launch_bounds__(THREADS) gemv_kernel(Params P) {
    extern __shared__ __align__(16) float xs[];  // [NS][K] fp32 activations
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int K = P.K;
    pdl_trigger();
    {  // before the producer of x has finished: pull this warp's first weight rows into L2
        const int g = blockIdx.x * WARPS + warp;
        const int per_group = (EPI == EPI_SILU) ? ROWS / 2 : ROWS;
        const int n_groups = (((EPI == EPI_SILU) ? P.N / 2 : P.N) + per_group - 1) / per_group;
        if (g < n_groups)
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
                int n;
                if constexpr (EPI == EPI_SILU) n = g * per_group + (r >> 1) + ((r & 1) ? P.N / 2 : 0);
                else n = g * ROWS + r;
                const char* row = reinterpret_cast<const char*>(P.W + (int64_t)min(n, P.N - 1) * K);
                for (int off = lane * 128; off < K * 2; off += 32 * 128) prefetch_l2(row + off);
            }
    }
    pdl_wait();
    // ---- activations -> shared memory (fp32), optionally normalised
    if constexpr (PRO == PRO_RMSNORM) {
        __shared__ float red[NS][WARPS];
        for (int s = 0; s < NS; ++s) {
            float ss = 0.f;
            for (int k = tid; k < K; k += THREADS) {
                float v = __bfloat162float(P.x[(int64_t)s * K + k]);
                if (P.residual) {
                    v += __bfloat162float(P.residual[(int64_t)s * K + k]);
                    v = __bfloat162float(__float2bfloat16_rn(v));  // the residual stream is bf16
                }
                xs[s * K + k] = v;
                ss = fmaf(v, v, ss);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
            if (lane == 0) red[s][warp] = ss;
        }
        __syncthreads();
        for (int s = 0; s < NS; ++s) {
            float ss = 0.f;
#pragma unroll
            for (int w = 0; w < WARPS; ++w) ss += red[s][w];
            const float inv = rsqrtf(ss / (float)K + P.eps);
            for (int k = tid; k < K; k += THREADS) {
                const float v = xs[s * K + k];
                if (blockIdx.x == 0 && P.residual_out) P.residual_out[(int64_t)s * K + k] = __float2bfloat16_rn(v);
                // y = bf16(h * inv * w), the arithmetic of ap_rmsnorm
                xs[s * K + k] = __bfloat162float(__float2bfloat16_rn(v * inv * __bfloat162float(P.ln_w[k])));
            }
        }
    } else {
        for (int i = tid; i < NS * K; i += THREADS) xs[i] = __bfloat162float(P.x[i]);
    }
    __syncthreads();

    // ---- persistent: warp-row groups g = blockIdx.x * WARPS + warp, + gridDim.x * WARPS, ...
    //      STORE / ARGMAX: weight rows g*ROWS ..; SILU: outputs g*ROWS/2 .., slot r = gate row (r even)
    //      or up row F + . (r odd) of output g*ROWS/2 + r/2
    const int n_out = (EPI == EPI_SILU) ? P.N / 2 : P.N;
    const int per_group = (EPI == EPI_SILU) ? ROWS / 2 : ROWS;
    const int n_groups = (n_out + per_group - 1) / per_group;
    const int chunks = K / 8;  // 16-byte chunks per row
    unsigned long long best[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) best[s] = 0;
    for (int g = blockIdx.x * WARPS + warp; g < n_groups; g += gridDim.x * WARPS) {
        const int row0 = g * ROWS, o0 = g * per_group;
        float acc[ROWS][NS];
#pragma unroll
        for (int r = 0; r < ROWS; ++r)
#pragma unroll
            for (int s = 0; s < NS; ++s) acc[r][s] = 0.f;
        const __nv_bfloat16* wrow[ROWS];
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            int n;
            if constexpr (EPI == EPI_SILU) n = o0 + (r >> 1) + ((r & 1) ? P.N / 2 : 0);
            else n = row0 + r;
            wrow[r] = P.W + (int64_t)min(n, P.N - 1) * K;  // clamped rows are computed and dropped
        }
        for (int c0 = lane; c0 < chunks; c0 += 32 * UNROLL) {
            uint4 w[UNROLL][ROWS];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u)
#pragma unroll
                for (int r = 0; r < ROWS; ++r) {
                    const int c = c0 + u * 32;
                    w[u][r] = c < chunks ? __ldcs(reinterpret_cast<const uint4*>(wrow[r]) + c) : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const int c = c0 + u * 32;
                if (c >= chunks) break;
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    float xv[8];
                    const float4 a = reinterpret_cast<const float4*>(xs + s * K + c * 8)[0];
                    const float4 b = reinterpret_cast<const float4*>(xs + s * K + c * 8)[1];
                    xv[0] = a.x; xv[1] = a.y; xv[2] = a.z; xv[3] = a.w; xv[4] = b.x; xv[5] = b.y; xv[6] = b.z; xv[7] = b.w;
#pragma unroll
                    for (int r = 0; r < ROWS; ++r) acc[r][s] += dot8(w[u][r], xv);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < ROWS; ++r)
#pragma unroll
            for (int s = 0; s < NS; ++s)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc[r][s] += __shfl_xor_sync(0xffffffffu, acc[r][s], o);

        if constexpr (EPI == EPI_STORE || EPI == EPI_ARGMAX) {
            if (P.y && lane == 0)
#pragma unroll
                for (int r = 0; r < ROWS; ++r)
                    if (row0 + r < P.N)
#pragma unroll
                        for (int s = 0; s < NS; ++s)
                            P.y[(int64_t)s * P.N + row0 + r] = __float2bfloat16_rn(acc[r][s]);
            if constexpr (EPI == EPI_ARGMAX) {  // bf16-rounded logits, ties -> lowest index (torch.argmax)
#pragma unroll
                for (int s = 0; s < NS; ++s)
#pragma unroll
                    for (int r = 0; r < ROWS; ++r)
                        if (row0 + r < P.N) {
                            const float v = __bfloat162float(__float2bfloat16_rn(acc[r][s]));
                            const unsigned long long key =
                                (unsigned long long)order_f32(v) << 32 | (uint32_t)~(uint32_t)(row0 + r);
                            best[s] = key > best[s] ? key : best[s];
                        }
            }
        } else {  // SILU
            const int F = P.N / 2;
            if (lane == 0)
#pragma unroll
                for (int j = 0; j < ROWS / 2; ++j) {
                    const int o = o0 + j;
                    if (o < F)
#pragma unroll
                        for (int s = 0; s < NS; ++s) {
                            // the gate/up GEMM output is bf16, then silu(g) * u as in ap_silu_mul
                            const float gt = __bfloat162float(__float2bfloat16_rn(acc[2 * j][s]));
                            const float up = __bfloat162float(__float2bfloat16_rn(acc[2 * j + 1][s]));
                            P.y[(int64_t)s * F + o] = __float2bfloat16_rn(gt / (1.f + __expf(-gt)) * up);
                        }
                }
        }
    }

    if constexpr (EPI == EPI_ARGMAX) {
        __shared__ unsigned long long cta_best[NS][WARPS];
#pragma unroll
        for (int s = 0; s < NS; ++s)
            if (lane == 0) cta_best[s][warp] = best[s];
        __syncthreads();
        if (tid < NS) {
            unsigned long long b = 0;
            for (int w = 0; w < WARPS; ++w) b = cta_best[tid][w] > b ? cta_best[tid][w] : b;
            atomicMax(P.arg + tid, b);
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            __shared__ int last;
            last = atomicAdd(P.counter, 1) == (int)gridDim.x - 1;
            if (last) {
                for (int s = 0; s < NS; ++s) {
                    const unsigned long long b = atomicExch(P.arg + s, 0ull);  // reset for the next call
                    P.tokens[s] = (int64_t)(uint32_t)~(uint32_t)(b & 0xffffffffu);
                }
                *P.counter = 0;
            }
        }
    }
}

template <int ROWS, int NS, int PRO, int EPI>
int launch(const Params& P, cudaStream_t st) {
    // SILU: a warp's ROWS weight rows are ROWS/2 (gate, up) pairs
    const int outs = (EPI == EPI_SILU) ? P.N / 2 : P.N;
    const int per_cta = WARPS * ((EPI == EPI_SILU) ? ROWS / 2 : ROWS);
    const size_t smem = (size_t)NS * P.K * 4;
    auto k = gemv_kernel<ROWS, NS, PRO, EPI>;
    static bool attr_set = false;
    if (!attr_set) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
    // persistent: at most one wave of resident CTAs, so the activation prologue runs once per CTA
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, THREADS, smem);
    const int cap = ap_device_sm_count() * (occ > 0 ? occ : 1);
    int grid = (outs + per_cta - 1) / per_cta;
    grid = grid < cap ? grid : cap;
    launch_ex(k, dim3(grid), dim3(THREADS), smem, st, 1, P);
    return launch_status("gemv_kernel");
}

template <int PRO, int EPI>
int dispatch_ns(const Params& P, int rows, cudaStream_t st) {
#define AP_GEMV_NS(R)                                                   \
    switch (P.NS) {                                                     \
        case 1: return launch<R, 1, PRO, EPI>(P, st);                   \
        case 2: return launch<R, 2, PRO, EPI>(P, st);                   \
        case 3: return launch<R, 3, PRO, EPI>(P, st);                   \
        default: return launch<R, 4, PRO, EPI>(P, st);                  \
    }
    if constexpr (EPI != EPI_SILU) {  // SILU needs (gate, up) row pairs
        if (rows == 1) { AP_GEMV_NS(1) }
    }
    if (rows == 2) { AP_GEMV_NS(2) }
    AP_GEMV_NS(4)
#undef AP_GEMV_NS
}

}  // namespace gemv
}  // namespace ap

using namespace ap;

extern "C" int ap_gemv(const void* W, const void* x, void* y, int32_t N, int32_t K, int32_t n_seq,
                       int32_t rows_per_warp, int32_t flags, const void* residual, void* residual_out,
                       const void* ln_w, float eps, void* arg_workspace, void* tokens, void* stream) {
    using namespace gemv;
    AP_REQUIRE(W && x && N > 0 && K > 0, AP_EPARAM, "bad GEMV operands");
    AP_REQUIRE(K % 8 == 0, AP_EPARAM, "K must be a multiple of 8 (16-byte rows)");
    AP_REQUIRE(n_seq >= 1 && n_seq <= MAX_NS, AP_EPARAM, "ap_gemv serves 1..4 activation rows");
    AP_REQUIRE(rows_per_warp == 1 || rows_per_warp == 2 || rows_per_warp == 4, AP_EPARAM, "rows_per_warp 1/2/4");
    AP_REQUIRE((int64_t)n_seq * K * 4 <= 200 * 1024, AP_EPARAM, "activations exceed shared memory");
    const int pro = flags & 1 ? PRO_RMSNORM : PRO_NONE;
    const int epi = (flags >> 1) & 3;
    AP_REQUIRE(epi <= EPI_ARGMAX, AP_EPARAM, "bad epilogue");
    AP_REQUIRE(pro == PRO_NONE || ln_w, AP_EPARAM, "RMSNORM prologue needs ln_w");
    AP_REQUIRE(epi != EPI_SILU || (N % 2 == 0 && rows_per_warp >= 2), AP_EPARAM,
               "SILU epilogue needs an even N ([gate; up]) and >= 2 rows per warp");
    AP_REQUIRE(epi != EPI_ARGMAX || (arg_workspace && tokens), AP_EPARAM, "ARGMAX needs its workspace and tokens");
    AP_REQUIRE(epi == EPI_ARGMAX || y, AP_EPARAM, "null output");
    Params P{};
    P.W = (const __nv_bfloat16*)W;
    P.x = (const __nv_bfloat16*)x;
    P.residual = (const __nv_bfloat16*)residual;
    P.residual_out = (__nv_bfloat16*)residual_out;
    AP_REQUIRE(!residual_out || (residual_out != residual && residual_out != x), AP_EPARAM,
               "residual_out must not alias the residual or x");
    P.ln_w = (const __nv_bfloat16*)ln_w;
    P.eps = eps;
    P.y = (__nv_bfloat16*)y;
    P.arg = (unsigned long long*)arg_workspace;                       // [4] u64, zero-initialised once
    P.counter = arg_workspace ? (int32_t*)((unsigned long long*)arg_workspace + MAX_NS) : nullptr;  // + int32
    P.tokens = (int64_t*)tokens;
    P.N = N;
    P.K = K;
    P.NS = n_seq;
    cudaStream_t st = as_stream(stream);
    if (pro == PRO_RMSNORM) {
        if (epi == EPI_STORE) return dispatch_ns<PRO_RMSNORM, EPI_STORE>(P, rows_per_warp, st);
        if (epi == EPI_SILU) return dispatch_ns<PRO_RMSNORM, EPI_SILU>(P, rows_per_warp, st);
        return dispatch_ns<PRO_RMSNORM, EPI_ARGMAX>(P, rows_per_warp, st);
    }
    if (epi == EPI_STORE) return dispatch_ns<PRO_NONE, EPI_STORE>(P, rows_per_warp, st);
    if (epi == EPI_SILU) return dispatch_ns<PRO_NONE, EPI_SILU>(P, rows_per_warp, st);
    return dispatch_ns<PRO_NONE, EPI_ARGMAX>(P, rows_per_warp, st);
}
