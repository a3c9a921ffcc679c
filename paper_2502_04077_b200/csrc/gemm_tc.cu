// Skinny tensor-core GEMM for batched decode: y[s][n] = sum_k x[s][k] W[n][k] for up to 16
// sequences (bf16 in / out, fp32 accumulate).  Not a reference function (the reference has no
// model): it carries the projections of the batch-5..16 decode engine (BASELINE cfg5), where the
// SIMT ap_gemv runs out of FMA throughput.
//
// tcgen05 formulation: M = 128 weight rows per MMA, N = 16 (the sequences, zero-padded by the
// tensor map's out-of-bounds fill), K = 16.  A stage is 128 rows x 256 K-elements of W (four TMA
// boxes {64, 128} in the 128-byte-swizzled K-major layout, 64 KB) plus the matching 16 x 256 slice
// of x (8 KB); one thread issues its 16 MMAs into a TMEM accumulator (128 lanes x 16 columns).
// Roles: warp 0 TMA producer, warp 1 MMA issuer, warps 2-5 epilogue (lane = weight row).
//
// Work split.  The (row tile, stage) sequence of the whole GEMM is cut into gridDim.x equal
// contiguous ranges, one per CTA (a persistent one-wave grid), so every SM streams the same number
// of bytes whatever N is.  A tile covered by several CTAs ("pieces") gets each piece's fp32 partial
// in a workspace slot; the last piece to finish (per-tile counter, self-resetting) adds them in
// piece order — deterministic — and writes bf16.  A tile covered by one CTA is written directly.
#include <cstdlib>

#include "common.cuh"
#include "tma.cuh"

namespace ap {
namespace gtc {

#ifndef GTC_SLABS
#define GTC_SLABS 2
#endif
#ifndef GTC_NST
#define GTC_NST 3
#endif
#ifndef GTC_CTAS
#define GTC_CTAS 1
#endif
constexpr int BM = 128, BN = 16, SLAB = 64, SLABS = GTC_SLABS;  // stage = SLABS slabs of 64 K-elements
constexpr int A_BOX = BM * SLAB * 2, B_BOX = BN * SLAB * 2;  // 16 KB, 2 KB
constexpr int STAGE = SLABS * (A_BOX + B_BOX);               // 36 KB
constexpr int NST = GTC_NST, NACC = 2;
constexpr int CTAS_PER_SM = GTC_CTAS;
constexpr int THREADS = 192;
// workspace: a fixed counter area first (so GEMMs of any shape can share one workspace: every one
// of them leaves its counters at zero), then the fp32 partials
constexpr int MAX_TILES = 4096;  // N <= 524288
constexpr int64_t COUNTER_BYTES = MAX_TILES * 4;

struct Params {
    __nv_bfloat16* y;        // [S][N]
    float* ws;               // [tiles][max_pieces][S][BM] partials
    int32_t* counters;       // [tiles], zero between launches
    int N, K, S, n_tiles, stages_per_tile, max_pieces;
    int grouped;             // W tensor map is the grouped 4-D view (one copy per stage)
    int trace;               // debug (ATTNPRED_GEMM_TRACE=1): per-CTA globaltimer events into g_trace
};

__device__ unsigned long long g_trace[160 * 12];
__device__ __forceinline__ void trace_event(const Params& P, int e) {
    if (P.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_trace[blockIdx.x * 12 + e] = t;
    }
}

struct Smem {
    static constexpr int off_stage = 0;  // [NST], 1024-aligned
    static constexpr int off_bar = NST * STAGE;
    static constexpr int total = off_bar + 8 * (2 * NST + 2 * NACC) + 16 + 1024;
};

// the CTA's contiguous range of the global (tile, stage) sequence
__device__ __forceinline__ void cta_range(const Params& P, int c, int64_t& g0, int64_t& g1) {
    const int64_t T = (int64_t)P.n_tiles * P.stages_per_tile;
    g0 = T * c / gridDim.x;
    g1 = T * (c + 1) / gridDim.x;
}
// first CTA whose range contains global stage g
__device__ __forceinline__ int owner_of(const Params& P, int64_t g) {
    const int64_t T = (int64_t)P.n_tiles * P.stages_per_tile;
    int c = (int)((g * gridDim.x) / T);
    // correct the rounding of the division (ranges are [T c / G, T (c + 1) / G))
    while (c > 0 && T * c / gridDim.x > g) --c;
    while (c + 1 < (int)gridDim.x && T * (c + 1) / gridDim.x <= g) ++c;
    return c;
}

__global__ void __launch_bounds__(THREADS, CTAS_PER_SM) gemm_tc_kernel(const __grid_constant__ CUtensorMap wmap,
                                                             const __grid_constant__ CUtensorMap xmap, Params P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::off_bar);
    uint64_t* full = bars;
    uint64_t* empty = bars + NST;
    uint64_t* acc_full = bars + 2 * NST;
    uint64_t* acc_empty = acc_full + NACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + NACC);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) trace_event(P, 0);
    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < NACC; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 4);
        }
    }
    if (warp == 0) tmem_alloc(tmem_slot, 32);
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    int64_t g0, g1;
    cta_range(P, blockIdx.x, g0, g1);
    const int spt = P.stages_per_tile;
    pdl_trigger();
    if (threadIdx.x == 0) trace_event(P, 1);

    if (warp == 0) {
        // ---------------------------------------------------------- TMA producer
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
            asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
            auto stage_coords = [&](int64_t g, int& tile, int& ks) {
                tile = (int)(g / spt);
                ks = (int)(g - (int64_t)tile * spt);
            };
            // The weights do not depend on the kernel before: the first NST stages' W boxes are in
            // flight while it drains; x (its output) follows after griddepcontrol.wait.
            const int n_pre = (int)((g1 - g0) < NST ? (g1 - g0) : NST);
            for (int i = 0; i < n_pre; ++i) {
                int tile, ks;
                stage_coords(g0 + i, tile, ks);
                uint8_t* dst = smem + Smem::off_stage + i * STAGE;
                mbar_arrive_tx(&full[i], STAGE);
                if (P.grouped) {
                    tma_load_4d(dst, &wmap, 0, 0, ks * SLABS, tile * (BM / 8), &full[i]);
                } else {
#pragma unroll
                    for (int sl = 0; sl < SLABS; ++sl)
                        tma_load_2d(dst + sl * A_BOX, &wmap, (ks * SLABS + sl) * SLAB, tile * BM, &full[i]);
                }
            }
            pdl_wait();
            trace_event(P, 2);
            for (int i = 0; i < n_pre; ++i) {
                int tile, ks;
                stage_coords(g0 + i, tile, ks);
                uint8_t* dst = smem + Smem::off_stage + i * STAGE + SLABS * A_BOX;
#pragma unroll
                for (int sl = 0; sl < SLABS; ++sl)
                    tma_load_2d(dst + sl * B_BOX, &xmap, (ks * SLABS + sl) * SLAB, 0, &full[i]);
            }
            int i = n_pre;
            for (int64_t g = g0 + n_pre; g < g1; ++g, ++i) {
                const int st = i % NST;
                mbar_wait(&empty[st], ((i / NST) & 1) ^ 1);
                int tile, ks;
                stage_coords(g, tile, ks);
                uint8_t* dst = smem + Smem::off_stage + st * STAGE;
                mbar_arrive_tx(&full[st], STAGE);
                if (P.grouped) tma_load_4d(dst, &wmap, 0, 0, ks * SLABS, tile * (BM / 8), &full[st]);
#pragma unroll
                for (int sl = 0; sl < SLABS; ++sl) {
                    const int kx = (ks * SLABS + sl) * SLAB;
                    if (!P.grouped) tma_load_2d(dst + sl * A_BOX, &wmap, kx, tile * BM, &full[st]);
                    tma_load_2d(dst + SLABS * A_BOX + sl * B_BOX, &xmap, kx, 0, &full[st]);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------- MMA issuer: one accumulator per piece
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_f16_f32(BM, BN, 1);  // bf16 x bf16 -> fp32
            int i = 0, piece = 0;
            for (int64_t g = g0; g < g1; ++piece) {
                const int tile = (int)(g / spt);
                const int64_t pend = (int64_t)(tile + 1) * spt < g1 ? (int64_t)(tile + 1) * spt : g1;
                const int ab = piece % NACC;
                mbar_wait(&acc_empty[ab], ((piece / NACC) & 1) ^ 1);  // (first use: free)
                tc_fence_after();
                bool first = true;
                for (; g < pend; ++g, ++i) {
                    const int st = i % NST;
                    mbar_wait(&full[st], (i / NST) & 1);
                    tc_fence_after();
                    if (i == 0) trace_event(P, 3);
                    const uint32_t a = smem_u32(smem + Smem::off_stage + st * STAGE);
                    const uint32_t b = a + SLABS * A_BOX;
#pragma unroll
                    for (int sl = 0; sl < SLABS; ++sl)
#pragma unroll
                        for (int kk = 0; kk < SLAB / 16; ++kk) {
                            const uint64_t ad = P.grouped ? desc_sw128_sbo(a + sl * 1024 + kk * 32, SLABS * 1024)
                                                          : desc_sw128(a + sl * A_BOX + kk * 32);
                            mma_f16(tmem_base + ab * BN, ad,
                                    desc_sw128(b + sl * B_BOX + kk * 32), idesc, first ? 0u : 1u);
                            first = false;
                        }
                    mma_commit(&empty[st]);
                }
                mma_commit(&acc_full[ab]);
            }
            trace_event(P, 4);
        }
    } else {
        // ---------------------------------------------------------- epilogue (lane = weight row of the tile)
        const int quad = warp & 3;
        const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16);
        const int row = quad * 32 + lane;
        int piece = 0;
        for (int64_t g = g0; g < g1; ++piece) {
            const int tile = (int)(g / spt);
            const int64_t tstart = (int64_t)tile * spt, tend = tstart + spt;
            const int64_t pend = tend < g1 ? tend : g1;
            const int ab = piece % NACC;
            mbar_wait(&acc_full[ab], (piece / NACC) & 1);
            tc_fence_after();
            if (threadIdx.x == 64 && piece == 0) trace_event(P, 5);
            uint32_t r[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                : "r"(lane_base + ab * BN));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[ab]);
            const int n = tile * BM + row;
            // pieces of this tile: the CTAs owning its first and last stage
            const int c_first = owner_of(P, tstart), c_last = owner_of(P, tend - 1);
            if (c_first == c_last) {  // the whole tile is this CTA's: bf16 straight out
                if (n < P.N)
#pragma unroll
                    for (int s = 0; s < BN; ++s)
                        if (s < P.S) P.y[(int64_t)s * P.N + n] = __float2bfloat16_rn(__uint_as_float(r[s]));
            } else {
                const int pidx = blockIdx.x - c_first, npieces = c_last - c_first + 1;
                // partials [tile][piece][row][16 sequences]: four 16-byte stores per row
                float4* slot = reinterpret_cast<float4*>(P.ws + (((int64_t)tile * P.max_pieces + pidx) * BM + row) * BN);
#pragma unroll
                for (int q = 0; q < BN / 4; ++q)
                    __stcg(slot + q, make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                                 __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3])));
                // four epilogue warps meet; the tile's last finisher adds the pieces in order
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (threadIdx.x == 64 && piece == 0) trace_event(P, 8);
                __shared__ int s_last;
                if (warp == 2 && lane == 0) {
                    // release the CTA's partials (ordered before the barrier) / acquire the others'
                    int prev;
                    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(P.counters + tile)
                                 : "memory");
                    s_last = prev == npieces - 1;
                    if (s_last) P.counters[tile] = 0;  // ready for the next launch
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (threadIdx.x == 64 && piece == 0) trace_event(P, 9);
                if (s_last) {
                    const float4* base =
                        reinterpret_cast<const float4*>(P.ws + ((int64_t)tile * P.max_pieces * BM + row) * BN);
                    float acc[BN];
#pragma unroll
                    for (int s = 0; s < BN; ++s) acc[s] = 0.f;
#pragma unroll 4
                    for (int pc = 0; pc < npieces; ++pc) {
                        float4 v[BN / 4];
#pragma unroll
                        for (int q = 0; q < BN / 4; ++q) v[q] = __ldcg(base + (int64_t)pc * (BM * BN / 4) + q);
#pragma unroll
                        for (int q = 0; q < BN / 4; ++q) {
                            acc[4 * q] += v[q].x;
                            acc[4 * q + 1] += v[q].y;
                            acc[4 * q + 2] += v[q].z;
                            acc[4 * q + 3] += v[q].w;
                        }
                    }
                    if (threadIdx.x == 64) trace_event(P, 10);
                    if (n < P.N)
#pragma unroll
                        for (int s = 0; s < BN; ++s)
                            if (s < P.S) P.y[(int64_t)s * P.N + n] = __float2bfloat16_rn(acc[s]);
                    if (threadIdx.x == 64) trace_event(P, 11);
                }
            }
            g = pend;
        }
        if (threadIdx.x == 64) trace_event(P, 6);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem_base, 32);
    if (threadIdx.x == 0) trace_event(P, 7);
}

struct Geometry {
    int n_tiles, stages_per_tile, grid, max_pieces;
};
static Geometry geometry(int N, int K) {
    Geometry G;
    G.n_tiles = (N + BM - 1) / BM;
    G.stages_per_tile = K / (SLAB * SLABS);
    const int64_t T = (int64_t)G.n_tiles * G.stages_per_tile;
    const int sms = ap_device_sm_count() * CTAS_PER_SM;
    G.grid = (int)(T < sms ? T : sms);
    const int64_t per = T / G.grid;  // >= 1
    G.max_pieces = (int)((G.stages_per_tile + per - 1) / per + 1);
    return G;
}

}  // namespace gtc
}  // namespace ap

using namespace ap;

extern "C" int64_t ap_gemm_tc_workspace_bytes(int32_t N, int32_t K, int32_t n_seq) {
    using namespace gtc;
    if (N <= 0 || K <= 0 || K % (SLAB * SLABS) != 0 || n_seq < 1 || n_seq > BN) return -1;
    (void)n_seq;
    const Geometry G = geometry(N, K);
    if (G.n_tiles > MAX_TILES) return -1;
    return COUNTER_BYTES + (int64_t)G.n_tiles * G.max_pieces * BN * BM * 4;
}

extern "C" int ap_gemm_tc(const void* W, const void* x, void* y, int32_t N, int32_t K, int32_t n_seq, void* workspace,
                          int64_t workspace_bytes, void* stream) {
    using namespace gtc;
    AP_REQUIRE(W && x && y && N > 0 && K > 0, AP_EPARAM, "bad GEMM operands");
    AP_REQUIRE(n_seq >= 1 && n_seq <= BN, AP_EPARAM, "ap_gemm_tc serves 1..16 sequences");
    AP_REQUIRE(K % (SLAB * SLABS) == 0, AP_EPARAM, "K must be a multiple of 256");
    const Geometry G = geometry(N, K);
    AP_REQUIRE(G.n_tiles <= MAX_TILES, AP_EPARAM, "N too large (at most %d rows)", MAX_TILES * BM);
    const int64_t need = COUNTER_BYTES + (int64_t)G.n_tiles * G.max_pieces * BN * BM * 4;
    AP_REQUIRE(workspace && workspace_bytes >= need, AP_EPARAM, "workspace too small (%lld bytes needed)",
               (long long)need);
    CUtensorMap wmap, xmap;
    static const int want_grouped = getenv("ATTNPRED_GEMM_GROUPED") ? atoi(getenv("ATTNPRED_GEMM_GROUPED")) : 1;
    const bool grouped = want_grouped && N % 8 == 0;
    if (grouped)
        AP_REQUIRE(make_tmap_bf16_sw128_grouped(&wmap, W, (uint64_t)N, (uint64_t)K, SLABS, BM / 8), AP_ECUDA,
                   "tensor map (W) failed");
    else
        AP_REQUIRE(make_tmap_bf16_sw128(&wmap, W, (uint64_t)N, (uint64_t)K, BM), AP_ECUDA, "tensor map (W) failed");
    AP_REQUIRE(make_tmap_bf16_sw128(&xmap, x, (uint64_t)n_seq, (uint64_t)K, BN), AP_ECUDA, "tensor map (x) failed");
    Params P{};
    P.y = (__nv_bfloat16*)y;
    P.counters = (int32_t*)workspace;
    P.ws = (float*)((char*)workspace + COUNTER_BYTES);
    P.N = N;
    P.K = K;
    P.S = n_seq;
    P.n_tiles = G.n_tiles;
    P.stages_per_tile = G.stages_per_tile;
    P.max_pieces = G.max_pieces;
    P.grouped = grouped;
    static const int trace = getenv("ATTNPRED_GEMM_TRACE") ? atoi(getenv("ATTNPRED_GEMM_TRACE")) : 0;
    P.trace = trace;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem::total);
        attr = true;
    }
    launch_ex(gemm_tc_kernel, dim3(G.grid), dim3(THREADS), Smem::total, as_stream(stream), 1, wmap, xmap, P);
    return launch_status("gemm_tc_kernel");
}

// debug: per-CTA event times of the last traced launch (ATTNPRED_GEMM_TRACE=1), 160 x 8 u64
extern "C" int ap_gemm_tc_trace(unsigned long long* host_out) {
    return cudaMemcpyFromSymbol(host_out, gtc::g_trace, sizeof(unsigned long long) * 160 * 12) == cudaSuccess ? AP_OK
                                                                                                           : AP_ECUDA;
}
