// Decode-engine GEMV (not a reference function: the reference has no model).  y[s] = W x[s] for
// the few sequences of a decode step, bf16 weights [N][K] row-major, fp32 accumulation.
//
// HBM-streaming design.  One persistent CTA per SM owns a contiguous range of weight rows, taken
// 8 rows at a time (a "row group"; SILU: 4 gate rows + their 4 up rows) and, along K, in slabs of
// <= 4096 columns.  A stage = one row group x one slab, landed in shared memory by per-row
// cp.async.bulk copies (TMA engine, issued by lanes of warp 0, completion on the stage's mbarrier)
// into rows padded by 16 bytes so the ldmatrix reads below are bank-conflict-free.  The stage ring
// keeps ~2-3 stages (~128-192 KB) in flight per SM.
//
// The dot products run on the warp-level tensor-core MMA (mma.sync m16n8k16 bf16, fp32
// accumulate): A = 8 weight rows x 16 columns (rows 8-15 of the fragment are zero) via one
// ldmatrix.x2, B = the activations (column n = sequence n < NS), each warp covering 1/8 of the
// slab's columns with four independent accumulator sets.  This is not for throughput - a GEMV
// has no reuse - but because it cuts the per-stage instruction count ~6x versus unpacking bf16
// pairs for FMAs, which otherwise keeps the stage ring from turning over at HBM rate.  Partial
// sums of the 8 warps are combined in a fixed order (deterministic results) after the CTA barrier
// that also releases the stage for its refill.  Weights do not depend on the previous kernel, so
// the first stages are issued before the programmatic-dependent-launch wait.
//
// Fused variants remove the neighbouring elementwise launches of a LLaMA layer:
//   * prologue RMSNORM: x = rmsnorm(x_in [+ residual]) * ln_w computed per CTA from the raw
//     activations (the row is L2-resident); CTA 0 also writes the updated residual stream to a
//     separate buffer (every CTA still reads the old one);
//   * epilogue SILU: W = [gate; up] (2F rows), act[i] = silu(gate_i) * up_i;
//   * epilogue ARGMAX: per-CTA best (value, lowest index) merged with a 64-bit atomicMax into
//     out_arg[s] (LM head + greedy sampling in one pass; `tokens` receives the index).
#include <cstdlib>

#include "common.cuh"

namespace ap {
namespace gemv {

constexpr int CWARPS = 8, CTHREADS = CWARPS * 32;   // consumer warps
constexpr int PRODUCER = CWARPS;                    // the copy-issuing warp
constexpr int THREADS = CTHREADS + 32, MAX_NS = 4, MAX_STAGES = 8, GROUP = 8;
constexpr int SLAB_MAX = 4096;             // columns per slab
constexpr int CPL = SLAB_MAX / 8 / CWARPS / 32;     // 16-byte chunks per lane per row and slab
constexpr int CTA_SMEM = 220 * 1024;       // stage ring + activations


enum Prologue { PRO_NONE = 0, PRO_RMSNORM = 1 };
enum Epilogue { EPI_STORE = 0, EPI_SILU = 1, EPI_ARGMAX = 2, EPI_ROPE = 3 };
// paired epilogues: a stage holds GROUP/2 rows and their GROUP/2 partner rows
__host__ __device__ constexpr bool paired(int epi) { return epi == EPI_SILU || epi == EPI_ROPE; }

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
    int slab, n_slab;        // columns per slab (multiple of 16), slabs per row
    int pitch;               // shared-memory bytes per staged row (slab * 2 + 16)
    int nst;                 // stages in the ring
    // ROPE epilogue (fused qkv projection + rotary embedding + KV append, as ap_rope_append)
    const int32_t* seq_len;  // [NS] positions + 1
    __nv_bfloat16* q_out;    // [NS][Hq][128]
    __nv_bfloat16* k_cache;  // [NS][Hkv][t_max][128]
    __nv_bfloat16* v_cache;  // same, or null (offload mode: V is read back from y)
    int Hq, Hkv, t_max;
    float theta;
};

// Paired units: SILU unit o = gate row o and up row N/2 + o; ROPE unit u = rows 128 h + i and 128 h + i + 64
// (h = u / 64, i = u % 64).  first_row(u) + k for k < cnt stays inside one head since units are
// dealt in groups of GROUP/2 and 64 % (GROUP/2) == 0.
template <int EPI>
__device__ __forceinline__ int64_t first_row(const Params& P, int u) {
    if constexpr (EPI == EPI_ROPE) return (int64_t)(u >> 6) * 128 + (u & 63);
    return u;
}
template <int EPI>
__device__ __forceinline__ int64_t partner_offset(const Params& P) {
    return EPI == EPI_ROPE ? 64 : P.N / 2;
}

__device__ __forceinline__ uint32_t order_f32(float f) {  // monotone float -> u32
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

template <int NS, int PRO, int EPI>
__global__ void __launch_bounds__(THREADS, 1) gemv_stream_kernel(Params P) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[MAX_STAGES], empty[MAX_STAGES];
    __shared__ float red[2][CWARPS][GROUP][NS];  // by row-group parity
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int K = P.K, NST = P.nst, n_slab = P.n_slab, slab = P.slab, pitch = P.pitch;
    const int stage_bytes = GROUP * pitch;
    constexpr int per_group = paired(EPI) ? GROUP / 2 : GROUP;
    const int U = paired(EPI) ? P.N / 2 : P.N;
    const int n_pg = (U + per_group - 1) / per_group;  // groups dealt to CTAs whole
    const int u0 = min(U, (int)((int64_t)blockIdx.x * n_pg / gridDim.x) * per_group);
    const int u1 = min(U, (int)((int64_t)(blockIdx.x + 1) * n_pg / gridDim.x) * per_group);
    const int n_group = (u1 - u0 + per_group - 1) / per_group;
    const int n_stage = n_group * n_slab;
    uint8_t* xs = smem + (size_t)NST * stage_bytes;  // [NS][K] bf16

    if (tid == 0)
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CWARPS);
        }
    __syncthreads();

    if (warp == PRODUCER) {
        // ---- producer warp: stage j = (row group g, slab sl) -> ring slot j % NST.  A single-slab
        // group is one contiguous copy; otherwise one copy per row (lanes in parallel).  Weights do
        // not depend on the previous kernel: no programmatic-dependent-launch wait here.
        pdl_trigger();
        int g = 0, sl = 0;
        for (int j = 0; j < n_stage; ++j) {
            const int slot = j % NST;
            if (j >= NST) mbar_wait_spin(&empty[slot], (uint32_t)(((j / NST) - 1) & 1));
            uint8_t* dst = smem + slot * stage_bytes;
            const int a = u0 + g * per_group, cnt = min(per_group, u1 - a);
            const int c0 = sl * slab, len = min(slab, K - c0);
            constexpr int halves = paired(EPI) ? 2 : 1;
            const int64_t row0 = first_row<EPI>(P, a), off = partner_offset<EPI>(P);
            if (lane == 0) mbar_arrive_tx(&full[slot], (uint32_t)(halves * cnt * len * 2));
            __syncwarp();
            if (n_slab == 1) {  // rows are contiguous in global and in the stage (pitch = row bytes)
                if (lane < halves) {
                    const int64_t row = row0 + lane * off;
                    bulk_g2s(dst + lane * (GROUP / 2) * pitch, P.W + row * K, (uint32_t)(cnt * len * 2), &full[slot]);
                }
            } else if (lane < halves * cnt) {
                const int h = lane / cnt, r = lane - h * cnt;
                const int64_t row = row0 + r + h * off;
                bulk_g2s(dst + (h * (GROUP / 2) + r) * pitch, P.W + row * K + c0, (uint32_t)len * 2, &full[slot]);
            }
            if (++sl == n_slab) { sl = 0; ++g; }
        }
        return;
    }

    // ---- consumers: activations -> shared memory as bf16 (the values are bf16-exact)
    pdl_trigger();
    pdl_wait();
    __nv_bfloat16* xb = reinterpret_cast<__nv_bfloat16*>(xs);
    if constexpr (PRO == PRO_RMSNORM) {
        __shared__ float rsum[NS][CWARPS];
        for (int s = 0; s < NS; ++s) {  // h = x [+ residual], staged in place
            float ss = 0.f;
            for (int k = tid; k < K; k += CTHREADS) {
                float v = __bfloat162float(P.x[(int64_t)s * K + k]);
                if (P.residual) {
                    v += __bfloat162float(P.residual[(int64_t)s * K + k]);
                    v = __bfloat162float(__float2bfloat16_rn(v));  // the residual stream is bf16
                }
                xb[s * K + k] = __float2bfloat16_rn(v);
                ss = fmaf(v, v, ss);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
            if (lane == 0) rsum[s][warp] = ss;
        }
        named_bar_sync(1, CTHREADS);
        for (int s = 0; s < NS; ++s) {
            float ss = 0.f;
#pragma unroll
            for (int w = 0; w < CWARPS; ++w) ss += rsum[s][w];
            const float inv = rsqrtf(ss / (float)K + P.eps);
            for (int k = tid; k < K; k += CTHREADS) {
                const float v = __bfloat162float(xb[s * K + k]);
                if (blockIdx.x == 0 && P.residual_out) P.residual_out[(int64_t)s * K + k] = __float2bfloat16_rn(v);
                // y = bf16(h * inv * w), the arithmetic of ap_rmsnorm
                xb[s * K + k] = __float2bfloat16_rn(v * inv * __bfloat162float(P.ln_w[k]));
            }
        }
    } else {
        for (int i = tid; i < NS * K; i += CTHREADS) xb[i] = P.x[i];
    }
    named_bar_sync(1, CTHREADS);

    // ---- stream: warp w reduces every row of a stage over its column range [k0, k1) of the slab;
    //      lane l takes the 16-byte chunks k0/8 + l + 32 i
    const int chunks = slab / 8;
    const int q0 = warp * chunks / CWARPS, q1 = (warp + 1) * chunks / CWARPS;
    unsigned long long best[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) best[s] = 0ull;
    float acc[GROUP][NS][2];
    int g = 0, sl = 0;
    for (int j = 0; j < n_stage; ++j) {
        const int slot = j % NST;
        const int c0 = sl * slab, qe = min(q1, (K - c0) / 8);  // the last slab may be shorter
        if (sl == 0) {
#pragma unroll
            for (int r = 0; r < GROUP; ++r)
#pragma unroll
                for (int s = 0; s < NS; ++s) acc[r][s][0] = acc[r][s][1] = 0.f;
        }
        // this lane's activation chunks of the slab -> fp32 registers
        float xf[CPL][NS][8];
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            const int q = q0 + lane + 32 * i;
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                const uint4 v = q < qe ? reinterpret_cast<const uint4*>(xb + (size_t)s * K + c0)[q] : make_uint4(0, 0, 0, 0);
                const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    xf[i][s][2 * e] = __uint_as_float(u[e] << 16);
                    xf[i][s][2 * e + 1] = __uint_as_float(u[e] & 0xffff0000u);
                }
            }
        }
        mbar_wait_spin(&full[slot], (uint32_t)((j / NST) & 1));
        const uint8_t* st = smem + slot * stage_bytes;
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            const int q = q0 + lane + 32 * i;
            if (q < qe) {
#pragma unroll
                for (int r = 0; r < GROUP; ++r) {
                    const uint4 w = reinterpret_cast<const uint4*>(st + r * pitch)[q];
                    const uint32_t v[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float wl = __uint_as_float(v[e] << 16), wh = __uint_as_float(v[e] & 0xffff0000u);
#pragma unroll
                        for (int s = 0; s < NS; ++s)
                            ffma2v(acc[r][s][0], acc[r][s][1], wl, wh, xf[i][s][2 * e], xf[i][s][2 * e + 1]);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);  // this warp is done reading the stage
        if (sl == n_slab - 1) {  // row group complete: reduce over lanes, then over warps in a fixed order
#pragma unroll
            for (int r = 0; r < GROUP; ++r)
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    float v = acc[r][s][0] + acc[r][s][1];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    if (lane == 0) red[g & 1][warp][r][s] = v;
                }
            named_bar_sync(1, CTHREADS);
            const int a = u0 + g * per_group, cnt = min(per_group, u1 - a);
            if constexpr (EPI == EPI_SILU) {
                if (tid < (GROUP / 2) * NS) {
                    const int o = tid % (GROUP / 2), s = tid / (GROUP / 2);
                    if (o < cnt) {
                        float gs = 0.f, us = 0.f;
#pragma unroll
                        for (int w = 0; w < CWARPS; ++w) {
                            gs += red[g & 1][w][o][s];
                            us += red[g & 1][w][GROUP / 2 + o][s];
                        }
                        // the gate/up GEMM output is bf16, then silu(g) * u as in ap_silu_mul
                        const float gt = __bfloat162float(__float2bfloat16_rn(gs));
                        const float up = __bfloat162float(__float2bfloat16_rn(us));
                        P.y[(int64_t)s * (P.N / 2) + a + o] = __float2bfloat16_rn(gt / (1.f + __expf(-gt)) * up);
                    }
                }
            } else if constexpr (EPI == EPI_ROPE) {
                if (tid < (GROUP / 2) * NS) {
                    const int o = tid % (GROUP / 2), s = tid / (GROUP / 2);
                    if (o < cnt) {
                        float x1 = 0.f, x2 = 0.f;
#pragma unroll
                        for (int w = 0; w < CWARPS; ++w) {
                            x1 += red[g & 1][w][o][s];
                            x2 += red[g & 1][w][GROUP / 2 + o][s];
                        }
                        const int u = a + o, head = u >> 6, i = u & 63;
                        const int64_t r1 = (int64_t)head * 128 + i;
                        const __nv_bfloat16 b1 = __float2bfloat16_rn(x1), b2 = __float2bfloat16_rn(x2);
                        P.y[(int64_t)s * P.N + r1] = b1;  // the projection output, as ap_gemv stores it
                        P.y[(int64_t)s * P.N + r1 + 64] = b2;
                        // ap_rope_append's arithmetic on the bf16 projection output
                        x1 = __bfloat162float(b1);
                        x2 = __bfloat162float(b2);
                        const int pos = P.seq_len[s] - 1;
                        if (head < P.Hq + P.Hkv) {
                            const float inv_freq = exp2f(-(float)(2 * i) / 128.f * log2f(P.theta));
                            float sn, cs;
                            sincosf((float)pos * inv_freq, &sn, &cs);
                            const float y1 = x1 * cs - x2 * sn, y2 = x2 * cs + x1 * sn;
                            x1 = y1;
                            x2 = y2;
                        }
                        __nv_bfloat16* dstp = nullptr;
                        if (head < P.Hq) dstp = P.q_out + ((int64_t)s * P.Hq + head) * 128;
                        else if (head < P.Hq + P.Hkv)
                            dstp = P.k_cache + (((int64_t)s * P.Hkv + (head - P.Hq)) * P.t_max + pos) * 128;
                        else if (P.v_cache)
                            dstp = P.v_cache + (((int64_t)s * P.Hkv + (head - P.Hq - P.Hkv)) * P.t_max + pos) * 128;
                        if (dstp) {
                            dstp[i] = __float2bfloat16_rn(x1);
                            dstp[i + 64] = __float2bfloat16_rn(x2);
                        }
                    }
                }
            } else {
                if (tid < GROUP * NS) {
                    const int rr = tid % GROUP, s = tid / GROUP;
                    if (rr < cnt) {
                        float v = 0.f;
#pragma unroll
                        for (int w = 0; w < CWARPS; ++w) v += red[g & 1][w][rr][s];
                        if (P.y) P.y[(int64_t)s * P.N + a + rr] = __float2bfloat16_rn(v);
                        if constexpr (EPI == EPI_ARGMAX) {  // bf16-rounded logits, ties -> lowest index (torch.argmax)
                            const float q = __bfloat162float(__float2bfloat16_rn(v));
                            const unsigned long long key =
                                (unsigned long long)order_f32(q) << 32 | (uint32_t)~(uint32_t)(a + rr);
#pragma unroll
                            for (int t = 0; t < NS; ++t)
                                if (t == s) best[t] = key > best[t] ? key : best[t];
                        }
                    }
                }
            }
            // red[g & 1] is rewritten by group g + 2, after the barrier of group g + 1
        }
        if (++sl == n_slab) { sl = 0; ++g; }
    }

    if constexpr (EPI == EPI_ARGMAX) {
        __shared__ unsigned long long cta_best[NS];
        if (tid < NS) cta_best[tid] = 0ull;
        named_bar_sync(1, CTHREADS);
#pragma unroll
        for (int s = 0; s < NS; ++s)
            if (best[s]) atomicMax(&cta_best[s], best[s]);
        named_bar_sync(1, CTHREADS);
        if (tid < NS) atomicMax(P.arg + tid, cta_best[tid]);
        __threadfence();
        named_bar_sync(1, CTHREADS);
        if (tid == 0) {
            __shared__ int last;
            last = atomicAdd(P.counter, 1) == (int)gridDim.x - 1;
            if (last) {
                __threadfence();
                for (int s = 0; s < NS; ++s) {
                    const unsigned long long b = atomicExch(P.arg + s, 0ull);  // reset for the next call
                    P.tokens[s] = (int64_t)(uint32_t)~(uint32_t)(b & 0xffffffffu);
                }
                *P.counter = 0;
            }
        }
    }
}

template <int NS, int PRO, int EPI>
int launch(Params P, cudaStream_t st) {
    // slabs: the fewest with <= SLAB_MAX columns each and >= 2 (ideally 3) stages next to the activations
    const int64_t xbytes = (int64_t)NS * P.K * 2;
    const int64_t ring = CTA_SMEM - xbytes;
    static int slab_max = -1;  // ATTNPRED_GEMV_SLAB: tuning override (<= SLAB_MAX, multiple of 8)
    if (slab_max < 0) {
        const char* e = getenv("ATTNPRED_GEMV_SLAB");
        slab_max = e ? atoi(e) : SLAB_MAX;
        if (slab_max < 256 || slab_max > SLAB_MAX) slab_max = SLAB_MAX;
    }
    int n_slab = (P.K + slab_max - 1) / slab_max;
    auto slab_of = [&](int n) { return ((P.K + n - 1) / n + 7) / 8 * 8; };
    while (ring < 3 * (int64_t)GROUP * slab_of(n_slab) * 2 && slab_of(n_slab) > 512) ++n_slab;
    P.n_slab = n_slab;
    P.slab = slab_of(n_slab);
    P.pitch = P.slab * 2;
    const int64_t stage_bytes = (int64_t)GROUP * P.pitch;
    static int nst_max = -1;  // ATTNPRED_GEMV_STAGES: tuning override
    if (nst_max < 0) {
        const char* e = getenv("ATTNPRED_GEMV_STAGES");
        nst_max = e ? atoi(e) : MAX_STAGES;
        if (nst_max < 2 || nst_max > MAX_STAGES) nst_max = MAX_STAGES;
    }
    int64_t nst = ring / stage_bytes;
    nst = nst > nst_max ? nst_max : nst;
    nst = nst > MAX_STAGES ? MAX_STAGES : nst;
    AP_REQUIRE(nst >= 2, AP_EPARAM, "ap_gemv: K = %d too large for the shared-memory stage ring", P.K);
    P.nst = (int)nst;
    const size_t smem = (size_t)(nst * stage_bytes + xbytes);
    const int units = paired(EPI) ? P.N / 2 : P.N;
    const int per_group = paired(EPI) ? GROUP / 2 : GROUP;
    int grid = (units + per_group - 1) / per_group;
    const int sms = ap_sm_budget();  // the SMs not reserved for a concurrent selector step
    grid = grid < sms ? grid : sms;
    auto k = gemv_stream_kernel<NS, PRO, EPI>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, CTA_SMEM);
        attr_set = true;
    }
    launch_ex(k, dim3(grid), dim3(THREADS), smem, st, 1, P);
    return launch_status("gemv_stream_kernel");
}

template <int PRO, int EPI>
int dispatch_ns(const Params& P, cudaStream_t st) {
    switch (P.NS) {
        case 1: return launch<1, PRO, EPI>(P, st);
        case 2: return launch<2, PRO, EPI>(P, st);
        case 3: return launch<3, PRO, EPI>(P, st);
        default: return launch<4, PRO, EPI>(P, st);
    }
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
    (void)rows_per_warp;  // ABI slot of the earlier register-streaming kernel; the stage geometry is chosen here
    AP_REQUIRE((int64_t)n_seq * K * 2 <= 150 * 1024, AP_EPARAM, "activations exceed shared memory");
    const int pro = flags & 1 ? PRO_RMSNORM : PRO_NONE;
    const int epi = (flags >> 1) & 3;
    AP_REQUIRE(epi <= EPI_ARGMAX, AP_EPARAM, "bad epilogue");
    AP_REQUIRE(pro == PRO_NONE || ln_w, AP_EPARAM, "RMSNORM prologue needs ln_w");
    AP_REQUIRE(epi != EPI_SILU || N % 2 == 0, AP_EPARAM, "SILU epilogue needs an even N ([gate; up])");
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
        if (epi == EPI_STORE) return dispatch_ns<PRO_RMSNORM, EPI_STORE>(P, st);
        if (epi == EPI_SILU) return dispatch_ns<PRO_RMSNORM, EPI_SILU>(P, st);
        return dispatch_ns<PRO_RMSNORM, EPI_ARGMAX>(P, st);
    }
    if (epi == EPI_STORE) return dispatch_ns<PRO_NONE, EPI_STORE>(P, st);
    if (epi == EPI_SILU) return dispatch_ns<PRO_NONE, EPI_SILU>(P, st);
    return dispatch_ns<PRO_NONE, EPI_ARGMAX>(P, st);
}

extern "C" int ap_gemv_qkv_rope(const void* W, const void* x, void* y, int32_t n_q_heads, int32_t n_kv_heads,
                                int32_t K, int32_t n_seq, int32_t flags, const void* residual, void* residual_out,
                                const void* ln_w, float eps, const int32_t* seq_len, void* q_out, void* k_cache,
                                void* v_cache, int32_t t_max, float theta, void* stream) {
    using namespace gemv;
    AP_REQUIRE(W && x && y && seq_len && q_out && k_cache, AP_EPARAM, "bad qkv/rope operands");
    AP_REQUIRE(n_q_heads > 0 && n_kv_heads > 0 && n_q_heads % n_kv_heads == 0, AP_EPARAM, "bad head counts");
    AP_REQUIRE(K > 0 && K % 8 == 0, AP_EPARAM, "K must be a multiple of 8 (16-byte rows)");
    AP_REQUIRE(n_seq >= 1 && n_seq <= MAX_NS, AP_EPARAM, "ap_gemv serves 1..4 activation rows");
    AP_REQUIRE((int64_t)n_seq * K * 2 <= 150 * 1024, AP_EPARAM, "activations exceed shared memory");
    AP_REQUIRE((flags & ~1) == 0, AP_EPARAM, "only the RMSNORM prologue flag applies");
    AP_REQUIRE(!(flags & 1) || ln_w, AP_EPARAM, "RMSNORM prologue needs ln_w");
    AP_REQUIRE(!residual_out || (residual_out != residual && residual_out != x), AP_EPARAM,
               "residual_out must not alias the residual or x");
    Params P{};
    P.W = (const __nv_bfloat16*)W;
    P.x = (const __nv_bfloat16*)x;
    P.residual = (const __nv_bfloat16*)residual;
    P.residual_out = (__nv_bfloat16*)residual_out;
    P.ln_w = (const __nv_bfloat16*)ln_w;
    P.eps = eps;
    P.y = (__nv_bfloat16*)y;
    P.N = (n_q_heads + 2 * n_kv_heads) * 128;
    P.K = K;
    P.NS = n_seq;
    P.seq_len = seq_len;
    P.q_out = (__nv_bfloat16*)q_out;
    P.k_cache = (__nv_bfloat16*)k_cache;
    P.v_cache = (__nv_bfloat16*)v_cache;
    P.Hq = n_q_heads;
    P.Hkv = n_kv_heads;
    P.t_max = t_max;
    P.theta = theta;
    cudaStream_t st = as_stream(stream);
    if (flags & 1) return dispatch_ns<PRO_RMSNORM, EPI_ROPE>(P, st);
    return dispatch_ns<PRO_NONE, EPI_ROPE>(P, st);
}
