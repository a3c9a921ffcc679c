// Kernel (4a) sparse decode attention over the selected blocks and (4b) the
// dense pass used for calibration rows and for the full-attention comparator.
//
// Semantics (SURVEY §8c "kernels with no reference implementation"):
//   scores = q . k / sqrt(d), softmax, . V          (attntap/model.py:70-74)
//   selection S = sink ∪ local ∪ middle blocks      (selector.py:122-149)
//   calibration row = max_pool(dense softmax row, b) (selector.py:112-117),
//     computed as exp(blockmax_logit - LSE) — exact by monotonicity of exp;
//   observed (fed-back) row on non-calibration steps: sparse_renorm mode —
//     probability under the sparse softmax over S at selected positions,
//     0 elsewhere (DESIGN.md §Observed-row semantics).
// Both kernels push the compressed row straight into the selector's history
// ring (the append of selector.py:117-120), so compression never re-reads a
// t-length row from HBM.
//
// Layout: K/V cache per layer [seq][kv_head][t_max][128] bf16 — a 16-token
// block of one head is 4 KiB contiguous.  A warp processes one block: lane =
// (token parity, 8-dim slice), 16-byte loads, half-warp shuffle reductions.
// Flash-decoding split over blocks; a combine kernel merges the splits.
#include <cooperative_groups.h>
#include <cuda.h>  // CUtensorMap (driver types only; the encoder comes via cudaGetDriverEntryPoint)
#include <cudaTypedefs.h>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tma.cuh"

namespace ap {

constexpr int HD = 128;                 // head dim
constexpr int ATT_THREADS = 256;        // 8 warps
constexpr int ATT_WARPS = ATT_THREADS / 32;
constexpr int KV_STAGE = 2 * 16 * 128 * 2;  // one 16-token block of K and of V, bf16 (sparse cluster staging)
constexpr float LOG2E = 1.4426950408889634f;

__device__ long long g_att_trace[16 * 16];  // debug: clock64 per phase, CTAs (split, 0, 0)
__device__ int g_att_trace_on;
// Phase traces are compiled in only with -DAP_ATT_TRACE (scripts/attn_trace.py, calib_trace.py build a
// variant library): the on/off flag is a global load, and on thread 0 of the traced CTAs it sat on the
// critical path of every launch (ncu: 11% of the sparse kernel's stall samples at the first trace point).
#ifdef AP_ATT_TRACE
#define ATT_TRACE2(e) \
    if (lane == 0 && blockIdx.y == 0 && blockIdx.z == 0 && g_att_trace_on && blockIdx.x < 16) g_att_trace[blockIdx.x * 16 + (e)] = clock64();
#define ATT_TRACE(e) \
    if (threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && g_att_trace_on) g_att_trace[blockIdx.x * 16 + (e)] = clock64();
#else
#define ATT_TRACE2(e) do { } while (0)
#define ATT_TRACE(e) do { } while (0)
#endif

struct AttnParams {
    int32_t n_seq, n_q_heads, n_kv_heads, t_max, n_splits, block;
    const __nv_bfloat16* q;       // [S][Hq][D]
    const __nv_bfloat16* k;       // [S][Hkv][t_max][D]
    const __nv_bfloat16* v;
    const int32_t* seq_len;       // [S]
    __nv_bfloat16* out;           // [S][Hq][D]
    float* lse;                   // [S][Hq] log2 units (nullable)
    float* partial;               // [S][Hq][n_splits][D+2]
    float* bmax;                  // [S][Hq][w_max] log2-unit block max logits (-inf = untouched)
    int32_t* counters;            // [S][Hq] split-completion counters (0 between launches)
    int32_t w_max;
    int32_t with_v, emit;
    // selector binding
    ap_selector sel;
    int32_t map_base, maps_per_seq, group;  // map(s, h) = s*maps_per_seq + map_base + h/group
    // paged V (offload mode, kernel 5): V blocks of the selection come from the page pool
    ap_vpages vp;
    int32_t paged, layer;
    int32_t sparse_units;  // emission from the selection's units only (sparse path)
};

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float (&f)[8]) {
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 t = __bfloat1622float2(p[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

// Per-warp running softmax state for NH heads; lane holds 8 dims (slice) of
// the accumulators for the tokens of its half-warp.
template <int NH, bool WITH_V>
struct WarpState {
    float m[NH], l[NH], acc[NH][8];
    __device__ void init() {
#pragma unroll
        for (int h = 0; h < NH; ++h) {
            m[h] = -INFINITY;
            l[h] = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[h][i] = 0.f;
        }
    }
};

// Process one 16-token block j for NH heads.  take(p) decides token membership.
// Writes the block max (log2 logits) of each head through bm_out(h, value) when EMIT.
//
// Lane layout: half = token parity, sub = 8-dim slice.  Each lane first forms
// partial dots for its 8 tokens x 8 dims, then a transpose-reduce across the
// 16 lanes of its half (xor 8, 4, 2: halving the live values each step, then
// xor 1) leaves lane `sub` holding the full dot of token (sub >> 1) — 8
// shuffles per head instead of 32, and one exp2 per lane instead of eight.
template <bool WITH_V>
__device__ __forceinline__ void load_block(const __nv_bfloat16* kh, const __nv_bfloat16* vh, int64_t j, int b,
                                           uint4 (&kv)[8], uint4 (&vv)[8]) {
    const int lane = threadIdx.x & 31, half = lane >> 4, sub = lane & 15;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
        const int64_t p = j * b + jj * 2 + half;
        kv[jj] = __ldg(reinterpret_cast<const uint4*>(kh + p * HD + sub * 8));
    }
    if constexpr (WITH_V) {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const int64_t p = j * b + jj * 2 + half;
            vv[jj] = __ldg(reinterpret_cast<const uint4*>(vh + p * HD + sub * 8));
        }
    }
}

// KSrc / VSrc: jj -> the 16 bytes (8 dims) of token jj*2 + half this lane holds (registers, or
// shared memory read just in time)
template <int NH, bool WITH_V, bool EMIT, typename KSrc, typename VSrc, typename Take, typename BmOut>
__device__ __forceinline__ void compute_block_src(KSrc kv, VSrc vv, int64_t j, int b, const float (&qf)[NH][8],
                                                  WarpState<NH, WITH_V>& st, Take take, BmOut bm_out);

template <int NH, bool WITH_V, bool EMIT, typename Take, typename BmOut>
__device__ __forceinline__ void compute_block(const uint4 (&kv)[8], const uint4 (&vv)[8], int64_t j, int b,
                                              const float (&qf)[NH][8], WarpState<NH, WITH_V>& st, Take take,
                                              BmOut bm_out) {
    compute_block_src<NH, WITH_V, EMIT>([&](int jj) { return kv[jj]; }, [&](int jj) { return vv[jj]; }, j, b, qf,
                                        st, take, bm_out);
}

template <int NH, bool WITH_V, bool EMIT, typename KSrc, typename VSrc, typename Take, typename BmOut>
__device__ __forceinline__ void compute_block_src(KSrc kv, VSrc vv, int64_t j, int b, const float (&qf)[NH][8],
                                                  WarpState<NH, WITH_V>& st, Take take, BmOut bm_out) {
    const int lane = threadIdx.x & 31, half = lane >> 4, sub = lane & 15;
    float d[NH][8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
        float kf[8];
        bf16x8_to_f32(kv(jj), kf);
#pragma unroll
        for (int h = 0; h < NH; ++h) {
            float a = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) a = fmaf(qf[h][i], kf[i], a);
            d[h][jj] = a;
        }
    }
    const bool b3 = (sub >> 3) & 1, b2 = (sub >> 2) & 1, b1 = (sub >> 1) & 1;
    const int my_jj = (sub >> 1) & 7;
    const bool my_sel = take(j * b + my_jj * 2 + half);
    float pm[NH];
    bool any = false;
#pragma unroll
    for (int h = 0; h < NH; ++h) {
        float e4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float send = b3 ? d[h][k] : d[h][k + 4];
            const float keep = b3 ? d[h][k + 4] : d[h][k];
            e4[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
        float e2[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const float send = b2 ? e4[k] : e4[k + 2];
            const float keep = b2 ? e4[k + 2] : e4[k];
            e2[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
        const float send = b1 ? e2[0] : e2[1];
        float e1 = (b1 ? e2[1] : e2[0]) + __shfl_xor_sync(0xffffffffu, send, 2);
        e1 += __shfl_xor_sync(0xffffffffu, e1, 1);
        const float sc = my_sel ? e1 : -INFINITY;
        float mx = sc;
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        if constexpr (EMIT) bm_out(h, mx);
        pm[h] = 0.f;
        if (mx == -INFINITY) continue;  // nothing selected in this block for this head (warp-uniform)
        any = true;
        const float m_new = fmaxf(st.m[h], mx);
        const float corr = exp2f(st.m[h] - m_new);
        pm[h] = exp2f(sc - m_new);  // 0 for unselected tokens
        // each token sits in two lanes (sub, sub^1): reduce over xor 16, 8, 4, 2 only
        float psum = pm[h];
        psum += __shfl_xor_sync(0xffffffffu, psum, 16);
        psum += __shfl_xor_sync(0xffffffffu, psum, 8);
        psum += __shfl_xor_sync(0xffffffffu, psum, 4);
        psum += __shfl_xor_sync(0xffffffffu, psum, 2);
        st.l[h] = st.l[h] * corr + psum;
        st.m[h] = m_new;
        if constexpr (WITH_V) {
#pragma unroll
            for (int i = 0; i < 8; ++i) st.acc[h][i] *= corr;
        }
    }
    if constexpr (WITH_V) {
        if (!any) return;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const int src = half * 16 + jj * 2;  // lane holding token jj of this half
            float pj[NH];
            bool nz = false;
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                pj[h] = __shfl_sync(0xffffffffu, pm[h], src);
                nz |= pj[h] != 0.f;
            }
            if (!nz) continue;  // unselected / beyond t: never touch its V (may be garbage)
            float vf[8];
            bf16x8_to_f32(vv(jj), vf);  // once per token, shared by every head
#pragma unroll
            for (int h = 0; h < NH; ++h)
#pragma unroll
                for (int i = 0; i < 8; ++i) st.acc[h][i] = fmaf(pj[h], vf[i], st.acc[h][i]);
        }
    }
}

template <int NH, bool WITH_V, bool EMIT, typename Take, typename BmOut>
__device__ __forceinline__ void process_block(const __nv_bfloat16* kh, const __nv_bfloat16* vh, int64_t j, int b,
                                              const float (&qf)[NH][8], WarpState<NH, WITH_V>& st, Take take,
                                              BmOut bm_out) {
    uint4 kv[8], vv[8];
    load_block<WITH_V>(kh, vh, j, b, kv, vv);
    compute_block<NH, WITH_V, EMIT>(kv, vv, j, b, qf, st, take, bm_out);
}

// Merge the 8 warps' states of a CTA and write the split partial (m, l, acc[128]).
template <int NH, bool WITH_V>
__device__ void write_partial(WarpState<NH, WITH_V>& st, float* smem, float* part_base /*[NH] stride*/,
                              int64_t head_stride) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, half = lane >> 4, sub = lane & 15;
    // combine the two half-warps (same dims, different tokens): they share m and l already
#pragma unroll
    for (int h = 0; h < NH; ++h)
#pragma unroll
        for (int i = 0; i < 8; ++i) st.acc[h][i] += __shfl_xor_sync(0xffffffffu, st.acc[h][i], 16);
    // smem: [warp][h][2 + 128]
    float* w = smem + warp * NH * (HD + 2);
#pragma unroll
    for (int h = 0; h < NH; ++h) {
        if (lane == 0) {
            w[h * (HD + 2) + 0] = st.m[h];
            w[h * (HD + 2) + 1] = st.l[h];
        }
        if (WITH_V && half == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) w[h * (HD + 2) + 2 + sub * 8 + i] = st.acc[h][i];
        }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < NH * (HD + 2); idx += ATT_THREADS) {
        const int h = idx / (HD + 2), e = idx % (HD + 2);
        float M = -INFINITY;
        for (int ww = 0; ww < ATT_WARPS; ++ww) M = fmaxf(M, smem[(ww * NH + h) * (HD + 2)]);
        float val = 0.f;
        if (e == 0) {
            val = M;
        } else if (M != -INFINITY) {
            for (int ww = 0; ww < ATT_WARPS; ++ww) {
                const float mw = smem[(ww * NH + h) * (HD + 2)];
                if (mw == -INFINITY) continue;
                val += smem[(ww * NH + h) * (HD + 2) + e] * exp2f(mw - M);
            }
        }
        if (e >= 2 && !WITH_V) continue;
        part_base[h * head_stride + e] = val;
    }
}

// ------------------------------------------------------------------ combine
// Executed by the LAST CTA to finish among the splits of a unit (flash-decoding
// reduction fused into the split kernel): merge the splits of heads
// [h0, h0 + nh) of sequence s; write out (bf16) and lse; when emit, write each
// map's compressed row max_h exp2(bm_h[j] - lse_h) (0 where untouched) into
// its ring slot and advance the map's ring state (selector.py:117-120).
__device__ void combine_heads(const AttnParams& P, int s, int h0, int nh) {
    __shared__ float s_w[8][64];
    __shared__ float s_lse[8], s_L[8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = P.seq_len[s];
    if (warp < nh) {  // warp per head: lanes over splits
        const float* part = P.partial + ((int64_t)s * P.n_q_heads + h0 + warp) * P.n_splits * (HD + 2);
        float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
        if (lane < P.n_splits) { m0 = __ldcg(part + lane * (HD + 2)); l0 = __ldcg(part + lane * (HD + 2) + 1); }
        if (lane + 32 < P.n_splits) { m1 = __ldcg(part + (lane + 32) * (HD + 2)); l1 = __ldcg(part + (lane + 32) * (HD + 2) + 1); }
        float M = fmaxf(m0, m1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        const float w0 = (m0 == -INFINITY) ? 0.f : exp2f(m0 - M), w1 = (m1 == -INFINITY) ? 0.f : exp2f(m1 - M);
        if (lane < P.n_splits) s_w[warp][lane] = w0;
        if (lane + 32 < P.n_splits) s_w[warp][lane + 32] = w1;
        float L = l0 * w0 + l1 * w1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
        if (lane == 0) {
            s_L[warp] = L;
            s_lse[warp] = M + log2f(L);
            if (P.lse) P.lse[(int64_t)s * P.n_q_heads + h0 + warp] = M + log2f(L);
        }
    }
    __syncthreads();
    if (P.with_v) {
        for (int idx = threadIdx.x; idx < nh * HD; idx += ATT_THREADS) {
            const int hh = idx / HD, d = idx % HD;
            const float* part = P.partial + ((int64_t)s * P.n_q_heads + h0 + hh) * P.n_splits * (HD + 2) + 2 + d;
            float o = 0.f;
            for (int sp = 0; sp < P.n_splits; ++sp) o = fmaf(__ldcg(part + sp * (HD + 2)), s_w[hh][sp], o);
            P.out[((int64_t)s * P.n_q_heads + h0 + hh) * HD + d] = __float2bfloat16_rn(o / s_L[hh]);
        }
    }
    if (P.emit) {
        const int64_t W = (t + P.block - 1) / P.block;
        for (int g0 = 0; g0 < nh; g0 += P.group) {
            const int map = s * P.maps_per_seq + P.map_base + (h0 + g0) / P.group;
            const ap_map_state ms = P.sel.state[map];
            const int Hh = P.sel.history;
            const int slot = (int)(ms.n_pushed % Hh);
            float* dst = P.sel.ring + ((int64_t)map * Hh + slot) * P.sel.w_max;
            float* bm0 = P.bmax + ((int64_t)s * P.n_q_heads + h0 + g0) * P.w_max;
            float mx = 0.f;  // max of the emitted row (forecaster operand scale)
            auto emit_block = [&](int64_t j) {
                float v = 0.f;
                for (int hh = 0; hh < P.group; ++hh) {
                    const float lg = __ldcg(bm0 + hh * (int64_t)P.w_max + j);
                    if (lg != -INFINITY) v = fmaxf(v, exp2f(lg - s_lse[g0 + hh]));
                    bm0[hh * (int64_t)P.w_max + j] = -INFINITY;  // untouched marker for the next step
                }
                dst[j] = v;
                mx = track_row_max(mx, v, P.sel.status);
            };
            if (P.sparse_units) {
                // only the selected blocks carry mass (sink, local, middle): zero the row, then write them
                for (int64_t j = threadIdx.x; j < W; j += ATT_THREADS) dst[j] = 0.f;
                __syncthreads();
                const int64_t sink_end = P.sel.sink < t ? P.sel.sink : t;
                const int64_t sb = (sink_end + P.block - 1) / P.block;
                int64_t lb = (t - P.sel.local > 0 ? t - P.sel.local : 0) / P.block;
                if (lb < sb) lb = sb;
                const int n_local = (int)(W - lb);
                const int n_mid = ms.n_mid;
                const int32_t* mid = P.sel.mid_blocks + (int64_t)map * (P.sel.k_mid > 0 ? P.sel.k_mid : 1);
                for (int u = threadIdx.x; u < (int)sb + n_local + n_mid; u += ATT_THREADS) {
                    const int64_t j = u < sb ? u : (u < sb + n_local ? lb + (u - sb) : mid[u - sb - n_local]);
                    emit_block(j);
                }
            } else {  // every block: the bm loads of 8 blocks x all heads in flight at once
                constexpr int U = 8;
                for (int64_t base = threadIdx.x; base < W; base += (int64_t)ATT_THREADS * U) {
                    float lg[U][8];
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int hh = 0; hh < 8; ++hh) {
                            const int64_t j = base + (int64_t)u * ATT_THREADS;
                            lg[u][hh] = (hh < P.group && j < W) ? __ldcg(bm0 + hh * (int64_t)P.w_max + j) : -INFINITY;
                        }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int64_t j = base + (int64_t)u * ATT_THREADS;
                        if (j >= W) break;
                        float v = 0.f;
#pragma unroll
                        for (int hh = 0; hh < 8; ++hh)
                            if (hh < P.group) {
                                if (lg[u][hh] != -INFINITY) v = fmaxf(v, exp2f(lg[u][hh] - s_lse[g0 + hh]));
                                bm0[hh * (int64_t)P.w_max + j] = -INFINITY;  // untouched marker for the next step
                            }
                        dst[j] = v;
                        mx = track_row_max(mx, v, P.sel.status);
                    }
                }
            }
            const int old_w = P.sel.slot_width[(int64_t)map * Hh + slot];
            for (int64_t j = W + threadIdx.x; j < old_w; j += ATT_THREADS) dst[j] = 0.f;  // zero beyond W
            mx = cta_max_nonneg(mx);
            if (threadIdx.x == 0) {
                P.sel.slot_xmax[(int64_t)map * Hh + slot] = mx;
                ap_map_state st = ms;
                P.sel.slot_width[(int64_t)map * Hh + slot] = (int32_t)W;
                st.n_pushed += 1;
                st.row_len = t;
                st.width = (int32_t)W;
                P.sel.state[map] = st;
            }
        }
    }
}

// Count this CTA's split as done; the last one (returns true) runs the combine.
// The counting atomic is acq_rel at gpu scope: after the CTA barrier it releases every thread's
// partial stores (release is cumulative over what the barrier ordered before it) and, for the last
// CTA, acquires the other splits' (read back with ld.cg, past L1).  No sequentially-consistent
// fences: under load they cost microseconds.
__device__ __forceinline__ bool last_split(int32_t* counter, int n_splits) {
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        int prev;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(counter) : "memory");
        s_last = (prev == n_splits - 1);
        if (s_last) *counter = 0;  // ready for the next launch (stream-ordered)
    }
    __syncthreads();
    return s_last;
}

// ------------------------------------------------------------------ dense
// grid (n_splits, Hkv, S); NH = Hq/Hkv q-heads per CTA share every K/V load.
template <int NH, bool WITH_V, bool EMIT>
__global__ void __launch_bounds__(ATT_THREADS) dense_partial_kernel(AttnParams P) {
    extern __shared__ float sm_att[];
    const int split = blockIdx.x, kvh = blockIdx.y, s = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, sub = lane & 15;
    const int64_t t = P.seq_len[s];
    const int b = P.block;
    const int64_t nblk = (t + b - 1) / b;
    const int64_t blk_per_split = (((int64_t)P.t_max + b - 1) / b + P.n_splits - 1) / P.n_splits;
    const int64_t j0 = split * blk_per_split, j1 = min(nblk, j0 + blk_per_split);
    const __nv_bfloat16* kh = P.k + ((int64_t)s * P.n_kv_heads + kvh) * P.t_max * HD;
    const __nv_bfloat16* vh = P.v + ((int64_t)s * P.n_kv_heads + kvh) * P.t_max * HD;
    const int h0 = kvh * NH;
    pdl_trigger();
    for (int64_t jp = j0 + warp; jp < j1 && jp < j0 + 2 * ATT_WARPS; jp += ATT_WARPS) {  // first blocks into L2
        prefetch_l2(reinterpret_cast<const char*>(kh + jp * b * HD) + lane * 128);
        if constexpr (WITH_V) prefetch_l2(reinterpret_cast<const char*>(vh + jp * b * HD) + lane * 128);
    }
    pdl_wait();  // q and the newest K/V token come from the kernel just before
    const float qscale = LOG2E * rsqrtf((float)HD);
    float qf[NH][8];
#pragma unroll
    for (int h = 0; h < NH; ++h) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(P.q + ((int64_t)s * P.n_q_heads + h0 + h) * HD + sub * 8));
        bf16x8_to_f32(u, qf[h]);
#pragma unroll
        for (int i = 0; i < 8; ++i) qf[h][i] *= qscale;
    }
    WarpState<NH, WITH_V> st;
    st.init();
    float* bm = P.bmax + ((int64_t)s * P.n_q_heads + h0) * P.w_max;
    // one block ahead: the next block's K/V loads are in flight while this one is computed
    uint4 kv[8], vv[8], kn[8], vn[8];
    int64_t j = j0 + warp;
    if (j < j1) load_block<WITH_V>(kh, vh, j, b, kv, vv);
    for (; j < j1; j += ATT_WARPS) {
        const int64_t jn = j + ATT_WARPS;
        if (jn < j1) load_block<WITH_V>(kh, vh, jn, b, kn, vn);
        compute_block<NH, WITH_V, EMIT>(kv, vv, j, b, qf, st, [&](int64_t p) { return p < t; },
                                        [&](int h, float v) { if (lane == 0) bm[h * (int64_t)P.w_max + j] = v; });
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            kv[q] = kn[q];
            if constexpr (WITH_V) vv[q] = vn[q];
        }
    }
    float* part = P.partial + (((int64_t)s * P.n_q_heads + h0) * P.n_splits + split) * (HD + 2);
    write_partial<NH, WITH_V>(st, sm_att, part, (int64_t)P.n_splits * (HD + 2));
    if (last_split(P.counters + (int64_t)s * P.n_q_heads + h0, P.n_splits)) combine_heads(P, s, h0, NH);
}

// ------------------------------------------------------------------ sparse
// grid (n_splits, maps per seq-layer, S); the NH = group q-heads of one map share its selection.
template <int NH, bool EMIT>
__global__ void __launch_bounds__(ATT_THREADS) sparse_partial_kernel(AttnParams P) {
    extern __shared__ float sm_att[];
    const int split = blockIdx.x, g = blockIdx.y, s = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, sub = lane & 15;
    const int64_t t = P.seq_len[s];
    const int b = P.block;
    const int map = s * P.maps_per_seq + P.map_base + g;
    const ap_map_state ms = P.sel.state[map];
    // selection over the row of length t (selector.py:122-147 with next_len = t)
    const int64_t sink_end = P.sel.sink < t ? P.sel.sink : t;
    const int64_t local_start = t - P.sel.local > 0 ? t - P.sel.local : 0;
    const int64_t sb = (sink_end + b - 1) / b;
    const int64_t eb = (t + b - 1) / b;
    int64_t lb = local_start / b;
    if (lb < sb) lb = sb;
    const int n_local = (int)(eb - lb);
    const int n_mid = ms.n_mid;
    const int n_units = (int)sb + n_local + n_mid;
    const int per = (n_units + P.n_splits - 1) / P.n_splits;
    const int u0 = split * per, u1 = min(n_units, u0 + per);
    const int32_t* mid = P.sel.mid_blocks + (int64_t)map * (P.sel.k_mid > 0 ? P.sel.k_mid : 1);
    const int h0 = g * NH;
    const int kvh = h0 / (P.n_q_heads / P.n_kv_heads);
    const __nv_bfloat16* kh = P.k + ((int64_t)s * P.n_kv_heads + kvh) * P.t_max * HD;
    const __nv_bfloat16* vh = P.v + ((int64_t)s * P.n_kv_heads + kvh) * P.t_max * HD;
    const float qscale = LOG2E * rsqrtf((float)HD);
    float qf[NH][8];
#pragma unroll
    for (int h = 0; h < NH; ++h) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(P.q + ((int64_t)s * P.n_q_heads + h0 + h) * HD + sub * 8));
        bf16x8_to_f32(u, qf[h]);
#pragma unroll
        for (int i = 0; i < 8; ++i) qf[h][i] *= qscale;
    }
    WarpState<NH, true> st;
    st.init();
    const int64_t mid_clip = ms.mid_clip;
    float* bm = P.bmax + ((int64_t)s * P.n_q_heads + h0) * P.w_max;
    for (int u = u0 + warp; u < u1; u += ATT_WARPS) {
        int64_t j;
        bool is_mid = false;
        if (u < sb) {
            j = u;
        } else if (u < sb + n_local) {
            j = lb + (u - sb);
        } else {
            j = mid[u - sb - n_local];
            is_mid = true;
        }
        auto take = [&](int64_t p) {
            if (p >= t) return false;
            if (p < sink_end || p >= local_start) return true;
            return is_mid && p < mid_clip;
        };
        const __nv_bfloat16* vsrc = vh;
        if (P.paged) {  // page of block j: sink | recent ring | middle page (prefetched, kernel 5)
            const int64_t vmap = ((int64_t)P.layer * P.n_seq + s) * P.n_kv_heads + kvh;
            const int npg = P.vp.sink_pages + P.vp.recent_pages + P.vp.k_cap;
            int page;
            if (is_mid) page = P.vp.sink_pages + P.vp.recent_pages + P.vp.mid_page[vmap * P.vp.k_cap + (u - sb - n_local)];
            else if (j < P.vp.sink_pages) page = (int)j;
            else page = P.vp.sink_pages + (int)(j % P.vp.recent_pages);
            // rebase so that vsrc + p*HD addresses token p of this block inside its page
            vsrc = reinterpret_cast<const __nv_bfloat16*>(P.vp.pages) + ((vmap * npg + page) * 16 - j * b) * HD;
        }
        process_block<NH, true, EMIT>(kh, vsrc, j, b, qf, st, take,
                                      [&](int h, float v) { if (lane == 0) bm[h * (int64_t)P.w_max + j] = v; });
    }
    float* part = P.partial + (((int64_t)s * P.n_q_heads + h0) * P.n_splits + split) * (HD + 2);
    write_partial<NH, true>(st, sm_att, part, (int64_t)P.n_splits * (HD + 2));
    if (last_split(P.counters + (int64_t)s * P.n_q_heads + h0, P.n_splits)) combine_heads(P, s, h0, NH);
}

// ------------------------------------------------------------------ sparse, one cluster per map
// The CL split CTAs of a map form a thread-block cluster: partials meet in distributed shared
// memory behind cluster barriers instead of a global workspace + completion counter, the CTA of
// rank h finalises q-head h, and every CTA emits the compressed-row values of its own blocks once
// the LSEs are known (the rest of the row was zeroed by the CTAs at the start, off the critical
// path).  Same arithmetic as sparse_partial_kernel + combine_heads.
template <int NH>
__device__ void merge_warps_to_smem(WarpState<NH, true>& st, float* scratch, float (*cpart)[HD + 2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, half = lane >> 4, sub = lane & 15;
#pragma unroll
    for (int h = 0; h < NH; ++h)
#pragma unroll
        for (int i = 0; i < 8; ++i) st.acc[h][i] += __shfl_xor_sync(0xffffffffu, st.acc[h][i], 16);
    float* w = scratch + warp * NH * (HD + 2);
#pragma unroll
    for (int h = 0; h < NH; ++h) {
        if (lane == 0) {
            w[h * (HD + 2) + 0] = st.m[h];
            w[h * (HD + 2) + 1] = st.l[h];
        }
        if (half == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) w[h * (HD + 2) + 2 + sub * 8 + i] = st.acc[h][i];
        }
    }
    __syncthreads();
    // per head: the CTA max and each warp's rescale factor, once
    __shared__ float s_scale[NH][ATT_WARPS];
    if (threadIdx.x < NH * ATT_WARPS) {
        const int h = threadIdx.x / ATT_WARPS, ww = threadIdx.x % ATT_WARPS;
        float M = -INFINITY;
#pragma unroll
        for (int v = 0; v < ATT_WARPS; ++v) M = fmaxf(M, scratch[(v * NH + h) * (HD + 2)]);
        const float mw = scratch[(ww * NH + h) * (HD + 2)];
        s_scale[h][ww] = mw == -INFINITY ? 0.f : exp2f(mw - M);
        if (ww == 0) cpart[h][0] = M;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < NH * (HD + 1); idx += ATT_THREADS) {
        const int h = idx / (HD + 1), e = 1 + idx % (HD + 1);  // l and the 128 accumulators
        float val = 0.f;
#pragma unroll
        for (int ww = 0; ww < ATT_WARPS; ++ww) val = fmaf(scratch[(ww * NH + h) * (HD + 2) + e], s_scale[h][ww], val);
        cpart[h][e] = val;
    }
}

// ------------------------------------------------------------------ tensor-core block path
// (sparse cluster kernel) One warp, one 16-token block, all NH <= 8 q-heads of the map:
// S = Q Kᵀ and O += P V as mma.sync m16n8k16 (bf16 in, fp32 accumulate); rows = q-heads (NH real
// of 16), K/V read from the warp's shared-memory stage with ldmatrix.  The stage holds K then V,
// each as two TMA boxes {64 dims, 16 tokens} in the 128-byte-swizzled layout (16-byte chunk c of
// token row r at chunk c ^ (r & 7)), so the 8 rows of every ldmatrix fragment hit distinct banks.
// Thread (g = lane/4, t = lane%4) holds row g.
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
// d += A(16x16, rows g / g+8) B(16x8); a1 = a3 = 0 (rows 8-15 are padding)
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
                 "{%0, %1, %2, %3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}

struct MmaState {
    float m, l;       // row g's running max (log2 units) and sum, replicated over the quad
    float o[16][4];   // O row g (o[nt][0..1] = dims nt*8 + 2t, +1); [2..3] = padding rows
    __device__ void init() {
        m = -INFINITY;
        l = 0.f;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) o[nt][e] = 0.f;
    }
};

// kb / vb: the block's K / V tile in shared memory (two swizzled 2 KB halves each).
// qa[kk][0/1]: the Q A-fragment (a0, a2) of k-step kk (zero for rows >= NH).
template <int NH, bool EMIT, typename Take, typename BmOut>
__device__ __forceinline__ void block_mma(uint32_t kb, uint32_t vb, int64_t j, int b, const uint32_t (&qa)[8][2],
                                          float qscale, MmaState& st, Take take, BmOut bm_out) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, mi = lane >> 3, r = lane & 7;
    float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    // K fragments: matrices (tokens 0-7 | 8-15) x (dims +0..7 | +8..15) of k-step kk
    const uint32_t krow = kb + (uint32_t)((((mi >> 1) << 3) | r) * 128);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        uint32_t bk[4];
        const int c = ((kk & 3) << 1) | (mi & 1);
        ldsm_x4(krow + (kk >> 2) * 2048 + ((c ^ r) << 4), bk);
        mma_bf16_16816(sc[0], qa[kk][0], qa[kk][1], bk[0], bk[1]);
        mma_bf16_16816(sc[1], qa[kk][0], qa[kk][1], bk[2], bk[3]);
    }
    const bool real = g < NH;
    float s[4];
    float mx = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int64_t p = j * b + nt * 8 + 2 * t + e;
            const float v = (real && take(p)) ? sc[nt][e] * qscale : -INFINITY;
            s[nt * 2 + e] = v;
            mx = fmaxf(mx, v);
        }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    if constexpr (EMIT) {
        if (real && t == 0) bm_out(g, mx);
    }
    float pr[4] = {0.f, 0.f, 0.f, 0.f};
    float corr = 1.f;
    if (mx != -INFINITY) {  // quad-uniform
        const float m_new = fmaxf(st.m, mx);
        corr = exp2f(st.m - m_new);  // 0 when st.m = -inf
#pragma unroll
        for (int e = 0; e < 4; ++e) pr[e] = exp2f(s[e] - m_new);  // 0 for masked tokens
        st.m = m_new;
    }
    float rs = (pr[0] + pr[1]) + (pr[2] + pr[3]);
    rs += __shfl_xor_sync(0xffffffffu, rs, 1);
    rs += __shfl_xor_sync(0xffffffffu, rs, 2);
    st.l = st.l * corr + rs;
    const bool any = __any_sync(0xffffffffu, mx != -INFINITY);
    if (!any) return;  // nothing selected in this block for any head: never touch its V
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
        st.o[nt][0] *= corr;
        st.o[nt][1] *= corr;
    }
    const uint32_t a0 = pack_bf16x2(pr[0], pr[1]), a2 = pack_bf16x2(pr[2], pr[3]);
    // V fragments (transposed): matrices (tokens 0-7 | 8-15) x (dims n0 + 0..7 | n0 + 8..15)
    const uint32_t vrow = vb + (uint32_t)((((mi & 1) << 3) | r) * 128);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        uint32_t bv[4];
        const int c = ((q & 3) << 1) | (mi >> 1);
        ldsm_x4_t(vrow + (q >> 2) * 2048 + ((c ^ r) << 4), bv);
        mma_bf16_16816(st.o[2 * q], a0, a2, bv[0], bv[1]);
        mma_bf16_16816(st.o[2 * q + 1], a0, a2, bv[2], bv[3]);
    }
}

// CTA merge of the warps' MmaStates into cpart[h] = (max, sum, acc[128]) (same result layout as
// merge_warps_to_smem).
template <int NH>
__device__ void merge_mma_to_smem(const MmaState& st, float* scratch, float (*cpart)[HD + 2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
    if (g < NH) {
        float* w = scratch + (warp * NH + g) * (HD + 2);
        if (t == 0) {
            w[0] = st.m;
            w[1] = st.l;
        }
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
            w[2 + nt * 8 + 2 * t] = st.o[nt][0];
            w[2 + nt * 8 + 2 * t + 1] = st.o[nt][1];
        }
    }
    __syncthreads();
    __shared__ float s_scale[NH][ATT_WARPS];
    if (threadIdx.x < NH * ATT_WARPS) {
        const int h = threadIdx.x / ATT_WARPS, ww = threadIdx.x % ATT_WARPS;
        float M = -INFINITY;
#pragma unroll
        for (int v = 0; v < ATT_WARPS; ++v) M = fmaxf(M, scratch[(v * NH + h) * (HD + 2)]);
        const float mw = scratch[(ww * NH + h) * (HD + 2)];
        s_scale[h][ww] = mw == -INFINITY ? 0.f : exp2f(mw - M);
        if (ww == 0) cpart[h][0] = M;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < NH * (HD + 1); idx += ATT_THREADS) {
        const int h = idx / (HD + 1), e = 1 + idx % (HD + 1);  // l and the 128 accumulators
        float val = 0.f;
#pragma unroll
        for (int ww = 0; ww < ATT_WARPS; ++ww) val = fmaf(scratch[(ww * NH + h) * (HD + 2) + e], s_scale[h][ww], val);
        cpart[h][e] = val;
    }
}

// Dense pass on tensor cores (output path, NH >= 2): grid (n_splits, Hkv, S) as dense_partial_kernel,
// each warp streaming its blocks through a 2-slot TMA ring (K/V boxes as in the sparse cluster
// kernel) into block_mma; partials combined by the last split (combine_heads).
template <int NH, bool EMIT>
__global__ void __launch_bounds__(ATT_THREADS, 1) dense_tc_kernel(const __grid_constant__ CUtensorMap kmap,
                                                               const __grid_constant__ CUtensorMap vmap,
                                                               AttnParams P) {
    extern __shared__ float sm_att[];  // [warps][NH][HD+2] merge scratch, then the staging rings
    __shared__ float cpart[NH][HD + 2];
    __shared__ __align__(8) uint64_t s_kvbar[ATT_WARPS][2];
    const int split = blockIdx.x, kvh = blockIdx.y, s = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = P.seq_len[s];
    const int b = P.block;
    const int64_t nblk = (t + b - 1) / b;
    const int64_t blk_per_split = (((int64_t)P.t_max + b - 1) / b + P.n_splits - 1) / P.n_splits;
    const int64_t j0 = split * blk_per_split, j1 = min(nblk, j0 + blk_per_split);
    const int h0 = kvh * NH;
    uint8_t* ring = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(sm_att + ATT_WARPS * NH * (HD + 2)) + 1023) & ~uintptr_t(1023));
    uint8_t* my_ring = ring + warp * 2 * KV_STAGE;
    if (lane == 0) {
        mbar_init(&s_kvbar[warp][0], 1);
        mbar_init(&s_kvbar[warp][1], 1);
    }
    __syncwarp();
    pdl_trigger();
    const int row0 = (int)(((int64_t)s * P.n_kv_heads + kvh) * P.t_max);
    auto issue = [&](int slot, int64_t j) {
        if (lane == 0) {
            uint8_t* d = my_ring + slot * KV_STAGE;
            const int row = row0 + (int)(j * b);
            mbar_arrive_tx(&s_kvbar[warp][slot], KV_STAGE);
            tma_load_2d(d, &kmap, 0, row, &s_kvbar[warp][slot]);
            tma_load_2d(d + 2048, &kmap, 64, row, &s_kvbar[warp][slot]);
            tma_load_2d(d + 4096, &vmap, 0, row, &s_kvbar[warp][slot]);
            tma_load_2d(d + 6144, &vmap, 64, row, &s_kvbar[warp][slot]);
        }
    };
    // the first two blocks of each warp before the programmatic-dependent-launch wait, unless they
    // hold the newest token (written by the kernel just before)
    bool issued[2] = {false, false};
    for (int i = 0; i < 2; ++i) {
        const int64_t j = j0 + warp + i * ATT_WARPS;
        if (j < j1 && j != nblk - 1) {
            issue(i, j);
            issued[i] = true;
        }
    }
    pdl_wait();
    const float qscale = LOG2E * rsqrtf((float)HD);
    uint32_t qa[8][2];
    {
        const int g = lane >> 2, t4 = lane & 3;
        const uint32_t* qrow =
            reinterpret_cast<const uint32_t*>(P.q + ((int64_t)s * P.n_q_heads + h0 + (g < NH ? g : 0)) * HD);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            qa[kk][0] = g < NH ? qrow[kk * 8 + t4] : 0u;
            qa[kk][1] = g < NH ? qrow[kk * 8 + 4 + t4] : 0u;
        }
    }
    for (int i = 0; i < 2; ++i) {
        const int64_t j = j0 + warp + i * ATT_WARPS;
        if (j < j1 && !issued[i]) issue(i, j);
    }
    MmaState st;
    st.init();
    float* bm = P.bmax + ((int64_t)s * P.n_q_heads + h0) * P.w_max;
    int i = 0;
    for (int64_t j = j0 + warp; j < j1; j += ATT_WARPS, ++i) {
        const int slot = i & 1;
        mbar_wait(&s_kvbar[warp][slot], (uint32_t)((i >> 1) & 1));
        const uint32_t kb = smem_u32(my_ring + slot * KV_STAGE);
        block_mma<NH, EMIT>(kb, kb + KV_STAGE / 2, j, b, qa, qscale, st, [&](int64_t p) { return p < t; },
                            [&](int h, float v) { bm[h * (int64_t)P.w_max + j] = v; });
        __syncwarp();
        if (j + 2 * ATT_WARPS < j1) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(slot, j + 2 * ATT_WARPS);
        }
    }
    merge_mma_to_smem<NH>(st, sm_att, cpart);
    __syncthreads();
    float* part = P.partial + (((int64_t)s * P.n_q_heads + h0) * P.n_splits + split) * (HD + 2);
    for (int idx = threadIdx.x; idx < NH * (HD + 2); idx += ATT_THREADS) {
        const int h = idx / (HD + 2), e = idx % (HD + 2);
        part[h * (int64_t)P.n_splits * (HD + 2) + e] = cpart[h][e];
    }
    if (last_split(P.counters + (int64_t)s * P.n_q_heads + h0, P.n_splits)) combine_heads(P, s, h0, NH);
}

// DSMEM push helpers: 32-bit shared::cluster address of a local variable in CTA `rank`, and
// register -> remote shared memory stores that complete_tx on the receiver's mbarrier.
__device__ __forceinline__ uint32_t mapa_u32(const void* p, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_v4(uint32_t addr, float a, float b, float c, float d, uint32_t mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                 :: "r"(addr), "f"(a), "f"(b), "f"(c), "f"(d), "r"(mbar) : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t addr, float a, float b, uint32_t mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];"
                 :: "r"(addr), "f"(a), "f"(b), "r"(mbar) : "memory");
}

// CL = cluster size = splits per map (2/4/8 portable, 16 with the non-portable opt-in); launched with
// the cluster dimension as a launch attribute.  The splits exchange their partials by pushing them
// (st.async) into the peers' shared memory: every rank receives every split's (m, l) of all NH heads,
// and rank h % CL the accumulators of q-head h; each waits on its own mbarrier only (no cluster-wide
// barrier on the critical path, nobody reads a peer's shared memory, so no exit barrier either).
template <int NH, bool EMIT, int CL>
__global__ void __launch_bounds__(ATT_THREADS) sparse_cluster_kernel(const __grid_constant__ CUtensorMap kmap,
                                                                     const __grid_constant__ CUtensorMap vmap,
                                                                     AttnParams P) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    constexpr int NFIN = (NH + CL - 1) / CL;                // q-heads a rank finalises (at most)
    __shared__ float cpart[NH][HD + 2];                     // this split's (m, l, acc) per head
    __shared__ __align__(16) float s_ml_in[CL][NH][2];      // every split's (m, l) per head
    __shared__ __align__(16) float s_acc_in[NFIN][CL][HD];  // every split's acc of the heads finalised here
    __shared__ __align__(8) uint64_t s_rx;                  // completes when all of the above has landed
    __shared__ float s_lse[NH];                             // LSE of every head
    __shared__ float s_w[NH][CL];                           // weight of split r in q-head h's output
    extern __shared__ float sm_att[];    // [warps][NH][HD+2] merge scratch, then [units][NH] block maxima
    const int split = (int)cluster.block_rank(), g = blockIdx.y, s = blockIdx.z;
    if (threadIdx.x == 0) {
        const int n_fin = split < NH ? (NH - split + CL - 1) / CL : 0;
        mbar_init(&s_rx, 1);
        mbar_arrive_tx(&s_rx, (uint32_t)(CL * NH * 2 * 4 + n_fin * CL * HD * 4));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // every peer's receive barrier must be initialised before anyone pushes: arrive now, wait (free by
    // then) just before the pushes.  The init is published by fence.mbarrier_init above, so the arrive
    // can be relaxed (a release arrive is a memory barrier on every thread: ncu put ~6% of the stall
    // samples here)
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    ATT_TRACE(0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    pdl_trigger();
    // Until pdl_wait: only data older than the previous kernel (positions, map state and selection,
    // the ring slot being replaced) — q and the newest K/V token come from the kernel just before.
    const int b = P.block;
    const int map = s * P.maps_per_seq + P.map_base + g;
    const int32_t* mid = P.sel.mid_blocks + (int64_t)map * (P.sel.k_mid > 0 ? P.sel.k_mid : 1);
    // the map's whole middle-block row is fetched together with the position and the map state (one
    // round trip instead of state -> ids), then sliced from shared memory
    const int per_max = (((P.sel.sink + b - 1) / b + P.sel.local / b + 2 + P.sel.k_mid) + CL - 1) / CL;
    int* s_mid = reinterpret_cast<int*>(sm_att + ATT_WARPS * NH * (HD + 2)) + per_max * (NH + 1);
    const int mv = (int)threadIdx.x < P.sel.k_mid ? __ldg(mid + threadIdx.x) : 0;  // in flight with the two below
    // 32-bit position arithmetic in the prologue (t < 2^31): 64-bit integer division is a ~100-cycle
    // software routine, and the prologue sits on the critical path of every layer
    const int t = P.seq_len[s];
    const ap_map_state ms = P.sel.state[map];
    if ((int)threadIdx.x < P.sel.k_mid) s_mid[threadIdx.x] = mv;
    for (int i = threadIdx.x + ATT_THREADS; i < P.sel.k_mid; i += ATT_THREADS) s_mid[i] = mid[i];  // k_mid > 256
    const int sink_end = P.sel.sink < t ? P.sel.sink : t;
    const int local_start = t - P.sel.local > 0 ? t - P.sel.local : 0;
    const int sb = (sink_end + b - 1) / b;
    const int eb = (t + b - 1) / b;
    int lb = local_start / b;
    if (lb < sb) lb = sb;
    const int n_local = (int)(eb - lb);
    const int n_units = (int)sb + n_local + ms.n_mid;
    const int per = (n_units + CL - 1) / CL;
    const int u0 = split * per, u1 = min(n_units, u0 + per);
#ifdef AP_ATT_TRACE
    if (threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && g_att_trace_on)
        g_att_trace[blockIdx.x * 16 + 12] = clock64() + (u1 & 0);  // after the state load is consumed
#endif
    const int h0 = g * NH;
    const int kvh = h0 / (P.n_q_heads / P.n_kv_heads);
    const __nv_bfloat16* kh = P.k + ((int64_t)s * P.n_kv_heads + kvh) * P.t_max * HD;
    const __nv_bfloat16* vh = P.v + ((int64_t)s * P.n_kv_heads + kvh) * P.t_max * HD;
    float* s_bm = sm_att + ATT_WARPS * NH * (HD + 2);  // [per][NH]

    const int Hh = P.sel.history;
    const int slot = (int)((uint32_t)ms.n_pushed % (uint32_t)Hh);  // n_pushed < 2^32
    float* dst = P.sel.ring + ((int64_t)map * Hh + slot) * P.sel.w_max;
    const int64_t W = eb;
    ATT_TRACE(13);
    if constexpr (EMIT) {  // zero this CTA's share of the whole ring row (rows are zero beyond their width;
                           // no dependent read of the slot's old width), refilled after the exchange
        const int Z = P.sel.w_max;
        const int z0 = Z * split / CL, z1 = Z * (split + 1) / CL;
        for (int j = z0 + threadIdx.x; j < z1; j += ATT_THREADS) dst[j] = 0.f;
        if (split == 0 && threadIdx.x == 0) P.sel.slot_xmax[(int64_t)map * Hh + slot] = 0.f;  // atomicMax'd later
    }
    // block id of each of this CTA's units (sink | local | middle), gathered once into shared memory
    int* s_blk = reinterpret_cast<int*>(s_bm + per * NH);
    ATT_TRACE(9);
    __syncthreads();  // s_mid landed
    ATT_TRACE(10);
    for (int i = threadIdx.x; i < u1 - u0; i += ATT_THREADS) {
        const int u = u0 + i;
        s_blk[i] = u < sb ? u : (u < sb + n_local ? (int)(lb + (u - sb)) : s_mid[u - sb - n_local]);
    }
    __syncthreads();
    ATT_TRACE(11);
    auto block_of = [&](int u, bool& is_mid) -> int64_t {
        is_mid = u >= sb + n_local;
        return s_blk[u - u0];
    };
    auto v_of = [&](int u, int64_t j, bool is_mid) -> const __nv_bfloat16* {
        if (!P.paged) return vh;
        // page of block j: sink | recent ring | middle page (prefetched, kernel 5); rebased so that
        // vsrc + p*HD addresses token p of this block inside its page
        const int64_t vmap = ((int64_t)P.layer * P.n_seq + s) * P.n_kv_heads + kvh;
        const int npg = P.vp.sink_pages + P.vp.recent_pages + P.vp.k_cap;
        int page;
        if (is_mid) page = P.vp.sink_pages + P.vp.recent_pages + P.vp.mid_page[vmap * P.vp.k_cap + (u - sb - n_local)];
        else if (j < P.vp.sink_pages) page = (int)j;
        else page = P.vp.sink_pages + (int)(j % P.vp.recent_pages);
        return reinterpret_cast<const __nv_bfloat16*>(P.vp.pages) + ((vmap * npg + page) * 16 - j * b) * HD;
    };
    // NH >= 2 (q-heads sharing a map): tensor-core path.  K/V staging: each warp owns a 2-slot ring
    // of 8 KB (K block | V block) filled by TMA, so the next block's copy is in flight while this one
    // is computed.  The first two blocks are requested before the programmatic-dependent-launch wait
    // unless they hold the newest token (written by the kernel just before) or their V lives in the
    // prefetched pages.  NH == 1 (one map per q-head): the SIMT path (one MMA row of 16 would be
    // busy) with the blocks prefetched into L2 and no staging, so the kernel's small shared-memory
    // footprint lets the next projection's CTAs start on the same SMs.
    constexpr bool TC = NH >= 2;
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(s_mid + P.sel.k_mid) + 1023) & ~uintptr_t(1023));
    uint8_t* my_ring = ring + warp * 2 * KV_STAGE;
    __shared__ __align__(8) uint64_t s_kvbar[ATT_WARPS][2];
    if (TC && lane == 0) {
        mbar_init(&s_kvbar[warp][0], 1);
        mbar_init(&s_kvbar[warp][1], 1);
    }
    __syncwarp();
    auto issue = [&](int slot, int u) {  // whole warp (lane 0 issues): four TMA boxes {64 dims, 16 tokens}
        bool is_mid;
        const int64_t j = block_of(u, is_mid);
        if (lane == 0) {
            uint8_t* d = my_ring + slot * KV_STAGE;
            const int krow = (int)(((int64_t)s * P.n_kv_heads + kvh) * P.t_max + j * b);
            int vrow = krow;
            if (P.paged) {  // page of block j (as v_of), row index in the page store
                const int64_t vm = ((int64_t)P.layer * P.n_seq + s) * P.n_kv_heads + kvh;
                const int npg = P.vp.sink_pages + P.vp.recent_pages + P.vp.k_cap;
                int page;
                if (is_mid) page = P.vp.sink_pages + P.vp.recent_pages + P.vp.mid_page[vm * P.vp.k_cap + (u - sb - n_local)];
                else if (j < P.vp.sink_pages) page = (int)j;
                else page = P.vp.sink_pages + (int)(j % P.vp.recent_pages);
                vrow = (int)((vm * npg + page) * 16);
            }
            mbar_arrive_tx(&s_kvbar[warp][slot], KV_STAGE);
            tma_load_2d(d, &kmap, 0, krow, &s_kvbar[warp][slot]);
            tma_load_2d(d + 2048, &kmap, 64, krow, &s_kvbar[warp][slot]);
            tma_load_2d(d + 4096, &vmap, 0, vrow, &s_kvbar[warp][slot]);
            tma_load_2d(d + 6144, &vmap, 64, vrow, &s_kvbar[warp][slot]);
        }
    };
    bool issued[2] = {false, false};
    if (TC && !P.paged)
        for (int i = 0; i < 2; ++i) {
            const int u = u0 + warp + i * ATT_WARPS;
            if (u >= u1) break;
            bool is_mid;
            if (block_of(u, is_mid) == eb - 1) continue;
            issue(i, u);
            issued[i] = true;
        }
    for (int u = u0 + warp + (TC ? 2 * ATT_WARPS : 0); u < u1; u += ATT_WARPS) {  // blocks into L2 (8 KB each)
        bool is_mid;
        const int64_t j = block_of(u, is_mid);
        const char* kb = reinterpret_cast<const char*>(kh + j * b * HD);
        const char* vb = reinterpret_cast<const char*>(vh + j * b * HD);
        prefetch_l2(kb + lane * 128);
        if (!P.paged) prefetch_l2(vb + lane * 128);
    }
    ATT_TRACE(1);
    pdl_wait();
    const float qscale = LOG2E * rsqrtf((float)HD);
    ATT_TRACE(2);
    const int64_t mid_clip = ms.mid_clip;
    auto take_of = [&](bool is_mid) {
        return [=](int64_t p) {
            if (p >= t) return false;
            if (p < sink_end || p >= local_start) return true;
            return is_mid && p < mid_clip;
        };
    };
    if constexpr (TC) {
        uint32_t qa[8][2];  // Q A-fragments (row g = q-head h0 + g), zero for padding rows
        {
            const int g = lane >> 2, t4 = lane & 3;
            const uint32_t* qrow =
                reinterpret_cast<const uint32_t*>(P.q + ((int64_t)s * P.n_q_heads + h0 + (g < NH ? g : 0)) * HD);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                qa[kk][0] = g < NH ? qrow[kk * 8 + t4] : 0u;
                qa[kk][1] = g < NH ? qrow[kk * 8 + 4 + t4] : 0u;
            }
        }
        MmaState st;
        st.init();
        for (int i = 0; i < 2; ++i) {
            const int u = u0 + warp + i * ATT_WARPS;
            if (u < u1 && !issued[i]) issue(i, u);
        }
        int i = 0;
        for (int u = u0 + warp; u < u1; u += ATT_WARPS, ++i) {
            bool is_mid;
            const int64_t j = block_of(u, is_mid);
            const int slot = i & 1;
            mbar_wait(&s_kvbar[warp][slot], (uint32_t)((i >> 1) & 1));
            const uint32_t kb = smem_u32(my_ring + slot * KV_STAGE);
            block_mma<NH, EMIT>(kb, kb + KV_STAGE / 2, j, b, qa, qscale, st, take_of(is_mid),
                                [&](int h, float v) { s_bm[(u - u0) * NH + h] = v; });
            __syncwarp();
            if (u + 2 * ATT_WARPS < u1) {  // refill this slot with the block after next
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(slot, u + 2 * ATT_WARPS);
            }
        }
        ATT_TRACE(3);
        merge_mma_to_smem<NH>(st, sm_att, cpart);
    } else {
        const int sub = lane & 15;
        float qf[NH][8];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(P.q + ((int64_t)s * P.n_q_heads + h0 + h) * HD + sub * 8));
            bf16x8_to_f32(u, qf[h]);
#pragma unroll
            for (int i = 0; i < 8; ++i) qf[h][i] *= qscale;
        }
        WarpState<NH, true> st;
        st.init();
        for (int u = u0 + warp; u < u1; u += ATT_WARPS) {
            bool is_mid;
            const int64_t j = block_of(u, is_mid);
            process_block<NH, true, EMIT>(kh, v_of(u, j, is_mid), j, b, qf, st, take_of(is_mid),
                                          [&](int h, float v) { if (lane == 0) s_bm[(u - u0) * NH + h] = v; });
        }
        ATT_TRACE(3);
        merge_warps_to_smem<NH>(st, sm_att, cpart);
    }
    __syncthreads();
    ATT_TRACE(4);
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    // push: (m, l) of head h to every rank; acc of head h (32 x 16 B) to rank h % CL
    if (threadIdx.x < CL * NH) {
        const int q = threadIdx.x / NH, h = threadIdx.x % NH;
        st_async_v2(mapa_u32(&s_ml_in[split][h][0], q), cpart[h][0], cpart[h][1], mapa_u32(&s_rx, q));
    }
    for (int idx = threadIdx.x; idx < NH * (HD / 4); idx += ATT_THREADS) {
        const int h = idx / (HD / 4), c = idx % (HD / 4), q = h % CL;
        const float* a = &cpart[h][2 + 4 * c];
        st_async_v4(mapa_u32(&s_acc_in[h / CL][split][4 * c], q), a[0], a[1], a[2], a[3], mapa_u32(&s_rx, q));
    }
    mbar_wait(&s_rx, 0);
    ATT_TRACE(5);
    if (threadIdx.x < NH) {  // LSE and split weights of every head
        const int h = threadIdx.x;
        float M = -INFINITY;
#pragma unroll
        for (int r = 0; r < CL; ++r) M = fmaxf(M, s_ml_in[r][h][0]);
        float wr[CL], L = 0.f;
#pragma unroll
        for (int r = 0; r < CL; ++r) {
            const float mr = s_ml_in[r][h][0];
            wr[r] = mr == -INFINITY ? 0.f : exp2f(mr - M);
            L += s_ml_in[r][h][1] * wr[r];
        }
        s_lse[h] = M + log2f(L);
#pragma unroll
        for (int r = 0; r < CL; ++r) s_w[h][r] = wr[r] / L;
    }
    __syncthreads();
    if (threadIdx.x < HD) {  // warps 0-3: rank r finalises q-heads r, r + CL, ... over the CL partials
        for (int h = split; h < NH; h += CL) {
            float o = 0.f;
#pragma unroll
            for (int r = 0; r < CL; ++r) o = fmaf(s_acc_in[h / CL][r][threadIdx.x], s_w[h][r], o);
            P.out[((int64_t)s * P.n_q_heads + h0 + h) * HD + threadIdx.x] = __float2bfloat16_rn(o);
            if (threadIdx.x == 0 && P.lse) P.lse[(int64_t)s * P.n_q_heads + h0 + h] = s_lse[h];
        }
        ATT_TRACE(6);
    } else if constexpr (EMIT) {  // warps 4-7, concurrently: the compressed-row values of this CTA's units
        const int et = threadIdx.x - HD;
        float lse[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) lse[h] = s_lse[h];
        float mx = 0.f;
        for (int u = u0 + et; u < u1; u += ATT_THREADS - HD) {
            bool is_mid;
            const int64_t j = block_of(u, is_mid);
            float v = 0.f;
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                const float lg = s_bm[(u - u0) * NH + h];
                if (lg != -INFINITY) v = fmaxf(v, exp2f(lg - lse[h]));
            }
            dst[j] = v;
            mx = track_row_max(mx, v, P.sel.status);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0 && mx > 0.f)  // per warp (non-negative floats order as ints)
            atomicMax(reinterpret_cast<int*>(P.sel.slot_xmax + (int64_t)map * Hh + slot), __float_as_int(mx));
        if (split == 0 && et == 0) {
            ap_map_state st2 = ms;
            P.sel.slot_width[(int64_t)map * Hh + slot] = (int32_t)W;
            st2.n_pushed += 1;
            st2.row_len = t;
            st2.width = (int32_t)W;
            P.sel.state[map] = st2;
        }
    }
    ATT_TRACE(7);
    ATT_TRACE(8);
}

template <int NH>
static void launch_dense(const AttnParams& P, bool with_v, bool emit, cudaStream_t st) {
    dim3 grid(P.n_splits, P.n_kv_heads, P.n_seq);
    const size_t sm = (size_t)ATT_WARPS * NH * (HD + 2) * sizeof(float);
    {
        if (with_v) {  // tensor-core output path
            CUtensorMap kmap, vmap;
            const uint64_t rows = (uint64_t)P.n_seq * P.n_kv_heads * P.t_max;
            if (make_tmap_bf16_sw128(&kmap, P.k, rows, HD, 16) && make_tmap_bf16_sw128(&vmap, P.v, rows, HD, 16)) {
                const size_t smtc = sm + 1024 + (size_t)ATT_WARPS * 2 * KV_STAGE;
                auto k = emit ? dense_tc_kernel<NH, true> : dense_tc_kernel<NH, false>;
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smtc);
                launch_ex(k, grid, dim3(ATT_THREADS), smtc, st, 1, kmap, vmap, P);
                return;
            }
        }
    }
    if (with_v && emit) launch_ex(dense_partial_kernel<NH, true, true>, grid, dim3(ATT_THREADS), sm, st, 1, P);
    else if (with_v) launch_ex(dense_partial_kernel<NH, true, false>, grid, dim3(ATT_THREADS), sm, st, 1, P);
    else launch_ex(dense_partial_kernel<NH, false, true>, grid, dim3(ATT_THREADS), sm, st, 1, P);
}

template <int NH, bool EMIT, int CL>
static int launch_cluster(const AttnParams& P, cudaStream_t st) {
    const int units_max = (P.sel.sink + P.block - 1) / P.block + P.sel.local / P.block + 2 + P.sel.k_mid;
    const size_t sm = ((size_t)ATT_WARPS * NH * (HD + 2) + (size_t)((units_max + CL - 1) / CL) * (NH + 1) +
                       (size_t)P.sel.k_mid) * sizeof(float) +
                      (NH >= 2 ? 1024 + (size_t)ATT_WARPS * 2 * KV_STAGE : 0);  // + the K/V staging rings (128 KB)
    auto k = sparse_cluster_kernel<NH, EMIT, CL>;
    if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (CL > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    // K (and V, or the offload page store) as [rows][128] bf16 for {64, 16} TMA boxes
    CUtensorMap kmap, vmap;
    const uint64_t kv_rows = (uint64_t)P.n_seq * P.n_kv_heads * P.t_max;
    bool ok = make_tmap_bf16_sw128(&kmap, P.k, kv_rows, HD, 16);
    if (P.paged) {
        const uint64_t npg = (uint64_t)(P.vp.sink_pages + P.vp.recent_pages + P.vp.k_cap);
        ok = ok && make_tmap_bf16_sw128(&vmap, P.vp.pages, (uint64_t)(P.layer + 1) * P.n_seq * P.n_kv_heads * npg * 16,
                                        HD, 16);
    } else {
        ok = ok && make_tmap_bf16_sw128(&vmap, P.v, kv_rows, HD, 16);
    }
    AP_REQUIRE(ok, AP_ECUDA, "tensor map for the sparse attention failed");
    launch_ex(k, dim3(CL, P.n_q_heads / NH, P.n_seq), dim3(ATT_THREADS), sm, st, CL, kmap, vmap, P);
    return AP_OK;
}

template <int NH>
static int launch_sparse(const AttnParams& P, bool emit, cudaStream_t st) {
    switch (P.n_splits) {  // cluster form: the splits of a map are one thread-block cluster
        case 2: return emit ? launch_cluster<NH, true, 2>(P, st) : launch_cluster<NH, false, 2>(P, st);
        case 4: return emit ? launch_cluster<NH, true, 4>(P, st) : launch_cluster<NH, false, 4>(P, st);
        case 8: return emit ? launch_cluster<NH, true, 8>(P, st) : launch_cluster<NH, false, 8>(P, st);
        case 16: return emit ? launch_cluster<NH, true, 16>(P, st) : launch_cluster<NH, false, 16>(P, st);
        default: break;
    }
    dim3 grid(P.n_splits, P.n_q_heads / NH, P.n_seq);
    const size_t sm = (size_t)ATT_WARPS * NH * (HD + 2) * sizeof(float);
    if (emit) sparse_partial_kernel<NH, true><<<grid, ATT_THREADS, sm, st>>>(P);
    else sparse_partial_kernel<NH, false><<<grid, ATT_THREADS, sm, st>>>(P);
    return AP_OK;
}

static int make_params(const ap_attn_layer* a, const ap_selector* sel, int32_t map_base, int32_t maps_per_seq,
                       int32_t group, AttnParams& P) {
    AP_REQUIRE(a && a->head_dim == HD, AP_EPARAM, "head_dim must be 128");
    AP_REQUIRE(a->n_q_heads % a->n_kv_heads == 0, AP_EPARAM, "n_q_heads must be a multiple of n_kv_heads");
    AP_REQUIRE(a->n_splits >= 1 && a->n_splits <= 64, AP_EPARAM, "n_splits must be in [1, 64]");
    AP_REQUIRE(a->block == 16, AP_EPARAM, "attention kernels assume 16-token blocks");
    AP_REQUIRE(a->t_max % a->block == 0, AP_EPARAM, "t_max must be a multiple of the block size");
    P.n_seq = a->n_seq; P.n_q_heads = a->n_q_heads; P.n_kv_heads = a->n_kv_heads; P.t_max = a->t_max;
    P.n_splits = a->n_splits; P.block = a->block;
    P.q = (const __nv_bfloat16*)a->q; P.k = (const __nv_bfloat16*)a->k_cache; P.v = (const __nv_bfloat16*)a->v_cache;
    P.seq_len = a->seq_len; P.out = (__nv_bfloat16*)a->out; P.lse = a->lse; P.partial = a->partial;
    P.bmax = a->bmax; P.w_max = a->w_max; P.counters = a->counters;
    AP_REQUIRE(a->counters != nullptr, AP_EPARAM, "counters workspace is required");
    // the kernels use P.block for the sink/local/middle units and the emitted width, the selector masks in
    // sel->block units and its ring rows are w_max wide: both must agree with the attention descriptor
    AP_REQUIRE(!sel || sel->block == a->block, AP_ECONFIG, "selector block size %d != attention block size %d",
               sel ? sel->block : 0, a->block);
    AP_REQUIRE(!sel || sel->w_max >= (a->t_max + a->block - 1) / a->block, AP_ECONFIG,
               "selector w_max %d < ceil(t_max / block) = %d", sel ? sel->w_max : 0,
               (a->t_max + a->block - 1) / a->block);
    if (sel) P.sel = *sel; else memset(&P.sel, 0, sizeof(P.sel));
    memset(&P.vp, 0, sizeof(P.vp));
    P.sparse_units = 0;
    P.paged = 0;
    P.layer = 0;
    P.map_base = map_base; P.maps_per_seq = maps_per_seq; P.group = group < 1 ? 1 : group;
    const int G = a->n_q_heads / a->n_kv_heads;
    AP_REQUIRE(G == 1 || G == 2 || G == 4 || G == 8, AP_EPARAM, "q-heads per kv-head must be 1, 2, 4 or 8");
    AP_REQUIRE(G % P.group == 0, AP_EPARAM, "selection group must divide the GQA group");
    return AP_OK;
}


// ------------------------------------------------------------------ L2 warm-up for the sparse pass
// One warp per map: the blocks the sparse pass of this layer will gather (sink | local | middle, as
// sparse_cluster_kernel enumerates them) are prefetched into L2 with evict_last priority, plus the map's
// state and middle-block ids.  Launched on a side stream at the start of the layer, it runs beside the
// qkv projection (which holds every SM's shared memory but leaves threads free), so the sparse pass's
// dependent loads and TMA block fetches hit L2 instead of HBM.  Reads only data older than this step's
// newest token (the newest block is written by the projection; its prefetch is skipped).
__global__ void __launch_bounds__(128) sparse_l2_prefetch_kernel(AttnParams P) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x * 4 + warp, s = blockIdx.y;
    const int maps = P.n_q_heads / P.group;
    if (g >= maps) return;
    const int64_t t = P.seq_len[s];
    const int b = P.block;
    const int map = s * P.maps_per_seq + P.map_base + g;
    const ap_map_state ms = P.sel.state[map];
    const int64_t sink_end = P.sel.sink < t ? P.sel.sink : t;
    const int64_t local_start = t - P.sel.local > 0 ? t - P.sel.local : 0;
    const int64_t sb = (sink_end + b - 1) / b, eb = (t + b - 1) / b;
    int64_t lb = local_start / b;
    if (lb < sb) lb = sb;
    const int n_local = (int)(eb - lb);
    const int n_units = (int)sb + n_local + ms.n_mid;
    const int32_t* mid = P.sel.mid_blocks + (int64_t)map * (P.sel.k_mid > 0 ? P.sel.k_mid : 1);
    const int kvh = (g * P.group) / (P.n_q_heads / P.n_kv_heads);
    const char* kh = reinterpret_cast<const char*>(P.k + ((int64_t)s * P.n_kv_heads + kvh) * P.t_max * HD);
    const char* vh = reinterpret_cast<const char*>(P.v + ((int64_t)s * P.n_kv_heads + kvh) * P.t_max * HD);
    for (int u = 0; u < n_units; ++u) {
        const int64_t j = u < sb ? u : (u < sb + n_local ? lb + (u - sb) : (int64_t)__ldg(mid + (u - sb - n_local)));
        if (j == eb - 1) continue;  // holds the newest token: written by the kernel before the sparse pass
        const int64_t off = j * b * HD * 2 + lane * 128;  // 16 tokens x 256 B = 32 lanes x 128 B
        asm volatile("prefetch.global.L2::evict_last [%0];" :: "l"(kh + off));
        if (!P.paged) asm volatile("prefetch.global.L2::evict_last [%0];" :: "l"(vh + off));
    }
}

// ------------------------------------------------------------------ calibration pass on tcgen05
// The K-only dense pass of calibration steps (every M-th step reads all of K: 64 MiB per layer at
// 32K for LLaMA-3.1-8B) as a TMA + tensor-core stream.  Per 128-token tile: two TMA boxes
// {64 dims, 128 tokens} land the K rows in the 128-byte-swizzled K-major layout tcgen05 reads
// directly; one thread issues 8 MMAs (M = 128 tokens, N = 16 (the NH q-heads of this KV head,
// zero-padded), K = 16 dims each, bf16 x bf16 -> fp32 in TMEM); four epilogue warps (lane =
// token) read the tile's logits, scale them to log2 units, take each 16-token block's max per head
// (the calibration row's compressed value is exp2(blockmax - LSE), by monotonicity) and fold the
// tokens into a per-thread online log-sum-exp.  Splits meet in the same last-CTA-done combine and
// emission as the SIMT dense kernel (combine_heads), so the outputs have the same layout and
// meaning.  Roles: warp 0 TMA producer, warp 1 MMA issuer, warps 2-5 epilogue (warps 6-7 only
// join the combine).
namespace ctc {

constexpr int TILE = 128, NST = 4, NACC = 4, NCOL = 16;
constexpr int STAGE_BYTES = TILE * HD * 2;  // 32 KB: two 16 KB swizzled boxes (dims 0-63 | 64-127)
constexpr int B_BYTES = 2 * NCOL * 128;     // q: two 64-dim atoms x 16 rows x 128 B

struct Smem {
    static constexpr int off_a = 0;                          // [NST] stages, 1024-aligned
    static constexpr int off_b = off_a + NST * STAGE_BYTES;  // q (B operand)
    static constexpr int off_red = off_b + B_BYTES;          // [4 warps][8 heads][2]
    static constexpr int off_lse = off_red + 4 * 8 * 2 * 4;  // [8] LSE per head (log2 units)
    static constexpr int off_bar = off_lse + 8 * 4;
    static constexpr int off_bm = off_bar + 8 * (2 * NST + 2 * NACC) + 16;  // [NH][tiles * 8] block maxima
    static int total(int nh, int max_tiles) { return off_bm + nh * max_tiles * (TILE / 16) * 4 + 1024; }
};

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// grid (n_splits, Hkv, S), one wave (every CTA resident; the splits of a KV head wait for each other
// once, for the LSE); 256 threads.  P.counters[s * Hq + h0]: split arrivals (self-resetting);
// partial[(s, h0, split)][2]: split's (m, l)-published epoch (= the map's n_pushed + 1 of this step).
template <int NH>
__global__ void __launch_bounds__(ATT_THREADS, 1) calib_tc_kernel(const __grid_constant__ CUtensorMap kmap,
                                                                  AttnParams P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::off_bar);
    uint64_t* full = bars;
    uint64_t* empty = bars + NST;
    uint64_t* acc_full = bars + 2 * NST;
    uint64_t* acc_empty = acc_full + NACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + NACC);
    float* red = reinterpret_cast<float*>(smem + Smem::off_red);
    float* s_lse = reinterpret_cast<float*>(smem + Smem::off_lse);
    float* s_bm = reinterpret_cast<float*>(smem + Smem::off_bm);
    const int split = blockIdx.x, kvh = blockIdx.y, s = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int h0 = kvh * NH;
    ATT_TRACE(0);
    pdl_trigger();
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
    if (warp == 0) tmem_alloc(tmem_slot, NACC * NCOL);
    // this step's map states (read before this CTA counts itself in, so before any update)
    const int Hh = P.sel.history;
    int64_t epoch = 0;
    pdl_wait();  // q and the newest K token come from earlier kernels in the stream
    {
        const int map0 = s * P.maps_per_seq + P.map_base + h0 / P.group;
        epoch = P.sel.state[map0].n_pushed + 1;
    }
    const int64_t t = P.seq_len[s];
    const int n_tiles = (int)((t + TILE - 1) / TILE);
    const int tile0 = (int)((int64_t)split * n_tiles / gridDim.x), tile1 = (int)((int64_t)(split + 1) * n_tiles / gridDim.x);
    const int my_blocks = (tile1 - tile0) * (TILE / 16);
    {  // q of this KV head's NH q-heads -> the swizzled B tile (rows >= NH zero)
        __nv_bfloat16* bq = reinterpret_cast<__nv_bfloat16*>(smem + Smem::off_b);
        for (int i = threadIdx.x; i < NCOL * HD; i += ATT_THREADS) {
            const int n = i / HD, d = i % HD;
            const __nv_bfloat16 v = n < NH ? P.q[((int64_t)s * P.n_q_heads + h0 + n) * HD + d] : __float2bfloat16_rn(0.f);
            const int atom = d >> 6, dd = d & 63;
            const int byte = atom * (NCOL * 128) + n * 128 + ((((dd >> 3) ^ (n & 7))) << 4) + (dd & 7) * 2;
            bq[byte >> 1] = v;
        }
    }
    fence_async_smem();  // the generic-proxy q writes -> visible to the tensor core
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    ATT_TRACE(1);
    const int64_t row0 = ((int64_t)s * P.n_kv_heads + kvh) * P.t_max;  // tensor-map row of token 0

    if (warp == 0) {
        // ---------------------------------------------------------- TMA producer
        if (lane == 0)
            for (int i = 0, tl = tile0; tl < tile1; ++i, ++tl) {
                const int st = i % NST;
                if (i >= NST) mbar_wait(&empty[st], ((i / NST) & 1) ^ 1);
                uint8_t* dst = smem + Smem::off_a + st * STAGE_BYTES;
                mbar_arrive_tx(&full[st], STAGE_BYTES);
                tma_load_2d(dst, &kmap, 0, (int)(row0 + (int64_t)tl * TILE), &full[st]);
                tma_load_2d(dst + STAGE_BYTES / 2, &kmap, 64, (int)(row0 + (int64_t)tl * TILE), &full[st]);
            }
    } else if (warp == 1) {
        // ---------------------------------------------------------- MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_f16_f32(TILE, NCOL, 1);  // bf16 x bf16 -> fp32
            const uint32_t b_addr = smem_u32(smem + Smem::off_b);
            for (int i = 0, tl = tile0; tl < tile1; ++i, ++tl) {
                const int st = i % NST, ab = i % NACC;
                mbar_wait(&full[st], (i / NST) & 1);
                mbar_wait(&acc_empty[ab], ((i / NACC) & 1) ^ 1);  // (first use: free)
                tc_fence_after();
                const uint32_t a_addr = smem_u32(smem + Smem::off_a + st * STAGE_BYTES);
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    const uint32_t ka = a_addr + (kk >> 2) * (STAGE_BYTES / 2) + (kk & 3) * 32;
                    const uint32_t kb = b_addr + (kk >> 2) * (NCOL * 128) + (kk & 3) * 32;
                    mma_f16(tmem_base + ab * NCOL, desc_sw128(ka), desc_sw128(kb), idesc, kk > 0);
                }
                mma_commit(&empty[st]);      // K tile consumed
                mma_commit(&acc_full[ab]);   // logits ready
            }
        }
    } else if (warp < 6) {
        // ---------------------------------------------------------- epilogue (lane = token of the tile)
        const int quad = warp & 3;
        const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16);
        const float qscale = LOG2E * rsqrtf((float)HD);
        float m[NH], l[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) { m[h] = -INFINITY; l[h] = 0.f; }
        for (int i = 0, tl = tile0; tl < tile1; ++i, ++tl) {
            const int ab = i % NACC;
            mbar_wait(&acc_full[ab], (i / NACC) & 1);
            tc_fence_after();
            float v[8];
            tmem_ld8(lane_base + ab * NCOL, v);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[ab]);
            const int64_t p = (int64_t)tl * TILE + quad * 32 + lane;
            const int jb = i * (TILE / 16) + quad * 2 + (lane >> 4);  // this CTA's block index
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                const float lg = p < t ? v[h] * qscale : -INFINITY;
                float bmx = lg;
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) bmx = fmaxf(bmx, __shfl_xor_sync(0xffffffffu, bmx, o));
                if ((lane & 15) == 0) s_bm[h * my_blocks + jb] = bmx;
                if (lg != -INFINITY) {
                    const float mn = fmaxf(m[h], lg);
                    l[h] = l[h] * exp2f(m[h] - mn) + exp2f(lg - mn);
                    m[h] = mn;
                }
            }
        }
        if (warp == 2) ATT_TRACE2(3);  // this epilogue warp's last tile
        // (m, l) of the split: over the 32 lanes, then the 4 warps
#pragma unroll
        for (int h = 0; h < NH; ++h) {
            float M = m[h];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
            float L = (m[h] == -INFINITY) ? 0.f : l[h] * exp2f(m[h] - M);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
            if (lane == 0) {
                red[(quad * 8 + h) * 2 + 0] = M;
                red[(quad * 8 + h) * 2 + 1] = L;
            }
        }
    }
    ATT_TRACE(2);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem_base, NACC * NCOL);
    if (threadIdx.x < NH) {
        const int h = threadIdx.x;
        float M = -INFINITY;
        for (int q = 0; q < 4; ++q) M = fmaxf(M, red[(q * 8 + h) * 2]);
        float L = 0.f;
        for (int q = 0; q < 4; ++q) {
            const float mq = red[(q * 8 + h) * 2];
            if (mq != -INFINITY) L += red[(q * 8 + h) * 2 + 1] * exp2f(mq - M);
        }
        float* part = P.partial + (((int64_t)s * P.n_q_heads + h0 + h) * P.n_splits + split) * (HD + 2);
        part[0] = M;
        part[1] = L;
    }
    const int64_t W = (t + P.block - 1) / P.block;
    ATT_TRACE(7);
    if (split == 0) {  // before split 0 publishes: the row maxima start from 0, the ring row is zero beyond W
        if (threadIdx.x < NH / P.group + (NH % P.group != 0)) {
            const int map = s * P.maps_per_seq + P.map_base + (h0 + threadIdx.x * P.group) / P.group;
            P.sel.slot_xmax[(int64_t)map * Hh + (int)((epoch - 1) % Hh)] = 0.f;
        }
        for (int g0 = 0; g0 < NH; g0 += P.group) {  // (rarely any)
            const int map = s * P.maps_per_seq + P.map_base + (h0 + g0) / P.group;
            const int slot = (int)((epoch - 1) % Hh);
            float* dst = P.sel.ring + ((int64_t)map * Hh + slot) * P.sel.w_max;
            const int old_w = P.sel.slot_width[(int64_t)map * Hh + slot];
            for (int64_t j = W + threadIdx.x; j < old_w; j += ATT_THREADS) dst[j] = 0.f;
        }
    }
    // ---- every split publishes its (m, l) with this step's epoch and combines all splits' itself (no
    // last-split hop: the LSE is ready one round trip after the slowest split's partials land)
    int* flag0 = reinterpret_cast<int*>(P.partial + ((int64_t)s * P.n_q_heads + h0) * P.n_splits * (HD + 2) + 2);
    __syncthreads();  // this split's partials (and split 0's resets) before its flag
    if (threadIdx.x == 0)
        asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(flag0 + split * (HD + 2)), "r"((int32_t)epoch) : "memory");
    if (warp == 0) {  // one warp waits for every split's epoch (lane = split), with back-off: 144 CTAs
                      // x 18 flags of acquire-polling otherwise crowd the flags' L2 lines
        for (int r0 = 0; r0 < P.n_splits; r0 += 32) {
            const int r = r0 + lane;
            int v = (int32_t)epoch;
            if (r < P.n_splits)
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag0 + r * (HD + 2)) : "memory");
                    if (v == (int32_t)epoch) break;
                    __nanosleep(64);
                }
        }
    }
    __syncthreads();
    if (warp < NH) {  // warp h: lanes over the splits
        const int h = warp;
        const float* part = P.partial + ((int64_t)s * P.n_q_heads + h0 + h) * P.n_splits * (HD + 2);
        float M = -INFINITY, L = 0.f;
        if (P.n_splits <= 32) {  // lane = split (the fixed order of the previous last-split combine)
            float ms = -INFINITY, ls = 0.f;
            if (lane < P.n_splits) {
                ms = __ldcg(part + lane * (HD + 2));
                ls = __ldcg(part + lane * (HD + 2) + 1);
            }
            M = ms;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
            L = (ms == -INFINITY) ? 0.f : ls * exp2f(ms - M);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
        } else {
            for (int r0 = 0; r0 < P.n_splits; r0 += 32) {
                const int r = r0 + lane;
                if (r < P.n_splits) {
                    const float ms = __ldcg(part + r * (HD + 2)), ls = __ldcg(part + r * (HD + 2) + 1);
                    if (ms != -INFINITY) {
                        const float mn = fmaxf(M, ms);
                        L = L * exp2f(M - mn) + ls * exp2f(ms - mn);
                        M = mn;
                    }
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {  // (m, l) over the lanes
                const float Mo = __shfl_xor_sync(0xffffffffu, M, o), Lo = __shfl_xor_sync(0xffffffffu, L, o);
                const float mn = fmaxf(M, Mo);
                L = (M == -INFINITY ? 0.f : L * exp2f(M - mn)) + (Mo == -INFINITY ? 0.f : Lo * exp2f(Mo - mn));
                M = mn;
            }
        }
        if (lane == 0) {
            const float lse = M + log2f(L);
            s_lse[h] = lse;
            if (split == 0 && P.lse) P.lse[(int64_t)s * P.n_q_heads + h0 + h] = lse;
        }
    }
    __syncthreads();
    ATT_TRACE(4);
    for (int g0 = 0; g0 < NH; g0 += P.group) {
        const int map = s * P.maps_per_seq + P.map_base + (h0 + g0) / P.group;
        const int slot = (int)((epoch - 1) % Hh);
        float* dst = P.sel.ring + ((int64_t)map * Hh + slot) * P.sel.w_max;
        float mx = 0.f;
        const int64_t jbase = (int64_t)tile0 * (TILE / 16);
        for (int jb = threadIdx.x; jb < my_blocks; jb += ATT_THREADS) {
            const int64_t j = jbase + jb;
            if (j >= W) break;
            float v = 0.f;
            for (int hh = 0; hh < P.group; ++hh) {
                const float lg = s_bm[(g0 + hh) * my_blocks + jb];
                if (lg != -INFINITY) v = fmaxf(v, exp2f(lg - s_lse[g0 + hh]));
            }
            dst[j] = v;
            mx = track_row_max(mx, v, P.sel.status);
        }
        mx = cta_max_nonneg(mx);
        if (threadIdx.x == 0)
            atomicMax(reinterpret_cast<int*>(P.sel.slot_xmax + (int64_t)map * Hh + slot), __float_as_int(mx));
    }
    ATT_TRACE(5);
    // ---- map state: the last CTA to finish emitting advances it (everyone has read the old one)
    __syncthreads();
    if (last_split(P.counters + (int64_t)s * P.n_q_heads + h0, P.n_splits)) {
        // every split is past its wait: clear the published epochs (the next layer's pass of this step
        // has the same epoch)
        for (int r = threadIdx.x; r < P.n_splits; r += ATT_THREADS) flag0[r * (HD + 2)] = 0;
        if (threadIdx.x == 0)
            for (int g0 = 0; g0 < NH; g0 += P.group) {
                const int map = s * P.maps_per_seq + P.map_base + (h0 + g0) / P.group;
                const int slot = (int)((epoch - 1) % Hh);
                ap_map_state st = P.sel.state[map];
                P.sel.slot_width[(int64_t)map * Hh + slot] = (int32_t)W;
                st.n_pushed += 1;
                st.row_len = t;
                st.width = (int32_t)W;
                P.sel.state[map] = st;
            }
    }
    ATT_TRACE(6);
}

template <int NH>
static int launch(AttnParams P, cudaStream_t st) {
    auto enc = tensor_map_encoder();
    AP_REQUIRE(enc != nullptr, AP_ECUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)HD, (cuuint64_t)P.n_seq * P.n_kv_heads * P.t_max};
    const cuuint64_t strides[1] = {(cuuint64_t)HD * 2};
    const cuuint32_t box[2] = {64, TILE}, estr[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(P.k), dims, strides, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    AP_REQUIRE(r == CUDA_SUCCESS, AP_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    auto k = calib_tc_kernel<NH>;
    // splits: one wave of one CTA per SM over the whole (KV head, sequence) grid (the splits of a KV
    // head wait for each other once, so they must all be resident)
    int splits = ap_sm_budget() / (P.n_kv_heads * P.n_seq);  // every split resident: not on reserved SMs
    AP_REQUIRE(splits >= 1, AP_EPARAM, "calibration pass: more (sequence, KV head) pairs than SMs");
    splits = splits > P.n_splits ? P.n_splits : splits;
    P.n_splits = splits;
    const int max_tiles = (P.t_max / TILE + 1 + splits - 1) / splits + 1;
    const int smem = Smem::total(NH, max_tiles);
    AP_REQUIRE(smem <= 227 * 1024, AP_EPARAM, "calibration pass: t_max too large for the block-max buffer");
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    launch_ex(k, dim3(splits, P.n_kv_heads, P.n_seq), dim3(ATT_THREADS), (size_t)smem, st, 1, map, P);
    return launch_status("calib_tc_kernel");
}

}  // namespace ctc

}  // namespace ap

using namespace ap;

static int g_calib_mode = -1;  // 1: TMA + tcgen05 calibration pass, 0: SIMT dense kernel
static bool calib_tc_enabled() {
    if (g_calib_mode < 0) {
        const char* e = getenv("ATTNPRED_CALIB_KERNEL");
        g_calib_mode = !(e && strcmp(e, "simt") == 0);
    }
    return g_calib_mode == 1;
}

extern "C" {

int ap_attn_set_calib_kernel(int mode) {
    const int prev = calib_tc_enabled() ? 1 : 0;
    g_calib_mode = mode ? 1 : 0;
    return prev;
}

int ap_attn_debug_trace(int on, long long* host_out) {
    if (host_out) return cudaMemcpyFromSymbol(host_out, g_att_trace, sizeof(long long) * 256) == cudaSuccess ? 0 : 5;
    return cudaMemcpyToSymbol(g_att_trace_on, &on, sizeof(int)) == cudaSuccess ? 0 : 5;
}

int ap_attn_dense(const ap_attn_layer* a, int with_v, const ap_selector* sel, int32_t map_base, int32_t maps_per_seq,
                  int32_t group, int emit, void* stream) {
    AttnParams P;
    int rc = make_params(a, sel, map_base, maps_per_seq, group, P);
    if (rc != AP_OK) return rc;
    AP_REQUIRE(with_v || emit, AP_EPARAM, "dense pass without V must emit the calibration row");
    P.with_v = with_v; P.emit = emit;
    AP_REQUIRE(!emit || sel, AP_EPARAM, "emit needs a selector");
    cudaStream_t st = as_stream(stream);
    const int G = a->n_q_heads / a->n_kv_heads;
    if (!with_v && calib_tc_enabled()) {  // calibration pass: TMA + tcgen05 (ATTNPRED_CALIB_KERNEL=simt: SIMT)
        switch (G) {
            case 1: return ctc::launch<1>(P, st);
            case 2: return ctc::launch<2>(P, st);
            case 4: return ctc::launch<4>(P, st);
            default: return ctc::launch<8>(P, st);
        }
    }
    switch (G) {
        case 1: launch_dense<1>(P, with_v, emit, st); break;
        case 2: launch_dense<2>(P, with_v, emit, st); break;
        case 4: launch_dense<4>(P, with_v, emit, st); break;
        default: launch_dense<8>(P, with_v, emit, st); break;
    }
    return launch_status("dense_partial_kernel");
}

int ap_attn_sparse_paged(const ap_attn_layer* a, const ap_selector* sel, int32_t map_base, int32_t maps_per_seq,
                         int32_t group, int emit, const ap_vpages* vp, int32_t layer, void* stream);

int ap_attn_sparse_prefetch(const ap_attn_layer* a, const ap_selector* sel, int32_t map_base, int32_t maps_per_seq,
                            int32_t group, void* stream) {
    AttnParams P;
    int rc = make_params(a, sel, map_base, maps_per_seq, group, P);
    if (rc != AP_OK) return rc;
    AP_REQUIRE(sel != nullptr, AP_EPARAM, "the L2 warm-up needs a selector");
    const int maps = P.n_q_heads / P.group;
    sparse_l2_prefetch_kernel<<<dim3((maps + 3) / 4, P.n_seq), 128, 0, as_stream(stream)>>>(P);
    return launch_status("sparse_l2_prefetch_kernel");
}

int ap_attn_sparse(const ap_attn_layer* a, const ap_selector* sel, int32_t map_base, int32_t maps_per_seq,
                   int32_t group, int emit, void* stream) {
    return ap_attn_sparse_paged(a, sel, map_base, maps_per_seq, group, emit, nullptr, 0, stream);
}

int ap_attn_sparse_paged(const ap_attn_layer* a, const ap_selector* sel, int32_t map_base, int32_t maps_per_seq,
                         int32_t group, int emit, const ap_vpages* vp, int32_t layer, void* stream) {
    AttnParams P;
    int rc = make_params(a, sel, map_base, maps_per_seq, group, P);
    if (rc != AP_OK) return rc;
    if (vp) {
        AP_REQUIRE(group == a->n_q_heads / a->n_kv_heads, AP_EPARAM, "paged V needs one selection map per KV head");
        AP_REQUIRE(vp->pages && vp->mid_page, AP_EPARAM, "bad paged-V descriptor");
        P.vp = *vp;
        P.paged = 1;
        P.layer = layer;
    }
    AP_REQUIRE(sel != nullptr, AP_EPARAM, "sparse attention needs a selector");
    P.with_v = 1; P.emit = emit; P.sparse_units = 1;
    cudaStream_t st = as_stream(stream);
    switch (P.group) {
        case 1: rc = launch_sparse<1>(P, emit, st); break;
        case 2: rc = launch_sparse<2>(P, emit, st); break;
        case 4: rc = launch_sparse<4>(P, emit, st); break;
        default: rc = launch_sparse<8>(P, emit, st); break;
    }
    if (rc != AP_OK) return rc;
    return launch_status("sparse_partial_kernel");
}

}  // extern "C"
