// Exact-boundary guard for the selector's top-k (kernel 3): makes the chosen middle blocks equal
// to those of the reference's float64 forecaster (selector.py:126-145 on predictor.py:185-216)
// instead of "equal except near-ties".
//
// The forecaster runs in fp32-class arithmetic (fp16x3 / fp32), so a block whose fp64 score sits
// within the device error of the k-th score can land on the wrong side of the boundary.  With a
// device error bound eps and band = rel * max(|tau|, floor * max|score|) >= 2 eps around the k-th
// device score tau:
//   A = {score > tau + band} is certainly in the reference's top k,
//   C = {score < tau - band} is certainly out,
//   B = the band.  If |B| > k - |A| the boundary is ambiguous: every block of B is re-scored in
//   fp64 from the history window (the reference's arithmetic, summed in a fixed order) and the
//   k - |A| best by (fp64 score desc, index asc) — selector.py:80's lexsort order — are taken.
// Detection runs inside the top-k kernel; the re-scoring is one persistent launch over
// (map, candidate) units, and the last unit of a map re-emits that map's block ids.
#pragma once

namespace ap {
namespace tie {

constexpr int CAP = 64;      // candidates per map; wider ambiguity falls back to the fp32 order (counted)
constexpr int HDR = 16;      // workspace header words
constexpr int REC_HDR = 16;  // per-map record header words
constexpr int REC = REC_HDR + 3 * CAP;  // + ids[CAP] int32 + scores[CAP] fp64
constexpr int NT = 256;

enum { H_UNITS = 0, H_NEXT = 1, H_DONE = 2, H_OVERFLOW = 3, H_MAPS = 4, H_CANDS = 5 };
enum { R_NA = 0, R_NEED, R_NB, R_KLO, R_KHI, R_PENDING, R_W, R_SINK_HI, R_LOCAL_LO, R_LOCAL_HI };

__host__ __device__ inline int64_t rec_off(int n_maps) { return (HDR + (int64_t)n_maps * CAP + 1) & ~int64_t(1); }
__host__ __device__ inline int64_t ws_words(int n_maps) { return rec_off(n_maps) + (int64_t)n_maps * REC; }

__device__ __forceinline__ float key_value(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// All threads of the top-k CTA.  keyfn(i) = the masked order key of block i (0 = masked).
// Returns the map's tie_n (0 unambiguous, NB re-scored candidates, -NB overflow).
template <int NTH, typename KeyFn>
__device__ int detect(const ap_selector& s, const Params& tp, int m, KeyFn keyfn, int W, int k, uint32_t T,
                      float amax, int sink_hi, int local_lo, int local_hi, int* scan_tmp, int* s_bcast) {
    const float tau = key_value(T);
    const float band = tp.rel * fmaxf(fabsf(tau), tp.floor * amax);
    const uint32_t khi = order_key(tau + band), klo = order_key(tau - band);
    const int per = (W + NTH - 1) / NTH, lo = min(W, (int)threadIdx.x * per), hi = min(W, lo + per);
    int na = 0, nb = 0;
    for (int i = lo; i < hi; ++i) {
        const uint32_t key = keyfn(i);
        na += key > khi;
        nb += key >= klo && key <= khi;
    }
    int NA = 0, NB = 0;
    block_excl_scan<NTH>(na, scan_tmp, NA);
    int pos = block_excl_scan<NTH>(nb, scan_tmp, NB);
    const int need = k - NA;
    if (NB <= need) return 0;
    int* ws = s.tie_ws;
    if (NB > CAP) {
        if (threadIdx.x == 0) atomicAdd(&ws[H_OVERFLOW], 1);
        return -NB;
    }
    int* rec = ws + rec_off(s.n_maps) + (int64_t)m * REC;
    for (int i = lo; i < hi; ++i) {
        const uint32_t key = keyfn(i);
        if (key >= klo && key <= khi) rec[REC_HDR + pos++] = i;  // ascending block ids
    }
    if (threadIdx.x == 0) {
        rec[R_NA] = NA;
        rec[R_NEED] = need;
        rec[R_NB] = NB;
        rec[R_KLO] = (int)klo;
        rec[R_KHI] = (int)khi;
        rec[R_PENDING] = NB;
        rec[R_W] = W;
        rec[R_SINK_HI] = sink_hi;
        rec[R_LOCAL_LO] = local_lo;
        rec[R_LOCAL_HI] = local_hi;
        *s_bcast = atomicAdd(&ws[H_UNITS], NB);
        atomicAdd(&ws[H_MAPS], 1);
        atomicAdd(&ws[H_CANDS], NB);
    }
    __syncthreads();
    const int ub = *s_bcast;
    for (int j = threadIdx.x; j < NB; j += NTH) ws[HDR + ub + j] = m * CAP + j;
    return NB;
}

// ------------------------------------------------------------------ fp64 re-scoring
// Shared memory (doubles): weights (w2 transposed to [k*9+tap][c]), the x window, the a1 window.
constexpr int SW1 = 0, SB1 = 144, SW2 = 160, SB2 = SW2 + 144 * 32, SW3 = SB2 + 32, SB3 = SW3 + 32;
constexpr int SX = SB3 + 8;                 // x window [68 rows][5 cols]
constexpr int A1S = 49;                     // a1 row stride (48 + 1: conflict-free interleaved rows)
constexpr int SA1 = SX + 68 * 5;            // a1 window [66 rows][A1S]
constexpr int SRED = SA1 + 66 * A1S;        // [NT/32] warp partials
constexpr int SMEM_DOUBLES = SRED + NT / 32 + 8;
constexpr int SMEM_BYTES = SMEM_DOUBLES * 8;

// score of block column `col` of map m: b3 + (1/H) sum_i sum_c w3[c] relu(s2[c][i][col]) in fp64,
// every product and sum in a fixed order (deterministic).  All threads.
__device__ double exact_score(const ap_selector& s, int m, int col, double* sm) {
    const ap_map_state st = s.state[m];
    const int H = s.history, W = st.width, pitch = s.w_max;
    const float* ring = s.ring + (int64_t)m * H * pitch;
    const int64_t n_pushed = st.n_pushed;
    const int first_real = n_pushed >= H ? 0 : (int)(H - n_pushed);
    const int tid = threadIdx.x, cp = tid >> 4, rg = tid & 15;
    double* sx = sm + SX;
    double* sa1 = sm + SA1;
    double acc = 0.0;
    for (int i0 = 0; i0 < H; i0 += 64) {
        const int nrows = min(64, H - i0);
        __syncthreads();
        for (int idx = tid; idx < (nrows + 4) * 5; idx += NT) {
            const int q = idx / 5, c = idx % 5, p = i0 - 2 + q, cc = col - 2 + c;
            double v = 0.0;
            if (p >= first_real && p < H && p >= 0 && cc >= 0 && cc < W) {
                int64_t r = (n_pushed - H + p) % H;
                if (r < 0) r += H;
                v = (double)ring[r * pitch + cc];
            }
            sx[idx] = v;
        }
        __syncthreads();
        for (int idx = tid; idx < (nrows + 2) * 48; idx += NT) {
            const int r = idx / 48, kd = idx % 48, kk = kd / 3, dj = kd % 3;
            const int p = i0 - 1 + r, c2 = col - 1 + dj;
            double a = 0.0;
            if (p >= 0 && p < H && c2 >= 0 && c2 < W) {  // conv2's zero padding of a1
                a = sm[SB1 + kk];
#pragma unroll
                for (int t = 0; t < 9; ++t) a = fma(sm[SW1 + kk * 9 + t], sx[(r + t / 3) * 5 + dj + t % 3], a);
                a = fmax(a, 0.0);
            }
            sa1[r * A1S + kd] = a;
        }
        __syncthreads();
        double s0[4], s1[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            s0[j] = sm[SB2 + 2 * cp];
            s1[j] = sm[SB2 + 2 * cp + 1];
        }
#pragma unroll 1
        for (int kk = 0; kk < 16; ++kk) {
#pragma unroll
            for (int t = 0; t < 9; ++t) {
                const int di = t / 3, dj = t % 3;
                const double2 w = *reinterpret_cast<const double2*>(&sm[SW2 + (kk * 9 + t) * 32 + 2 * cp]);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const double av = sa1[(rg + 16 * j + di) * A1S + kk * 3 + dj];
                    s0[j] = fma(w.x, av, s0[j]);
                    s1[j] = fma(w.y, av, s1[j]);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (rg + 16 * j < nrows) {
                acc = fma(sm[SW3 + 2 * cp], fmax(s0[j], 0.0), acc);
                acc = fma(sm[SW3 + 2 * cp + 1], fmax(s1[j], 0.0), acc);
            }
        }
    }
    // fixed-order block reduction
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __syncthreads();
    if ((tid & 31) == 0) sm[SRED + (tid >> 5)] = acc;
    __syncthreads();
    double tot = 0.0;
    for (int w = 0; w < NT / 32; ++w) tot += sm[SRED + w];
    return sm[SB3] + tot / H;
}

// Re-emit map m's middle blocks: A plus the `need` best re-scored candidates, ascending.
__device__ void finalize(const ap_selector& s, int m, int* flags /*[CAP] smem*/, int* scan_tmp) {
    const int* rec = s.tie_ws + rec_off(s.n_maps) + (int64_t)m * REC;
    const int NB = __ldcg(rec + R_NB), need = __ldcg(rec + R_NEED), W = __ldcg(rec + R_W);
    const uint32_t klo = (uint32_t)__ldcg(rec + R_KLO), khi = (uint32_t)__ldcg(rec + R_KHI);
    const int sink_hi = __ldcg(rec + R_SINK_HI), local_lo = __ldcg(rec + R_LOCAL_LO),
              local_hi = __ldcg(rec + R_LOCAL_HI);
    const int* ids = rec + REC_HDR;
    const double* sc = reinterpret_cast<const double*>(rec + REC_HDR + CAP);
    if ((int)threadIdx.x < NB) {
        const int j = threadIdx.x, id = __ldcg(ids + j);
        const double v = __ldcg(sc + j);
        int rank = 0;
        for (int l = 0; l < NB; ++l) {
            const double u = __ldcg(sc + l);
            rank += (u > v) || (u == v && __ldcg(ids + l) < id);
        }
        flags[j] = rank < need;
    }
    __syncthreads();
    const float* row = s.scores + (int64_t)m * s.w_max;
    auto keyof = [&](int i) -> uint32_t {
        const bool masked = i < sink_hi || (i >= local_lo && i < local_hi);
        return masked ? 0u : order_key(row[i]);
    };
    const int per = (W + NT - 1) / NT, lo = min(W, (int)threadIdx.x * per), hi = min(W, lo + per);
    int c0 = 0;  // first candidate at or after lo
    while (c0 < NB && __ldcg(ids + c0) < lo) ++c0;
    int n_sel = 0, c = c0;
    for (int i = lo; i < hi; ++i) {
        const uint32_t key = keyof(i);
        if (key > khi) ++n_sel;
        else if (key >= klo && key <= khi) n_sel += flags[c++];
    }
    int total = 0;
    int pos = block_excl_scan<NT>(n_sel, scan_tmp, total);
    const int words = (s.w_max + 31) / 32;
    uint32_t* mask = s.mid_mask + (int64_t)m * words;
    int32_t* mid = s.mid_blocks + (int64_t)m * (s.k_mid > 0 ? s.k_mid : 1);
    for (int w = threadIdx.x; w < words; w += NT) mask[w] = 0u;
    __syncthreads();
    c = c0;
    for (int i = lo; i < hi; ++i) {
        const uint32_t key = keyof(i);
        bool take = key > khi;
        if (!take && key >= klo && key <= khi) take = flags[c++];
        if (take) {
            mid[pos++] = i;
            atomicOr(&mask[i >> 5], 1u << (i & 31));
        }
    }
}

__global__ void __launch_bounds__(NT) refine_kernel(ap_selector s, Params tp) {
    extern __shared__ double sm[];
    __shared__ int s_unit, s_last;
    __shared__ int flags[CAP];
    __shared__ int scan_tmp[NT / 32 + 2];
    int* ws = s.tie_ws;
    bool staged = false;
    for (;;) {
        if (threadIdx.x == 0) s_unit = atomicAdd(&ws[H_NEXT], 1);
        __syncthreads();
        const int u = s_unit;
        if (u >= __ldcg(&ws[H_UNITS])) break;
        if (!staged) {  // weights as fp64 (exact: they are fp32 values); w2 as [k*9+tap][c]
            for (int i = threadIdx.x; i < 144; i += NT) sm[SW1 + i] = (double)tp.w[i];
            for (int i = threadIdx.x; i < 16; i += NT) sm[SB1 + i] = (double)tp.w[144 + i];
            for (int i = threadIdx.x; i < 4608; i += NT) {
                const int c = i / 144, kt = i % 144;
                sm[SW2 + kt * 32 + c] = (double)tp.w[160 + i];
            }
            for (int i = threadIdx.x; i < 32; i += NT) {
                sm[SB2 + i] = (double)tp.w[4768 + i];
                sm[SW3 + i] = (double)tp.w[4800 + i];
            }
            if (threadIdx.x == 0) sm[SB3] = (double)tp.w[4832];
            staged = true;
            __syncthreads();
        }
        const int m = u / CAP, j = u % CAP;
        int* rec = ws + rec_off(s.n_maps) + (int64_t)m * REC;
        const int col = __ldcg(rec + REC_HDR + j);
        const double v = exact_score(s, m, col, sm);
        if (threadIdx.x == 0) {
            reinterpret_cast<double*>(rec + REC_HDR + CAP)[j] = v;
            __threadfence();
            s_last = atomicSub(rec + R_PENDING, 1) == 1;
            if (s_last) __threadfence();
        }
        __syncthreads();
        if (s_last) finalize(s, m, flags, scan_tmp);
        __syncthreads();
    }
    if (threadIdx.x == 0) {  // the last CTA out resets the work list for the next step
        __threadfence();
        if (atomicAdd(&ws[H_DONE], 1) == (int)gridDim.x - 1) {
            ws[H_UNITS] = 0;
            ws[H_NEXT] = 0;
            ws[H_DONE] = 0;
            __threadfence();
        }
    }
}

}  // namespace tie
}  // namespace ap
