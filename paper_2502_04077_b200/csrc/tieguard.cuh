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
// Detection runs inside the top-k kernel.  Re-scoring is one persistent launch over units of
// (map, candidate, group of history rows): a candidate's 16 row groups run on different CTAs, the
// last group of a candidate sums the partials in a fixed order, and the last candidate of a map
// re-emits that map's block ids.
#pragma once

namespace ap {
namespace tie {

constexpr int CAP = 64;      // candidates per map; wider ambiguity falls back to the fp32 order (counted)
constexpr int NG = 16;       // history-row groups per candidate (units)
constexpr int MAX_RG = 8;    // rows per group: the guard covers H <= NG * MAX_RG = 128
constexpr int HDR = 16;      // workspace header words
constexpr int REC_HDR = 16;  // per-map record header words
// record: header | ids[CAP] | cpend[CAP] | scores[CAP] fp64 | parts[CAP][NG] fp64
constexpr int OFF_IDS = REC_HDR, OFF_CPEND = OFF_IDS + CAP, OFF_SC = OFF_CPEND + CAP, OFF_PARTS = OFF_SC + 2 * CAP;
constexpr int REC = OFF_PARTS + 2 * CAP * NG;
constexpr int NT = 128;      // refine CTA: 4 warps, lane = conv2 output channel

enum { H_UNITS = 0, H_NEXT = 1, H_DONE = 2, H_OVERFLOW = 3, H_MAPS = 4, H_CANDS = 5, H_SELDONE = 6 };
enum { R_NA = 0, R_NEED, R_NB, R_KLO, R_KHI, R_PENDING, R_W, R_SINK_HI, R_LOCAL_LO, R_LOCAL_HI };

__host__ __device__ inline int64_t units_cap(int n_maps) { return (int64_t)n_maps * CAP * NG; }
__host__ __device__ inline int64_t rec_off(int n_maps) { return (HDR + units_cap(n_maps) + 1) & ~int64_t(1); }
__host__ __device__ inline int64_t ws_words(int n_maps) { return rec_off(n_maps) + (int64_t)n_maps * REC; }

// fp64 weight image (g_w64, written by ap_set_weights): w1[144] b1[16] w2t[144][32] b2[32] w3[32] b3
constexpr int W64_W1 = 0, W64_B1 = 144, W64_W2T = 160, W64_B2 = 4768, W64_W3 = 4800, W64_B3 = 4832;

__device__ __forceinline__ float key_value(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// All threads of the top-k CTA.  keyfn(i) = the masked order key of block i (0 = masked).
// Returns the map's tie_n (0 unambiguous, NB re-scored candidates, -NB overflow).
template <int NTH, typename KeyFn, class G = CtaGroup>
__device__ int detect(const ap_selector& s, const Params& tp, int m, KeyFn keyfn, int W, int k, uint32_t T,
                      float amax, int sink_hi, int local_lo, int local_hi, int* scan_tmp, int* s_bcast,
                      const G& grp = G{}) {
    const float tau = key_value(T);
    const float band = tp.rel * fmaxf(fabsf(tau), tp.floor * amax);
    const uint32_t khi = order_key(tau + band), klo = order_key(tau - band);
    const int tid = grp.tid();
    const int per = (W + NTH - 1) / NTH, lo = min(W, tid * per), hi = min(W, lo + per);
    int na = 0, nb = 0;
    for (int i = lo; i < hi; ++i) {
        const uint32_t key = keyfn(i);
        na += key > khi;
        nb += key >= klo && key <= khi;
    }
    int NA = 0, NB = 0;
    group_excl_scan<NTH>(na, scan_tmp, NA, grp);
    int pos = group_excl_scan<NTH>(nb, scan_tmp, NB, grp);
    const int need = k - NA;
    if (NB <= need) return 0;
    int* ws = s.tie_ws;
    if (NB > CAP || s.history > NG * MAX_RG) {
        if (tid == 0) atomicAdd(&ws[H_OVERFLOW], 1);
        return -NB;
    }
    int* rec = ws + rec_off(s.n_maps) + (int64_t)m * REC;
    for (int i = lo; i < hi; ++i) {
        const uint32_t key = keyfn(i);
        if (key >= klo && key <= khi) rec[OFF_IDS + pos++] = i;  // ascending block ids
    }
    for (int j = tid; j < NB; j += NTH) rec[OFF_CPEND + j] = NG;
    if (tid == 0) {
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
        *s_bcast = atomicAdd(&ws[H_UNITS], NB * NG);
        atomicAdd(&ws[H_MAPS], 1);
        atomicAdd(&ws[H_CANDS], NB);
    }
    __threadfence();  // the record before its units: a fused consumer may take a unit as soon as it is listed
    grp.sync();
    const int ub = *s_bcast;
    // units listed as value + 1 (0 = not written yet; the consumer clears its entry for the next step)
    for (int u = tid; u < NB * NG; u += NTH) st_volatile(ws + HDR + ub + u, (m * CAP + u / NG) * NG + u % NG + 1);
    return NB;
}

// The same for a thread group holding the map's keys in registers (thread t: blocks [i0, i0 + IPT),
// i0 = t * IPT; key 0 = masked): the common unambiguous case costs one barrier and no global loads.
// red: >= 2 * NTH / 32 ints of scratch shared memory.
template <int NTH, int IPT, class G>
__device__ int detect_regs(const ap_selector& s, const Params& tp, int m, const uint32_t (&key)[IPT], int i0, int W,
                           int k, uint32_t T, float amax, int sink_hi, int local_lo, int local_hi, int* scan_tmp,
                           int* red, int* s_bcast, const G& grp) {
    const float tau = key_value(T);
    const float band = tp.rel * fmaxf(fabsf(tau), tp.floor * amax);
    const uint32_t khi = order_key(tau + band), klo = order_key(tau - band);
    const int tid = grp.tid(), lane = tid & 31, warp = tid >> 5;
    int na = 0, nb = 0;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
        na += key[q] > khi;
        nb += key[q] >= klo && key[q] <= khi;
    }
    const int wa = (int)__reduce_add_sync(0xffffffffu, (unsigned)na), wb = (int)__reduce_add_sync(0xffffffffu, (unsigned)nb);
    if (lane == 0) {
        red[warp] = wa;
        red[NTH / 32 + warp] = wb;
    }
    grp.sync();
    int NA = 0, NB = 0;
#pragma unroll
    for (int w = 0; w < NTH / 32; ++w) {
        NA += red[w];
        NB += red[NTH / 32 + w];
    }
    grp.sync();  // (red is reused by the caller)
    const int need = k - NA;
    if (NB <= need) return 0;
    int* ws = s.tie_ws;
    if (NB > CAP || s.history > NG * MAX_RG) {
        if (tid == 0) atomicAdd(&ws[H_OVERFLOW], 1);
        return -NB;
    }
    int tot = 0;
    int pos = group_excl_scan<NTH>(nb, scan_tmp, tot, grp);
    int* rec = ws + rec_off(s.n_maps) + (int64_t)m * REC;
#pragma unroll
    for (int q = 0; q < IPT; ++q)
        if (key[q] >= klo && key[q] <= khi) rec[OFF_IDS + pos++] = i0 + q;  // ascending block ids
    for (int j = tid; j < NB; j += NTH) rec[OFF_CPEND + j] = NG;
    if (tid == 0) {
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
        *s_bcast = atomicAdd(&ws[H_UNITS], NB * NG);
        atomicAdd(&ws[H_MAPS], 1);
        atomicAdd(&ws[H_CANDS], NB);
    }
    __threadfence();  // the record before its units: a fused consumer may take a unit as soon as it is listed
    grp.sync();
    const int ub = *s_bcast;
    for (int u = tid; u < NB * NG; u += NTH) st_volatile(ws + HDR + ub + u, (m * CAP + u / NG) * NG + u % NG + 1);
    return NB;
}

// The same for one warp holding a map's keys in registers (sel_topk_warp_kernel: block q * 32 + lane in
// key[q]).  All lanes of the warp.
template <int IPT>
__device__ int detect_warp(const ap_selector& s, const Params& tp, int m, const uint32_t (&key)[IPT], int W, int k,
                           uint32_t T, float amax, int sink_hi, int local_lo, int local_hi) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const float tau = key_value(T);
    const float band = tp.rel * fmaxf(fabsf(tau), tp.floor * amax);
    const uint32_t khi = order_key(tau + band), klo = order_key(tau - band);
    int na = 0, nb = 0;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
        na += key[q] > khi;
        nb += key[q] >= klo && key[q] <= khi;
    }
    const int NA = (int)__reduce_add_sync(FULL, (unsigned)na), NB = (int)__reduce_add_sync(FULL, (unsigned)nb);
    const int need = k - NA;
    if (NB <= need) return 0;
    int* ws = s.tie_ws;
    if (NB > CAP || s.history > NG * MAX_RG) {
        if (lane == 0) atomicAdd(&ws[H_OVERFLOW], 1);
        return -NB;
    }
    int* rec = ws + rec_off(s.n_maps) + (int64_t)m * REC;
    const unsigned lt = (1u << lane) - 1u;
    int pos = 0;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {  // ascending block ids
        const bool in = key[q] >= klo && key[q] <= khi;
        const unsigned bm = __ballot_sync(FULL, in);
        if (in) rec[OFF_IDS + pos + __popc(bm & lt)] = q * 32 + lane;
        pos += __popc(bm);
    }
    for (int j = lane; j < NB; j += 32) rec[OFF_CPEND + j] = NG;
    int ub = 0;
    if (lane == 0) {
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
        ub = atomicAdd(&ws[H_UNITS], NB * NG);
        atomicAdd(&ws[H_MAPS], 1);
        atomicAdd(&ws[H_CANDS], NB);
    }
    ub = __shfl_sync(FULL, ub, 0);
    __threadfence();
    for (int u = lane; u < NB * NG; u += 32) st_volatile(ws + HDR + ub + u, (m * CAP + u / NG) * NG + u % NG + 1);
    return NB;
}

// ------------------------------------------------------------------ fp64 re-scoring
// sum over history rows [g*RG, g*RG+RG) of r_i = sum_c w3[c] relu(s2[c][i][col]), in fp64, fixed order.
// x window [RG+4 rows][5 cols], a1 window [RG+2 rows][16 ch][3 cols] in shared memory; warp w takes
// rows w, w+4, ..., lane = output channel c (conv2 = a 144-term dot per lane, weights w2t[kt][c]
// coalesced across lanes, a1 values broadcast).  All threads.
template <class G = CtaGroup>
__device__ double group_partial(const ap_selector& s, const double* __restrict__ w64, int m, int col, int g,
                                double* sx, double* sa1, double* srow, const G& grp = G{}) {
    const ap_map_state st = s.state[m];
    const int H = s.history, W = st.width, pitch = s.w_max;
    const int RG = (H + NG - 1) / NG;
    const int r0 = g * RG, nr = max(0, min(H, r0 + RG) - r0);
    if (nr == 0) return 0.0;
    const float* ring = s.ring + (int64_t)m * H * pitch;
    const int64_t n_pushed = st.n_pushed;
    const int first_real = n_pushed >= H ? 0 : (int)(H - n_pushed);
    const int tid = grp.tid(), lane = tid & 31, warp = tid >> 5;
    for (int idx = tid; idx < (nr + 4) * 5; idx += NT) {  // x rows r0-2 .. r0+nr+1, cols col-2 .. col+2
        const int q = idx / 5, c = idx % 5, p = r0 - 2 + q, cc = col - 2 + c;
        double v = 0.0;
        if (p >= first_real && p < H && p >= 0 && cc >= 0 && cc < W) {
            int64_t r = (n_pushed - H + p) % H;
            if (r < 0) r += H;
            v = (double)ring[r * pitch + cc];
        }
        sx[idx] = v;
    }
    grp.sync();
    for (int idx = tid; idx < (nr + 2) * 48; idx += NT) {  // a1 rows r0-1 .. r0+nr, cols col-1 .. col+1
        const int r = idx / 48, kd = idx % 48, kk = kd / 3, dj = kd % 3;
        const int p = r0 - 1 + r, c2 = col - 1 + dj;
        double a = 0.0;
        if (p >= 0 && p < H && c2 >= 0 && c2 < W) {  // conv2's zero padding of a1
            double e = w64[W64_B1 + kk], o = 0.0;
#pragma unroll
            for (int t = 0; t < 9; t += 2) e = fma(w64[W64_W1 + kk * 9 + t], sx[(r + t / 3) * 5 + dj + t % 3], e);
#pragma unroll
            for (int t = 1; t < 9; t += 2) o = fma(w64[W64_W1 + kk * 9 + t], sx[(r + t / 3) * 5 + dj + t % 3], o);
            a = fmax(e + o, 0.0);
        }
        sa1[r * 48 + kd] = a;
    }
    grp.sync();
    for (int ri = warp; ri < nr; ri += NT / 32) {
        double e = w64[W64_B2 + lane], o = 0.0;  // two chains: even / odd input channels
#pragma unroll 4
        for (int kk = 0; kk < 16; kk += 2) {
#pragma unroll
            for (int t = 0; t < 9; ++t) {
                const int di = t / 3, dj = t % 3;
                e = fma(w64[W64_W2T + (kk * 9 + t) * 32 + lane], sa1[(ri + di) * 48 + kk * 3 + dj], e);
                o = fma(w64[W64_W2T + ((kk + 1) * 9 + t) * 32 + lane], sa1[(ri + di) * 48 + (kk + 1) * 3 + dj], o);
            }
        }
        double r = w64[W64_W3 + lane] * fmax(e + o, 0.0);
#pragma unroll
        for (int off = 16; off; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
        if (lane == 0) srow[ri] = r;
    }
    grp.sync();
    double tot = 0.0;
    for (int ri = 0; ri < nr; ++ri) tot += srow[ri];  // fixed order
    return tot;
}

// Re-emit map m's middle blocks: A plus the `need` best re-scored candidates, ascending.
template <class G = CtaGroup>
__device__ void finalize(const ap_selector& s, int m, int* flags /*[CAP] smem*/, int* scan_tmp, const G& grp = G{}) {
    const int tid = grp.tid();
    const int* rec = s.tie_ws + rec_off(s.n_maps) + (int64_t)m * REC;
    const int NB = __ldcg(rec + R_NB), need = __ldcg(rec + R_NEED), W = __ldcg(rec + R_W);
    const uint32_t klo = (uint32_t)__ldcg(rec + R_KLO), khi = (uint32_t)__ldcg(rec + R_KHI);
    const int sink_hi = __ldcg(rec + R_SINK_HI), local_lo = __ldcg(rec + R_LOCAL_LO),
              local_hi = __ldcg(rec + R_LOCAL_HI);
    const int* ids = rec + OFF_IDS;
    const double* sc = reinterpret_cast<const double*>(rec + OFF_SC);
    for (int j = tid; j < NB; j += NT) {
        const int id = __ldcg(ids + j);
        const double v = __ldcg(sc + j);
        int rank = 0;
        for (int l = 0; l < NB; ++l) {
            const double u = __ldcg(sc + l);
            rank += (u > v) || (u == v && __ldcg(ids + l) < id);
        }
        flags[j] = rank < need;
    }
    grp.sync();
    const float* row = s.scores + (int64_t)m * s.w_max;
    auto keyof = [&](int i) -> uint32_t {
        const bool masked = i < sink_hi || (i >= local_lo && i < local_hi);
        return masked ? 0u : order_key(row[i]);
    };
    const int per = (W + NT - 1) / NT, lo = min(W, (int)tid * per), hi = min(W, lo + per);
    int c0 = 0;  // first candidate at or after lo
    while (c0 < NB && __ldcg(ids + c0) < lo) ++c0;
    int n_sel = 0, c = c0;
    for (int i = lo; i < hi; ++i) {
        const uint32_t key = keyof(i);
        if (key > khi) ++n_sel;
        else if (key >= klo && key <= khi) n_sel += flags[c++];
    }
    int total = 0;
    int pos = group_excl_scan<NT>(n_sel, scan_tmp, total, grp);
    const int words = (s.w_max + 31) / 32;
    uint32_t* mask = s.mid_mask + (int64_t)m * words;
    int32_t* mid = s.mid_blocks + (int64_t)m * (s.k_mid > 0 ? s.k_mid : 1);
    for (int w = tid; w < words; w += NT) mask[w] = 0u;
    grp.sync();
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

// One unit of the fp64 re-scoring ((map * CAP + candidate) * NG + group): the group's partial, the
// candidate's score once its last group is in, the map's re-emission once its last candidate is.
// All threads of grp (NT of them).
template <class G>
__device__ void refine_unit(const ap_selector& s, const Params& tp, int unit, double* sx, double* sa1, double* srow,
                            int* flags, int* scan_tmp, int* s_last, const G& grp) {
    int* ws = s.tie_ws;
    const double* w64 = tp.w64;
    const int g = unit % NG, j = (unit / NG) % CAP, m = unit / (NG * CAP);
    int* rec = ws + rec_off(s.n_maps) + (int64_t)m * REC;
    const int col = __ldcg(rec + OFF_IDS + j);
    const double part = group_partial(s, w64, m, col, g, sx, sa1, srow, grp);
    if (grp.tid() == 0) {
        double* parts = reinterpret_cast<double*>(rec + OFF_PARTS) + j * NG;
        parts[g] = part;
        __threadfence();
        *s_last = 0;
        if (atomicSub(rec + OFF_CPEND + j, 1) == 1) {  // last group of this candidate
            __threadfence();
            double tot = 0.0;
            for (int q = 0; q < NG; ++q) tot += __ldcg(parts + q);  // fixed order
            reinterpret_cast<double*>(rec + OFF_SC)[j] = w64[W64_B3] + tot / s.history;
            __threadfence();
            *s_last = atomicSub(rec + R_PENDING, 1) == 1;  // last candidate of this map
            if (*s_last) __threadfence();
        }
    }
    grp.sync();
    if (*s_last) finalize(s, m, flags, scan_tmp, grp);
    grp.sync();
}

// Shared-memory scratch of one re-scoring group.
struct RefineSmem {
    double sx[(MAX_RG + 4) * 5];
    double sa1[(MAX_RG + 2) * 48];
    double srow[MAX_RG];
    int flags[CAP];
    int scan_tmp[NT / 32 + 2];
    int unit, val, last;
};

// Separate-launch form (after the top-k kernel: every unit is listed before this starts).  A template
// so that only the translation unit launching it (topk.cu) instantiates it.
template <int = 0>
__global__ void __launch_bounds__(NT) refine_kernel(ap_selector s, Params tp) {
    __shared__ RefineSmem sm;
    int* ws = s.tie_ws;
    // units are dealt statically (unit u on CTA u % gridDim.x: the list is complete when this launch
    // starts), so CTAs without a unit — all of them on most steps — leave after one read, with no
    // contended atomics
    const int n_units = __ldcg(&ws[H_UNITS]);
    if ((int)blockIdx.x >= n_units) return;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        if (threadIdx.x == 0) {
            sm.val = __ldcg(&ws[HDR + u]) - 1;
            ws[HDR + u] = 0;  // cleared for the next step
        }
        __syncthreads();
        refine_unit(s, tp, sm.val, sm.sx, sm.sa1, sm.srow, sm.flags, sm.scan_tmp, &sm.last, CtaGroup{});
    }
    if (threadIdx.x == 0) {  // the last CTA out resets the work list for the next step
        __threadfence();
        const int active = n_units < (int)gridDim.x ? n_units : (int)gridDim.x;
        if (atomicAdd(&ws[H_DONE], 1) == active - 1) {
            ws[H_UNITS] = 0;
            ws[H_DONE] = 0;
            __threadfence();
        }
    }
}

}  // namespace tie
}  // namespace ap
