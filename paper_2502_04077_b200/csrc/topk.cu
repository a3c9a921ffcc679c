// Kernel (3): per-row top-k block selection as a block-wide radix select.
//
// Reference: selector.topk (selector.py:73-81) — the k largest values,
// descending, ties broken toward the lower index (lexsort on (index,
// -value)), -0.0 == +0.0 — and the sink/local masking + min(K, available)
// of selector.step (selector.py:134-145).
//
// Values map to order-preserving unsigned keys; an 8-bit-digit radix select
// finds the k-th largest key T; then one ordered pass takes every key > T and
// the lowest-index keys == T until k are taken.  Output ids are ascending,
// which is the set the reference returns.  Bit-exact on identical inputs.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "select.cuh"

namespace ap {

template <typename KeyT>
struct KeyTraits;
template <> struct KeyTraits<uint32_t> { static constexpr int kPasses = 4; };
template <> struct KeyTraits<unsigned long long> { static constexpr int kPasses = 8; };

// keyfn(i) -> KeyT for i in [0, n).  Returns T and the number of keys == T to take.
template <int NT, typename KeyT, typename KeyFn>
__device__ void radix_select(KeyFn keyfn, int n, int k, int* hist /*[256]*/, int* scan_tmp, KeyT& T_out,
                             int& take_eq_out) {
    KeyT prefix = 0, hi_mask = 0;
    int remaining = k;
#pragma unroll 1
    for (int pass = KeyTraits<KeyT>::kPasses - 1; pass >= 0; --pass) {
        const int shift = pass * 8;
        for (int d = threadIdx.x; d < 256; d += NT) hist[d] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += NT) {
            KeyT key = keyfn(i);
            if (((key ^ prefix) & hi_mask) == 0) atomicAdd(&hist[(int)((key >> shift) & 0xFF)], 1);
        }
        __syncthreads();
        // suffix scan over digits 255..0: thread d (<256) owns digit 255-d
        int c = threadIdx.x < 256 ? hist[255 - threadIdx.x] : 0;
        int total = 0;
        int excl = block_excl_scan<NT>(c, scan_tmp, total);
        // the digit where the cumulative count first reaches `remaining`
        if (threadIdx.x < 256 && excl < remaining && excl + c >= remaining) {
            scan_tmp[NT / 32] = 255 - threadIdx.x;
            scan_tmp[NT / 32 + 1] = excl;
        }
        __syncthreads();
        const int digit = scan_tmp[NT / 32];
        remaining -= scan_tmp[NT / 32 + 1];
        prefix |= (KeyT)digit << shift;
        hi_mask |= (KeyT)0xFF << shift;
        __syncthreads();
    }
    T_out = prefix;
    take_eq_out = remaining;
}

// Ordered emission: ids of keys > T plus the first take_eq keys == T, ascending.
// Returns the count (== k).  emit(rank, id) is called once per selected id.
template <int NT, typename KeyT, typename KeyFn, typename Emit>
__device__ int ordered_emit(KeyFn keyfn, int n, KeyT T, int take_eq, int* scan_tmp, Emit emit) {
    const int per = (n + NT - 1) / NT;
    const int lo = threadIdx.x * per;
    const int hi = lo + per < n ? lo + per : n;
    int n_eq = 0;
    for (int i = lo; i < hi; ++i) n_eq += (keyfn(i) == T);
    int tot = 0;
    int eq_base = block_excl_scan<NT>(n_eq, scan_tmp, tot);
    int n_sel = 0;
    int eq_rank = eq_base;
    for (int i = lo; i < hi; ++i) {
        KeyT key = keyfn(i);
        if (key > T) {
            ++n_sel;
        } else if (key == T) {
            n_sel += (eq_rank < take_eq);
            ++eq_rank;
        }
    }
    int total = 0;
    int out_base = block_excl_scan<NT>(n_sel, scan_tmp, total);
    eq_rank = eq_base;
    int pos = out_base;
    for (int i = lo; i < hi; ++i) {
        KeyT key = keyfn(i);
        bool take = false;
        if (key > T) {
            take = true;
        } else if (key == T) {
            take = eq_rank < take_eq;
            ++eq_rank;
        }
        if (take) emit(pos++, i);
    }
    return total;
}

template <typename V>
struct ValueKey {
    const V* v;
    __device__ auto operator()(int i) const { return order_key(v[i]); }
};

template <int NT, typename V>
__global__ void __launch_bounds__(NT) topk_rows_kernel(const V* __restrict__ values, int64_t row_stride, int n,
                                                       int k, int32_t* __restrict__ out_ids, int64_t out_stride,
                                                       int32_t* __restrict__ out_count) {
    using KeyT = decltype(order_key(V(0)));
    __shared__ int hist[256];
    __shared__ int scan_tmp[NT / 32 + 2];
    const int64_t r = blockIdx.x;
    ValueKey<V> kf{values + r * row_stride};
    int32_t* ids = out_ids + r * out_stride;
    if (k <= 0) {
        if (threadIdx.x == 0) out_count[r] = 0;
        return;
    }
    KeyT T;
    int take_eq;
    radix_select<NT, KeyT>(kf, n, k, hist, scan_tmp, T, take_eq);
    int total = ordered_emit<NT, KeyT>(kf, n, T, take_eq, scan_tmp, [&](int pos, int i) { ids[pos] = i; });
    if (threadIdx.x == 0) out_count[r] = total;
}

// ------------------------------------------------------ selector tail kernel
struct MaskedScoreKey {
    const float* scores;
    int sink_lo, sink_hi, local_lo, local_hi;  // masked covering block ranges [lo, hi)
    __device__ uint32_t operator()(int i) const {
        bool masked = (i >= sink_lo && i < sink_hi) || (i >= local_lo && i < local_hi);
        return masked ? order_key(-INFINITY) : order_key(scores[i]);
    }
};

template <int NT>
__global__ void __launch_bounds__(NT) sel_topk_kernel(ap_selector s, tie::Params tp) {
    __shared__ int hist[256];
    __shared__ int scan_tmp[NT / 32 + 2];
    __shared__ int s_nan, s_amax, s_bcast;
    const int m = blockIdx.x;
    ap_map_state st = s.state[m];
    const bool update = (st.counter % s.update_interval) == 0;
    const int words = (s.w_max + 31) / 32;
    uint32_t* mask = s.mid_mask + (int64_t)m * words;
    int32_t* mid = s.mid_blocks + (int64_t)m * (s.k_mid > 0 ? s.k_mid : 1);
    if (threadIdx.x == 0) {
        s_nan = 0;
        s_amax = 0;
    }
    __syncthreads();
    int count = st.n_mid;
    int tie_n = 0;
    if (update && s.k_mid > 0 && st.width > 0) {
        const int W = st.width;
        const int b = s.block;
        const int64_t t = st.row_len;
        const int64_t nl = t + 1;
        // covering blocks of sink [0, min(sink, nl)) and local [max(0, nl-local), nl) — selector.py:84-88,134-142
        MaskedScoreKey kf;
        kf.scores = s.scores + (int64_t)m * s.w_max;
        const int64_t sink_end = s.sink < nl ? s.sink : nl;
        kf.sink_lo = 0;
        kf.sink_hi = sink_end > 0 ? (int)cdiv64(sink_end, b) : 0;
        const int64_t ls = nl - s.local > 0 ? nl - s.local : 0;
        kf.local_lo = ls < nl ? (int)(ls / b) : 0;
        kf.local_hi = ls < nl ? (int)cdiv64(nl, b) : 0;
        if (kf.sink_hi > W) kf.sink_hi = W;
        if (kf.local_hi > W) kf.local_hi = W;
        // available = #finite after masking (selector.py:143)
        int n_masked_local = 0;
        float amax = 0.f;
        for (int i = threadIdx.x; i < W; i += NT) {
            bool masked = (i >= kf.sink_lo && i < kf.sink_hi) || (i >= kf.local_lo && i < kf.local_hi);
            float v = kf.scores[i];
            if (v != v) s_nan = 1;
            n_masked_local += masked || (v == -INFINITY);
            if (!masked && fabsf(v) <= 3.402823466e38f) amax = fmaxf(amax, fabsf(v));
        }
        atomicMax(&s_amax, __float_as_int(amax));  // non-negative floats order as ints
        int n_masked = 0;
        block_excl_scan<NT>(n_masked_local, scan_tmp, n_masked);
        if (s_nan) raise_status(s.status, AP_ENUMERIC);
        const int available = W - n_masked;
        // per-map middle budget (budget allocation policy; selector.py:47-50 per map), capped by the pitch
        const int kcap = s.k_map ? min(max(s.k_map[m], 0), s.k_mid) : s.k_mid;
        const int k = kcap < available ? kcap : available;
        for (int w = threadIdx.x; w < words; w += NT) mask[w] = 0u;
        __syncthreads();
        if (k > 0) {
            uint32_t T;
            int take_eq;
            radix_select<NT, uint32_t>(kf, W, k, hist, scan_tmp, T, take_eq);
            count = ordered_emit<NT, uint32_t>(kf, W, T, take_eq, scan_tmp, [&](int pos, int i) {
                mid[pos] = i;
                atomicOr(&mask[i >> 5], 1u << (i & 31));
            });
            if (tp.enabled && s.tie_ws)
                tie_n = tie::detect<NT>(s, tp, m, kf, W, k, T, __int_as_float(s_amax), kf.sink_hi, kf.local_lo,
                                        kf.local_hi, scan_tmp, &s_bcast);
        } else {
            count = 0;
        }
        if (threadIdx.x == 0) {
            st.n_mid = count;
            st.mid_clip = t;
            st.r_pushed = st.n_pushed;
            st.r_width = st.width;
            st.r_wgen = tp.wgen ? *tp.wgen : 0;
            st.tie_n = tie_n;
        }
    } else if (update && s.k_mid <= 0) {
        for (int w = threadIdx.x; w < words; w += NT) mask[w] = 0u;
        if (threadIdx.x == 0) st.n_mid = 0;
    }
    if (threadIdx.x == 0) {
        st.counter += 1;
        s.state[m] = st;
    }
}


// Register-resident variant for rows of <= NT * IPT blocks (the usual case: W = 2048 at 32K): thread
// t owns blocks [t * IPT, t * IPT + IPT), loaded once; the radix passes and the ordered emission run
// on registers (the generic kernel re-reads the row from global memory on every pass).
#ifdef AP_TOPK_TRACE  // profiling only: CTA 0's phase clocks of the last launch
__device__ long long g_topk_trace[16];
#define TOPK_TRACE(e) if (blockIdx.x == 0 && threadIdx.x == 0) g_topk_trace[e] = clock64();
#else
#define TOPK_TRACE(e)
#endif
template <int NT, int IPT>
__global__ void __launch_bounds__(NT) sel_topk_reg_kernel(ap_selector s, tie::Params tp) {
    TOPK_TRACE(0);
    __shared__ int hist[256];
    __shared__ int scan_tmp[NT / 32 + 2];
    __shared__ int s_nan, s_amax, s_bcast;
    __shared__ unsigned s_kmn, s_kmx;  // key range of the unmasked blocks
    const int m = blockIdx.x;
    ap_map_state st = s.state[m];
    const bool update = (st.counter % s.update_interval) == 0;
    const int words = (s.w_max + 31) / 32;
    uint32_t* mask = s.mid_mask + (int64_t)m * words;
    int32_t* mid = s.mid_blocks + (int64_t)m * (s.k_mid > 0 ? s.k_mid : 1);
    if (threadIdx.x == 0) {
        s_nan = 0;
        s_amax = 0;
        s_kmn = 0xffffffffu;
        s_kmx = 0u;
    }
    __syncthreads();
    TOPK_TRACE(1);
    int count = st.n_mid;
    int tie_n = 0;
    if (update && s.k_mid > 0 && st.width > 0) {
        const int W = st.width;
        const int b = s.block;
        const int64_t t = st.row_len;
        const int64_t nl = t + 1;
        // covering blocks of sink [0, min(sink, nl)) and local [max(0, nl-local), nl) — selector.py:84-88,134-142
        const int64_t sink_end = s.sink < nl ? s.sink : nl;
        int sink_hi = sink_end > 0 ? (int)cdiv64(sink_end, b) : 0;
        const int64_t ls = nl - s.local > 0 ? nl - s.local : 0;
        const int local_lo = ls < nl ? (int)(ls / b) : 0;
        int local_hi = ls < nl ? (int)cdiv64(nl, b) : 0;
        sink_hi = sink_hi > W ? W : sink_hi;
        local_hi = local_hi > W ? W : local_hi;
        const float* sc = s.scores + (int64_t)m * s.w_max;
        const int i0 = threadIdx.x * IPT;
        uint32_t key[IPT];
        int n_masked_local = 0;
        bool nan = false;
        float amax = 0.f;
#pragma unroll
        for (int q = 0; q < IPT; ++q) {
            const int i = i0 + q;
            const float v = i < W ? sc[i] : -INFINITY;
            nan |= v != v;
            const bool masked = i >= W || (i < sink_hi) || (i >= local_lo && i < local_hi);
            key[q] = masked ? 0u : order_key(v);  // 0 sorts below every real key (and is never taken)
            n_masked_local += i < W && (masked || v == -INFINITY);
            if (!masked && fabsf(v) <= 3.402823466e38f) amax = fmaxf(amax, fabsf(v));
        }
        if (nan) s_nan = 1;
        atomicMax(&s_amax, __float_as_int(amax));  // non-negative floats order as ints
        {
            unsigned kmn = 0xffffffffu, kmx = 0u;
#pragma unroll
            for (int q = 0; q < IPT; ++q)
                if (key[q]) {
                    kmn = min(kmn, key[q]);
                    kmx = max(kmx, key[q]);
                }
            kmn = __reduce_min_sync(0xffffffffu, kmn);
            kmx = __reduce_max_sync(0xffffffffu, kmx);
            if ((threadIdx.x & 31) == 0) {
                atomicMin(&s_kmn, kmn);
                atomicMax(&s_kmx, kmx);
            }
        }
        int n_masked = 0;
        block_excl_scan<NT>(n_masked_local, scan_tmp, n_masked);
        if (s_nan) raise_status(s.status, AP_ENUMERIC);
        const int available = W - n_masked;
        TOPK_TRACE(2);
        // per-map middle budget (budget allocation policy; selector.py:47-50 per map), capped by the pitch
        const int kcap = s.k_map ? min(max(s.k_map[m], 0), s.k_mid) : s.k_mid;
        const int k = kcap < available ? kcap : available;
        for (int w = threadIdx.x; w < words; w += NT) mask[w] = 0u;
        if (k > 0) {
            // radix select of the k-th largest key, 8 bits per pass.  Every unmasked key lies in [kmn, kmx],
            // so the bytes above their highest differing bit are common: those passes are skipped.
            // (Warp-aggregating equal digits with __match_any_sync measured slower: 147.5 vs 118.8 us.)
            const uint32_t kmn = s_kmn, kmx = s_kmx;
            const int top = (kmn ^ kmx) ? 31 - __clz(kmn ^ kmx) : -1;
            const int first = top >= 0 ? top / 8 : -1;
            uint32_t hi_mask = first >= 3 ? 0u : (0xffffffffu << ((first + 1) * 8));
            uint32_t prefix = kmx & hi_mask;
            int remaining = k;
#pragma unroll 1
            for (int pass = first; pass >= 0; --pass) {
                const int shift = pass * 8;
                for (int d = threadIdx.x; d < 256; d += NT) hist[d] = 0;
                __syncthreads();
#pragma unroll
                for (int q = 0; q < IPT; ++q)
                    if (key[q] != 0u && ((key[q] ^ prefix) & hi_mask) == 0) atomicAdd(&hist[(key[q] >> shift) & 0xFF], 1);
                __syncthreads();
                const int c = threadIdx.x < 256 ? hist[255 - threadIdx.x] : 0;
                int total = 0;
                const int excl = block_excl_scan<NT>(c, scan_tmp, total);
                if (threadIdx.x < 256 && excl < remaining && excl + c >= remaining) {
                    scan_tmp[NT / 32] = 255 - threadIdx.x;
                    scan_tmp[NT / 32 + 1] = excl;
                }
                __syncthreads();
                const int digit = scan_tmp[NT / 32];
                remaining -= scan_tmp[NT / 32 + 1];
                prefix |= (uint32_t)digit << shift;
                hi_mask |= 0xFFu << shift;
                __syncthreads();
            }
            const uint32_t T = prefix;
            const int take_eq = remaining;
            TOPK_TRACE(3);
#ifdef AP_TOPK_TRACE
            if (blockIdx.x == 0 && threadIdx.x == 0) g_topk_trace[8] = first + 1;
#endif
            // ordered emission: keys > T and the lowest-index take_eq keys == T, ascending
            int n_eq = 0;
#pragma unroll
            for (int q = 0; q < IPT; ++q) n_eq += key[q] == T;
            int tot = 0;
            const int eq_base = block_excl_scan<NT>(n_eq, scan_tmp, tot);
            int n_sel = 0, eq_rank = eq_base;
#pragma unroll
            for (int q = 0; q < IPT; ++q) {
                if (key[q] > T) ++n_sel;
                else if (key[q] == T) { n_sel += eq_rank < take_eq; ++eq_rank; }
            }
            int total = 0;
            int pos = block_excl_scan<NT>(n_sel, scan_tmp, total);
            eq_rank = eq_base;
            uint32_t bits[(IPT + 31) / 32 + 1] = {};  // this thread's ids span IPT / 32 (+1) mask words
#pragma unroll
            for (int q = 0; q < IPT; ++q) {
                bool take = false;
                if (key[q] > T) take = true;
                else if (key[q] == T) { take = eq_rank < take_eq; ++eq_rank; }
                if (take) {
                    mid[pos++] = i0 + q;
                    bits[((i0 + q) >> 5) - (i0 >> 5)] |= 1u << ((i0 + q) & 31);
                }
            }
            __syncthreads();  // the mask words were cleared above by other threads
#pragma unroll
            for (int wq = 0; wq < (IPT + 31) / 32 + 1; ++wq)
                if (bits[wq]) atomicOr(&mask[(i0 >> 5) + wq], bits[wq]);
            count = total;
            TOPK_TRACE(4);
            if (tp.enabled && s.tie_ws) {
                auto kf = [&](int i) -> uint32_t {
                    const bool masked = (i < sink_hi) || (i >= local_lo && i < local_hi);
                    return masked ? 0u : order_key(sc[i]);
                };
                tie_n = tie::detect<NT>(s, tp, m, kf, W, k, T, __int_as_float(s_amax), sink_hi, local_lo, local_hi,
                                        scan_tmp, &s_bcast);
            }
            TOPK_TRACE(5);
        } else {
            count = 0;
        }
        if (threadIdx.x == 0) {
            st.n_mid = count;
            st.mid_clip = t;
            st.r_pushed = st.n_pushed;
            st.r_width = st.width;
            st.r_wgen = tp.wgen ? *tp.wgen : 0;
            st.tie_n = tie_n;
        }
    } else if (update && s.k_mid <= 0) {
        for (int w = threadIdx.x; w < words; w += NT) mask[w] = 0u;
        if (threadIdx.x == 0) st.n_mid = 0;
    }
    if (threadIdx.x == 0) {
        st.counter += 1;
        s.state[m] = st;
    }
    TOPK_TRACE(6);
}

template <int NT, int IPT>
__global__ void __launch_bounds__(NT) sel_topk_band_kernel(ap_selector s, tie::Params tp) {
    __shared__ SelSmem<NT, IPT> sh;
    select_map<NT, IPT>(s, tp, blockIdx.x, CtaGroup{}, sh);
}

// Warp-per-map variant (opt-in, slower: see launch_sel_topk) for rows of <= 32 * IPT blocks (W = 2049 at 32K needs IPT 72): lane l owns blocks
// q * 32 + l, so a ballot over one q covers 32 consecutive blocks — exactly one word of the bitmask and
// a run of ascending ids.  The k-th largest key comes from a 32-step binary search on the key bits (a
// warp reduction per step, no CTA barriers); ties are ranked by ballots in index order.  Same results
// as sel_topk_reg_kernel (the CTA form is kept for the generic path and A/B checks).
template <int IPT>
__global__ void __launch_bounds__(64) sel_topk_warp_kernel(ap_selector s, tie::Params tp) {
    static_assert(IPT % 8 == 0, "eight counting chains");
    const int lane = threadIdx.x & 31;
    const int m = blockIdx.x * 2 + (threadIdx.x >> 5);
    if (m >= s.n_maps) return;
    const unsigned FULL = 0xffffffffu;
    ap_map_state st = s.state[m];
    const bool update = (st.counter % s.update_interval) == 0;
    const int words = (s.w_max + 31) / 32;
    uint32_t* mask = s.mid_mask + (int64_t)m * words;
    int32_t* mid = s.mid_blocks + (int64_t)m * (s.k_mid > 0 ? s.k_mid : 1);
    int count = st.n_mid, tie_n = 0;
    if (update && s.k_mid > 0 && st.width > 0) {
        const int W = st.width, b = s.block;
        const int64_t t = st.row_len, nl = t + 1;
        // covering blocks of sink [0, min(sink, nl)) and local [max(0, nl-local), nl) — selector.py:84-88,134-142
        const int64_t sink_end = s.sink < nl ? s.sink : nl;
        int sink_hi = sink_end > 0 ? (int)cdiv64(sink_end, b) : 0;
        const int64_t ls = nl - s.local > 0 ? nl - s.local : 0;
        const int local_lo = ls < nl ? (int)(ls / b) : 0;
        int local_hi = ls < nl ? (int)cdiv64(nl, b) : 0;
        sink_hi = sink_hi > W ? W : sink_hi;
        local_hi = local_hi > W ? W : local_hi;
        const float* sc = s.scores + (int64_t)m * s.w_max;
        uint32_t key[IPT];
        int n_masked = 0;
        bool nan = false;
        float amax = 0.f;
#pragma unroll
        for (int q = 0; q < IPT; ++q) {
            const int i = q * 32 + lane;
            const float v = i < W ? sc[i] : -INFINITY;
            nan |= v != v;
            const bool masked = i >= W || i < sink_hi || (i >= local_lo && i < local_hi);
            key[q] = masked ? 0u : order_key(v);  // 0 sorts below every real key (and is never taken)
            n_masked += i < W && (masked || v == -INFINITY);
            if (!masked && fabsf(v) <= 3.402823466e38f) amax = fmaxf(amax, fabsf(v));
        }
        if (__any_sync(FULL, nan) && lane == 0) raise_status(s.status, AP_ENUMERIC);
        n_masked = __reduce_add_sync(FULL, n_masked);
        amax = __uint_as_float(__reduce_max_sync(FULL, __float_as_uint(amax)));  // non-negative: bits order
        const int available = W - n_masked;
        const int kcap = s.k_map ? min(max(s.k_map[m], 0), s.k_mid) : s.k_mid;
        const int k = kcap < available ? kcap : available;
        for (int w = lane; w < words; w += 32) mask[w] = 0u;
        count = 0;
        if (k > 0) {
            // T = the k-th largest key: the largest T with #(key >= T) >= k, bit by bit from the top
            uint32_t T = 0;
#pragma unroll 1
            for (int bit = 31; bit >= 0; --bit) {
                const uint32_t cand = T | (1u << bit);
                int c[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // independent chains (IPT is a multiple of 8)
#pragma unroll
                for (int q = 0; q < IPT; ++q) c[q & 7] += key[q] >= cand;
                const int cs = ((c[0] + c[1]) + (c[2] + c[3])) + ((c[4] + c[5]) + (c[6] + c[7]));
                if ((int)__reduce_add_sync(FULL, (unsigned)cs) >= k) T = cand;
            }
            int n_gt = 0;
#pragma unroll
            for (int q = 0; q < IPT; ++q) n_gt += key[q] > T;
            const int take_eq = k - (int)__reduce_add_sync(FULL, (unsigned)n_gt);
            // ordered emission: keys > T and the lowest-index take_eq keys == T, ascending
            const unsigned lt = (1u << lane) - 1u;
            int eq_before = 0, pos = 0;
            __syncwarp();  // mask words cleared above by other lanes
#pragma unroll
            for (int q = 0; q < IPT; ++q) {
                const unsigned eqm = __ballot_sync(FULL, key[q] == T);
                const bool take = key[q] > T || (key[q] == T && eq_before + __popc(eqm & lt) < take_eq);
                const unsigned tm = __ballot_sync(FULL, take);
                eq_before += __popc(eqm);
                if (take) mid[pos + __popc(tm & lt)] = q * 32 + lane;
                if (lane == 0 && tm) mask[q] = tm;
                pos += __popc(tm);
            }
            count = pos;
            if (tp.enabled && s.tie_ws) tie_n = tie::detect_warp<IPT>(s, tp, m, key, W, k, T, amax, sink_hi,
                                                                      local_lo, local_hi);
        }
        st.n_mid = count;
        st.mid_clip = t;
        st.r_pushed = st.n_pushed;
        st.r_width = st.width;
        st.r_wgen = tp.wgen ? *tp.wgen : 0;
        st.tie_n = tie_n;
    } else if (update && s.k_mid <= 0) {
        for (int w = lane; w < words; w += 32) mask[w] = 0u;
        st.n_mid = 0;
    }
    st.counter += 1;
    __syncwarp();
    if (lane == 0) s.state[m] = st;
}

void launch_sel_topk(const ap_selector& s, const tie::Params& tp, cudaStream_t stream) {
    static int warp_form = -1, radix_form = 0;
    if (warp_form < 0) {
        // opt-in (ATTNPRED_TOPK_KERNEL=warp): measured 27 us slower per 256-map launch at 32K than the
        // CTA form (graph replay, scripts/dbg/forecast_knobs.py: 145.4 vs 118.8 us with the forecaster);
        // ATTNPRED_TOPK_KERNEL=radix: the 8-bit radix CTA form the range-bin kernel replaced
        const char* e = getenv("ATTNPRED_TOPK_KERNEL");
        warp_form = e && strcmp(e, "warp") == 0;
        radix_form = e && strcmp(e, "radix") == 0;
    }
    const unsigned wgrid = (unsigned)((s.n_maps + 1) / 2);
    if (warp_form && s.w_max <= 32 * 16) sel_topk_warp_kernel<16><<<wgrid, 64, 0, stream>>>(s, tp);
    else if (warp_form && s.w_max <= 32 * 72) sel_topk_warp_kernel<72><<<wgrid, 64, 0, stream>>>(s, tp);
    else if (!radix_form && s.w_max <= 256 * 8) sel_topk_band_kernel<256, 8><<<s.n_maps, 256, 0, stream>>>(s, tp);
    else if (!radix_form && s.w_max <= 256 * 16) sel_topk_band_kernel<256, 16><<<s.n_maps, 256, 0, stream>>>(s, tp);
    else if (s.w_max <= 256 * 8) sel_topk_reg_kernel<256, 8><<<s.n_maps, 256, 0, stream>>>(s, tp);
    else if (s.w_max <= 256 * 16) sel_topk_reg_kernel<256, 16><<<s.n_maps, 256, 0, stream>>>(s, tp);
    else sel_topk_kernel<256><<<s.n_maps, 256, 0, stream>>>(s, tp);
    if (tp.enabled && s.tie_ws) {
        static int grid = 0;
        if (!grid) grid = 4 * ap_device_sm_count();
        tie::refine_kernel<><<<grid, tie::NT, 0, stream>>>(s, tp);
    }
}

}  // namespace ap

using namespace ap;

#ifdef AP_TOPK_TRACE
extern "C" int ap_debug_topk_trace(long long* host_out) {
    return cudaMemcpyFromSymbol(host_out, g_topk_trace, sizeof(long long) * 16) == cudaSuccess ? AP_OK : AP_ECUDA;
}
#endif

extern "C" int64_t ap_sel_tie_ws_bytes(int32_t n_maps) {
    return n_maps < 1 ? 0 : 4 * tie::ws_words(n_maps);
}

extern "C" int ap_sel_tie_stats(const int32_t* tie_ws, int32_t* host_out3) {
    // cumulative [overflow maps, refined maps, re-scored candidates] since the workspace was zeroed
    AP_REQUIRE(tie_ws && host_out3, AP_EPARAM, "null pointer");
    return cudaMemcpy(host_out3, tie_ws + tie::H_OVERFLOW, 3 * sizeof(int32_t), cudaMemcpyDeviceToHost) ==
                   cudaSuccess ? AP_OK : AP_ECUDA;
}

extern "C" int ap_topk(const void* values, int dtype, int64_t n_rows, int64_t row_stride, int32_t n, int32_t k,
                       int32_t* out_ids, int64_t out_stride, int32_t* out_count, int32_t* status, void* stream) {
    (void)status;
    AP_REQUIRE(k <= n, AP_EPARAM, "k=%d exceeds vector length %d", k, n);
    AP_REQUIRE(n >= 0 && n_rows >= 0 && n_rows <= 0x7fffffff, AP_EPARAM, "bad sizes");
    if (n_rows == 0) return AP_OK;
    cudaStream_t st = as_stream(stream);
    if (dtype == AP_F32)
        topk_rows_kernel<512, float><<<(unsigned)n_rows, 512, 0, st>>>((const float*)values, row_stride, n, k,
                                                                       out_ids, out_stride, out_count);
    else if (dtype == AP_F64)
        topk_rows_kernel<512, double><<<(unsigned)n_rows, 512, 0, st>>>((const double*)values, row_stride, n, k,
                                                                        out_ids, out_stride, out_count);
    else
        AP_REQUIRE(false, AP_EPARAM, "values must be float32 or float64");
    return launch_status("ap_topk");
}
