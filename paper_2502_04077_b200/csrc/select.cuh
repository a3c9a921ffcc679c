// One map's top-k selection (kernel 3's body) for any thread group: the standalone top-k kernel runs
// it with a whole CTA per map, the fused forecaster (forecast_wsm.cuh) with four warps of each of its
// CTAs on the maps whose last chunk that CTA finished.
#pragma once

#include "tieguard.cuh"

namespace ap {

#ifdef AP_SEL_TRACE  // profiling only: clock64 phase stamps of map 0's selection (the last launch)
__device__ long long g_sel_trace[16];
extern "C" int ap_debug_sel_trace(long long* host_out) {
    return cudaMemcpyFromSymbol(host_out, g_sel_trace, 16 * sizeof(long long)) == cudaSuccess ? 0 : 5;
}
#define SEL_TRACE(e) if (m == 0 && tid == 0) g_sel_trace[e] = clock64();
#else
#define SEL_TRACE(e)
#endif

// Nested search bands around the previous k-th score tau: half-widths 2^-2, 2^-4, 2^-6, 2^-8 of |tau|
// (how far the boundary moves between two updates depends on the rows: on the decode engine's maps
// the 2^-2 band holds the new boundary 99.9% of the time with ~34 keys, on tightly clustered synthetic
// scores the 2^-8 band does with ~20; scripts/dbg/topk_stats.py)
constexpr int TK_NB = 4;
__device__ __forceinline__ float tk_band(int i) { return i == 0 ? 0.25f : i == 1 ? 0.0625f : i == 2 ? 0.015625f : 0.00390625f; }
#ifdef AP_TOPK_STATS  // profiling only: [maps, boundary inside the band, fast path taken, sum of band sizes]
__device__ int g_topk_stats[4];
extern "C" int ap_debug_topk_stats(int* host_out) {
    const cudaError_t e = cudaMemcpyFromSymbol(host_out, g_topk_stats, 4 * sizeof(int));
    int z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_topk_stats, z, sizeof(z));
    return e == cudaSuccess ? 0 : 5;
}
#endif

// Band variant (the default for rows of <= NT * IPT blocks).  Scores move little between two updates
// of a map (an incremental forecast changes five of H history rows), so the boundary is first looked
// for in a narrow band around the previous update's k-th score (ap_map_state.prev_kth): one counting
// pass gives the keys above the band and in it; if the k-th key falls inside a band of at most TK_CAND
// keys, those are ranked against each other by (key desc, index asc) — selector.py:80's order — and the
// selection is exact after ~6 CTA barriers.  Otherwise (first update, calibration jumps, heavy ties) the
// 8-bit radix passes of sel_topk_reg_kernel run on the same registers.  The radix form alone spent
// 19.7k cycles per map on CTA 0 (scripts/dbg/topk_trace.py), most of it in same-address shared atomics:
// the scores' bulk shares a few digits.
constexpr int TK_CAND = 128;

template <int NT, int IPT>
struct SelSmem {  // shared memory of one map's selection by an NT-thread group
    int hist[256];
    int scan_tmp[NT / 32 + 2];
    __align__(16) unsigned long long c_pk[TK_CAND + 2];  // band keys packed (key << 32 | ~id): one compare orders them
    uint32_t mask[NT * IPT / 32 + 1];
    int nan, amax, nmask, cnt, bcast;
    int above[TK_NB], band[TK_NB];  // per search band: keys above it, keys in it
    unsigned kmn, kmx, tmin;
};

// Map m's update (or counter tick) by the NT threads of grp; rows of <= NT * IPT blocks.
template <int NT, int IPT, class G>
__device__ void select_map(const ap_selector& s, const tie::Params& tp, int m, const G& grp, SelSmem<NT, IPT>& sh) {
    static_assert(IPT <= 32 && IPT % 4 == 0, "one take bit per key, 16-byte loads");
    int* hist = sh.hist;
    int* scan_tmp = sh.scan_tmp;
    unsigned long long* c_pk = sh.c_pk;
    uint32_t* s_mask = sh.mask;
    int &s_nan = sh.nan, &s_amax = sh.amax, &s_nmask = sh.nmask, &s_cnt = sh.cnt, &s_bcast = sh.bcast;
    int* s_above = sh.above;
    int* s_band = sh.band;
    unsigned &s_kmn = sh.kmn, &s_kmx = sh.kmx, &s_tmin = sh.tmin;
    const int tid = grp.tid(), lane = tid & 31;
    // the row's scores are requested before the map state they depend on arrives (one round trip, not two)
    const float* sc = s.scores + (int64_t)m * s.w_max;
    const int i0 = tid * IPT;
    float vals[IPT];
    if (i0 + IPT <= s.w_max) {  // 16-byte loads (w_max % 4 == 0, i0 % 4 == 0); L2: other CTAs wrote them
#pragma unroll
        for (int v4 = 0; v4 < IPT / 4; ++v4) {
            const float4 f = __ldcg(reinterpret_cast<const float4*>(sc + i0) + v4);
            vals[4 * v4] = f.x; vals[4 * v4 + 1] = f.y; vals[4 * v4 + 2] = f.z; vals[4 * v4 + 3] = f.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < IPT; ++q) vals[q] = i0 + q < s.w_max ? __ldcg(sc + i0 + q) : -INFINITY;
    }
    SEL_TRACE(0);
    ap_map_state st = s.state[m];
    const bool update = (st.counter % s.update_interval) == 0;
    SEL_TRACE(6);
    const int words = (s.w_max + 31) / 32;
    uint32_t* mask = s.mid_mask + (int64_t)m * words;
    int32_t* mid = s.mid_blocks + (int64_t)m * (s.k_mid > 0 ? s.k_mid : 1);
    int count = st.n_mid;
    int tie_n = 0;
    uint32_t kth = st.prev_kth;
    if (update && s.k_mid > 0 && st.width > 0) {
        for (int w = tid; w < words; w += NT) s_mask[w] = 0u;
        if (tid == 0) {
            s_nan = 0; s_amax = 0; s_nmask = 0; s_cnt = 0;
            for (int i = 0; i < TK_NB; ++i) s_above[i] = s_band[i] = 0;
            s_kmn = 0xffffffffu; s_kmx = 0u; s_tmin = 0xffffffffu;
        }
        const int W = st.width;
        const unsigned b = (unsigned)s.block;
        const int64_t t = st.row_len;
        // covering blocks of sink [0, min(sink, nl)) and local [max(0, nl-local), nl) — selector.py:84-88,134-142
        // (32-bit: positions < 2^31; 64-bit division is a ~100-cycle software routine on the critical path)
        const unsigned nl = (unsigned)(t + 1);
        const unsigned sink_end = (unsigned)s.sink < nl ? (unsigned)s.sink : nl;
        int sink_hi = (int)((sink_end + b - 1) / b);
        const unsigned ls = nl > (unsigned)s.local ? nl - (unsigned)s.local : 0u;
        const int local_lo = ls < nl ? (int)(ls / b) : 0;  // (an empty local window covers no block)
        int local_hi = ls < nl ? (int)((nl + b - 1) / b) : 0;
        sink_hi = sink_hi > W ? W : sink_hi;
        local_hi = local_hi > W ? W : local_hi;
        // this thread's blocks [i0, i0 + IPT) as bit masks: inside the row, and selectable (not sink / local)
        auto span = [&](int lo, int hi) -> uint32_t {  // bits q with lo <= i0 + q < hi
            const int a = max(lo - i0, 0), z = min(hi - i0, IPT);
            if (a >= z) return 0u;
            const uint32_t upto = z >= 32 ? 0xffffffffu : (1u << z) - 1u;
            return upto & ~((1u << a) - 1u);
        };
        const uint32_t in_row = span(0, W);
        const uint32_t live = in_row & ~(span(0, sink_hi) | span(local_lo, local_hi));
        uint32_t key[IPT];
        int nm = 0;
        bool nan = false;
        float amax = 0.f;
#pragma unroll
        for (int q = 0; q < IPT; ++q) {
            const float v = vals[q];
            const bool r = (in_row >> q) & 1u, l = (live >> q) & 1u;
            nan |= r && v != v;
            key[q] = l ? order_key(v) : 0u;  // 0 sorts below every real key (and is never taken)
            nm += r && (!l || v == -INFINITY);
            if (l && fabsf(v) <= 3.402823466e38f) amax = fmaxf(amax, fabsf(v));
        }
        SEL_TRACE(7);
        uint32_t lo_b[TK_NB], hi_b[TK_NB];  // search bands (empty without a previous boundary)
        const float tau = tie::key_value(kth);
#pragma unroll
        for (int i = 0; i < TK_NB; ++i) {
            const float d = fmaxf(tk_band(i) * fabsf(tau), 1e-30f);
            lo_b[i] = kth ? order_key(tau - d) : 1u;
            hi_b[i] = kth ? order_key(tau + d) : 0u;
        }
        int na[TK_NB], nb[TK_NB];
#pragma unroll
        for (int i = 0; i < TK_NB; ++i) na[i] = nb[i] = 0;
#pragma unroll
        for (int q = 0; q < IPT; ++q)
#pragma unroll
            for (int i = 0; i < TK_NB; ++i) {
                na[i] += key[q] > hi_b[i];
                nb[i] += key[q] >= lo_b[i] && key[q] <= hi_b[i];
            }
        grp.sync();  // shared state initialised
        SEL_TRACE(1);
        // CTA reductions: one shared atomic per warp
        nm = (int)__reduce_add_sync(0xffffffffu, (unsigned)nm);
#pragma unroll
        for (int i = 0; i < TK_NB; ++i) {
            na[i] = (int)__reduce_add_sync(0xffffffffu, (unsigned)na[i]);
            nb[i] = (int)__reduce_add_sync(0xffffffffu, (unsigned)nb[i]);
        }
        const unsigned am = __reduce_max_sync(0xffffffffu, __float_as_uint(amax));  // non-negative floats
        if (__any_sync(0xffffffffu, nan) && lane == 0) s_nan = 1;
        if (lane == 0) {
            atomicAdd(&s_nmask, nm);
#pragma unroll
            for (int i = 0; i < TK_NB; ++i) {
                if (na[i]) atomicAdd(&s_above[i], na[i]);
                if (nb[i]) atomicAdd(&s_band[i], nb[i]);
            }
            atomicMax(&s_amax, (int)am);
        }
        grp.sync();
        SEL_TRACE(2);
        if (s_nan) raise_status(s.status, AP_ENUMERIC);
        const int available = W - s_nmask;
        const int kcap = s.k_map ? min(max(s.k_map[m], 0), s.k_mid) : s.k_mid;
        const int k = kcap < available ? kcap : available;
        uint32_t take = 0u;  // bit q: block i0 + q is selected
        if (k > 0) {
            // the narrowest band that brackets the k-th key and is small enough to rank directly
            int sel_b = -1;
#pragma unroll
            for (int i = 0; i < TK_NB; ++i)
                if (s_above[i] < k && s_above[i] + s_band[i] >= k && s_band[i] <= TK_CAND) sel_b = i;
            const int above = sel_b >= 0 ? s_above[sel_b] : 0, band = sel_b >= 0 ? s_band[sel_b] : 0;
            uint32_t blo = 1u, bhi = 0u;
#pragma unroll
            for (int i = 0; i < TK_NB; ++i)
                if (i == sel_b) {
                    blo = lo_b[i];
                    bhi = hi_b[i];
                }
#ifdef AP_SEL_TRACE
            if (m == 0 && tid == 0) {
                g_sel_trace[8] = sel_b;
                g_sel_trace[9] = band;
                g_sel_trace[10] = s_band[0];
                g_sel_trace[11] = s_above[0];
                g_sel_trace[12] = k;
                g_sel_trace[13] = s_band[3];
            }
#endif
#ifdef AP_TOPK_STATS
            if (tid == 0) {
                atomicAdd(&g_topk_stats[0], 1);
                if (sel_b >= 0) atomicAdd(&g_topk_stats[1], 1);
                if (sel_b >= 0) atomicAdd(&g_topk_stats[2], 1);
                atomicAdd(&g_topk_stats[3], band);
            }
#endif
            if (sel_b >= 0) {
                // fast path: the k-th key is in the band; rank the band's keys among themselves
                const int need = k - above;
                // gather the band's keys by a scan of the per-thread counts (same-address shared atomics
                // serialise), packed as key << 32 | ~id so that "ahead in (key desc, index asc)" is one compare
                uint32_t inband = 0u;
#pragma unroll
                for (int q = 0; q < IPT; ++q)
                    if (key[q] >= blo && key[q] <= bhi) inband |= 1u << q;
                int tot_b = 0;
                int slot = group_excl_scan1<NT>(__popc(inband), scan_tmp, tot_b, grp);
#pragma unroll
                for (int q = 0; q < IPT; ++q)
                    if ((inband >> q) & 1u) c_pk[slot++] = (unsigned long long)key[q] << 32 | (uint32_t)~(uint32_t)(i0 + q);
                if (tid == 0) c_pk[band] = 0ull;  // pad to a pair (0 is behind every real entry)
                grp.sync();
                if (tid < band) {  // one thread per band key: how many band keys are ahead of it
                    const unsigned long long mine = c_pk[tid];
                    const ulonglong2* pk = reinterpret_cast<const ulonglong2*>(c_pk);
                    int rank = 0;
#pragma unroll 4
                    for (int j = 0; j < (band + 1) / 2; ++j) {
                        const ulonglong2 v = pk[j];
                        rank += (v.x > mine) + (v.y > mine);
                    }
                    const int iq = (int)~(uint32_t)mine;
                    if (rank < need) atomicOr(&s_mask[iq >> 5], 1u << (iq & 31));
                }
                grp.sync();
                // (the band's chosen ids are already in the mask image; `take` adds the keys above the band)
#pragma unroll
                for (int q = 0; q < IPT; ++q)
                    if (key[q] > bhi || ((inband >> q) & 1u && (s_mask[(i0 + q) >> 5] >> ((i0 + q) & 31)) & 1u))
                        take |= 1u << q;
            } else {
                // radix select of the k-th largest key, 8 bits per pass, skipping the bytes every unmasked
                // key shares (they all lie in [kmn, kmx], taken here: this path is rare)
                unsigned kmn = 0xffffffffu, kmx = 0u;
#pragma unroll
                for (int q = 0; q < IPT; ++q)
                    if (key[q]) {
                        kmn = min(kmn, key[q]);
                        kmx = max(kmx, key[q]);
                    }
                kmn = __reduce_min_sync(0xffffffffu, kmn);
                kmx = __reduce_max_sync(0xffffffffu, kmx);
                if (lane == 0) {
                    atomicMin(&s_kmn, kmn);
                    atomicMax(&s_kmx, kmx);
                }
                grp.sync();
                kmn = s_kmn;
                kmx = s_kmx;
                const int top = (kmn ^ kmx) ? 31 - __clz(kmn ^ kmx) : -1;
                const int first = top >= 0 ? top / 8 : -1;
                uint32_t hi_mask = first >= 3 ? 0u : (0xffffffffu << ((first + 1) * 8));
                uint32_t prefix = kmx & hi_mask;
                int remaining = k;
#pragma unroll 1
                for (int pass = first; pass >= 0; --pass) {
                    const int shift = pass * 8;
                    for (int d = tid; d < 256; d += NT) hist[d] = 0;
                    grp.sync();
#pragma unroll
                    for (int q = 0; q < IPT; ++q)
                        if (key[q] != 0u && ((key[q] ^ prefix) & hi_mask) == 0) atomicAdd(&hist[(key[q] >> shift) & 0xFF], 1);
                    grp.sync();
                    int c = 0;
                    for (int d = tid * 256 / NT; d < (tid + 1) * 256 / NT; ++d) c += hist[255 - d];
                    int total = 0;
                    int run = group_excl_scan<NT>(c, scan_tmp, total, grp);
                    for (int d = tid * 256 / NT; d < (tid + 1) * 256 / NT; ++d) {
                        const int hd = hist[255 - d];
                        if (run < remaining && run + hd >= remaining) {
                            scan_tmp[NT / 32] = 255 - d;
                            scan_tmp[NT / 32 + 1] = run;
                        }
                        run += hd;
                    }
                    grp.sync();
                    remaining -= scan_tmp[NT / 32 + 1];
                    prefix |= (uint32_t)scan_tmp[NT / 32] << shift;
                    hi_mask |= 0xFFu << shift;
                    grp.sync();
                }
                const uint32_t T = prefix;  // keys > T, and the lowest-index `remaining` keys == T
                int n_eq = 0;
#pragma unroll
                for (int q = 0; q < IPT; ++q) n_eq += key[q] == T;
                int te = 0;
                int eq_rank = group_excl_scan<NT>(n_eq, scan_tmp, te, grp);
#pragma unroll
                for (int q = 0; q < IPT; ++q) {
                    if (key[q] > T) {
                        take |= 1u << q;
                    } else if (key[q] == T) {
                        if (eq_rank < remaining) take |= 1u << q;
                        ++eq_rank;
                    }
                }
            }
            // ordered emission (ascending ids) and the bitmask image in shared memory
            int total = 0;
            SEL_TRACE(3);
            int pos = group_excl_scan1<NT>(__popc(take), scan_tmp, total, grp);
            unsigned tmin = 0xffffffffu;
#pragma unroll
            for (int q = 0; q < IPT; ++q)
                if (take & (1u << q)) {
                    mid[pos++] = i0 + q;
                    tmin = min(tmin, key[q]);
                }
            if (take && 32 % IPT == 0) {  // all of this thread's ids lie in one mask word
                uint32_t w = 0u;
#pragma unroll
                for (int q = 0; q < IPT; ++q)
                    if (take & (1u << q)) w |= 1u << ((i0 + q) & 31);
                atomicOr(&s_mask[i0 >> 5], w);
            } else if (take) {
                uint32_t bits[(IPT + 31) / 32 + 1] = {};
#pragma unroll
                for (int q = 0; q < IPT; ++q)
                    if (take & (1u << q)) bits[((i0 + q) >> 5) - (i0 >> 5)] |= 1u << ((i0 + q) & 31);
#pragma unroll
                for (int wq = 0; wq < (IPT + 31) / 32 + 1; ++wq)
                    if (bits[wq]) atomicOr(&s_mask[(i0 >> 5) + wq], bits[wq]);
            }
            tmin = __reduce_min_sync(0xffffffffu, tmin);
            if (lane == 0 && tmin != 0xffffffffu) atomicMin(&s_tmin, tmin);
            count = total;
        } else {
            count = 0;
        }
        grp.sync();
        for (int w = tid; w < words; w += NT) mask[w] = s_mask[w];
        SEL_TRACE(4);
        kth = k > 0 ? s_tmin : 0u;
        if (k > 0 && tp.enabled && s.tie_ws)  // (the keys are still in registers: no second read of the row)
            tie_n = tie::detect_regs<NT, IPT>(s, tp, m, key, i0, W, k, kth, __int_as_float(s_amax), sink_hi, local_lo,
                                              local_hi, scan_tmp, hist, &s_bcast, grp);
        if (tid == 0) {
            st.n_mid = count;
            st.mid_clip = t;
            st.r_pushed = st.n_pushed;
            st.r_width = st.width;
            st.r_wgen = tp.wgen ? *tp.wgen : 0;
            st.tie_n = tie_n;
            SEL_TRACE(5);
            st.prev_kth = kth;
        }
    } else if (update && s.k_mid <= 0) {
        for (int w = tid; w < words; w += NT) mask[w] = 0u;
        if (tid == 0) st.n_mid = 0;
    }
    if (tid == 0) {
        st.counter += 1;
        s.state[m] = st;
    }
}

}  // namespace ap
