// Kernel (5): cross-token prefetch of the predicted critical V blocks from
// pinned host memory into a per-(layer, sequence, KV-head) device page pool.
//
// Reference contract: the cross_token schedule of prefetchsim._schedule_point
// (prefetchsim.py:126-151): the blocks predicted at step t are transferred
// while the model computes, total = max(compute, predict + transfer), and the
// device holds only the budget (resident = B * bytes/token/layer * L,
// prefetchsim.py:130-134).  The reference only models this; here it is real:
//
//   * K stays resident on the device (the calibration pass, every M-th step,
//     reads all of K: selector.py:112-116); V is offloaded to pinned host
//     memory (written through by the append kernel).
//   * Device V per map: [sink blocks | recent ring | middle pages].  Sink and
//     the local window are device-resident; middle pages hold the selected
//     middle blocks.
//   * After the selector predicts step t+1's middle blocks (at the end of step
//     t), this kernel diffs them against the blocks already resident, keeps
//     the pages of blocks selected again (the delta cache), and gathers only
//     the new blocks from mapped host memory with 16-byte loads — launched per
//     layer on a side stream so layer l's transfer overlaps layers < l of the
//     next token.
#include "common.cuh"

namespace ap {

constexpr int PF_THREADS = 256;
constexpr int BLOCK_V_BYTES = 16 * 128 * 2;  // one 16-token block of one head, bf16

__device__ __forceinline__ int lower_bound_i32(const int32_t* a, int n, int32_t x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// grid (n_kv_heads, n_seq): one CTA per map of `layer`.
__global__ void __launch_bounds__(PF_THREADS) prefetch_kernel(ap_selector sel, ap_vpages vp, int32_t layer,
                                                             int32_t n_seq, int32_t n_kv, int32_t maps_per_seq) {
    __shared__ int32_t s_new[128], s_old[128], s_oldp[128], s_newp[128];
    __shared__ int32_t s_fetch_blk[128], s_fetch_pg[128];
    __shared__ uint32_t s_used[4];
    __shared__ int s_warp[PF_THREADS / 32 + 2];
    __shared__ int s_nfetch;
    const int h = blockIdx.x, s = blockIdx.y;
    const int smap = s * maps_per_seq + layer * n_kv + h;   // selector map (KV-group selection)
    const int64_t vmap = ((int64_t)layer * n_seq + s) * n_kv + h;
    const int kcap = vp.k_cap;
    const int n_new = sel.state[smap].n_mid;
    const int n_old = vp.old_n[vmap];
    const int32_t* mid = sel.mid_blocks + (int64_t)smap * (sel.k_mid > 0 ? sel.k_mid : 1);
    const int tid = threadIdx.x;
    if (tid < 4) s_used[tid] = 0u;
    for (int i = tid; i < n_new; i += PF_THREADS) s_new[i] = mid[i];
    for (int i = tid; i < n_old; i += PF_THREADS) {
        s_old[i] = vp.old_blocks[vmap * kcap + i];
        s_oldp[i] = vp.old_pages[vmap * kcap + i];
    }
    __syncthreads();
    // kept blocks reuse their page; mark used pages
    int need = 0;
    for (int i = tid; i < n_new; i += PF_THREADS) {
        const int k = lower_bound_i32(s_old, n_old, s_new[i]);
        if (k < n_old && s_old[k] == s_new[i]) {
            s_newp[i] = s_oldp[k];
            atomicOr(&s_used[s_oldp[k] >> 5], 1u << (s_oldp[k] & 31));
        } else {
            s_newp[i] = -1;
        }
    }
    __syncthreads();
    // fetch list in block order; free pages in page order; the r-th fetch takes the r-th free page
    const int i = tid;
    need = (i < n_new && s_newp[i] < 0) ? 1 : 0;
    int total = 0;
    const int rank = block_excl_scan<PF_THREADS>(need, s_warp, total);
    const int pg_i = i;  // candidate page for the free-page scan
    const int is_free = (pg_i < kcap && !((s_used[pg_i >> 5] >> (pg_i & 31)) & 1u)) ? 1 : 0;
    int n_free = 0;
    const int frank = block_excl_scan<PF_THREADS>(is_free, s_warp, n_free);
    if (is_free && frank < 128) s_fetch_pg[frank] = pg_i;  // staging: free page list
    __syncthreads();
    if (need) {
        const int pg = s_fetch_pg[rank];
        s_fetch_blk[rank] = s_new[i];
        s_newp[i] = pg;
    }
    if (tid == 0) s_nfetch = total;
    __syncthreads();
    // publish the new resident set (page per middle block, aligned with mid_blocks) and remember it
    for (int k = tid; k < n_new; k += PF_THREADS) {
        vp.mid_page[vmap * kcap + k] = s_newp[k];
        vp.old_blocks[vmap * kcap + k] = s_new[k];
        vp.old_pages[vmap * kcap + k] = s_newp[k];
    }
    if (tid == 0) vp.old_n[vmap] = n_new;
    // gather the new blocks: host (mapped, pinned) -> device pages, 16-byte loads, 4 blocks in flight
    const int nf = s_nfetch;
    const uint4* hv = reinterpret_cast<const uint4*>(vp.host_v) + vmap * (vp.host_t_max * 128 * 2 / 16);
    uint4* pages = reinterpret_cast<uint4*>(vp.pages) + vmap * (int64_t)(vp.sink_pages + vp.recent_pages + kcap) *
                                                             (BLOCK_V_BYTES / 16);
    constexpr int V16 = BLOCK_V_BYTES / 16;  // 256 uint4 per block
    for (int f0 = 0; f0 < nf; f0 += 4) {
        uint4 v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (f0 + q < nf) v[q] = hv[(int64_t)s_fetch_blk[f0 + q] * V16 + tid];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (f0 + q < nf)
                pages[(int64_t)(vp.sink_pages + vp.recent_pages + s_fetch_pg[f0 + q]) * V16 + tid] = v[q];
    }
    if (tid == 0 && vp.bytes_copied) atomicAdd(reinterpret_cast<unsigned long long*>(vp.bytes_copied),
                                               (unsigned long long)nf * BLOCK_V_BYTES);
}

// Append the step's V row to the paged store (sink page when pos < sink, the
// recent ring otherwise) and write it through to host V; K goes to the
// resident cache as usual (ap_rope_append with v_cache = NULL does that).
__global__ void v_append_kernel(const __nv_bfloat16* __restrict__ qkv, int Hq, int Hkv, const int32_t* seq_len,
                                ap_vpages vp, int32_t layer, int32_t n_seq) {
    const int s = blockIdx.y, h = blockIdx.x, i = threadIdx.x;  // 128 threads: one per dim
    const int pos = seq_len[s] - 1;
    const int64_t vmap = ((int64_t)layer * n_seq + s) * Hkv + h;
    const __nv_bfloat16 v = qkv[((int64_t)s * (Hq + 2 * Hkv) + Hq + Hkv + h) * 128 + i];
    __nv_bfloat16* host = reinterpret_cast<__nv_bfloat16*>(const_cast<void*>(vp.host_v));
    host[(vmap * vp.host_t_max + pos) * 128 + i] = v;
    const int blk = pos / 16;
    const int page = blk < vp.sink_pages ? blk : vp.sink_pages + blk % vp.recent_pages;
    __nv_bfloat16* pages = reinterpret_cast<__nv_bfloat16*>(vp.pages);
    pages[((vmap * (vp.sink_pages + vp.recent_pages + vp.k_cap) + page) * 16 + pos % 16) * 128 + i] = v;
}

// Fill the device-resident pages (sink blocks and the recent ring) of every map
// from host V after a synthetic prefill of length t.
__global__ void v_pages_init_kernel(ap_vpages vp, int64_t t, int64_t n_vmaps) {
    const int64_t vmap = blockIdx.x;
    if (vmap >= n_vmaps) return;
    constexpr int V16 = BLOCK_V_BYTES / 16;
    const uint4* hv = reinterpret_cast<const uint4*>(vp.host_v) + vmap * (vp.host_t_max * 128 * 2 / 16);
    uint4* pages = reinterpret_cast<uint4*>(vp.pages) + vmap * (int64_t)(vp.sink_pages + vp.recent_pages + vp.k_cap) * V16;
    const int64_t nblk = (t + 15) / 16;
    for (int b = 0; b < vp.sink_pages && b < nblk; ++b)
        for (int e = threadIdx.x; e < V16; e += blockDim.x) pages[(int64_t)b * V16 + e] = hv[(int64_t)b * V16 + e];
    for (int64_t b = (nblk > vp.recent_pages ? nblk - vp.recent_pages : 0); b < nblk; ++b) {
        if (b < vp.sink_pages) continue;
        const int page = vp.sink_pages + (int)(b % vp.recent_pages);
        for (int e = threadIdx.x; e < V16; e += blockDim.x) pages[(int64_t)page * V16 + e] = hv[b * V16 + e];
    }
    if (threadIdx.x == 0) vp.old_n[vmap] = 0;
}

}  // namespace ap

using namespace ap;

extern "C" {

int ap_prefetch(const ap_selector* sel, const ap_vpages* vp, int32_t layer, int32_t n_seq, int32_t n_kv_heads,
                int32_t maps_per_seq, void* stream) {
    AP_REQUIRE(sel && vp && vp->pages && vp->host_v, AP_EPARAM, "bad prefetch descriptors");
    AP_REQUIRE(vp->k_cap >= sel->k_mid && vp->k_cap <= 128, AP_EPARAM, "k_cap must be in [k_mid, 128]");
    AP_REQUIRE(sel->block == 16, AP_EPARAM, "prefetch assumes 16-token blocks");
    dim3 grid(n_kv_heads, n_seq);
    prefetch_kernel<<<grid, PF_THREADS, 0, as_stream(stream)>>>(*sel, *vp, layer, n_seq, n_kv_heads, maps_per_seq);
    return launch_status("ap_prefetch");
}

int ap_v_append(const void* qkv, int32_t n_q_heads, int32_t n_kv_heads, const int32_t* seq_len, const ap_vpages* vp,
                int32_t layer, int32_t n_seq, void* stream) {
    AP_REQUIRE(vp && vp->pages, AP_EPARAM, "bad paged-V descriptor");
    v_append_kernel<<<dim3(n_kv_heads, n_seq), 128, 0, as_stream(stream)>>>((const __nv_bfloat16*)qkv, n_q_heads,
                                                                            n_kv_heads, seq_len, *vp, layer, n_seq);
    return launch_status("ap_v_append");
}

int ap_v_pages_init(const ap_vpages* vp, int64_t t, int64_t n_vmaps, void* stream) {
    AP_REQUIRE(vp && vp->pages && vp->host_v, AP_EPARAM, "bad paged-V descriptor");
    v_pages_init_kernel<<<(unsigned)n_vmaps, 256, 0, as_stream(stream)>>>(*vp, t, n_vmaps);
    return launch_status("ap_v_pages_init");
}

}  // extern "C"
