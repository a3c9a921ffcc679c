// Merged-band warp-specialised forecaster kernel (tensor-core precisions) — included by
// predictor.cu after forecast_ws.cuh, whose role structure it keeps (one 16-warp CTA per SM:
// producer warp, MMA warp, 4 epilogue warps, 10 conv1 warps; mbarrier handshakes).
//
// What changes: the per-band handoffs (metadata, copies, three role handshakes) dominate the
// warp-specialised kernel — with every arithmetic step disabled a launch still costs ~70 us at
// the bench shape — and an incremental task used to be two bands (history rows {0, 1} and
// [lo2, H)).  Here a band holds up to MO = 5 output rows in at most two contiguous segments, so an
// incremental update (2 + 3 rows at one new history row per step) is ONE band, and a full
// recompute is 13 bands instead of 22.  Accumulators are exact: output row k of the band owns
// TMEM columns [32 k, 32 k + 32); each conv2 MMA covers only the output rows its a1 row feeds
// (N = 32 / 64 / 96 over a sub-range of the stacked [di = 2, 1, 0] B tile) and always
// accumulates — the epilogue clears the columns after reading them.
#pragma once

namespace ap {
namespace wsm {

#ifndef AP_WSM_NCONV
#define AP_WSM_NCONV 10
#endif
#ifndef AP_CNT_SLEEP
#define AP_CNT_SLEEP 64
#endif
#ifndef AP_WSM_NX
#define AP_WSM_NX 4
#endif
#ifndef AP_WSM_LAYOUT
#define AP_WSM_LAYOUT 1
#endif
#if AP_WSM_LAYOUT
// Warp w runs on scheduler w % 4.  Scheduler 1 (warps 1, 5, 9, 13) hosts only the MMA issuer, the
// quadrant-1 epilogue warp, the producer and an idle warp, so the single thread that issues every
// tcgen05.mma does not share its issue slots with conv1 warps; the 9 conv1 warps fill schedulers 0, 2, 3.
#ifndef AP_WSM_CONV13
#define AP_WSM_CONV13 0  // 1: warp 13 is a tenth conv1 warp (shares scheduler 1 with the MMA issuer)
#endif
constexpr int NCONV = 9 + AP_WSM_CONV13;
#else
constexpr int NCONV = AP_WSM_NCONV;         // conv1 warps (16 measured slower: shared-memory port)
#endif
constexpr int MO = 5;                       // output rows per band
constexpr int MA = MO + 4;                  // a1 tile rows per band (2 segments x (n + 2))
constexpr int MX = MO + 8;                  // x tile rows per band (2 segments x (n + 4))
constexpr int NX = AP_WSM_NX;               // x tile stages
constexpr int NA = 2;                       // a1 tile / accumulator stages
constexpr int NEPI = 4;
#if AP_WSM_LAYOUT
constexpr int WARP_PROD = 9, WARP_MMA = 1, EPI0 = 0;
constexpr int NT = 16 * 32;
enum { R_PROD, R_MMA, R_EPI, R_CONV, R_IDLE };
__device__ __forceinline__ int role_of(int w) {
    return w == WARP_PROD ? R_PROD : w == WARP_MMA ? R_MMA : (w == 0 || w == 2 || w == 3 || w == 5) ? R_EPI
         : (w == 13 && !AP_WSM_CONV13) ? R_IDLE : R_CONV;
}
__device__ __forceinline__ int conv_rank(int w) {  // warps 4, 6, 7, 8, 10, 11, 12, 14, 15 (, 13) -> 0..8 (, 9)
    return w == 13 ? 9 : w == 4 ? 0 : w < 9 ? w - 5 : w < 13 ? w - 6 : w - 7;
}
#else
constexpr int WARP_PROD = 0, WARP_MMA = 1, EPI0 = 2, CONV0 = 6;
constexpr int NT = (CONV0 + NCONV) * 32;
enum { R_PROD, R_MMA, R_EPI, R_CONV, R_IDLE };
__device__ __forceinline__ int role_of(int w) {
    return w == WARP_PROD ? R_PROD : w == WARP_MMA ? R_MMA : w < EPI0 + NEPI ? R_EPI : R_CONV;
}
__device__ __forceinline__ int conv_rank(int w) { return w - CONV0; }
#endif
constexpr int NCONV_T = NCONV * 32;
// Fused selection (FUSE): once a CTA has no more bands, its warps split into four groups of four that run
// kernel 3 (top-k + exact-boundary guard) on the CTA's maps (map m on CTA m % gridDim.x) as soon as every
// chunk of the map is forecast, then help with the guard's fp64 re-scoring.
constexpr int SEL_NT = 128;                 // guard re-scoring group (tie::NT)
constexpr int SEL_IPT = 8;                  // selection by the whole CTA: rows of <= NT * 8 = 4096 blocks
constexpr int NGRP = NT / SEL_NT;
constexpr int QN = 256;                     // arrival queue: ((map + 1) << 3 | arrivals) events, 1 = end
constexpr int BAR_EPI = 7, BAR_GRP0 = 8;    // named barriers: epilogue warps at the end, select group g
struct RtGroup {  // select group g: threads [128 g, 128 g + 128), named barrier BAR_GRP0 + g
    int g;
    __device__ __forceinline__ int tid() const { return (int)threadIdx.x - g * SEL_NT; }
    __device__ __forceinline__ void sync() const {
        asm volatile("bar.sync %0, %1;" :: "r"(BAR_GRP0 + g), "n"(SEL_NT) : "memory");
    }
};
constexpr int TMEM = 512;
constexpr int ACC_COLS = MO * 32;           // 160
constexpr int PLANE_M = MA * A1C * 16;      // one 8-channel fp16 plane of the a1 tile
static_assert(NA * ACC_COLS <= TMEM, "TMEM budget");

__device__ long long g_trace[64 * 16];  // debug bit 16: CTA 0 timeline of its first 64 bands
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// debug bit 32: per-CTA globaltimer stamps in ws::g_prof[cta * 8 + e] (entry, setup done, producer's last
// band issued, exit) and the CTA's band count
#define WSM_CTA(e, v) \
    if ((dbg & 32) && (threadIdx.x & 31) == 0 && blockIdx.x < 320) ws::g_prof[blockIdx.x * 8 + (e)] = (v);
#define WSM_TRACE(b, e) \
    if ((dbg & 16) && blockIdx.x == 0 && (b) < 64) g_trace[(b) * 16 + (e)] = clock64();

// real a1 rows of the steady-state incremental band: tile row, first output (band index), outputs fed, B block
__host__ __device__ constexpr int STD_R(int i) { return i + 1; }
__host__ __device__ constexpr int STD_O(int i) { return i < 2 ? 0 : i == 2 ? 1 : i < 6 ? 2 : 3; }
__host__ __device__ constexpr int STD_N(int i) { return i == 2 || i == 3 ? 1 : i == 5 ? 3 : 2; }
__host__ __device__ constexpr int STD_B(int i) { return i == 0 ? 1 : i == 3 ? 2 : i == 4 ? 1 : 0; }

struct Meta {  // producer -> conv1 (per x stage) and conv1 -> MMA / epilogue (per a1 stage)
    int valid, map, chunk, W, first, last, full, lo2, base_slot, first_real, aexp;
    int n_out, n_x, n_a1;
    int out_slot[MO];     // ring slot of output row k (segment 0 outputs, then segment 1)
    int x_lim[MX];        // x tile row q: valid columns [0, x_lim) (0: row outside the history / missing)
    int a1_r[MA];         // real a1 rows: tile row, history position, x tile row of position p - 1,
    int a1_p[MA];         //   first output row fed (band index) and how many (1-3), B block of it
    int a1_x[MA];
    int a1_o[MA], a1_n[MA], a1_b[MA];
};

struct EpiInfo {  // MMA issuer -> epilogue (info[] is refilled by conv1 as soon as the MMAs complete)
    int valid, map, chunk, W, first, last, full, lo2, base_slot, aexp, n_out;
    int out_slot[MO];
};

struct EOld {  // conv1 -> epilogue: per column of a task's first band, the running sum and the old r
    double S[TW];      // of the rows the task recomputes (read before any of them is rewritten)
    float osum[TW];
};

struct Smem {
    static constexpr int kB = 2 * 3 * B96_BYTES;
    static constexpr int kA1 = 4 * PLANE_M;
    static constexpr int kX = MX * XC4 * 4;
    static constexpr int off_b = 0;
    static constexpr int off_a1 = off_b + kB;                                   // [NA]
    static constexpr int off_x = off_a1 + NA * kA1;                             // [NX]
    static constexpr int off_meta = off_x + NX * kX;                            // Meta[NX]
    static constexpr int off_info = off_meta + NX * (int)sizeof(Meta);          // Meta[NA] (conv1 -> MMA / epi)
    static constexpr int off_ainfo = off_info + NA * (int)sizeof(Meta);         // EpiInfo[NA]
    static constexpr int off_eold = (off_ainfo + NA * (int)sizeof(EpiInfo) + 15) / 16 * 16;  // EOld[NA]
    // FUSE, after the last band: per select group SelSmem + RefineSmem over the (then idle) a1 tiles
    static constexpr int kSel = ((int)sizeof(SelSmem<NT, SEL_IPT>) + 15) / 16 * 16;
    static constexpr int kGrp = ((int)sizeof(tie::RefineSmem) + 15) / 16 * 16;
    static constexpr int off_grp = off_a1;
    // arrival queue int[QN], tail, head
    static constexpr int off_q = (off_eold + NA * (int)sizeof(EOld) + 15) / 16 * 16;
    static constexpr int off_bar = (off_q + (QN + 4) * 4 + 7) / 8 * 8;
    // x_full[NX], x_empty[NX], a1_full[NA], a1_empty[NA], acc_full[NA], acc_empty[NA], eold_empty[NA], tmem slot
    static constexpr int total = off_bar + 8 * (2 * NX + 5 * NA) + 16;
};

// FUSE: a map is complete after NEPI * n_chunks arrivals — each epilogue warp at a task's last band, the
// producer NEPI at once for a skipped task.  Arrivals are queued in shared memory (CTA-scope release
// only: no device-scope fence on the forecasting warps' path) to the counter warp (warp 13, otherwise
// idle), which drains a batch, publishes it with one device-scope fence and counts it into
// ap_selector.fused_done.  Map m is selected by CTA m % gridDim.x, whose select group waits for the
// map's count (maps complete in task order, so each CTA's one or two maps come due at different times;
// handing a map to whichever CTA counted it last instead piles the maps onto the slowest counters).
__device__ __forceinline__ void ring_push(int* q, int cap, int v) {  // q[cap] = tail, q[cap + 1] = head
    const int slot = atomicAdd(&q[cap], 1);
    while (slot - ld_volatile(&q[cap + 1]) >= cap) __nanosleep(64);
    st_volatile(&q[slot % cap], v);
}
__device__ __forceinline__ void sel_arrive(uint8_t* smem, int map, int n, int dbg) {
    if (!(dbg & 256)) __threadfence_block();  // the arriving warp's score stores before the event
    ring_push(reinterpret_cast<int*>(smem + Smem::off_q), QN, ((map + 1) << 3) | n);
}

// Output rows of band bi of a task: the task's row list is [0, H) (full) or {0, 1} ∪ [lo2, H)
// (incremental), taken MO at a time; a band is one or two contiguous segments.
__device__ __forceinline__ int band_count(int full, int lo2, int H) {
    const int n = full ? H : 2 + H - lo2;
    return (n + MO - 1) / MO;
}
__device__ __forceinline__ void band_segs(int full, int lo2, int H, int bi, int (&so)[2], int (&sn)[2], int& nseg) {
    const int n = full ? H : 2 + H - lo2;
    const int i0 = bi * MO, i1 = min(n, i0 + MO);
    auto pos = [&](int i) { return (full || i < 2) ? i : lo2 + i - 2; };
    if (!full && i0 < 2 && i1 > 2) {
        nseg = 2; so[0] = i0; sn[0] = 2 - i0; so[1] = lo2; sn[1] = i1 - 2;
    } else {
        nseg = 1; so[0] = pos(i0); sn[0] = i1 - i0; so[1] = 0; sn[1] = 0;
    }
}

static_assert(Smem::kSel + NGRP * Smem::kGrp <= NA * Smem::kA1, "select scratch fits the a1 tiles");

template <int PREC, bool FUSE>
__global__ void __launch_bounds__(NT, 1) conv_forecast_wsm_kernel(ConvParams P) {
    extern __shared__ __align__(1024) uint8_t smem[];
    Meta* meta = reinterpret_cast<Meta*>(smem + Smem::off_meta);
    Meta* info = reinterpret_cast<Meta*>(smem + Smem::off_info);
    EpiInfo* ainfo = reinterpret_cast<EpiInfo*>(smem + Smem::off_ainfo);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::off_bar);
    uint64_t* x_full = bars;
    uint64_t* x_empty = bars + NX;
    uint64_t* a1_full = bars + 2 * NX;
    uint64_t* a1_empty = a1_full + NA;
    uint64_t* acc_full = a1_empty + NA;
    uint64_t* acc_empty = acc_full + NA;
    uint64_t* eold_empty = acc_empty + NA;
    EOld* eold = reinterpret_cast<EOld*>(smem + Smem::off_eold);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(eold_empty + NA);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int H = P.H;
    const bool sel = P.state != nullptr;
    const int dbg = P.debug;  // profiling only: 1 no conv1 arithmetic, 2 no MMAs, 4 no epilogue arithmetic,
                              // 64 no accumulator clearing, 128 / 256 no fence at fused arrival counting / queuing
    if (tid == 0) WSM_CTA(0, gtimer());

    {  // B operands once per persistent CTA; barriers; TMEM
        const uint4* src = g_bpack96;
        uint4* dst = reinterpret_cast<uint4*>(smem + Smem::off_b);
        for (int i = tid; i < Smem::kB / 16; i += (int)blockDim.x) dst[i] = src[i];
        if (FUSE)
            for (int i = tid; i < QN + 4; i += (int)blockDim.x) reinterpret_cast<int*>(smem + Smem::off_q)[i] = 0;
        if (tid == 0) {
            for (int s = 0; s < NX; ++s) {
                mbar_init(&x_full[s], 1);
                mbar_init(&x_empty[s], NCONV);
            }
            for (int a = 0; a < NA; ++a) {
                mbar_init(&a1_full[a], NCONV);
                mbar_init(&a1_empty[a], 1);
                mbar_init(&acc_full[a], 2);
                mbar_init(&acc_empty[a], NEPI);
                mbar_init(&eold_empty[a], NEPI);
            }
        }
        if (warp == WARP_PROD) tmem_alloc(tmem_slot, TMEM);
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }
    const uint32_t tmem_base = *tmem_slot;
    if (tid == 0) WSM_CTA(1, gtimer());

    const int role = role_of(warp);
    if (role == R_PROD) {
        // ------------------------------------------------------------------ producer (whole warp)
        const int G = gridDim.x, n_tasks = P.n_maps * P.n_chunks;
        const float b1max = g_b1abs[0], w1max = g_w1abs[0];
        const bool pre_xm = sel && P.slot_xmax && H <= 64;
        int b = 0;
        for (int task0 = blockIdx.x;; task0 += 32 * G) {
            const int t = task0 + lane * G;
            const bool have = t < n_tasks;
            const int map = have ? t / P.n_chunks : 0, chunk = have ? t - map * P.n_chunks : 0;
            ap_map_state st{};
            if (have && P.state) st = P.state[map];
            const Task T = have ? plan_task(P, st, chunk) : Task{true, true, false, 0, 0, 0};
            const bool live = have && !T.skip;
            if (FUSE && have && !live) sel_arrive(smem, map, NEPI, dbg);  // nothing to forecast: the whole count
            const int base_slot = sel ? slot_of(row_index(T.n_pushed, H, 0), H) : 0;
            const int first_real = (!sel || T.n_pushed >= H) ? 0 : (int)(H - T.n_pushed);
            unsigned todo = __ballot_sync(0xffffffffu, live);
            auto load_xm = [&](int mp, float& va, float& vb) {
                const float* src = P.slot_xmax + (int64_t)mp * H;
                va = lane < H ? src[lane] : 0.f;
                vb = lane + 32 < H ? src[lane + 32] : 0.f;
            };
            float ca = 0.f, cb = 0.f;
            if (pre_xm && todo) load_xm(__shfl_sync(0xffffffffu, map, __ffs(todo) - 1), ca, cb);
            while (todo) {
                const int l = __ffs(todo) - 1;
                todo &= todo - 1;
                float na = 0.f, nb_ = 0.f;
                {
                    const int nmap = __shfl_sync(0xffffffffu, map, todo ? __ffs(todo) - 1 : 0);
                    if (pre_xm && todo) load_xm(nmap, na, nb_);
                }
                const int q_map = __shfl_sync(0xffffffffu, map, l), q_chunk = __shfl_sync(0xffffffffu, chunk, l);
                const int q_W = __shfl_sync(0xffffffffu, T.W, l), q_full = __shfl_sync(0xffffffffu, (int)T.full, l);
                const int q_lo2 = __shfl_sync(0xffffffffu, T.lo2, l);
                const int q_base = __shfl_sync(0xffffffffu, base_slot, l);
                const int q_fr = __shfl_sync(0xffffffffu, first_real, l);
                const int nb = band_count(q_full, q_lo2, H);
                const int w0 = q_chunk * TW;
                const int c_lo = max(0, w0 - 4), c_hi = min(P.pitch, w0 + TW + 4);
                const float* ring = P.ring + (int64_t)q_map * P.map_stride;
                int pa = lane - q_base, pb = lane + 32 - q_base;  // history positions of slots lane, lane + 32
                pa += pa < 0 ? H : 0;
                pb += pb < 0 ? H : 0;
                auto slot_p = [&](int p) { return sel ? (q_base + p >= H ? q_base + p - H : q_base + p) : p; };
                for (int bi = 0; bi < nb; ++bi, ++b) {
                    const int s = b % NX;
                    if (b >= NX) mbar_wait(&x_empty[s], ((b / NX) & 1) ^ 1);
                    int so[2], sn[2], nseg;
                    band_segs(q_full, q_lo2, H, bi, so, sn, nseg);
                    const int n_out = sn[0] + sn[1];
                    const int nx0 = sn[0] + 4, n_x = nx0 + (nseg > 1 ? sn[1] + 4 : 0);
                    Meta& m = meta[s];
                    // lane q < n_x: x tile row q (segment k, position so_k - 2 + local row)
                    const int xk = lane < nx0 ? 0 : 1, xq = lane - (xk ? nx0 : 0);
                    const int p = (xk ? so[1] : so[0]) - 2 + xq;
                    const bool xrow = lane < n_x && p >= 0 && p < H && p >= q_fr && c_hi > c_lo;
                    const int slot = slot_p(p);
                    if (lane < MX) m.x_lim[lane] = xrow ? q_W : 0;
                    if (lane < n_out) m.out_slot[lane] = slot_p(lane < sn[0] ? so[0] + lane : so[1] + lane - sn[0]);
                    {   // lane i < MA: a1 tile row i (segment k, position so_k - 1 + local row), real rows compacted
                        const int n_a0 = sn[0] + 2, ak = lane < n_a0 ? 0 : 1, ar = lane - (ak ? n_a0 : 0);
                        const int ao = ak ? so[1] : so[0], an = ak ? sn[1] : sn[0];
                        const int ap = ao - 1 + ar;
                        const bool real = lane < n_a0 + (nseg > 1 ? sn[1] + 2 : 0) && ap >= 0 && ap < H;
                        const unsigned rm = __ballot_sync(0xffffffffu, real);
                        if (real) {
                            const int k = __popc(rm & ((1u << lane) - 1));
                            const int oa = max(ap - 1, ao), ob = min(ap + 1, ao + an - 1);
                            m.a1_r[k] = lane;
                            m.a1_p[k] = ap;
                            m.a1_x[k] = (ak ? nx0 : 0) + ar;  // x tile row of position ap - 1
                            m.a1_o[k] = (ak ? sn[0] : 0) + (oa - ao);
                            m.a1_n[k] = ob - oa + 1;
                            m.a1_b[k] = oa - ap + 1;
                        }
                        if (lane == 0) m.n_a1 = __popc(rm);
                    }
                    const unsigned nrows = __popc(__ballot_sync(0xffffffffu, xrow));
                    if (P.slot_xmax) {  // operand scale from the rows' maxima recorded when they were written
                        float xm;
                        if (pre_xm) {
                            auto in_band = [&](int pp) {
                                bool in = false;
                                for (int k = 0; k < nseg; ++k)
                                    in |= pp >= max(max(so[k] - 2, q_fr), 0) && pp < min(so[k] + sn[k] + 2, H);
                                return in;
                            };
                            xm = (lane < H && in_band(pa)) ? ca : 0.f;
                            if (lane + 32 < H && in_band(pb)) xm = fmaxf(xm, cb);
                        } else {
                            xm = xrow ? P.slot_xmax[(int64_t)q_map * H + slot] : 0.f;
                        }
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) xm = fmaxf(xm, __shfl_xor_sync(0xffffffffu, xm, o));
                        if (lane == 0) m.aexp = f16_scale_exp(fmaf(w1max, xm, b1max));
                    } else if (lane == 0) {
                        m.aexp = 0;  // explicit grids: set by conv1 from a scan of the landed tile
                    }
                    if (lane == 0) {
                        m.valid = 1; m.map = q_map; m.chunk = q_chunk; m.W = q_W;
                        m.first = bi == 0; m.last = bi == nb - 1;
                        m.full = q_full; m.lo2 = q_lo2; m.base_slot = q_base; m.first_real = q_fr;
                        m.n_out = n_out; m.n_x = n_x;
                        mbar_arrive_tx(&x_full[s], nrows * (uint32_t)(c_hi - c_lo) * 4);
                    }
                    __syncwarp();
                    if (xrow)
                        bulk_g2s(reinterpret_cast<float*>(smem + Smem::off_x + s * Smem::kX) + lane * XC4 + (c_lo - (w0 - 4)),
                                 ring + (int64_t)slot * P.pitch + c_lo, (uint32_t)(c_hi - c_lo) * 4, &x_full[s]);
                    if (lane == 0) WSM_TRACE(b, 0);
                }
                ca = na;
                cb = nb_;
            }
            if (task0 + 32 * G >= n_tasks) break;
        }
        if (lane == 0) {
            WSM_CTA(2, gtimer());
            WSM_CTA(4, b);
        }
        {  // end of work: an invalid band tells the consumers to stop
            const int s = b % NX;
            if (b >= NX) mbar_wait(&x_empty[s], ((b / NX) & 1) ^ 1);
            if (lane == 0) {
                meta[s].valid = 0;
                mbar_arrive(&x_full[s]);
            }
        }
    } else if (role == R_MMA) {
        // ------------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t b_addr = smem_u32(smem + Smem::off_b);
            uint64_t bdesc[2][3];
#pragma unroll
            for (int hl = 0; hl < 2; ++hl)
#pragma unroll
                for (int dj = 0; dj < 3; ++dj) bdesc[hl][dj] = umma_desc(b_addr + (hl * 3 + dj) * B96_BYTES, 1536, 128);
            for (int b = 0;; ++b) {
                const int a = b % NA, ph = (b / NA) & 1;
                mbar_wait(&a1_full[a], ph);
                const Meta& I = info[a];
                mbar_wait(&acc_empty[a], ph);  // phase 0: the epilogue's start-up arrive (columns cleared)
                EpiInfo& E = ainfo[a];  // free: the epilogue finished band b - NA
                E.valid = I.valid;
                if (!I.valid) {
                    mbar_arrive(&acc_full[a]);
                    mbar_arrive(&acc_full[a]);
                    break;
                }
                E.map = I.map; E.chunk = I.chunk; E.W = I.W; E.first = I.first; E.last = I.last; E.full = I.full;
                E.lo2 = I.lo2; E.base_slot = I.base_slot; E.aexp = I.aexp; E.n_out = I.n_out;
                for (int k = 0; k < MO; ++k) E.out_slot[k] = I.out_slot[k];
                tc_fence_after();
                WSM_TRACE(b, 4);
                const uint32_t a1_addr = smem_u32(smem + Smem::off_a1 + a * Smem::kA1);
                const uint32_t d0 = tmem_base + a * ACC_COLS;
                // The steady-state incremental band (one new history row: outputs {0, 1} | {H-3, H-1}) always
                // has the same 7-row schedule; issuing it from a compile-time table keeps the single MMA
                // thread to a few instructions per MMA (descriptor = base + constant), which is what paced
                // the band: the generic loop spent ~75 cycles per MMA against a ~48-cycle tensor-pipe floor.
                bool std_band = I.n_a1 == 7 && !(dbg & 2);
#pragma unroll
                for (int i = 0; i < 7; ++i)
                    std_band = std_band && I.a1_r[i] == STD_R(i) && I.a1_o[i] == STD_O(i) && I.a1_n[i] == STD_N(i) &&
                               I.a1_b[i] == STD_B(i);
                if (std_band) {
                    const uint64_t A0 = umma_desc(a1_addr, PLANE_M, 128);
                    const uint64_t AL = A0 + (uint64_t)((2 * PLANE_M) >> 4);
#pragma unroll
                    for (int i = 0; i < 7; ++i) {
                        const uint32_t d = d0 + STD_O(i) * 32;
                        const uint32_t idesc = idesc_f16_f32(TW, 32 * STD_N(i), 0);
                        const uint64_t boff = (uint64_t)(STD_B(i) * 32);
#pragma unroll
                        for (int dj = 0; dj < 3; ++dj) {
                            const uint64_t off = (uint64_t)(STD_R(i) * A1C + dj);  // pixel (16-byte) units
                            if constexpr (PREC == AP_PREC_F16X3) {
                                mma_f16_afill(d, A0 + off, bdesc[0][dj] + boff, idesc, 1);
                                mma_f16_alast(d, A0 + off, bdesc[1][dj] + boff, idesc, 1);
                                mma_f16(d, AL + off, bdesc[0][dj] + boff, idesc, 1);
                            } else {
                                mma_f16(d, A0 + off, bdesc[0][dj] + boff, idesc, 1);
                            }
                        }
                    }
                }
                for (int i = 0; i < ((dbg & 2) || std_band ? 0 : I.n_a1); ++i) {
                    const uint32_t d = d0 + I.a1_o[i] * 32;
                    const uint32_t idesc = idesc_f16_f32(TW, 32 * I.a1_n[i], 0);
                    const uint64_t boff = (uint64_t)((I.a1_b[i] * 32 * 16) >> 4);
                    const int r = I.a1_r[i];
#pragma unroll
                    for (int dj = 0; dj < 3; ++dj) {
                        const uint32_t pix = (uint32_t)(r * A1C + dj) * 16;
                        const uint64_t a_hi = umma_desc(a1_addr + pix, PLANE_M, 128);
                        if constexpr (PREC == AP_PREC_F16X3) {
                            // a_hi feeds two MMAs: read its tile once, keep it in the A collector
                            const uint64_t a_lo = umma_desc(a1_addr + 2 * PLANE_M + pix, PLANE_M, 128);
                            mma_f16_afill(d, a_hi, bdesc[0][dj] + boff, idesc, 1);
                            mma_f16_alast(d, a_hi, bdesc[1][dj] + boff, idesc, 1);
                            mma_f16(d, a_lo, bdesc[0][dj] + boff, idesc, 1);
                        } else {
                            mma_f16(d, a_hi, bdesc[0][dj] + boff, idesc, 1);
                        }
                    }
                }
                WSM_TRACE(b, 5);
                mma_commit(&a1_empty[a]);   // a1 tile consumed -> conv1 may refill it
                mma_commit(&acc_full[a]);   // accumulators ready
                mbar_arrive(&acc_full[a]);  // releases info[a] to the epilogue
            }
        }
    } else if (role == R_EPI) {
        // ------------------------------------------------------------------ epilogue
        const int quad = warp & 3, pix = quad * 32 + lane;
        const int wexp = g_wexp;
        const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16);
        for (int c = 0; c < NA * ACC_COLS; c += 32) tmem_zero32(lane_base + c);  // accumulate-only MMAs
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0)
            for (int a = 0; a < NA; ++a) {
                mbar_arrive(&acc_empty[a]);
                mbar_arrive(&eold_empty[a]);
            }
        double S = 0.0, Snew = 0.0;
        float osum = 0.f;
        for (int b = 0;; ++b) {
            const int a = b % NA, ph = (b / NA) & 1;
            mbar_wait(&acc_full[a], ph);
            const EpiInfo& I = ainfo[a];
            if (!I.valid) break;
            if (warp == EPI0 && lane == 0) WSM_TRACE(b, 6);
            tc_fence_after();
            const int W = I.W, col = I.chunk * TW + pix;
            const bool live = col < W;
            float* rmap = P.rmap + (int64_t)I.map * P.map_stride + col;
            const int64_t at = (int64_t)I.map * P.pitch + col;
            if (I.first) {  // the task's old running sum / old r of its recomputed rows, gathered by conv1
                S = (I.full || !P.rsum || !live) ? 0.0 : eold[a].S[pix];
                osum = (I.full || !live) ? 0.f : eold[a].osum[pix];
                Snew = 0.0;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&eold_empty[a]);
            {
                const int e = I.aexp + wexp;
                const bool one_mul = e >= -126 && e <= 126;
                const float u = one_mul ? pow2f(-e) : pow2f(-I.aexp), u2 = one_mul ? 1.f : pow2f(-wexp);
                const uint32_t t0 = lane_base + a * ACC_COLS;
                float bsum = 0.f;
                const int n_out = (dbg & 4) ? 0 : I.n_out;
                uint32_t ra[16], rb[16];
                tmem_ld16_start(t0, ra);
                for (int k = 0; k < n_out; ++k) {
                    tmem_ld16_start(t0 + k * 32 + 16, rb);
                    tmem_ld_wait(ra);
                    tmem_ld_wait(rb);
                    if (k == 0 && warp == EPI0 && lane == 0) WSM_TRACE(b, 8);
                    if (!one_mul) {  // scale too extreme for one multiply (never for attention rows)
#pragma unroll
                        for (int n = 0; n < 16; ++n) {
                            ra[n] = __float_as_uint(__uint_as_float(ra[n]) * u2);
                            rb[n] = __float_as_uint(__uint_as_float(rb[n]) * u2);
                        }
                    }
                    // r = sum_c w3[c] relu(acc[c] * u + b2[c]), channel pairs on the packed FMA pipe
                    float r0 = 0.f, r1 = 0.f;
#pragma unroll
                    for (int n = 0; n < 16; n += 2) {
                        float s0 = c_w[OFF_B2 + n], s1 = c_w[OFF_B2 + n + 1];
                        ffma2(s0, s1, __uint_as_float(ra[n]), __uint_as_float(ra[n + 1]), u);
                        ffma2v(r0, r1, fmaxf(s0, 0.f), fmaxf(s1, 0.f), c_w[OFF_W3 + n], c_w[OFF_W3 + n + 1]);
                    }
                    if (k + 1 < n_out) tmem_ld16_start(t0 + (k + 1) * 32, ra);  // next row's first half
#pragma unroll
                    for (int n = 0; n < 16; n += 2) {
                        float s0 = c_w[OFF_B2 + 16 + n], s1 = c_w[OFF_B2 + 16 + n + 1];
                        ffma2(s0, s1, __uint_as_float(rb[n]), __uint_as_float(rb[n + 1]), u);
                        ffma2v(r0, r1, fmaxf(s0, 0.f), fmaxf(s1, 0.f), c_w[OFF_W3 + 16 + n], c_w[OFF_W3 + 16 + n + 1]);
                    }
                    const float r = r0 + r1;
                    if (live) {
                        rmap[(int64_t)I.out_slot[k] * P.pitch] = r;
                        bsum += r;
                    }
                }
                if (n_out > 0) tmem_ld_wait(ra);
                if (warp == EPI0 && lane == 0) WSM_TRACE(b, 9);
                for (int k = 0; k < ((dbg & 64) ? 0 : n_out); ++k) tmem_zero32(t0 + k * 32);  // cleared for the next band
                Snew += (double)bsum;
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            const bool last = I.last;
            const int mapi = I.map;
            const int64_t sat = (int64_t)I.map * P.score_stride + col;
            if (warp == EPI0 && lane == 0) WSM_TRACE(b, 7);
            __syncwarp();  // every lane has read ainfo[a]: the MMA issuer refills it once all four warps arrive
            if (lane == 0) mbar_arrive(&acc_empty[a]);  // (ainfo[a] is not read after this)
            if (last && live) {
                S += Snew - (double)osum;
                if (P.rsum) P.rsum[at] = S;
                P.scores[sat] = c_w[OFF_B3] + (float)S / (float)H;
            }
            if (FUSE && last) {
                __syncwarp();
                if (lane == 0) sel_arrive(smem, mapi, 1, dbg);
            }
        }
        if (FUSE) {  // every epilogue warp's arrivals are in: no more maps complete in this CTA
            asm volatile("bar.sync %0, %1;" :: "n"(BAR_EPI), "n"(NEPI * 32) : "memory");
            if (warp == EPI0 && lane == 0) ring_push(reinterpret_cast<int*>(smem + Smem::off_q), QN, 1);
        }
    } else if (FUSE && role == R_IDLE) {
        // ------------------------------------------------------------------ arrival counter (warp 13, lane 0)
        if (lane == 0) {
            int* q = reinterpret_cast<int*>(smem + Smem::off_q);
            int head = 0;
            bool end = false;
            while (!end) {
                int evs[16], n_ev = 0, v;
                while (n_ev < 16 && (v = ld_volatile(&q[head % QN])) != 0) {
                    st_volatile(&q[head % QN], 0);
                    ++head;
                    evs[n_ev++] = v;
                }
                if (!n_ev) {
                    __nanosleep(AP_CNT_SLEEP);  // rarely: this warp shares a scheduler with the MMA issuer
                    continue;
                }
                st_volatile(&q[QN + 1], head);
                if (!(dbg & 128)) __threadfence();  // the arrivals' score stores (CTA-ordered before the events) before the counts
                for (int i = 0; i < n_ev; ++i) {
                    if (evs[i] == 1) end = true;
                    else atomicAdd(&P.sel.fused_done[(evs[i] >> 3) - 1], evs[i] & 7);
                }
            }
        }
    } else if (role == R_CONV) {
        // ------------------------------------------------------------------ conv1 workers
        const int ct = conv_rank(warp) * 32 + lane;
        const int cw = ct >> 5;
        for (int b = 0;; ++b) {
            const int s = b % NX, a = b % NA;
            mbar_wait(&x_full[s], (b / NX) & 1);  // tile landed
            Meta& m = meta[s];
            if (!m.valid) {
                if (b >= NA) mbar_wait(&a1_empty[a], ((b / NA) & 1) ^ 1);
                if (ct == 0) info[a].valid = 0;
                __syncwarp();
                if (lane == 0) mbar_arrive(&a1_full[a]);
                break;
            }
            const float* xs = reinterpret_cast<const float*>(smem + Smem::off_x + s * Smem::kX);
            const int W = m.W, w0 = m.chunk * TW;
            if (!P.slot_xmax) {  // explicit grids: operand scale from max|x| over the landed tile (+ finiteness)
                float xmax = 0.f;
                bool bad = false;
                const int cbase = w0 - 4;
                for (int i = ct; i < m.n_x * (XC4 / 4); i += NCONV_T) {
                    const int q = i / (XC4 / 4), k = i - q * (XC4 / 4);
                    const int lim = m.x_lim[q];
                    const float4 v = reinterpret_cast<const float4*>(xs + q * XC4)[k];
                    const float e4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int xc = 4 * k + u, c = cbase + xc;
                        if (xc >= 2 && xc < TW + 6 && (unsigned)c < (unsigned)lim) {
                            bad |= !(fabsf(e4[u]) <= 3.402823466e38f);
                            xmax = fmaxf(xmax, fabsf(e4[u]));
                        }
                    }
                }
                if (__any_sync(0xffffffffu, bad) && lane == 0) raise_status(P.status, AP_ENUMERIC);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) xmax = fmaxf(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
                // the ten conv1 warps agree through an atomic max in the metadata, then a named barrier
                if (lane == 0 && xmax > 0.f) atomicMax(reinterpret_cast<int*>(&m.aexp), __float_as_int(xmax));
                asm volatile("bar.sync 1, %0;" :: "r"(NCONV_T) : "memory");
                const float xm = __int_as_float(*reinterpret_cast<volatile int*>(&m.aexp));
                asm volatile("bar.sync 1, %0;" :: "r"(NCONV_T) : "memory");  // everyone read it
                if (ct == 0) m.aexp = f16_scale_exp(fmaf(g_w1abs[0], xm, g_b1abs[0]));
                asm volatile("bar.sync 1, %0;" :: "r"(NCONV_T) : "memory");
            }
            const int aexp = m.aexp;
            const float ascale = pow2f(aexp);
            if (ct == 0) WSM_TRACE(b, 1);
            // first band of an incremental task: old running sum and old r of the rows it rewrites,
            // one column per thread (loads issued now, stored after the a1 tile)
            const bool gather = m.first && !m.full && ct < TW && w0 + ct < W;
            double g_S = 0.0;
            float g_os = 0.f, ov[8];  // loads issued now, summed after the a1 tile (latency under conv1)
            int n_old = 0;
            if (gather) {
                const int col = w0 + ct;
                const float* rm = P.rmap + (int64_t)m.map * P.map_stride + col;
                if (P.rsum) g_S = __ldcg(P.rsum + (int64_t)m.map * P.pitch + col);
                n_old = 2 + H - m.lo2;  // positions {0, 1} ∪ [lo2, H)
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int pp = k < 2 ? k : m.lo2 + k - 2;
                    int sl = sel ? m.base_slot + pp : pp;
                    sl = sl >= H ? sl - H : sl;
                    ov[k] = k < n_old ? __ldcg(rm + (int64_t)sl * P.pitch) : 0.f;
                }
            }
            if (b >= NA) mbar_wait(&a1_empty[a], ((b / NA) & 1) ^ 1);
            if (ct == 0) WSM_TRACE(b, 2);
            uint8_t* a1t = smem + Smem::off_a1 + a * Smem::kA1;
            // Two a1 pixels per thread, HALF apart (packed FFMA2), real a1 rows only: consecutive lanes own
            // consecutive pixels, so every 16-byte tile store of a warp is one contiguous 512-byte run and
            // every x load one contiguous 128-byte run (adjacent pixel pairs per thread cost twice the
            // shared-memory wavefronts, and the port is what this kernel is bound by alongside the MMAs)
            constexpr int HALF = A1C / 2;
            const int n_items = (dbg & 1) ? 0 : m.n_a1 * HALF;
            for (int i = ct; i < n_items; i += NCONV_T) {
                const int rr = i / HALF, ac = i - rr * HALF;
                const int ar = m.a1_r[rr], xb = m.a1_x[rr];
                const int c = w0 - 1 + ac;  // pixel columns c, c + HALF
                float xw[3][3], xv[3][3];
#pragma unroll
                for (int di = 0; di < 3; ++di) {
                    const int lim = m.x_lim[xb + di];
                    const float* xr = xs + (xb + di) * XC4 + ac + 2;
#pragma unroll
                    for (int e = 0; e < 3; ++e) {
                        xw[di][e] = ((unsigned)(c - 1 + e) < (unsigned)lim) ? xr[e] : 0.f;
                        xv[di][e] = ((unsigned)(c + HALF - 1 + e) < (unsigned)lim) ? xr[HALF + e] : 0.f;
                    }
                }
                // pixels outside [0, W) are conv2's zero padding: a zero scale clears them
                const float sc0 = (unsigned)c < (unsigned)W ? ascale : 0.f;
                const float sc1 = (unsigned)(c + HALF) < (unsigned)W ? ascale : 0.f;
                const int px = ar * A1C + ac;
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                    float v0[8], v1[8];  // scaled relu(a1) of pixels c, c+1, channels 8g ..
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int ch = g * 8 + q;
                        float s0 = c_w[OFF_B1 + ch], s1 = s0;
#pragma unroll
                        for (int k = 0; k < 9; ++k)
                            ffma2(s0, s1, xw[k / 3][k % 3], xv[k / 3][k % 3], c_w[OFF_W1 + ch * 9 + k]);
                        v0[q] = fmaxf(s0 * sc0, 0.f);  // relu(s) * 2^aexp (scale > 0, exact)
                        v1[q] = fmaxf(s1 * sc1, 0.f);
                    }
                    uint4 h0, l0, h1, l1;
                    if constexpr (PREC == AP_PREC_F16X3) {
                        split_f16x2(v0[0], v0[1], h0.x, l0.x); split_f16x2(v0[2], v0[3], h0.y, l0.y);
                        split_f16x2(v0[4], v0[5], h0.z, l0.z); split_f16x2(v0[6], v0[7], h0.w, l0.w);
                        split_f16x2(v1[0], v1[1], h1.x, l1.x); split_f16x2(v1[2], v1[3], h1.y, l1.y);
                        split_f16x2(v1[4], v1[5], h1.z, l1.z); split_f16x2(v1[6], v1[7], h1.w, l1.w);
                    } else {  // single fp16 operand: round to nearest
                        h0 = make_uint4(pack_f16x2(v0[0], v0[1]), pack_f16x2(v0[2], v0[3]), pack_f16x2(v0[4], v0[5]),
                                        pack_f16x2(v0[6], v0[7]));
                        h1 = make_uint4(pack_f16x2(v1[0], v1[1]), pack_f16x2(v1[2], v1[3]), pack_f16x2(v1[4], v1[5]),
                                        pack_f16x2(v1[6], v1[7]));
                    }
                    *reinterpret_cast<uint4*>(a1t + g * PLANE_M + px * 16) = h0;
                    *reinterpret_cast<uint4*>(a1t + g * PLANE_M + (px + HALF) * 16) = h1;
                    if constexpr (PREC == AP_PREC_F16X3) {
                        *reinterpret_cast<uint4*>(a1t + (2 + g) * PLANE_M + px * 16) = l0;
                        *reinterpret_cast<uint4*>(a1t + (2 + g) * PLANE_M + (px + HALF) * 16) = l1;
                    }
                }
            }
            if (gather) {
#pragma unroll
                for (int k = 0; k < 8; ++k) g_os += ov[k];
                const float* rm = P.rmap + (int64_t)m.map * P.map_stride + w0 + ct;
                for (int k = 8; k < n_old; ++k) {  // more than 6 new rows since the last update (rare)
                    const int pp = m.lo2 + k - 2;
                    int sl = sel ? m.base_slot + pp : pp;
                    sl = sl >= H ? sl - H : sl;
                    g_os += __ldcg(rm + (int64_t)sl * P.pitch);
                }
            }
            mbar_wait(&eold_empty[a], (b / NA) & 1);  // completion 0 = start-up; then the epilogue read band b - NA's
            if (gather) {
                eold[a].S[ct] = g_S;
                eold[a].osum[ct] = g_os;
            }
            // metadata for the MMA issuer / epilogue (the x stage is released below)
            {
                const int* src = reinterpret_cast<const int*>(&m);
                int* dst = reinterpret_cast<int*>(&info[a]);
                for (int i = ct; i < (int)(sizeof(Meta) / 4); i += NCONV_T) dst[i] = src[i];
            }
            fence_async_smem();  // a1 tile -> visible to the tensor core's async proxy
            __syncwarp();
            if (ct == 0) WSM_TRACE(b, 3);
            if (lane == 0) {
                mbar_arrive(&a1_full[a]);
                mbar_arrive(&x_empty[s]);
            }
            (void)cw;
        }
    }

    if (FUSE) {
        // ------------------------------------------------------------------ selection (kernel 3)
        // this CTA has no more bands: the whole CTA selects maps blockIdx.x + j * gridDim.x, each once all
        // its chunks' arrivals are counted; then groups of four warps help with the guard's re-scoring
        auto& sh = *reinterpret_cast<SelSmem<NT, SEL_IPT>*>(smem + Smem::off_grp);
        const RtGroup grp{warp / 4};
        const int gt = grp.tid();
        auto& rs = *reinterpret_cast<tie::RefineSmem*>(smem + Smem::off_grp + Smem::kSel + grp.g * Smem::kGrp);
        const int target = NEPI * P.n_chunks;
        __syncthreads();  // every role is done (the last MMAs too): the a1 tiles are free for the scratch
        if (tid == 0) WSM_CTA(5, gtimer());
        for (int m = blockIdx.x; m < P.n_maps; m += gridDim.x) {
            if (tid == 0) {
                while (ld_volatile(&P.sel.fused_done[m]) != target) __nanosleep(128);
                __threadfence();  // every chunk's scores before the selection reads them
            }
            __syncthreads();
            select_map<NT, SEL_IPT>(P.sel, P.tp, m, CtaGroup{}, sh);
            if (tid == 0) P.sel.fused_done[m] = 0;  // every arrival of this launch is in: reset for the next
        }
        if (tid == 0) WSM_CTA(6, gtimer());
        int* ws = P.sel.tie_ws;
        if (P.tp.enabled && ws) {
            // exact-boundary guard: fp64 re-scoring units of every CTA's maps, taken from the shared list as
            // they appear, until all CTAs have selected all their maps and the list is drained
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                atomicAdd(&ws[tie::H_SELDONE], 1);
            }
            for (;;) {
                if (gt == 0) {
                    const int u = atomicAdd(&ws[tie::H_NEXT], 1);
                    int val = 0;
                    for (;;) {
                        const int done = ld_volatile(&ws[tie::H_SELDONE]);
                        __threadfence();
                        if (u < ld_volatile(&ws[tie::H_UNITS])) {
                            while ((val = ld_volatile(&ws[tie::HDR + u])) == 0) __nanosleep(32);
                            st_volatile(&ws[tie::HDR + u], 0);
                            break;
                        }
                        if (done == (int)gridDim.x) break;  // the list is final and u is past its end
                        __nanosleep(256);
                    }
                    rs.val = val - 1;
                }
                grp.sync();
                const int unit = rs.val;
                if (unit < 0) break;
                __threadfence();
                tie::refine_unit(P.sel, P.tp, unit, rs.sx, rs.sa1, rs.srow, rs.flags, rs.scan_tmp, &rs.last, grp);
            }
            __syncthreads();
            if (tid == 0) {  // the last CTA out resets the work list for the next step
                __threadfence();
                if (atomicAdd(&ws[tie::H_DONE], 1) == (int)gridDim.x - 1) {
                    ws[tie::H_UNITS] = 0;
                    ws[tie::H_NEXT] = 0;
                    ws[tie::H_DONE] = 0;
                    ws[tie::H_SELDONE] = 0;
                    __threadfence();
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) WSM_CTA(3, gtimer());
    if (warp == WARP_PROD) tmem_dealloc(tmem_base, TMEM);
}

}  // namespace wsm
}  // namespace ap
