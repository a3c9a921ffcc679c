// Warp-specialised forecaster kernel (tensor-core precisions) — included by predictor.cu
// after the shared definitions (weights in constant memory, packed B tiles, task
// planning, band geometry).
//
// One CTA (16 warps) per SM, persistent over (map, 128-column chunk) tasks; each
// task is processed as bands of <= MAXO history rows.  Roles, connected by
// mbarrier handshakes so no role ever waits on a CTA-wide barrier:
//   warp 0      producer (whole warp): plans 32 tasks at a time (map state loads in
//               parallel), publishes band metadata and starts lane-parallel
//               cp.async.bulk copies of the band's history rows into an x ring; the
//               fp16 operand scale comes from the per-slot row maxima the ring
//               writers recorded (selector mode) or from a scan of the landed tile
//               two bands behind (explicit grids);
//   warp 1      MMA: per band, tcgen05.cp the dj-shifted a1 windows into the TMEM
//               ring and issues the conv2 MMAs (A from TMEM) into one of two TMEM
//               accumulator buffers; commits release the a1 tile and publish the
//               accumulators;
//   warps 2-5   epilogue (one per TMEM lane quadrant, lane = column): bias, ReLU,
//               w3 dot -> r, r-map store, running-sum update S += r_new - r_old,
//               and at the end of a task the chunk forecast b3 + S / H;
//   warps 6-15  conv1 (FMA pipe) + fp16 hi/lo split into a double-buffered a1 tile.
// Band b's MMAs overlap band b+1's conv1 and band b-1's epilogue.
#pragma once

namespace ap {
namespace ws {

__device__ unsigned long long g_prof[16 * 160];  // debug bit 8: per-CTA cycle counters per role phase
__device__ long long g_trace[64 * 8];             // debug bit 16: CTA 0 timeline of its first 64 bands
#define WS_TRACE(b, e) if ((dbg & 16) && blockIdx.x == 0 && (b) < 64) g_trace[(b) * 8 + (e)] = clock64();

constexpr int NT = 512;
constexpr int NX = 6;                       // x tile stages
constexpr int SCAN_LAG = 2;                 // the producer scans band b - SCAN_LAG after issuing band b
constexpr int NA = 2;                       // a1 tile / accumulator stages
constexpr int WARP_PROD = 0, WARP_MMA = 1, EPI0 = 2, NEPI = 4, CONV0 = 6, NCONV = 10;
constexpr int NCONV_T = NCONV * 32;
constexpr int TMEM = 512;
// Accumulator window per band: output positions o0-2 .. o0+n_out+1 (slot q = o - (o0-2)); a1 row ar
// (position o0-1+ar) feeds slots ar, ar+1, ar+2 through one N=96 MMA per (dj, term).  Real outputs
// are slots 2 .. n_out+1; the edge slots collect partial sums of rows outside the band (ignored).
constexpr int NSLOT = MAXO + 4;
constexpr int ACC_COLS = NSLOT * 32;        // 224
static_assert(NA * ACC_COLS <= TMEM, "TMEM budget");

struct BandInfo {  // conv1 -> MMA -> epilogue
    int valid, map, chunk, W, first, last, full, lo2, base_slot, first_real, o0, n_out, aexp;
    int out_slot[MAXO];
};

template <int PREC>
struct Smem {
    static constexpr int kB = 2 * 3 * B96_BYTES;
    static constexpr int kA1 = 4 * PLANE;
    static constexpr int kX = MAXX * XC4 * 4;
    static constexpr int off_b = 0;
    static constexpr int off_a1 = off_b + kB;                                   // [NA]
    static constexpr int off_x = off_a1 + NA * kA1;                             // [NX]
    static constexpr int off_meta = off_x + NX * kX;                            // BandMeta[NX]
    static constexpr int off_info = (off_meta + NX * (int)sizeof(BandMeta) + 15) / 16 * 16;   // BandInfo[NA] (conv1)
    static constexpr int off_ainfo = off_info + NA * (int)sizeof(BandInfo);     // BandInfo[NA] (accumulators)
    static constexpr int off_bar = (off_ainfo + NA * (int)sizeof(BandInfo) + 15) / 16 * 16;
    // mbarriers: x_full[NX], x_ready[NX], x_empty[NX], a1_full[NA], a1_empty[NA], acc_full[NA], acc_empty[NA]
    static constexpr int total = off_bar + 8 * (3 * NX + 4 * NA) + 16;
};


template <int PREC>
__global__ void __launch_bounds__(NT, 1) conv_forecast_ws_kernel(ConvParams P) {
    using L = Smem<PREC>;
    extern __shared__ __align__(1024) uint8_t smem[];
    BandMeta* meta = reinterpret_cast<BandMeta*>(smem + L::off_meta);
    BandInfo* info = reinterpret_cast<BandInfo*>(smem + L::off_info);
    BandInfo* ainfo = reinterpret_cast<BandInfo*>(smem + L::off_ainfo);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::off_bar);
    uint64_t* x_full = bars;            // bulk copies landed (producer)
    uint64_t* x_ready = bars + NX;      // tile scanned, operand scale published (conv1)
    uint64_t* x_empty = bars + 2 * NX;
    uint64_t* a1_full = bars + 3 * NX;
    uint64_t* a1_empty = a1_full + NA;
    uint64_t* acc_full = a1_empty + NA;
    uint64_t* acc_empty = acc_full + NA;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * NX + 4 * NA);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int H = P.H;
    const bool sel = P.state != nullptr;
    const int dbg = P.debug;

    {  // B operands once per persistent CTA; barriers; TMEM
        const uint4* src = g_bpack96;
        uint4* dst = reinterpret_cast<uint4*>(smem + L::off_b);
        for (int i = tid; i < L::kB / 16; i += NT) dst[i] = src[i];
        if (tid == 0) {
            for (int s = 0; s < NX; ++s) {
                mbar_init(&x_full[s], 1);
                mbar_init(&x_ready[s], 1);
                mbar_init(&x_empty[s], NCONV);
            }
            for (int a = 0; a < NA; ++a) {
                mbar_init(&a1_full[a], NCONV);
                mbar_init(&a1_empty[a], 1);
                mbar_init(&acc_full[a], 2);
                mbar_init(&acc_empty[a], NEPI);
            }
        }
        if (warp == WARP_PROD) tmem_alloc(tmem_slot, TMEM);
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }
    const uint32_t tmem_base = *tmem_slot;

    if (warp == WARP_PROD) {
        // ------------------------------------------------------------------ producer (whole warp)
        // Lane l plans task task0 + l*G of this CTA's strided work list (map state loads and task
        // planning for 32 tasks in parallel); the warp then walks the live tasks in order, and for
        // each band lane 0 publishes the metadata while lane q starts the bulk copy of x row q.
        const int G = gridDim.x, n_tasks = P.n_maps * P.n_chunks;
        const float b1max = g_b1abs[0], w1max = g_w1abs[0];
        unsigned long long t_wait = 0, t_plan = 0, t_scan = 0;
        // Band j's copies have landed: max|x| over its conv input window (+ finiteness check) ->
        // the fp16 operand scale of its a1 tile, then release it to conv1.  Runs one band behind
        // the copies so the bulk-copy latency is hidden.
        auto finalize = [&](int j) {
            long long f0 = clock64();
            const int s = j % NX;
            mbar_wait(&x_full[s], (j / NX) & 1);
            BandMeta& m = meta[s];
            const float* xs = reinterpret_cast<const float*>(smem + L::off_x + s * L::kX);
            const int n_x = m.n_out + 4, cbase = m.chunk * TW - 4;
            float xmax = 0.f;
            bool bad = false;
            for (int i = lane; i < n_x * (XC4 / 4); i += 32) {  // float4 i: row q, tile columns [4k, 4k+4)
                const int q = i / (XC4 / 4), k = i - q * (XC4 / 4);
                const int lim = m.x_lim[q];
                const float4 v = reinterpret_cast<const float4*>(xs + q * XC4)[k];
                const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int xc = 4 * k + u, c = cbase + xc;
                    if (xc >= 2 && xc < TW + 6 && (unsigned)c < (unsigned)lim) {
                        bad |= !(fabsf(e[u]) <= 3.402823466e38f);  // NaN or inf
                        xmax = fmaxf(xmax, fabsf(e[u]));
                    }
                }
            }
            if (__any_sync(0xffffffffu, bad) && lane == 0) raise_status(P.status, AP_ENUMERIC);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) xmax = fmaxf(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
            if (lane == 0) {
                m.aexp = f16_scale_exp(fmaf(w1max, xmax, b1max));
                mbar_arrive(&x_ready[s]);
            }
            __syncwarp();
            t_scan += clock64() - f0;
        };
        const bool pre_xm = sel && P.slot_xmax && H <= 64;
        int b = 0;
        for (int task0 = blockIdx.x;; task0 += 32 * G) {
            long long tp0 = clock64();
            const int t = task0 + lane * G;
            const bool have = t < n_tasks;
            const int map = have ? t / P.n_chunks : 0, chunk = have ? t - map * P.n_chunks : 0;
            ap_map_state st{};
            if (have && P.state) st = P.state[map];
            const Task T = have ? plan_task(P, st, chunk) : Task{true, true, false, 0, 0, 0};
            const bool live = have && !T.skip;
            const int base_slot = sel ? slot_of(row_index(T.n_pushed, H, 0), H) : 0;
            const int first_real = (!sel || T.n_pushed >= H) ? 0 : (int)(H - T.n_pushed);
            unsigned todo = __ballot_sync(0xffffffffu, live);
            // Row maxima of a task's map (H <= 64: lane l holds slots l and l + 32), loaded one task
            // ahead so no band waits on global memory for its operand scale.
            auto load_xm = [&](int mp, float& va, float& vb) {
                const float* src = P.slot_xmax + (int64_t)mp * H;
                va = lane < H ? src[lane] : 0.f;
                vb = lane + 32 < H ? src[lane + 32] : 0.f;
            };
            float ca = 0.f, cb = 0.f;
            if (pre_xm && todo) load_xm(__shfl_sync(0xffffffffu, map, __ffs(todo) - 1), ca, cb);
            t_plan += clock64() - tp0;
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
                // bands: [0, rb0) in MAXO-row pieces, then (incremental) [lo2, H)  (band_of order)
                const int rb0 = q_full ? H : 2, nb0 = (rb0 + MAXO - 1) / MAXO;
                const int nb = nb0 + (q_full ? 0 : (H - q_lo2 + MAXO - 1) / MAXO);
                const int w0 = q_chunk * TW;
                const int c_lo = max(0, w0 - 4), c_hi = min(P.pitch, w0 + TW + 4);
                const float* ring = P.ring + (int64_t)q_map * P.map_stride;
                int pa = lane - q_base, pb = lane + 32 - q_base;  // history positions of slots lane, lane + 32
                pa += pa < 0 ? H : 0;
                pb += pb < 0 ? H : 0;
                for (int bi = 0; bi < nb; ++bi, ++b) {
                    const int s = b % NX;
                    long long t0 = clock64();
                    if (b >= NX) mbar_wait(&x_empty[s], ((b / NX) & 1) ^ 1);
                    long long t1 = clock64();
                    int o0, o1;
                    if (bi < nb0) { o0 = bi * MAXO; o1 = min(rb0, o0 + MAXO); }
                    else { o0 = q_lo2 + (bi - nb0) * MAXO; o1 = min(H, o0 + MAXO); }
                    const int n_out = o1 - o0;
                    BandMeta& m = meta[s];
                    // lane q < n_out + 4: x row q (position o0 - 2 + q)
                    const int p = o0 - 2 + lane;
                    const bool xrow = lane < n_out + 4 && p >= 0 && p < H && p >= q_fr && c_hi > c_lo;
                    const int slot = sel ? (q_base + p >= H ? q_base + p - H : q_base + p) : p;
                    if (lane < MAXX) m.x_lim[lane] = xrow ? q_W : 0;
                    if (lane < MAXO) m.out_slot[lane] = sel ? (q_base + o0 + lane >= H ? q_base + o0 + lane - H
                                                                                       : q_base + o0 + lane)
                                                            : o0 + lane;
                    const unsigned nrows = __popc(__ballot_sync(0xffffffffu, xrow));
                    if (P.slot_xmax) {  // operand scale from the rows' maxima recorded when they were written
                        float xm;
                        if (pre_xm) {
                            const int plo = max(max(o0 - 2, q_fr), 0), phi = min(o0 + n_out + 2, H);
                            xm = (lane < H && pa >= plo && pa < phi) ? ca : 0.f;
                            if (lane + 32 < H && pb >= plo && pb < phi) xm = fmaxf(xm, cb);
                        } else {
                            xm = xrow ? P.slot_xmax[(int64_t)q_map * H + slot] : 0.f;
                        }
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) xm = fmaxf(xm, __shfl_xor_sync(0xffffffffu, xm, o));
                        if (lane == 0) m.aexp = f16_scale_exp(fmaf(w1max, xm, b1max));
                    }
                    if (lane == 0) {
                        m.valid = 1; m.map = q_map; m.chunk = q_chunk; m.W = q_W;
                        m.first = bi == 0; m.last = bi == nb - 1;
                        m.full = q_full; m.lo2 = q_lo2; m.base_slot = q_base; m.first_real = q_fr;
                        m.o0 = o0; m.n_out = n_out;
                        mbar_arrive_tx(&x_full[s], nrows * (uint32_t)(c_hi - c_lo) * 4);
                    }
                    __syncwarp();
                    if (xrow)
                        bulk_g2s(reinterpret_cast<float*>(smem + L::off_x + s * L::kX) + lane * XC4 + (c_lo - (w0 - 4)),
                                 ring + (int64_t)slot * P.pitch + c_lo, (uint32_t)(c_hi - c_lo) * 4, &x_full[s]);
                    if (lane == 0) WS_TRACE(b, 0);
                    t_wait += t1 - t0;
                    t_plan += clock64() - t1;
                    if (!P.slot_xmax && b >= SCAN_LAG) finalize(b - SCAN_LAG);
                }
                ca = na;
                cb = nb_;
            }
            if (task0 + 32 * G >= n_tasks) break;
        }
        if (!P.slot_xmax)
            for (int j = max(0, b - SCAN_LAG); j < b; ++j) finalize(j);
        {  // end of work: an invalid band tells the consumers to stop
            const int s = b % NX;
            if (b >= NX) mbar_wait(&x_empty[s], ((b / NX) & 1) ^ 1);
            if (lane == 0) {
                meta[s].valid = 0;
                mbar_arrive(P.slot_xmax ? &x_full[s] : &x_ready[s]);
            }
        }
        if ((dbg & 8) && lane == 0) {
            g_prof[blockIdx.x * 16 + 0] = t_wait;
            g_prof[blockIdx.x * 16 + 1] = t_plan;
            g_prof[blockIdx.x * 16 + 7] = t_scan;
        }
    } else if (warp == WARP_MMA) {
        // ------------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_f16_f32(TW, 96, 0);
            constexpr uint32_t idesc64 = idesc_f16_f32(TW, 64, 0), idesc32 = idesc_f16_f32(TW, 32, 0);
            const uint32_t b_addr = smem_u32(smem + L::off_b);
            uint64_t bdesc[2][3];
#pragma unroll
            for (int hl = 0; hl < 2; ++hl)
#pragma unroll
                for (int dj = 0; dj < 3; ++dj) bdesc[hl][dj] = umma_desc(b_addr + (hl * 3 + dj) * B96_BYTES, 1536, 128);
            unsigned long long m_wa1 = 0, m_wacc = 0;
            for (int b = 0;; ++b) {
                const int a = b % NA, ph = (b / NA) & 1;
                long long m0 = clock64();
                mbar_wait(&a1_full[a], ph);
                long long m1 = clock64();
                const BandInfo I = info[a];
                // accumulators of buffer a were read by the epilogue (round 0: free at start-up)
                mbar_wait(&acc_empty[a], ph);
                m_wa1 += m1 - m0;
                m_wacc += clock64() - m1;
                if (!I.valid) {
                    if (dbg & 8) {
                        g_prof[blockIdx.x * 16 + 11] = m_wa1;
                        g_prof[blockIdx.x * 16 + 12] = m_wacc;
                    }
                    ainfo[a].valid = 0;
                    mbar_arrive(&acc_full[a]);
                    mbar_arrive(&acc_full[a]);
                    break;
                }
                tc_fence_after();
                WS_TRACE(b, 4);
                ainfo[a] = I;
                const uint32_t a1_addr = smem_u32(smem + L::off_a1 + a * L::kA1);
                // Slot q's first writer initialises it (accumulate = 0): the first real a1 row
                // initialises its whole window; every later row initialises only its newest slot
                // (ar+2) through an extra N=32 MMA, so accumulators never need clearing.
                bool first_row = true;
                for (int ar = 0; ar < ((dbg & 2) ? 0 : I.n_out + 2); ++ar) {
                    const int pos = I.o0 - 1 + ar;
                    if (pos < 0 || pos >= H) continue;  // zero padding row: contributes nothing
                    const uint32_t d_tmem = tmem_base + a * ACC_COLS + ar * 32;
#pragma unroll
                    for (int dj = 0; dj < 3; ++dj) {
                        const uint32_t pix = (uint32_t)(ar * A1C + dj) * 16;
                        const uint64_t a_hi = umma_desc(a1_addr + pix, PLANE, 128);
                        if (dj == 0 && first_row) {
                            mma_f16(d_tmem, a_hi, bdesc[0][0], idesc, 0);
                        } else if (dj == 0) {
                            mma_f16(d_tmem, a_hi, bdesc[0][0], idesc64, 1);                  // slots ar, ar+1
                            mma_f16(d_tmem + 64, a_hi, bdesc[0][0] + (1024 >> 4), idesc32, 0);  // slot ar+2 (rows 64..95)
                        } else {
                            mma_f16(d_tmem, a_hi, bdesc[0][dj], idesc, 1);
                        }
                        if constexpr (PREC == AP_PREC_F16X3) {
                            const uint64_t a_lo = umma_desc(a1_addr + 2 * PLANE + pix, PLANE, 128);
                            mma_f16(d_tmem, a_hi, bdesc[1][dj], idesc, 1);
                            mma_f16(d_tmem, a_lo, bdesc[0][dj], idesc, 1);
                        }
                    }
                    first_row = false;
                }
                WS_TRACE(b, 5);
                mma_commit(&a1_empty[a]);   // a1 tile consumed -> conv1 may refill it
                mma_commit(&acc_full[a]);   // accumulators ready
                mbar_arrive(&acc_full[a]);  // releases ainfo[a]
            }
        }
    } else if (warp >= EPI0 && warp < EPI0 + NEPI) {
        // ------------------------------------------------------------------ epilogue
        const int quad = warp & 3, pix = quad * 32 + lane;
        const int wexp = g_wexp;
        const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16);
        // start-up: both accumulator buffers are free
        __syncwarp();
        if (lane == 0)
            for (int a = 0; a < NA; ++a) mbar_arrive(&acc_empty[a]);
        // Running sum of this column: the stored value (incremental task) or 0 (full task), plus the
        // new r of every recomputed slot, minus the values those slots held.  The old values are
        // loaded at the task's first band (before any of its stores) and subtracted at its last.
        constexpr int NOLD = 8;
        double S = 0.0, Snew = 0.0;
        float oldv[NOLD];
        unsigned long long e_wait = 0, e_work = 0, e_math = 0;
        long long e_t = clock64();
        for (int b = 0;; ++b) {
            const int a = b % NA, ph = (b / NA) & 1;
            long long e0 = clock64();
            e_work += e0 - e_t;
            mbar_wait(&acc_full[a], ph);
            e_t = clock64();
            e_wait += e_t - e0;
            const BandInfo I = ainfo[a];
            if (warp == EPI0 && lane == 0) WS_TRACE(b, 6);
            if (!I.valid) {
                if ((dbg & 8) && warp == EPI0 && lane == 0) {
                    g_prof[blockIdx.x * 16 + 2] = e_wait;
                    g_prof[blockIdx.x * 16 + 3] = e_work;
                    g_prof[blockIdx.x * 16 + 10] = e_math;
                }
                break;
            }
            tc_fence_after();
            const int W = I.W, col = I.chunk * TW + pix;
            const bool live = col < W;
            float* rmap = P.rmap + (int64_t)I.map * P.map_stride + col;
            const int64_t at = (int64_t)I.map * P.pitch + col;
            if (I.first) {
                S = (I.full || !P.rsum || !live) ? 0.0 : P.rsum[at];  // first used at the last band
                Snew = 0.0;
                const int n_old = (I.full || !live) ? 0 : 2 + H - I.lo2;  // positions {0, 1} ∪ [lo2, H)
                auto slot_at = [&](int k) {
                    const int p = k < 2 ? k : I.lo2 + k - 2;
                    const int sl = sel ? I.base_slot + p : p;
                    return sl >= H ? sl - H : sl;
                };
#pragma unroll
                for (int k = 0; k < NOLD; ++k) oldv[k] = k < n_old ? rmap[(int64_t)slot_at(k) * P.pitch] : 0.f;
                for (int k = NOLD; k < n_old; ++k) Snew -= (double)rmap[(int64_t)slot_at(k) * P.pitch];  // > NOLD - 4 new rows
            }
            long long q0 = clock64();
            if (!(dbg & 4)) {
                const int e = I.aexp + wexp;
                const bool one_mul = e >= -126 && e <= 126;
                const float u = one_mul ? pow2f(-e) : pow2f(-I.aexp), u2 = one_mul ? 1.f : pow2f(-wexp);
                // 16-column pieces (row j = c / 2, channels 16 (c % 2) ..) ping-pong between two register
                // sets: piece c+1's TMEM load overlaps piece c's math
                const int n_pc = 2 * I.n_out;
                const uint32_t t0 = lane_base + a * ACC_COLS + 2 * 32;
                uint32_t ra[16], rb[16];
                tmem_ld16_start(t0, ra);
                tmem_ld_wait(ra);
                float r0 = 0.f, r1 = 0.f, bsum = 0.f;  // bsum: this band's new r (one fp64 add per band)
#pragma unroll
                for (int c = 0; c < 2 * MAXO; ++c) {
                    if (c >= n_pc) break;
                    uint32_t (&cur)[16] = (c & 1) ? rb : ra;
                    uint32_t (&nxt)[16] = (c & 1) ? ra : rb;
                    if (c + 1 < n_pc) tmem_ld16_start(t0 + (c + 1) * 16, nxt);
                    if (!one_mul) {  // scale too extreme for one multiply (never for attention rows)
#pragma unroll
                        for (int n = 0; n < 16; ++n) cur[n] = __float_as_uint(__uint_as_float(cur[n]) * u2);
                    }
                    // r += sum_c w3[c] relu(acc[c] * u + b2[c]), channel pairs on the packed FMA pipe
                    const int ch0 = (c & 1) * 16;
#pragma unroll
                    for (int n = 0; n < 16; n += 2) {
                        float s0 = c_w[OFF_B2 + ch0 + n], s1 = c_w[OFF_B2 + ch0 + n + 1];
                        ffma2(s0, s1, __uint_as_float(cur[n]), __uint_as_float(cur[n + 1]), u);
                        ffma2v(r0, r1, fmaxf(s0, 0.f), fmaxf(s1, 0.f), c_w[OFF_W3 + ch0 + n], c_w[OFF_W3 + ch0 + n + 1]);
                    }
                    if (c & 1) {  // row complete
                        const float r = r0 + r1;
                        if (live) {
                            rmap[(int64_t)I.out_slot[c >> 1] * P.pitch] = r;
                            bsum += r;
                        }
                        r0 = r1 = 0.f;
                    }
                    if (c + 1 < n_pc) tmem_ld_wait(nxt);
                }
                Snew += (double)bsum;
            }
            e_math += clock64() - q0;
            tc_fence_before();  // our tcgen05.ld reads of buffer a are complete before it is reused
            __syncwarp();
            if (warp == EPI0 && lane == 0) WS_TRACE(b, 7);
            const bool last = I.last;  // read before the release: the MMA issuer refills the info slot after it
            const int64_t sat = (int64_t)I.map * P.score_stride + col;
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[a]);
            if (last && live) {
                float osum = 0.f;
#pragma unroll
                for (int k = 0; k < NOLD; ++k) osum += oldv[k];
                S += Snew - (double)osum;
                if (P.rsum) P.rsum[at] = S;
                P.scores[sat] = c_w[OFF_B3] + (float)S / (float)H;
            }
        }
    } else {
        // ------------------------------------------------------------------ conv1 workers
        const int ct = tid - CONV0 * 32;
        unsigned long long c_wx = 0, c_wa = 0, c_work = 0;
        long long c_t = clock64();
        for (int b = 0;; ++b) {
            const int s = b % NX;
            long long c0 = clock64();
            c_work += c0 - c_t;
            mbar_wait(P.slot_xmax ? &x_full[s] : &x_ready[s], (b / NX) & 1);  // tile landed / scanned
            c_t = clock64();
            c_wx += c_t - c0;
            const BandMeta& m = meta[s];
            const int a = b % NA;
            if (!m.valid && (dbg & 8) && ct == 0) {
                g_prof[blockIdx.x * 16 + 4] = c_wx;
                g_prof[blockIdx.x * 16 + 5] = c_wa;
                g_prof[blockIdx.x * 16 + 6] = c_work;
            }
            if (!m.valid) {
                if (b >= NA) mbar_wait(&a1_empty[a], ((b / NA) & 1) ^ 1);
                if (ct == 0) info[a].valid = 0;
                __syncwarp();
                if (lane == 0) mbar_arrive(&a1_full[a]);
                break;
            }
            const float* xs = reinterpret_cast<const float*>(smem + L::off_x + s * L::kX);
            const int W = m.W, w0 = m.chunk * TW, n_out = m.n_out, n_a1 = n_out + 2, n_x = n_out + 4;
            const int aexp = m.aexp;
            const float ascale = pow2f(aexp);
            long long ca = clock64();
            if (b >= NA) mbar_wait(&a1_empty[a], ((b / NA) & 1) ^ 1);
            long long cb = clock64();
            if (ct == 0) WS_TRACE(b, 2);
            c_wa += cb - ca;
            c_work -= cb - ca;
            uint8_t* a1t = smem + L::off_a1 + a * L::kA1;
            // Two adjacent a1 pixels per thread (packed FFMA2, shared x window).  Only rows inside the
            // history are computed: conv2's zero-padding rows (position < 0 or >= H) are never read.
            const int ar_lo = max(0, 1 - m.o0), ar_hi = min(n_a1, H + 1 - m.o0);
            constexpr int PAIRS = A1C / 2;
            for (int i = ct; i < ((dbg & 1) ? 0 : (ar_hi - ar_lo) * PAIRS); i += NCONV_T) {
                const int rr = i / PAIRS, ar = ar_lo + rr, ac = 2 * (i - rr * PAIRS);
                const int c = w0 - 1 + ac;  // pixel columns c, c + 1
                float xw[3][4];
#pragma unroll
                for (int di = 0; di < 3; ++di) {
                    const int lim = m.x_lim[ar + di];
                    const float* xr = xs + (ar + di) * XC4 + ac + 2;
#pragma unroll
                    for (int e = 0; e < 4; ++e) xw[di][e] = ((unsigned)(c - 1 + e) < (unsigned)lim) ? xr[e] : 0.f;
                }
                // pixels outside [0, W) are conv2's zero padding: a zero scale clears them
                const float sc0 = (unsigned)c < (unsigned)W ? ascale : 0.f;
                const float sc1 = (unsigned)(c + 1) < (unsigned)W ? ascale : 0.f;
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
                            ffma2(s0, s1, xw[k / 3][k % 3], xw[k / 3][k % 3 + 1], c_w[OFF_W1 + ch * 9 + k]);
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
                    *reinterpret_cast<uint4*>(a1t + g * PLANE + px * 16) = h0;
                    *reinterpret_cast<uint4*>(a1t + g * PLANE + px * 16 + 16) = h1;
                    if constexpr (PREC == AP_PREC_F16X3) {
                        *reinterpret_cast<uint4*>(a1t + (2 + g) * PLANE + px * 16) = l0;
                        *reinterpret_cast<uint4*>(a1t + (2 + g) * PLANE + px * 16 + 16) = l1;
                    }
                }
            }
            if (ct == 0) {
                BandInfo& I = info[a];
                I.valid = 1; I.map = m.map; I.chunk = m.chunk; I.W = W; I.first = m.first; I.last = m.last;
                I.full = m.full; I.lo2 = m.lo2; I.base_slot = m.base_slot; I.first_real = m.first_real;
                I.o0 = m.o0; I.n_out = n_out; I.aexp = aexp;
                for (int j = 0; j < MAXO; ++j) I.out_slot[j] = m.out_slot[j];
            }
            fence_async_smem();  // a1 tile -> visible to the tensor core's async proxy
            __syncwarp();
            if (ct == 0) WS_TRACE(b, 3);
            if (ct == NCONV_T - 32) WS_TRACE(b, 1);
            if (lane == 0) {
                mbar_arrive(&a1_full[a]);
                mbar_arrive(&x_empty[s]);
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == WARP_PROD) tmem_dealloc(tmem_base, TMEM);
}

}  // namespace ws
}  // namespace ap
