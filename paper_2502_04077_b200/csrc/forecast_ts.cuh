// Register-fed forecaster kernel (tensor-core precisions) — included by predictor.cu after the
// shared definitions (weights in constant memory, packed B tiles, task planning, band geometry).
//
// Why this shape: in the shared-memory-operand form (forecast_ws.cuh) every conv2 MMA re-reads
// its 4 KB A tile (a shifted a1 row) and 3 KB B tile from shared memory, and with the conv1
// tile writes that traffic alone saturates the SM's 128 B/clk shared-memory port (~3 k cycles per
// 3-row band).  Here conv1 never touches shared memory on the way out: the conv1 warps compute
// a1 in registers, lane = pixel, and write it straight into tensor memory with tcgen05.st as the
// A operand of "TS" MMAs (A from TMEM), once per column shift dj (two register shuffles make the
// shifts).  Shared memory then only carries the x tiles (TMA bulk copies) and the constant B
// tiles, and the MMAs run at the tensor pipe's rate.
//
// One CTA (19 warps) per SM, persistent over (map, 128-column chunk) tasks, each task processed
// as bands of <= MAXO history rows.  Roles, connected by mbarriers:
//   warps 0-1   producers (alternate bands): task planning (32 tasks at a time, lane-parallel
//               state loads), band metadata into a ring, lane-parallel cp.async.bulk copies of the
//               band's x rows;
//               operand scale from the per-slot row maxima the ring writers recorded (selector
//               mode) or from a scan of the landed tile (explicit grids);
//   warp 2      MMA: per real a1 row of a band, 3 column shifts x (1 or 3 precision terms) TS MMAs
//               whose N covers exactly the band's output rows that a1 row feeds (32/64/96);
//               commits free the a1 row's TMEM slot and publish the accumulators;
//   warps 3-6   epilogue (one per TMEM lane quadrant, lane = column): bias, ReLU, w3 dot -> r,
//               r-map store, running-sum update; clears its accumulator columns for the next use;
//   warps 7-18  conv1: three groups of four quadrant warps take a1 row pairs in turn; lane l of the
//               quadrant-q warp computes a1 at column w0 + 32 q + l - 1 (16 channels, packed
//               FFMA2), ReLU + fp16 hi/lo split, then tcgen05.st of the three shifted A tiles.
#pragma once

namespace ap {
namespace ts {

constexpr int NG = 3;                               // conv1 groups (four quadrant warps each)
constexpr int NCW = 4 * NG;                         // conv1 warps
constexpr int NPROD = 2;                            // producer warps (bands dealt round-robin)
constexpr int WARP_PROD = 0, WARP_MMA = NPROD, EPI0 = NPROD + 1, NEPI = 4, CONV0 = EPI0 + NEPI;
constexpr int NWARP = CONV0 + NCW;
constexpr int NT = NWARP * 32;
constexpr int NX = 4;                               // x tile stages
constexpr int NBI = 8;                              // band-metadata ring
constexpr int NAR = 6;                              // a1 rows resident in TMEM (A operand ring)
constexpr int ACOLS = 48;                           // per a1 row: hi dj0..2, lo dj0..2 (8 columns each)
constexpr int NACC = 2;                             // accumulator buffers
constexpr int ACC_COLS = MAXO * 32;                 // exact: one 32-column slot per output row
constexpr int ACC0 = NAR * ACOLS;
constexpr int TMEM = 512;
static_assert(ACC0 + NACC * ACC_COLS <= TMEM, "TMEM budget");

__device__ long long g_trace[64 * 8];  // debug bit 16: CTA 0 timeline of its first 64 bands
#define TS_TRACE(b, e) \
    if ((dbg & 16) && blockIdx.x == 0 && (b) < 64) g_trace[(b) * 8 + (e)] = clock64();

constexpr int BND_WARP = 2 * 2 * 16;      // per conv warp: [row][column][16 words]

struct Smem {
    static constexpr int kB = 2 * 3 * B96_BYTES;
    static constexpr int kX = MAXX * XC4 * 4;
    static constexpr int off_b = 0;
    static constexpr int off_x = off_b + kB;                                    // [NX] x tiles
    static constexpr int off_meta = off_x + NX * kX;                            // BandMeta[NBI]
    static constexpr int off_bnd = (off_meta + NBI * (int)sizeof(BandMeta) + 15) / 16 * 16;
    // per conv warp: the two columns right of its 32 (both rows, hi | lo words)
    static constexpr int kBnd = NCW * BND_WARP * 4;
    static constexpr int off_w1 = off_bnd + kBnd;                               // w1 [16][9], b1 [16] (fp32)
    static constexpr int off_zero = off_w1 + 160 * 4;                           // an all-zero x row
    static constexpr int off_bar = off_zero + XC4 * 4;
    // x_full[NX], x_ready[NX], x_empty[NX], bi_empty[NBI], meta_full[NBI], a_full[NAR], a_empty[NAR],
    // acc_full[NACC], acc_empty[NACC], tmem slot
    static constexpr int n_bar = 3 * NX + 2 * NBI + 2 * NAR + 2 * NACC;
    static constexpr int total = off_bar + 8 * n_bar + 16;
};

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
                    "r"(v[7]) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// relu(v) as fp16 hi + lo (hi = v truncated to 11 significant bits, exact; lo = the remainder,
// rounded once); for v <= 0 both are 0.  Two channels per 32-bit word, channel 2i in the low half.
__device__ __forceinline__ void split_relu_f16x2(float v0, float v1, uint32_t& hi2, uint32_t& lo2) {
    const float h0 = __uint_as_float(__float_as_uint(v0) & 0xffffe000u);
    const float h1 = __uint_as_float(__float_as_uint(v1) & 0xffffe000u);
    asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(hi2) : "f"(h1), "f"(h0));
    asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(lo2) : "f"(v1 - h1), "f"(v0 - h0));
}
__device__ __forceinline__ uint32_t relu_f16x2_rn(float v0, float v1) {
    uint32_t r;
    asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v1), "f"(v0));
    return r;
}

// Real a1 rows of a band: history positions [o0 - 1, o0 + n_out] inside [0, H)
__device__ __forceinline__ void a1_rows(int o0, int n_out, int H, int& p_lo, int& n_rows) {
    p_lo = max(o0 - 1, 0);
    const int p_hi = min(o0 + n_out, H - 1);
    n_rows = p_hi - p_lo + 1;
}

template <int PREC>
__global__ void __launch_bounds__(NT, 1) conv_forecast_ts_kernel(ConvParams P) {
    constexpr bool X3 = PREC == AP_PREC_F16X3;
    extern __shared__ __align__(1024) uint8_t smem[];
    BandMeta* meta = reinterpret_cast<BandMeta*>(smem + Smem::off_meta);
    uint32_t* bnd = reinterpret_cast<uint32_t*>(smem + Smem::off_bnd);
    float* s_w1 = reinterpret_cast<float*>(smem + Smem::off_w1);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::off_bar);
    uint64_t* x_full = bars;                 // bulk copies landed (producer)
    uint64_t* x_ready = bars + NX;           // tile scanned, operand scale published (explicit grids)
    uint64_t* x_empty = bars + 2 * NX;       // conv1 done with the tile
    uint64_t* bi_empty = bars + 3 * NX;      // epilogue done with the band's metadata
    uint64_t* meta_full = bi_empty + NBI;    // band metadata published (MMA / epilogue; never lag-aliased)
    uint64_t* a_full = meta_full + NBI;      // a1 row written to TMEM (4 quadrant warps)
    uint64_t* a_empty = a_full + NAR;        // MMAs reading the a1 row completed (commit)
    uint64_t* acc_full = a_empty + NAR;      // accumulators complete (commit + MMA thread)
    uint64_t* acc_empty = acc_full + NACC;   // epilogue read and cleared them
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + NACC);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int H = P.H;
    const bool sel = P.state != nullptr;
    const int dbg = P.debug;

    {  // B operands once per persistent CTA; barriers; TMEM
        const uint4* src = g_bpack96;
        uint4* dst = reinterpret_cast<uint4*>(smem + Smem::off_b);
        for (int i = tid; i < Smem::kB / 16; i += NT) dst[i] = src[i];
        for (int i = tid; i < 160; i += NT) s_w1[i] = c_w[OFF_W1 + i];  // w1 then b1 (APW1 order)
        for (int i = tid; i < XC4; i += NT) reinterpret_cast<float*>(smem + Smem::off_zero)[i] = 0.f;
        if (tid == 0) {
            for (int s = 0; s < NX; ++s) {
                mbar_init(&x_full[s], 1);
                mbar_init(&x_ready[s], 1);
                mbar_init(&x_empty[s], NCW);
            }
            for (int i = 0; i < NBI; ++i) {
                mbar_init(&bi_empty[i], NEPI);
                mbar_init(&meta_full[i], 1);
            }
            for (int k = 0; k < NAR; ++k) {
                mbar_init(&a_full[k], 4);
                mbar_init(&a_empty[k], 1);
            }
            for (int a = 0; a < NACC; ++a) {
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

    if (warp < WARP_PROD + NPROD) {
        // ------------------------------------------------------------------ producers (whole warps)
        // Both walk the CTA's task / band sequence; producer p publishes the bands b = p mod NPROD.
        const int pw = warp - WARP_PROD;
        const int G = gridDim.x, n_tasks = P.n_maps * P.n_chunks;
        const float b1max = g_b1abs[0], w1max = g_w1abs[0];
        // explicit grids: max|x| over the landed tile (+ finiteness) -> operand scale, one band behind
        auto finalize = [&](int j) {
            const int s = j % NX;
            mbar_wait_spin(&x_full[s], (j / NX) & 1);
            BandMeta& m = meta[j % NBI];
            const float* xs = reinterpret_cast<const float*>(smem + Smem::off_x + s * Smem::kX);
            const int n_x = m.n_out + 4, cbase = m.chunk * TW - 4;
            float xmax = 0.f;
            bool bad = false;
            for (int i = lane; i < n_x * (XC4 / 4); i += 32) {
                const int q = i / (XC4 / 4), k = i - q * (XC4 / 4);
                const int lim = m.x_lim[q];
                const float4 v = reinterpret_cast<const float4*>(xs + q * XC4)[k];
                const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int xc = 4 * k + u, c = cbase + xc;
                    if (xc >= 2 && xc < TW + 6 && (unsigned)c < (unsigned)lim) {
                        bad |= !(fabsf(e[u]) <= 3.402823466e38f);
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
        };
        const bool pre_xm = sel && P.slot_xmax && H <= 64;
        int b = 0, b_own = -1;  // b_own: this producer's previous band (explicit grids: scanned one band behind)
        for (int task0 = blockIdx.x;; task0 += 32 * G) {
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
                const int rb0 = q_full ? H : 2, nb0 = (rb0 + MAXO - 1) / MAXO;
                const int nb = nb0 + (q_full ? 0 : (H - q_lo2 + MAXO - 1) / MAXO);
                const int w0 = q_chunk * TW;
                const int c_lo = max(0, w0 - 4), c_hi = min(P.pitch, w0 + TW + 4);
                const float* ring = P.ring + (int64_t)q_map * P.map_stride;
                int pa = lane - q_base, pb = lane + 32 - q_base;  // history positions of slots lane, lane + 32
                pa += pa < 0 ? H : 0;
                pb += pb < 0 ? H : 0;
                for (int bi = 0; bi < nb; ++bi, ++b) {
                    if (b % NPROD != pw) continue;
                    const int s = b % NX, mi = b % NBI;
                    if (b >= NX) mbar_wait_spin(&x_empty[s], ((b / NX) & 1) ^ 1);
                    if (b >= NBI) mbar_wait_spin(&bi_empty[mi], ((b / NBI) & 1) ^ 1);
                    int o0, o1;
                    if (bi < nb0) { o0 = bi * MAXO; o1 = min(rb0, o0 + MAXO); }
                    else { o0 = q_lo2 + (bi - nb0) * MAXO; o1 = min(H, o0 + MAXO); }
                    const int n_out = o1 - o0;
                    BandMeta& m = meta[mi];
                    const int p = o0 - 2 + lane;  // lane q < n_out + 4: x row q (position o0 - 2 + q)
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
                    // x tile columns outside the copied range [c_lo, c_hi) read as zero
                    float* xt = reinterpret_cast<float*>(smem + Smem::off_x + s * Smem::kX);
                    const int gap_l = c_lo - (w0 - 4), gap_r = (w0 + TW + 4) - c_hi;
                    if (gap_l > 0 || gap_r > 0) {
                        if (gap_l > 0)
                            for (int i = lane; i < MAXX * 4; i += 32)
                                if ((i & 3) < gap_l) xt[(i >> 2) * XC4 + (i & 3)] = 0.f;
                        if (gap_r > 0)
                            for (int i = lane; i < MAXX * gap_r; i += 32) {
                                const int q = i / gap_r, k = i - q * gap_r;
                                xt[q * XC4 + XC4 - 1 - k] = 0.f;
                            }
                        fence_async_smem();  // generic zero writes ordered before later bulk copies into the stage
                    }
                    // (tile rows that are not copied read as zero: conv1 points them at a zero row)
                    if (lane == 0) {
                        m.valid = 1; m.map = q_map; m.chunk = q_chunk; m.W = q_W;
                        m.first = bi == 0; m.last = bi == nb - 1;
                        m.full = q_full; m.lo2 = q_lo2; m.base_slot = q_base; m.first_real = q_fr;
                        m.o0 = o0; m.n_out = n_out;
                        mbar_arrive(&meta_full[mi]);
                        mbar_arrive_tx(&x_full[s], nrows * (uint32_t)(c_hi - c_lo) * 4);
                    }
                    __syncwarp();
                    if (xrow)
                        bulk_g2s(xt + lane * XC4 + (c_lo - (w0 - 4)), ring + (int64_t)slot * P.pitch + c_lo,
                                 (uint32_t)(c_hi - c_lo) * 4, &x_full[s]);
                    if (lane == 0) TS_TRACE(b, 0);
                    if (!P.slot_xmax && b_own >= 0) finalize(b_own);
                    b_own = b;
                }
                ca = na;
                cb = nb_;
            }
            if (task0 + 32 * G >= n_tasks) break;
        }
        if (!P.slot_xmax && b_own >= 0) finalize(b_own);
        if (b % NPROD == pw) {  // end of work: an invalid band tells the consumers to stop
            const int s = b % NX, mi = b % NBI;
            if (b >= NX) mbar_wait_spin(&x_empty[s], ((b / NX) & 1) ^ 1);
            if (b >= NBI) mbar_wait_spin(&bi_empty[mi], ((b / NBI) & 1) ^ 1);
            if (lane == 0) {
                meta[mi].valid = 0;
                mbar_arrive(&meta_full[mi]);
                mbar_arrive(&x_full[s]);
                mbar_arrive(&x_ready[s]);
            }
        }
    } else if (warp == WARP_MMA) {
        // ------------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t b_addr = smem_u32(smem + Smem::off_b);
            uint64_t bdesc[2][3];
#pragma unroll
            for (int hl = 0; hl < 2; ++hl)
#pragma unroll
                for (int dj = 0; dj < 3; ++dj) bdesc[hl][dj] = umma_desc(b_addr + (hl * 3 + dj) * B96_BYTES, 1536, 128);
            int seq = 0;
            for (int b = 0;; ++b) {
                const int ab = b % NACC;
                mbar_wait_spin(&meta_full[b % NBI], (b / NBI) & 1);
                const BandMeta& m = meta[b % NBI];
                if (!m.valid) break;
                const int o0 = m.o0, n_out = m.n_out;
                int p_lo, n_rows;
                a1_rows(o0, n_out, H, p_lo, n_rows);
                mbar_wait_spin(&acc_empty[ab], (b / NACC) & 1);  // completion 0 = the epilogue's start-up arrive
                TS_TRACE(b, 4);
                const uint32_t d0 = tmem_base + ACC0 + ab * ACC_COLS;
                for (int i = 0; i < n_rows; ++i, ++seq) {
                    const int k = seq % NAR;
                    mbar_wait_spin(&a_full[k], (seq / NAR) & 1);
                    tc_fence_after();
                    const int p = p_lo + i;
                    const int oa = max(p - 1, o0), ob = min(p + 1, o0 + n_out - 1);
                    const int nb = ob - oa + 1, blk = oa - p + 1;  // B rows stacked di = 2, 1, 0
                    const uint32_t d = d0 + (oa - o0) * 32, idesc = idesc_f16_f32(TW, 32 * nb, 0);
                    const uint32_t a0 = tmem_base + k * ACOLS;
                    const uint64_t boff = (uint64_t)((blk * 32 * 16) >> 4);
#pragma unroll
                    for (int dj = 0; dj < ((dbg & 2) ? 0 : 3); ++dj) {
                        mma_f16_ts(d, a0 + dj * 8, bdesc[0][dj] + boff, idesc, 1);
                        if constexpr (X3) {
                            mma_f16_ts(d, a0 + dj * 8, bdesc[1][dj] + boff, idesc, 1);       // hi x lo(w)
                            mma_f16_ts(d, a0 + 24 + dj * 8, bdesc[0][dj] + boff, idesc, 1);  // lo(a) x hi
                        }
                    }
                    mma_commit(&a_empty[k]);  // a1 row consumed -> its TMEM slot may be rewritten
                }
                TS_TRACE(b, 5);
                mma_commit(&acc_full[ab]);
                mbar_arrive(&acc_full[ab]);
            }
        }
    } else if (warp >= EPI0 && warp < EPI0 + NEPI) {
        // ------------------------------------------------------------------ epilogue
        const int quad = warp & 3, pix = quad * 32 + lane;
        const int wexp = g_wexp;
        const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16);
        // start-up: clear every accumulator column this warp owns; both buffers are then free
        for (int c = ACC0; c < ACC0 + NACC * ACC_COLS; c += 32) tmem_zero32(lane_base + c);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0)
            for (int a = 0; a < NACC; ++a) mbar_arrive(&acc_empty[a]);
        constexpr int NOLD = 8;
        double S = 0.0, Snew = 0.0;
        float oldv[NOLD];
        for (int b = 0;; ++b) {
            const int ab = b % NACC, mi = b % NBI;
            mbar_wait_spin(&meta_full[mi], (b / NBI) & 1);
            const BandMeta I = meta[mi];
            if (!I.valid) break;
            const int W = I.W, col = I.chunk * TW + pix;
            const bool live = col < W;
            float* rmap = P.rmap + (int64_t)I.map * P.map_stride + col;
            const int64_t at = (int64_t)I.map * P.pitch + col;
            if (I.first) {  // old values of the rows this task rewrites (loads overlap the MMAs)
                S = (I.full || !P.rsum || !live) ? 0.0 : P.rsum[at];
                Snew = 0.0;
                const int n_old = (I.full || !live) ? 0 : 2 + H - I.lo2;  // positions {0, 1} ∪ [lo2, H)
                auto slot_at = [&](int k) {
                    const int p = k < 2 ? k : I.lo2 + k - 2;
                    const int sl = sel ? I.base_slot + p : p;
                    return sl >= H ? sl - H : sl;
                };
#pragma unroll
                for (int k = 0; k < NOLD; ++k) oldv[k] = k < n_old ? rmap[(int64_t)slot_at(k) * P.pitch] : 0.f;
                for (int k = NOLD; k < n_old; ++k) Snew -= (double)rmap[(int64_t)slot_at(k) * P.pitch];
            }
            mbar_wait_spin(&acc_full[ab], (b / NACC) & 1);
            tc_fence_after();
            if (warp == EPI0 && lane == 0) TS_TRACE(b, 6);
            {
                // aexp: re-read after acc_full (explicit grids publish it after the rest of the metadata)
                const int aexp = *reinterpret_cast<volatile int*>(&meta[mi].aexp);
                const int e = aexp + wexp;
                const bool one_mul = e >= -126 && e <= 126;
                const float u = one_mul ? pow2f(-e) : pow2f(-aexp), u2 = one_mul ? 1.f : pow2f(-wexp);
                const uint32_t t0 = lane_base + ACC0 + ab * ACC_COLS;
                float bsum = 0.f;
                for (int j = 0; j < ((dbg & 4) ? 0 : I.n_out); ++j) {
                    uint32_t ra[16], rb[16];
                    tmem_ld16_start(t0 + j * 32, ra);
                    tmem_ld16_start(t0 + j * 32 + 16, rb);
                    tmem_ld_wait(ra);
                    tmem_ld_wait(rb);
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
                        float q0 = c_w[OFF_B2 + 16 + n], q1 = c_w[OFF_B2 + 16 + n + 1];
                        ffma2(q0, q1, __uint_as_float(rb[n]), __uint_as_float(rb[n + 1]), u);
                        ffma2v(r0, r1, fmaxf(q0, 0.f), fmaxf(q1, 0.f), c_w[OFF_W3 + 16 + n], c_w[OFF_W3 + 16 + n + 1]);
                    }
                    const float r = r0 + r1;
                    if (live) {
                        rmap[(int64_t)meta[mi].out_slot[j] * P.pitch] = r;
                        bsum += r;
                    }
                    tmem_zero32(t0 + j * 32);  // cleared for the next band's accumulate-only MMAs
                }
                Snew += (double)bsum;
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (warp == EPI0 && lane == 0) TS_TRACE(b, 7);
            if (lane == 0) {
                mbar_arrive(&acc_empty[ab]);
                mbar_arrive(&bi_empty[mi]);
            }
            if (I.last && live) {
                float osum = 0.f;
#pragma unroll
                for (int k = 0; k < NOLD; ++k) osum += oldv[k];
                S += Snew - (double)osum;
                if (P.rsum) P.rsum[at] = S;
                P.scores[(int64_t)I.map * P.score_stride + col] = c_w[OFF_B3] + (float)S / (float)H;
            }
        }
    } else {
        // ------------------------------------------------------------------ conv1 workers
        // Work unit = two consecutive a1 rows of a band (the last unit of a band may hold one), dealt
        // round-robin over the NG groups across bands; the four quadrant warps of a group each cover
        // 32 columns of the unit's rows, independently (each computes the two columns right of its
        // range itself, so the shifted tiles need no cross-warp exchange).
        const int cw = warp - CONV0, grp = cw >> 2, quad = warp & 3;
        const float* xzero = reinterpret_cast<const float*>(smem + Smem::off_zero);
        const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16);
        int seq = 0, useq = 0;  // a1 rows / units of all bands so far
        for (int b = 0;; ++b) {
            const int s = b % NX;
            mbar_wait_spin(P.slot_xmax ? &x_full[s] : &x_ready[s], (b / NX) & 1);  // tile landed / scanned
            const BandMeta& m = meta[b % NBI];
            if (!m.valid) break;
            if (lane == 0 && cw == 0) TS_TRACE(b, 2);
            const float* xs = reinterpret_cast<const float*>(smem + Smem::off_x + s * Smem::kX);
            const int W = m.W, w0 = m.chunk * TW, o0 = m.o0;
            const float ascale = pow2f(m.aexp);
            int p_lo, n_rows;
            a1_rows(o0, m.n_out, H, p_lo, n_rows);
            const int n_units = (n_rows + 1) >> 1;
            const bool masked = !sel;  // explicit grids: the caller's row padding is not known to be zero
            for (int u = (grp - useq % NG + NG) % NG; u < n_units; u += NG) {
                const bool two = 2 * u + 1 < n_rows;
                const int sq0 = seq + 2 * u, k0 = sq0 % NAR, k1 = (sq0 + 1) % NAR;
                const int p0 = p_lo + 2 * u, ar = p0 - (o0 - 1);  // x tile rows ar .. ar + 3 = positions p0-1 .. p0+2
                // x window of this lane's column, 4 rows (rows p0 - 1 + r), pre-scaled by 2^aexp
                auto xwin = [&](int cc, float (&xw)[4][3]) {
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int lim = (ar + r < MAXX) ? m.x_lim[ar + r] : 0;
                        const float* xr = (lim > 0 ? xs + (ar + r) * XC4 : xzero) + (cc - (w0 - 4)) - 1;
#pragma unroll
                        for (int e = 0; e < 3; ++e) {
                            float v = (r < 3 || two) ? xr[e] : 0.f;
                            if (masked && !((unsigned)(cc - 1 + e) < (unsigned)lim)) v = 0.f;
                            xw[r][e] = v * ascale;
                        }
                    }
                };
                const int c = w0 + 32 * quad + lane - 1;  // lane l: a1 at column c, rows p0 and p0 + 1
                uint32_t hi[2][8], lo[2][8];
                if (dbg & 1) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) hi[0][q] = hi[1][q] = lo[0][q] = lo[1][q] = 0u;
                } else {
                    float xw[4][3];
                    xwin(c, xw);
                    float a[2][16];
#pragma unroll
                    for (int ch = 0; ch < 16; ++ch) a[0][ch] = a[1][ch] = c_w[OFF_B1 + ch] * ascale;
#pragma unroll
                    for (int t = 0; t < 9; ++t)
#pragma unroll
                        for (int ch = 0; ch < 16; ++ch)  // the two rows on the packed FMA pipe
                            ffma2(a[0][ch], a[1][ch], xw[t / 3][t % 3], xw[t / 3 + 1][t % 3], c_w[OFF_W1 + ch * 9 + t]);
                    const bool inside = (unsigned)c < (unsigned)W;  // conv2's zero padding outside [0, W)
#pragma unroll
                    for (int r = 0; r < 2; ++r)
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            if constexpr (X3) split_relu_f16x2(a[r][2 * q], a[r][2 * q + 1], hi[r][q], lo[r][q]);
                            else { hi[r][q] = relu_f16x2_rn(a[r][2 * q], a[r][2 * q + 1]); lo[r][q] = 0u; }
                            if (!inside) hi[r][q] = lo[r][q] = 0u;
                        }
                }
                // the two columns right of this warp's 32 (w0 + 32 q + 31, + 32), needed by the shifted
                // tiles: lane l -> column e = l / 16, channel l % 16, both rows; packed into the warp's
                // scratch as [row][column][hi words 0-7 | lo words 8-15]
                uint32_t* bw = bnd + (warp - CONV0) * BND_WARP;
                if (!(dbg & 1)) {
                    const int e = lane >> 4, ch = lane & 15, cc = w0 + 32 * quad + 31 + e;
                    float xw[4][3];
                    xwin(cc, xw);
                    float a0 = s_w1[144 + ch] * ascale, a1v = a0;
#pragma unroll
                    for (int t = 0; t < 9; ++t) {
                        const float w = s_w1[ch * 9 + t];
                        a0 = fmaf(w, xw[t / 3][t % 3], a0);
                        a1v = fmaf(w, xw[t / 3 + 1][t % 3], a1v);
                    }
                    const bool inside = (unsigned)cc < (unsigned)W;
                    __half* bh = reinterpret_cast<__half*>(bw);
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        const float v = inside ? (r ? a1v : a0) : 0.f;
                        __half hh, hl;
                        if constexpr (X3) {
                            const float h = __uint_as_float(__float_as_uint(v) & 0xffffe000u);
                            hh = __float2half_rn(fmaxf(h, 0.f));
                            hl = __float2half_rn(fmaxf(v - h, 0.f));
                        } else {
                            hh = __float2half_rn(fmaxf(v, 0.f));
                            hl = __float2half_rn(0.f);
                        }
                        bh[((r * 2 + e) * 16) * 2 + ch] = hh;  // word ch / 2, half ch % 2 (channel 2i low)
                        bh[((r * 2 + e) * 16 + 8) * 2 + ch] = hl;
                    }
                }
                __syncwarp();
                // per row: shifted copies built in registers, then (slot free) six stores and a_full
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    if (r == 1 && !two) break;
                    uint32_t sh[2][8], sl[2][8];  // dj = 1, 2: lane m <- column w0 + 32 q + m - 1 + dj
#pragma unroll
                    for (int dj = 1; dj < 3; ++dj) {
                        const int e = max(lane - (32 - dj), 0);  // tail lanes: right column e
                        const bool tail = lane >= 32 - dj;
                        const uint32_t* src = bw + (r * 2 + e) * 16;
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const uint32_t vh = __shfl_down_sync(0xffffffffu, hi[r][q], dj);
                            sh[dj - 1][q] = tail ? src[q] : vh;
                            if constexpr (X3) {
                                const uint32_t vl = __shfl_down_sync(0xffffffffu, lo[r][q], dj);
                                sl[dj - 1][q] = tail ? src[8 + q] : vl;
                            }
                        }
                    }
                    const int sqr = sq0 + r, kr = sqr % NAR;
                    if (sqr >= NAR) mbar_wait_spin(&a_empty[kr], ((sqr / NAR) & 1) ^ 1);  // previous occupant read
                    tc_fence_after();
                    const uint32_t ta = lane_base + kr * ACOLS;
                    tmem_st8(ta, hi[r]);  // dj = 0: lane m <- column w0 + 32 q + m - 1
                    tmem_st8(ta + 8, sh[0]);
                    tmem_st8(ta + 16, sh[1]);
                    if constexpr (X3) {
                        tmem_st8(ta + 24, lo[r]);
                        tmem_st8(ta + 32, sl[0]);
                        tmem_st8(ta + 40, sl[1]);
                    }
                    tmem_st_wait();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&a_full[kr]);
                }
            }
            seq += n_rows;
            useq += n_units;
            if (lane == 0 && cw == 0) TS_TRACE(b, 3);
            __syncwarp();
            if (lane == 0) mbar_arrive(&x_empty[s]);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == WARP_PROD) tmem_dealloc(tmem_base, TMEM);
}

}  // namespace ts
}  // namespace ap
