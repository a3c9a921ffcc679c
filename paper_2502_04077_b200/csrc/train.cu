// Forecaster training on the device: exact gradients of the MSE loss (predictor.backward,
// predictor.py:219-251) for a batch of equal-shape samples, and the Adam update of
// predictor.train (predictor.py:371-391).
//
// This is not the decode hot path: plain SIMT kernels in fp64 (the
// reference's arithmetic type), channel planes [n][C][H][W] so a warp reads consecutive
// columns of a plane, and every reduction over pixels in a fixed order (deterministic).
// The reference's im2col / col2im matrices are never formed: the conv2 input gradient is
// the transposed convolution with the flipped, channel-swapped kernel, and the weight
// gradients are direct 3x3 correlations of the output gradient with the layer input.
#include "common.cuh"

namespace ap {
namespace {

// fp64 throughout, like the reference (B200 keeps full-rate-ish FP64; training is off the decode
// path), and every reduction in a fixed order: two runs give bit-identical weights.
using real = double;

constexpr int C1 = 16, C2 = 32;
constexpr int OFF_W1 = 0, OFF_B1 = 144, OFF_W2 = 160, OFF_B2 = 4768, OFF_W3 = 4800, OFF_B3 = 4832;
constexpr int CT = 64;                         // corr2 tile columns
constexpr int CORR_CTAS = 296;                 // persistent CTAs of the d w2 reduction (2 per SM)
constexpr int CORR_OUT = C2 * C1 * 9 + C2;     // d_w2 then d_b2
constexpr int C1_CHUNKS = 148;                 // pixel chunks of the d w1 reduction
constexpr int HEAD_OUT = 2 + C2;               // loss, d_b3, d_w3[32] per head CTA

struct TrainWs {
    real* w2t;    // [16][32][9] flipped, channel-swapped w2 (conv2 input gradient)
    real* a1;     // [n][16][H][W] relu(s1)
    real* s2;     // [n][32][H][W] conv2 pre-activations
    real* dout;   // [n][W] d loss / d out
    real* ds2;    // [n][32][H][W]
    real* ds1;    // [n][16][H][W]
    real* part2;  // [CORR_CTAS][CORR_OUT]
    real* part1;  // [16][C1_CHUNKS][10]
    real* parth;  // [n * ceil(W/32)][HEAD_OUT]
};

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

size_t carve(TrainWs* ws, void* base, int64_t n, int64_t H, int64_t W) {
    const int64_t px = n * H * W;
    const size_t sizes[9] = {C1 * C2 * 9, (size_t)(C1 * px), (size_t)(C2 * px), (size_t)(n * W), (size_t)(C2 * px),
                             (size_t)(C1 * px), (size_t)CORR_CTAS * CORR_OUT, (size_t)C1 * C1_CHUNKS * 10,
                             (size_t)(n * ((W + 31) / 32)) * HEAD_OUT};
    real** dst[9] = {&ws->w2t, &ws->a1, &ws->s2, &ws->dout, &ws->ds2, &ws->ds1, &ws->part2, &ws->part1, &ws->parth};
    size_t off = 0;
    for (int i = 0; i < 9; ++i) {
        if (ws) *dst[i] = reinterpret_cast<real*>(static_cast<char*>(base) + off);
        off += align_up(sizes[i] * sizeof(real));
    }
    return off;
}

__device__ __forceinline__ real warp_sum(real v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void prep_weights_kernel(const real* __restrict__ w, real* __restrict__ w2t) {
    // w2t[k][c][tap] = w2[c][k][8 - tap]
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < C1 * C2 * 9; i += blockDim.x * gridDim.x) {
        const int tap = i % 9, c = (i / 9) % C2, k = i / (9 * C2);
        w2t[i] = w[OFF_W2 + (c * C1 + k) * 9 + (8 - tap)];
    }
}

// out[n][co][p] = bias[co] + sum_{ci, tap} w[co][ci][tap] * in[n][ci][p + off(tap)]  (zero pad 1)
// RELU: out = max(out, 0).  mask != nullptr: out = mask[n][co][p] > 0 ? out : 0.
// Each thread computes PX consecutive columns of one row, so every weight read from shared
// memory (a warp-wide broadcast) feeds PX FMAs and each input row segment of PX+2 values
// feeds 3·PX taps.  NT threads per CTA (measured: 64 for conv2, 128 for the others).
template <int CI, int CO, int PX, bool RELU, int NT>
__global__ void __launch_bounds__(NT) conv3x3_kernel(const real* __restrict__ in, const real* __restrict__ w,
                                                     const real* __restrict__ bias, const real* __restrict__ mask,
                                                     real* __restrict__ out, int H, int W) {
    __shared__ real sw[CO * CI * 9];
    for (int i = threadIdx.x; i < CO * CI * 9; i += blockDim.x) sw[i] = w[i];
    __syncthreads();
    const int x0 = (blockIdx.x * blockDim.x + threadIdx.x) * PX;
    const int y = blockIdx.y, n = blockIdx.z;
    if (x0 >= W) return;
    const int64_t plane = (int64_t)H * W;
    real acc[CO][PX];
#pragma unroll
    for (int co = 0; co < CO; ++co)
#pragma unroll
        for (int q = 0; q < PX; ++q) acc[co][q] = bias ? bias[co] : 0.0;
#pragma unroll 1
    for (int ci = 0; ci < CI; ++ci) {
        const real* src = in + ((int64_t)n * CI + ci) * plane;
        real v[3][PX + 2];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const int yy = y + r - 1;
#pragma unroll
            for (int j = 0; j < PX + 2; ++j) {
                const int xx = x0 + j - 1;
                v[r][j] = (yy >= 0 && yy < H && xx >= 0 && xx < W) ? src[(int64_t)yy * W + xx] : 0.0;
            }
        }
#pragma unroll
        for (int co = 0; co < CO; ++co)
#pragma unroll
            for (int t = 0; t < 9; ++t) {
                const real wt = sw[(co * CI + ci) * 9 + t];
#pragma unroll
                for (int q = 0; q < PX; ++q) acc[co][q] = fma(wt, v[t / 3][q + t % 3], acc[co][q]);
            }
    }
#pragma unroll
    for (int co = 0; co < CO; ++co)
#pragma unroll
        for (int q = 0; q < PX; ++q) {
            const int x = x0 + q;
            if (x >= W) continue;
            const int64_t o = ((int64_t)n * CO + co) * plane + (int64_t)y * W + x;
            real r = RELU ? fmax(acc[co][q], 0.0) : acc[co][q];
            if (mask && !(mask[o] > 0.0)) r = 0.0;
            out[o] = r;
        }
}

template <int CI, int CO, int PX, bool RELU, int NT>
void launch_conv(const real* in, const real* w, const real* bias, const real* mask, real* out, int n, int H, int W,
                 cudaStream_t st) {
    const dim3 grid((W + NT * PX - 1) / (NT * PX), H, n);
    conv3x3_kernel<CI, CO, PX, RELU, NT><<<grid, NT, 0, st>>>(in, w, bias, mask, out, H, W);
}

// z[c][lane] = mean_h relu(s2) of one column (predictor.py:196-198); shared by the training head and
// the inference-only fp64 forward so both form `out` with the same operations in the same order.
__device__ __forceinline__ void head_z(const real* __restrict__ s2, real (*zs)[33], int n, int x, bool live,
                                       int H, int W) {
    const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
    const int64_t plane = (int64_t)H * W;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int c = grp * 4 + j;
        real s = 0.0;
        if (live) {
            const real* src = s2 + ((int64_t)n * C2 + c) * plane + x;
            for (int y = 0; y < H; ++y) s += fmax(src[(int64_t)y * W], 0.0);
        }
        zs[c][lane] = s / H;
    }
}

// out = w3 . z + b3 (predictor.py:199)
__device__ __forceinline__ real head_out(const real* __restrict__ w, const real (*zs)[33], int lane) {
    real out = 0.0;
#pragma unroll
    for (int c = 0; c < C2; ++c) out = fma(w[OFF_W3 + c], zs[c][lane], out);
    return out + w[OFF_B3];
}

// Inference only: out[n][x] of predictor.forward in fp64 (one warp group per 32 columns).
__global__ void __launch_bounds__(256) head_fwd_kernel(const real* __restrict__ s2, const real* __restrict__ w,
                                                       real* __restrict__ out, int64_t out_stride, int H, int W) {
    __shared__ real zs[C2][33];
    const int lane = threadIdx.x & 31;
    const int x = blockIdx.x * 32 + lane, n = blockIdx.y;
    head_z(s2, zs, n, x, x < W, H, W);
    __syncthreads();
    if (threadIdx.x < 32 && x < W) out[(int64_t)n * out_stride + x] = head_out(w, zs, lane);
}

// z = mean_h relu(s2), out = w3.z + b3, the loss and d out; per-CTA partials of the loss,
// d b3 = sum d out and d w3 = sum z * d out (predictor.py:196-199,230-238).  CTA = 32 columns x
// 8 channel groups of 4: each thread sums its 4 channel planes down one column, z goes through
// shared memory to the group-0 warp, which forms out / resid / d out.
__global__ void __launch_bounds__(256) head_kernel(const real* __restrict__ s2, const real* __restrict__ w,
                                                   const real* __restrict__ target, real* __restrict__ dout,
                                                   real* __restrict__ parth, int H, int W) {
    __shared__ real zs[C2][33];
    __shared__ real ds[32];
    const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
    const int x = blockIdx.x * 32 + lane, n = blockIdx.y;
    const bool live = x < W;
    real* part = parth + ((int64_t)n * gridDim.x + blockIdx.x) * HEAD_OUT;
    head_z(s2, zs, n, x, live, H, W);
    __syncthreads();
    if (grp == 0) {
        const real out = head_out(w, zs, lane);
        const real resid = live ? out - target[(int64_t)n * W + x] : 0.0;
        const real d = 2.0 * resid / W;
        ds[lane] = d;
        if (live) dout[(int64_t)n * W + x] = d;
        const real l = warp_sum(resid * resid);
        const real db3 = warp_sum(d);
        if (lane == 0) {
            part[0] = l / W;
            part[1] = db3;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int c = grp * 4 + j;
        const real g = warp_sum(zs[c][lane] * ds[lane]);
        if (lane == 0) part[2 + c] = g;
    }
}

// loss_sum += sum of per-sample losses; grads[b3], grads[w3] += column sums.  One warp per
// output: lane-strided partial sums then a fixed shuffle tree (deterministic).
__global__ void head_finish_kernel(const real* __restrict__ parth, int n_samples, int xblocks,
                                   real* __restrict__ grads, real* __restrict__ loss_sum) {
    const int j = blockIdx.x, lane = threadIdx.x;
    const int64_t total = (int64_t)n_samples * xblocks;
    real s = 0.0;
    for (int64_t k = lane; k < total; k += 32) s += parth[k * HEAD_OUT + j];
    s = warp_sum(s);
    if (lane == 0) {
        if (j == 0) *loss_sum += s;
        else if (j == 1) grads[OFF_B3] += s;
        else grads[OFF_W3 + j - 2] += s;
    }
}

// d s2 = [s2 > 0] * w3[c] * d out[x] / H  (predictor.py:239-240)
__global__ void ds2_kernel(const real* __restrict__ s2, const real* __restrict__ w, const real* __restrict__ dout,
                           real* __restrict__ ds2, int H, int W, int64_t total) {
    const int64_t plane = (int64_t)H * W;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t nc = i / plane;
        const int c = (int)(nc % C2);
        const int64_t n = nc / C2;
        const int x = (int)(i % W);
        ds2[i] = s2[i] > 0.0 ? w[OFF_W3 + c] * dout[n * W + x] / H : 0.0;
    }
}

// d w1[k][tap] = sum_p d s1[k][p] * x_pad[p + off(tap)], d b1[k] = sum_p d s1[k][p].
// Grid (C1_CHUNKS, 16): fixed pixel assignment, warp-shuffle + shared-memory tree, one
// partial per (k, chunk) — no atomics.
__global__ void __launch_bounds__(256) corr1_kernel(const real* __restrict__ ds1, const real* __restrict__ x,
                                                    real* __restrict__ part1, int n_samples, int H, int W) {
    const int k = blockIdx.y;
    const int64_t plane = (int64_t)H * W, total = (int64_t)n_samples * plane;
    real acc[10];
#pragma unroll
    for (int i = 0; i < 10; ++i) acc[i] = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = i / plane, p = i % plane;
        const int y = (int)(p / W), xc = (int)(p % W);
        const real g = ds1[(n * C1 + k) * plane + p];
        if (g == 0.0) continue;  // relu-masked pixels contribute nothing
        acc[9] += g;
        const real* src = x + n * plane;
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            const int yy = y + t / 3 - 1, xx = xc + t % 3 - 1;
            if (yy >= 0 && yy < H && xx >= 0 && xx < W) acc[t] = fma(g, src[(int64_t)yy * W + xx], acc[t]);
        }
    }
    __shared__ real red[8][10];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const real v = warp_sum(acc[i]);
        if (lane == 0) red[wid][i] = v;
    }
    __syncthreads();
    if (threadIdx.x < 10) {
        real s = 0.0;
        for (int w8 = 0; w8 < 8; ++w8) s += red[w8][threadIdx.x];
        part1[((int64_t)k * gridDim.x + blockIdx.x) * 10 + threadIdx.x] = s;
    }
}

__global__ void corr1_finish_kernel(const real* __restrict__ part1, int chunks, real* __restrict__ grads) {
    const int j = threadIdx.x;  // k * 10 + i
    if (j >= C1 * 10) return;
    const int k = j / 10, i = j % 10;
    real s = 0.0;
    for (int c = 0; c < chunks; ++c) s += part1[((int64_t)k * chunks + c) * 10 + i];
    grads[i < 9 ? OFF_W1 + k * 9 + i : OFF_B1 + k] += s;
}

// d w2 / d b2 as a shared-memory tiled reduction: the 4608 outputs d_w2[a][b][tap] =
// sum_p d_s2[a][p] * a1_pad[b][p + off(tap)] form a 32 x 144 GEMM over pixels.  A persistent
// CTA walks 64-column row tiles (d_s2 rows [32][64], a1 rows y-1..y+1 with halo [16][3][66] in
// shared memory); thread t owns a-pair t/16 and b = t%16 (2 x 9 taps + 2 bias sums), sliding a
// 3-wide register window along the row so each pixel costs 2 + 3 shared loads for 18 FMAs.
// Per-CTA partials go to a [grid][4640] buffer and are summed in a fixed order.
__global__ void __launch_bounds__(256) corr2_tiled_kernel(const real* __restrict__ ds2, const real* __restrict__ a1,
                                                          real* __restrict__ partial, int n_samples, int H, int W) {
    __shared__ real As[C2][CT + 1];
    __shared__ real Bs[C1][3][CT + 2];
    const int tid = threadIdx.x, b = tid % 16, a0 = (tid / 16) * 2;
    real acc[2][9], bias[2] = {0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int t = 0; t < 9; ++t) acc[i][t] = 0.0;
    const int xt = (W + CT - 1) / CT;
    const int64_t n_tiles = (int64_t)n_samples * H * xt, plane = (int64_t)H * W;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int x0 = (int)(tile % xt) * CT;
        const int y = (int)((tile / xt) % H);
        const int64_t n = tile / ((int64_t)xt * H);
        __syncthreads();
        for (int i = tid; i < C2 * CT; i += 256) {
            const int c = i / CT, x = x0 + i % CT;
            As[c][i % CT] = x < W ? ds2[(n * C2 + c) * plane + (int64_t)y * W + x] : 0.0;
        }
        for (int i = tid; i < C1 * 3 * (CT + 2); i += 256) {
            const int c = i / (3 * (CT + 2)), r = (i / (CT + 2)) % 3, xx = x0 - 1 + i % (CT + 2), yy = y - 1 + r;
            Bs[c][r][i % (CT + 2)] =
                (yy >= 0 && yy < H && xx >= 0 && xx < W) ? a1[(n * C1 + c) * plane + (int64_t)yy * W + xx] : 0.0;
        }
        __syncthreads();
        real win[3][3];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            win[r][0] = Bs[b][r][0];
            win[r][1] = Bs[b][r][1];
        }
#pragma unroll 4
        for (int p = 0; p < CT; ++p) {
#pragma unroll
            for (int r = 0; r < 3; ++r) win[r][2] = Bs[b][r][p + 2];
            const real g0 = As[a0][p], g1 = As[a0 + 1][p];
            bias[0] += g0;
            bias[1] += g1;
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    acc[0][r * 3 + c] = fma(g0, win[r][c], acc[0][r * 3 + c]);
                    acc[1][r * 3 + c] = fma(g1, win[r][c], acc[1][r * 3 + c]);
                }
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                win[r][0] = win[r][1];
                win[r][1] = win[r][2];
            }
        }
    }
    real* out = partial + (int64_t)blockIdx.x * CORR_OUT;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
#pragma unroll
        for (int t = 0; t < 9; ++t) out[((a0 + i) * C1 + b) * 9 + t] = acc[i][t];
        if (b == 0) out[C2 * C1 * 9 + a0 + i] = bias[i];
    }
}

// grads[OFF_W2 + j] += sum over CTAs of partial[cta][j] (j < 4608), then d_b2; fixed order.
__global__ void corr2_finish_kernel(const real* __restrict__ partial, int n_parts, real* __restrict__ grads) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= CORR_OUT) return;
    real s = 0.0;
    for (int k = 0; k < n_parts; ++k) s += partial[(int64_t)k * CORR_OUT + j];
    grads[(j < C2 * C1 * 9 ? OFF_W2 + j : OFF_B2 + (j - C2 * C1 * 9))] += s;
}

// Adam (predictor.py:381-391), fp64, no FMA contraction so it rounds like numpy.
__global__ void adam_kernel(double* __restrict__ w, double* __restrict__ m, double* __restrict__ v,
                            const double* __restrict__ gsum, int n, double batch, double lr, double beta1,
                            double beta2, double eps, double corr1, double corr2) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += blockDim.x * gridDim.x) {
        const double g = __ddiv_rn(gsum[i], batch);
        const double mt = __dadd_rn(__dmul_rn(m[i], beta1), __dmul_rn(__dadd_rn(1.0, -beta1), g));
        const double vt = __dadd_rn(__dmul_rn(v[i], beta2), __dmul_rn(__dmul_rn(__dadd_rn(1.0, -beta2), g), g));
        m[i] = mt;
        v[i] = vt;
        const double step = __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mt, corr1)), __dadd_rn(__dsqrt_rn(__ddiv_rn(vt, corr2)), eps));
        w[i] = __dadd_rn(w[i], -step);
    }
}

int grid_for(int64_t work, int threads) {
    int64_t b = (work + threads - 1) / threads;
    return (int)(b < 148 * 8 ? (b < 1 ? 1 : b) : 148 * 8);
}

}  // namespace
}  // namespace ap

using namespace ap;

extern "C" {

int64_t ap_train_workspace_bytes(int32_t n_samples, int32_t H, int32_t W) {
    if (n_samples < 1 || H < 1 || W < 1) return 0;
    return (int64_t)carve(nullptr, nullptr, n_samples, H, W);
}

int ap_train_backward(const double* grids, const double* targets, int32_t n_samples, int32_t H, int32_t W,
                      const double* weights, double* grads, double* loss_sum, void* workspace,
                      int64_t workspace_bytes, void* stream) {
    AP_REQUIRE(n_samples >= 1 && H >= 1 && W >= 1, AP_EPARAM, "bad batch shape");
    AP_REQUIRE(grids && targets && weights && grads && loss_sum && workspace, AP_EPARAM, "null pointer");
    AP_REQUIRE(H <= 65535 && n_samples <= 65535, AP_EPARAM, "H and n_samples must be <= 65535");
    AP_REQUIRE(workspace_bytes >= ap_train_workspace_bytes(n_samples, H, W), AP_EPARAM, "workspace too small");
    cudaStream_t st = as_stream(stream);
    TrainWs ws;
    carve(&ws, workspace, n_samples, H, W);
    const int64_t px = (int64_t)n_samples * H * W;
    prep_weights_kernel<<<8, 512, 0, st>>>(weights, ws.w2t);
    launch_conv<1, C1, 2, true, 128>(grids, weights + OFF_W1, weights + OFF_B1, nullptr, ws.a1, n_samples, H, W, st);
    launch_conv<C1, C2, 1, false, 64>(ws.a1, weights + OFF_W2, weights + OFF_B2, nullptr, ws.s2, n_samples, H, W, st);
    const int xblocks = (W + 31) / 32;
    head_kernel<<<dim3(xblocks, n_samples), 256, 0, st>>>(ws.s2, weights, targets, ws.dout, ws.parth, H, W);
    head_finish_kernel<<<HEAD_OUT, 32, 0, st>>>(ws.parth, n_samples, xblocks, grads, loss_sum);
    ds2_kernel<<<grid_for(C2 * px, 256), 256, 0, st>>>(ws.s2, weights, ws.dout, ws.ds2, H, W, C2 * px);
    corr2_tiled_kernel<<<CORR_CTAS, 256, 0, st>>>(ws.ds2, ws.a1, ws.part2, n_samples, H, W);
    corr2_finish_kernel<<<(CORR_OUT + 255) / 256, 256, 0, st>>>(ws.part2, CORR_CTAS, grads);
    // d a1 = conv2^T(d s2); d s1 = [a1 > 0] * d a1  (predictor.py:243-245; a1 > 0 <=> s1 > 0)
    launch_conv<C2, C1, 2, false, 128>(ws.ds2, ws.w2t, nullptr, ws.a1, ws.ds1, n_samples, H, W, st);
    corr1_kernel<<<dim3(C1_CHUNKS, C1), 256, 0, st>>>(ws.ds1, grids, ws.part1, n_samples, H, W);
    corr1_finish_kernel<<<1, 192, 0, st>>>(ws.part1, C1_CHUNKS, grads);
    return launch_status("ap_train_backward");
}

int64_t ap_forward_f64_workspace_bytes(int32_t n_grids, int32_t H, int32_t W) {
    if (n_grids < 1 || H < 1 || W < 1) return 0;
    return (int64_t)align_up(sizeof(real) * (size_t)(C1 + C2) * n_grids * H * W);
}

int ap_predict_forward_f64(const double* grids, int32_t n_grids, int32_t H, int32_t W, const double* weights,
                           double* out, int64_t out_stride, void* workspace, int64_t workspace_bytes, void* stream) {
    AP_REQUIRE(n_grids >= 0 && H >= 1 && W >= 1, AP_EPARAM, "bad grid shape");
    AP_REQUIRE(H <= 65535 && n_grids <= 65535 && out_stride >= W, AP_EPARAM, "bad sizes");
    if (n_grids == 0) return AP_OK;
    AP_REQUIRE(grids && weights && out && workspace, AP_EPARAM, "null pointer");
    AP_REQUIRE(workspace_bytes >= ap_forward_f64_workspace_bytes(n_grids, H, W), AP_EPARAM, "workspace too small");
    cudaStream_t st = as_stream(stream);
    real* a1 = static_cast<real*>(workspace);
    real* s2 = a1 + (int64_t)C1 * n_grids * H * W;
    // the same conv kernels and head arithmetic as ap_train_backward, so `out` here equals the
    // forward that backward differentiates bit for bit
    launch_conv<1, C1, 2, true, 128>(grids, weights + OFF_W1, weights + OFF_B1, nullptr, a1, n_grids, H, W, st);
    launch_conv<C1, C2, 1, false, 64>(a1, weights + OFF_W2, weights + OFF_B2, nullptr, s2, n_grids, H, W, st);
    head_fwd_kernel<<<dim3((W + 31) / 32, n_grids), 256, 0, st>>>(s2, weights, out, out_stride, H, W);
    return launch_status("ap_predict_forward_f64");
}

int ap_adam_step(double* weights, double* m, double* v, const double* grad_sum, int32_t n_params, double batch,
                 double lr, double beta1, double beta2, double eps, int64_t step, void* stream) {
    AP_REQUIRE(weights && m && v && grad_sum && n_params >= 0, AP_EPARAM, "bad Adam arguments");
    AP_REQUIRE(step >= 1, AP_EPARAM, "Adam step counts from 1");
    const double corr1 = 1.0 - pow(beta1, (double)step), corr2 = 1.0 - pow(beta2, (double)step);
    adam_kernel<<<grid_for(n_params, 256), 256, 0, as_stream(stream)>>>(weights, m, v, grad_sum, n_params, batch,
                                                                        lr, beta1, beta2, eps, corr1, corr2);
    return launch_status("ap_adam_step");
}

}  // extern "C"
