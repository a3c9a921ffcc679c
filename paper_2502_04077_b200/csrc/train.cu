// Forecaster training on the device: exact gradients of the MSE loss (predictor.backward,
// predictor.py:219-251) for a batch of equal-shape samples, and the Adam update of
// predictor.train (predictor.py:371-391).
//
// This is not the decode hot path: the kernels are plain SIMT,
// fp32 arithmetic with fp64 accumulation of every reduction over pixels, one thread per
// pixel for the convolutions (channel planes [n][C][H][W], so a warp reads 32 consecutive
// columns of a plane) and one CTA row per output channel group for the weight gradients.
// The reference's im2col / col2im matrices are never formed: the conv2 input gradient is
// the transposed convolution with the flipped, channel-swapped kernel, and the weight
// gradients are direct 3x3 correlations of the output gradient with the layer input.
#include "common.cuh"

namespace ap {
namespace {

constexpr int C1 = 16, C2 = 32;
constexpr int OFF_W1 = 0, OFF_B1 = 144, OFF_W2 = 160, OFF_B2 = 4768, OFF_W3 = 4800, OFF_B3 = 4832;

struct TrainWs {
    float* wf;    // 4833 fp32 weights
    float* w2t;   // [16][32][9] flipped, channel-swapped w2 (conv2 input gradient)
    float* a1;    // [n][16][H][W] relu(s1)
    float* s2;    // [n][32][H][W] conv2 pre-activations
    float* dout;  // [n][W] d loss / d out
    float* ds2;   // [n][32][H][W]
    float* ds1;   // [n][16][H][W]
    double* part; // [CORR_CTAS][CORR_OUT] per-CTA d_w2 / d_b2 partials
};

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

size_t carve(TrainWs* ws, void* base, int64_t n, int64_t H, int64_t W) {
    const int64_t px = n * H * W;
    const size_t sizes[8] = {AP_PARAM_COUNT * 4, 16 * 32 * 9 * 4, (size_t)(C1 * px) * 4, (size_t)(C2 * px) * 4,
                             (size_t)(n * W) * 4, (size_t)(C2 * px) * 4, (size_t)(C1 * px) * 4,
                             (size_t)296 * (32 * 16 * 9 + 32) * 8};
    float** dst[8] = {&ws->wf, &ws->w2t, &ws->a1, &ws->s2, &ws->dout, &ws->ds2, &ws->ds1,
                      reinterpret_cast<float**>(&ws->part)};
    size_t off = 0;
    for (int i = 0; i < 8; ++i) {
        if (ws) *dst[i] = reinterpret_cast<float*>(static_cast<char*>(base) + off);
        off += align_up(sizes[i]);
    }
    return off;
}

__global__ void prep_weights_kernel(const double* __restrict__ w, float* __restrict__ wf, float* __restrict__ w2t) {
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < AP_PARAM_COUNT; i += blockDim.x * gridDim.x)
        wf[i] = (float)w[i];
    // w2t[k][c][tap] = w2[c][k][8 - tap]
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < C1 * C2 * 9; i += blockDim.x * gridDim.x) {
        const int tap = i % 9, c = (i / 9) % C2, k = i / (9 * C2);
        w2t[i] = (float)w[OFF_W2 + (c * C1 + k) * 9 + (8 - tap)];
    }
}

// out[n][co][p] = bias[co] + sum_{ci, tap} w[co][ci][tap] * in[n][ci][p + off(tap)]  (zero pad 1)
// RELU: out = max(out, 0).  mask != nullptr: out = mask[n][co][p] > 0 ? out : 0.
// Each thread computes PX consecutive columns of one row, so every weight read from shared
// memory (a warp-wide broadcast) feeds PX FMAs and each input row segment of PX+2 values
// feeds 3·PX taps.
template <int CI, int CO, int PX, bool RELU>
__global__ void __launch_bounds__(64) conv3x3_kernel(const float* __restrict__ in, const float* __restrict__ w,
                                                     const float* __restrict__ bias, const float* __restrict__ mask,
                                                     float* __restrict__ out, int H, int W) {
    __shared__ float sw[CO * CI * 9];
    for (int i = threadIdx.x; i < CO * CI * 9; i += blockDim.x) sw[i] = w[i];
    __syncthreads();
    const int x0 = (blockIdx.x * blockDim.x + threadIdx.x) * PX;
    const int y = blockIdx.y, n = blockIdx.z;
    if (x0 >= W) return;
    const int64_t plane = (int64_t)H * W;
    float acc[CO][PX];
#pragma unroll
    for (int co = 0; co < CO; ++co)
#pragma unroll
        for (int q = 0; q < PX; ++q) acc[co][q] = bias ? bias[co] : 0.f;
#pragma unroll 1
    for (int ci = 0; ci < CI; ++ci) {
        const float* src = in + ((int64_t)n * CI + ci) * plane;
        float v[3][PX + 2];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const int yy = y + r - 1;
#pragma unroll
            for (int j = 0; j < PX + 2; ++j) {
                const int xx = x0 + j - 1;
                v[r][j] = (yy >= 0 && yy < H && xx >= 0 && xx < W) ? src[(int64_t)yy * W + xx] : 0.f;
            }
        }
#pragma unroll
        for (int co = 0; co < CO; ++co)
#pragma unroll
            for (int t = 0; t < 9; ++t) {
                const float wt = sw[(co * CI + ci) * 9 + t];
#pragma unroll
                for (int q = 0; q < PX; ++q) acc[co][q] = fmaf(wt, v[t / 3][q + t % 3], acc[co][q]);
            }
    }
#pragma unroll
    for (int co = 0; co < CO; ++co)
#pragma unroll
        for (int q = 0; q < PX; ++q) {
            const int x = x0 + q;
            if (x >= W) continue;
            const int64_t o = ((int64_t)n * CO + co) * plane + (int64_t)y * W + x;
            float r = RELU ? fmaxf(acc[co][q], 0.f) : acc[co][q];
            if (mask && !(mask[o] > 0.f)) r = 0.f;
            out[o] = r;
        }
}

template <int CI, int CO, int PX, bool RELU>
void launch_conv(const float* in, const float* w, const float* bias, const float* mask, float* out, int n, int H,
                 int W, cudaStream_t st) {
    const dim3 grid((W + 64 * PX - 1) / (64 * PX), H, n);
    conv3x3_kernel<CI, CO, PX, RELU><<<grid, 64, 0, st>>>(in, w, bias, mask, out, H, W);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// z = mean_h relu(s2), out = w3.z + b3, the loss and d out, d w3 = sum z * d out, d b3 = sum d out
// (predictor.py:196-199,230-238).  CTA = 32 columns x 8 channel groups of 4: each thread sums its
// 4 channel planes down one column, z goes through shared memory to the group-0 warp, which forms
// out / resid / d out; then every thread reduces z * d out for its channels.
__global__ void __launch_bounds__(256) head_kernel(const float* __restrict__ s2, const float* __restrict__ wf,
                                                   const float* __restrict__ target, float* __restrict__ dout,
                                                   double* __restrict__ grads, double* __restrict__ loss_sum,
                                                   int H, int W) {
    __shared__ float zs[C2][33];
    __shared__ float ds[32];
    const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
    const int x = blockIdx.x * 32 + lane, n = blockIdx.y;
    const bool live = x < W;
    const int64_t plane = (int64_t)H * W;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int c = grp * 4 + j;
        float s = 0.f;
        if (live) {
            const float* src = s2 + ((int64_t)n * C2 + c) * plane + x;
            for (int y = 0; y < H; ++y) s += fmaxf(src[(int64_t)y * W], 0.f);
        }
        zs[c][lane] = s / (float)H;
    }
    __syncthreads();
    if (grp == 0) {
        float out = wf[OFF_B3];
#pragma unroll
        for (int c = 0; c < C2; ++c) out = fmaf(wf[OFF_W3 + c], zs[c][lane], out);
        const float resid = live ? out - target[(int64_t)n * W + x] : 0.f;
        const float d = 2.f * resid / (float)W;
        ds[lane] = d;
        if (live) dout[(int64_t)n * W + x] = d;
        const double l = warp_sum((double)resid * resid / W);
        const double db3 = warp_sum((double)d);
        if (lane == 0) {
            atomicAdd(loss_sum, l);
            atomicAdd(grads + OFF_B3, db3);
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int c = grp * 4 + j;
        const double g = warp_sum((double)zs[c][lane] * ds[lane]);
        if (lane == 0) atomicAdd(grads + OFF_W3 + c, g);
    }
}

// d s2 = [s2 > 0] * w3[c] * d out[x] / H  (predictor.py:239-240)
__global__ void ds2_kernel(const float* __restrict__ s2, const float* __restrict__ wf, const float* __restrict__ dout,
                           float* __restrict__ ds2, int H, int W, int64_t total) {
    const int64_t plane = (int64_t)H * W;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t nc = i / plane;
        const int c = (int)(nc % C2);
        const int64_t n = nc / C2;
        const int x = (int)(i % W);
        ds2[i] = s2[i] > 0.f ? wf[OFF_W3 + c] * dout[n * W + x] / (float)H : 0.f;
    }
}

// g_w[a][b][tap] += sum_p A[n][a][p] * B[n][b][p + off(tap)]   (zero pad 1)
// g_b[a]         += sum_p A[n][a][p]                              (when b-group 0)
// Grid: (pixel chunks, CA * CB / BG).  Each thread keeps BG*9 + 1 fp32 partials over its
// pixels (a few hundred terms), the CTA reduces them in fp64 and adds them atomically.
template <int CA, int CB, int BG>
__global__ void __launch_bounds__(256) corr_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                   double* __restrict__ gw, double* __restrict__ gb, int n_samples,
                                                   int H, int W) {
    const int a = blockIdx.y / (CB / BG), b0 = (blockIdx.y % (CB / BG)) * BG;
    const int64_t plane = (int64_t)H * W, total = (int64_t)n_samples * plane;
    float acc[BG * 9 + 1];
#pragma unroll
    for (int i = 0; i < BG * 9 + 1; ++i) acc[i] = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = i / plane, p = i % plane;
        const int y = (int)(p / W), x = (int)(p % W);
        const float g = A[(n * CA + a) * plane + p];
        if (g == 0.f) continue;  // relu-masked pixels contribute nothing
        acc[BG * 9] += g;
#pragma unroll
        for (int j = 0; j < BG; ++j) {
            const float* src = B + (n * CB + b0 + j) * plane;
#pragma unroll
            for (int t = 0; t < 9; ++t) {
                const int yy = y + t / 3 - 1, xx = x + t % 3 - 1;
                if (yy >= 0 && yy < H && xx >= 0 && xx < W) acc[j * 9 + t] = fmaf(g, src[(int64_t)yy * W + xx], acc[j * 9 + t]);
            }
        }
    }
    __shared__ double red[8][BG * 9 + 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < BG * 9 + 1; ++i) {
        double v = warp_sum((double)acc[i]);
        if (lane == 0) red[wid][i] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < BG * 9 + 1; i += blockDim.x) {
        double s = 0.0;
        for (int w8 = 0; w8 < (int)(blockDim.x >> 5); ++w8) s += red[w8][i];
        if (i < BG * 9) {
            atomicAdd(gw + (a * CB + b0 + i / 9) * 9 + i % 9, s);
        } else if (b0 == 0) {
            atomicAdd(gb + a, s);
        }
    }
}

// d w2 / d b2 as a shared-memory tiled reduction: the 4608 outputs d_w2[a][b][tap] =
// sum_p d_s2[a][p] * a1_pad[b][p + off(tap)] form a 32 x 144 GEMM over pixels.  A persistent
// CTA walks 64-column row tiles (d_s2 rows [32][64], a1 rows y-1..y+1 with halo [16][3][66] in
// shared memory); thread t owns a-pair t/16 and b = t%16 (2 x 9 taps = 18 fp32 accumulators),
// sliding a 3-wide register window along the row so each pixel costs 2 + 3 shared loads for
// 18 FMAs.  Each tile's fp32 sums are folded into fp64 registers; per-CTA partials go to a
// [grid][4640] fp64 buffer and are summed in a fixed order (run-to-run deterministic).
constexpr int CT = 64;        // tile columns
constexpr int CORR_CTAS = 296;
constexpr int CORR_OUT = C2 * C1 * 9 + C2;  // d_w2 then d_b2

__global__ void __launch_bounds__(256) corr2_tiled_kernel(const float* __restrict__ ds2, const float* __restrict__ a1,
                                                          double* __restrict__ partial, int n_samples, int H, int W) {
    __shared__ float As[C2][CT + 1];
    __shared__ float Bs[C1][3][CT + 2];
    const int tid = threadIdx.x, b = tid % 16, a0 = (tid / 16) * 2;
    double tot[2][10];  // per-tile fp32 sums folded into fp64 (tiles are 64 pixels)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int t = 0; t < 10; ++t) tot[i][t] = 0.0;
    const int xt = (W + CT - 1) / CT;
    const int64_t n_tiles = (int64_t)n_samples * H * xt, plane = (int64_t)H * W;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int x0 = (int)(tile % xt) * CT;
        const int y = (int)((tile / xt) % H);
        const int64_t n = tile / ((int64_t)xt * H);
        __syncthreads();
        for (int i = tid; i < C2 * CT; i += 256) {
            const int c = i / CT, x = x0 + i % CT;
            As[c][i % CT] = x < W ? ds2[(n * C2 + c) * plane + (int64_t)y * W + x] : 0.f;
        }
        for (int i = tid; i < C1 * 3 * (CT + 2); i += 256) {
            const int c = i / (3 * (CT + 2)), r = (i / (CT + 2)) % 3, xx = x0 - 1 + i % (CT + 2), yy = y - 1 + r;
            Bs[c][r][i % (CT + 2)] =
                (yy >= 0 && yy < H && xx >= 0 && xx < W) ? a1[(n * C1 + c) * plane + (int64_t)yy * W + xx] : 0.f;
        }
        __syncthreads();
        float acc[2][9], bias[2] = {0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int t = 0; t < 9; ++t) acc[i][t] = 0.f;
        float win[3][3];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            win[r][0] = Bs[b][r][0];
            win[r][1] = Bs[b][r][1];
        }
#pragma unroll 4
        for (int p = 0; p < CT; ++p) {
#pragma unroll
            for (int r = 0; r < 3; ++r) win[r][2] = Bs[b][r][p + 2];
            const float g0 = As[a0][p], g1 = As[a0 + 1][p];
            bias[0] += g0;
            bias[1] += g1;
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    acc[0][r * 3 + c] = fmaf(g0, win[r][c], acc[0][r * 3 + c]);
                    acc[1][r * 3 + c] = fmaf(g1, win[r][c], acc[1][r * 3 + c]);
                }
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                win[r][0] = win[r][1];
                win[r][1] = win[r][2];
            }
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
#pragma unroll
            for (int t = 0; t < 9; ++t) tot[i][t] += acc[i][t];
            tot[i][9] += bias[i];
        }
    }
    double* out = partial + (int64_t)blockIdx.x * CORR_OUT;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
#pragma unroll
        for (int t = 0; t < 9; ++t) out[((a0 + i) * C1 + b) * 9 + t] = tot[i][t];
        if (b == 0) out[C2 * C1 * 9 + a0 + i] = tot[i][9];
    }
}

// grads[OFF_W2 + j] += sum over CTAs of partial[cta][j] (j < 4608), then d_b2; fixed order.
__global__ void corr2_finish_kernel(const double* __restrict__ partial, int n_parts, double* __restrict__ grads) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= CORR_OUT) return;
    double s = 0.0;
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

int ap_train_backward(const float* grids, const float* targets, int32_t n_samples, int32_t H, int32_t W,
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
    prep_weights_kernel<<<8, 512, 0, st>>>(weights, ws.wf, ws.w2t);
    launch_conv<1, C1, 4, true>(grids, ws.wf + OFF_W1, ws.wf + OFF_B1, nullptr, ws.a1, n_samples, H, W, st);
    launch_conv<C1, C2, 2, false>(ws.a1, ws.wf + OFF_W2, ws.wf + OFF_B2, nullptr, ws.s2, n_samples, H, W, st);
    head_kernel<<<dim3((W + 31) / 32, n_samples), 256, 0, st>>>(ws.s2, ws.wf, targets, ws.dout, grads, loss_sum, H, W);
    ds2_kernel<<<grid_for(C2 * px, 256), 256, 0, st>>>(ws.s2, ws.wf, ws.dout, ws.ds2, H, W, C2 * px);
    const int chunks = grid_for(px, 256) / 4 + 1;
    corr2_tiled_kernel<<<CORR_CTAS, 256, 0, st>>>(ws.ds2, ws.a1, ws.part, n_samples, H, W);
    corr2_finish_kernel<<<(CORR_OUT + 255) / 256, 256, 0, st>>>(ws.part, CORR_CTAS, grads);
    // d a1 = conv2^T(d s2); d s1 = [a1 > 0] * d a1  (predictor.py:243-245; a1 > 0 <=> s1 > 0)
    launch_conv<C2, C1, 4, false>(ws.ds2, ws.w2t, nullptr, ws.a1, ws.ds1, n_samples, H, W, st);
    corr_kernel<C1, 1, 1><<<dim3(chunks, C1), 256, 0, st>>>(ws.ds1, grids, grads + OFF_W1, grads + OFF_B1, n_samples,
                                                            H, W);
    return launch_status("ap_train_backward");
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
