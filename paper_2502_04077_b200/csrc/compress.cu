// Kernel (1): block-wise max-pool compression and the history-ring append.
//
// Reference: compress.max_pool (compress.py:28-40), compress.expand_indices
// (compress.py:43-57), the history append of selector.step
// (selector.py:112-120) and the observed-row masking of the evaluation loop
// (evaluation.py:109-112).  Max is exact, so every output here is bit-exact
// against the float64 oracle for float32/float64 inputs.
#include "common.cuh"

namespace ap {

// max over positions [j*b, j*b+b) of v(p) where v(p) = row[p] for p < t and
// take(p), else 0 (zero padding / unselected).  Returns the max in double.
template <typename T, typename Take>
__device__ __forceinline__ double block_max(const T* row, int64_t t, int b, int64_t j, Take take) {
    const int64_t lo = j * (int64_t)b;
    const int64_t hi = lo + b;
    const int64_t end = hi < t ? hi : t;
    double m = 0.0;
    bool have = false;
    for (int64_t p = lo; p < end; ++p) {
        double v = take(p) ? to_f64(row[p]) : 0.0;
        m = have ? np_max(m, v) : v;
        have = true;
    }
    if (end < hi) m = have ? np_max(m, 0.0) : 0.0;  // zero pad of the tail block
    return m;
}

// Fast path: fp32 rows, b == 16, 16-byte aligned rows, every position taken.
__device__ __forceinline__ float block_max16_f32(const float* row, int64_t t, int64_t j) {
    const int64_t lo = j * 16;
    if (lo + 16 <= t) {
        const float4* p = reinterpret_cast<const float4*>(row + lo);
        float4 a = __ldg(p), c = __ldg(p + 1), d = __ldg(p + 2), e = __ldg(p + 3);
        float m = np_max(np_max(np_max(a.x, a.y), np_max(a.z, a.w)), np_max(np_max(c.x, c.y), np_max(c.z, c.w)));
        m = np_max(m, np_max(np_max(np_max(d.x, d.y), np_max(d.z, d.w)), np_max(np_max(e.x, e.y), np_max(e.z, e.w))));
        return m;
    }
    float m = row[lo];
    for (int64_t p = lo + 1; p < t; ++p) m = np_max(m, row[p]);
    return np_max(m, 0.0f);
}

struct TakeAll {
    __device__ bool operator()(int64_t) const { return true; }
};

template <typename T, typename O>
__global__ void max_pool_kernel(const T* __restrict__ rows, int64_t n_rows, int64_t row_stride, int64_t t,
                                int b, O* __restrict__ out, int64_t out_stride, int64_t W) {
    const int64_t i = blockIdx.y;
    const T* row = rows + i * row_stride;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < W; j += (int64_t)gridDim.x * blockDim.x) {
        double m = block_max(row, t, b, j, TakeAll{});
        out[i * out_stride + j] = (O)m;
    }
}

__global__ void max_pool_f32_b16_kernel(const float* __restrict__ rows, int64_t row_stride, int64_t t,
                                        float* __restrict__ out, int64_t out_stride, int64_t W) {
    const int64_t i = blockIdx.y;
    const float* row = rows + i * row_stride;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < W; j += (int64_t)gridDim.x * blockDim.x)
        out[i * out_stride + j] = block_max16_f32(row, t, j);
}

__global__ void expand_kernel(const int32_t* __restrict__ blocks, int32_t n_blocks, int32_t b, int64_t t,
                              int64_t* __restrict__ tokens, int32_t* __restrict__ n_tokens, int32_t* status) {
    __shared__ int warp_tot[9];
    const int64_t nb = cdiv64(t, b);
    int64_t base = 0;
    for (int32_t c0 = 0; c0 < n_blocks; c0 += 256) {
        const int32_t i = c0 + threadIdx.x;
        int len = 0;
        int64_t j = -1;
        if (i < n_blocks) {
            j = blocks[i];
            if (j < 0 || j >= nb) {
                raise_status(status, AP_EPARAM);
            } else {
                int64_t end = j * b + b < t ? j * b + b : t;
                len = (int)(end - j * b);
            }
        }
        int total = 0;
        int off = block_excl_scan<256>(len, warp_tot, total);
        for (int q = 0; q < len; ++q) tokens[base + off + q] = j * b + q;
        base += total;
    }
    if (threadIdx.x == 0) *n_tokens = (int32_t)base;
}

// ------------------------------------------------------------------ selector
__global__ void sel_reset_kernel(ap_selector s) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < s.n_maps) {
        ap_map_state z;
        z.n_pushed = 0; z.r_pushed = -1; z.row_len = 0; z.counter = 0; z.mid_clip = 0;
        z.width = 0; z.r_width = 0; z.n_mid = 0; z.r_wgen = 0; z.tie_n = 0; z.prev_kth = 0;
        s.state[i] = z;
    }
    // slot content unknown after a reset: the first push into a slot zero-fills [W, w_max), so ring rows
    // are always zero beyond their own width (the forecaster relies on it instead of per-slot masks)
    if (i < (int64_t)s.n_maps * s.history) s.slot_width[i] = s.w_max;
    const int64_t words = (s.w_max + 31) / 32;
    for (int64_t k = i; k < (int64_t)s.n_maps * words; k += (int64_t)gridDim.x * blockDim.x) s.mid_mask[k] = 0u;
    if (i == 0) *s.status = 0;
}

// Previous selection of a map (selector.py:122-147): sink ∪ local over
// next_len, plus middle blocks clipped to mid_clip.
struct PrevSelection {
    int64_t nl, sink_end, local_start, mid_clip;
    int b;
    const uint32_t* mask;
    __device__ bool operator()(int64_t p) const {
        if (p < sink_end) return true;
        if (p >= local_start && p < nl) return true;
        int64_t j = p / b;
        return p < mid_clip && ((mask[j >> 5] >> (j & 31)) & 1u);
    }
};

// One CTA per map: compress the map's row and append it to the ring.
template <typename T>
__global__ void sel_push_kernel(ap_selector s, const T* __restrict__ rows, int64_t row_stride, int64_t t,
                                int mode) {
    const int m = blockIdx.x;
    ap_map_state st = s.state[m];
    const int b = s.block;
    const int64_t W = cdiv64(t, b);
    const int H = s.history;
    const int slot = (int)(st.n_pushed % H);
    float* dst = s.ring + ((int64_t)m * H + slot) * s.w_max;
    const T* row = rows + (int64_t)m * row_stride;
    const bool calibrate = (st.counter % s.calib_period) == 0;
    const bool masked = (mode == 1) && !calibrate && st.n_pushed > 0 && st.row_len > 0;
    float mx = 0.f;  // max |x| of the row (forecaster operand scale)
    if (masked) {
        PrevSelection sel;
        sel.nl = st.row_len + 1;
        sel.sink_end = s.sink < sel.nl ? s.sink : sel.nl;
        sel.local_start = sel.nl - s.local > 0 ? sel.nl - s.local : 0;
        sel.mid_clip = st.mid_clip;
        sel.b = b;
        sel.mask = s.mid_mask + (int64_t)m * ((s.w_max + 31) / 32);
        for (int64_t j = threadIdx.x; j < W; j += blockDim.x) {
            const float v = (float)block_max(row, t, b, j, sel);
            dst[j] = v;
            mx = track_row_max(mx, v, s.status);
        }
    } else {
        for (int64_t j = threadIdx.x; j < W; j += blockDim.x) {
            const float v = (float)block_max(row, t, b, j, TakeAll{});
            dst[j] = v;
            mx = track_row_max(mx, v, s.status);
        }
    }
    const int old_w = s.slot_width[(int64_t)m * H + slot];
    for (int64_t j = W + threadIdx.x; j < old_w; j += blockDim.x) dst[j] = 0.f;  // keep the row zero beyond W
    mx = cta_max_nonneg(mx);
    if (threadIdx.x == 0) {
        s.slot_xmax[(int64_t)m * H + slot] = mx;
        s.slot_width[(int64_t)m * H + slot] = (int32_t)W;
        st.n_pushed += 1;
        st.row_len = t;
        st.width = (int32_t)W;
        s.state[m] = st;
    }
}

__global__ void sel_push_f32_b16_kernel(ap_selector s, const float* __restrict__ rows, int64_t row_stride,
                                        int64_t t) {
    const int m = blockIdx.x;
    ap_map_state st = s.state[m];
    const int64_t W = cdiv64(t, 16);
    const int H = s.history;
    const int slot = (int)(st.n_pushed % H);
    float* dst = s.ring + ((int64_t)m * H + slot) * s.w_max;
    const float* row = rows + (int64_t)m * row_stride;
    float mx = 0.f;
    for (int64_t j = threadIdx.x; j < W; j += blockDim.x) {
        const float v = block_max16_f32(row, t, j);
        dst[j] = v;
        mx = track_row_max(mx, v, s.status);
    }
    const int old_w = s.slot_width[(int64_t)m * H + slot];
    for (int64_t j = W + threadIdx.x; j < old_w; j += blockDim.x) dst[j] = 0.f;  // keep the row zero beyond W
    mx = cta_max_nonneg(mx);
    if (threadIdx.x == 0) {
        s.slot_xmax[(int64_t)m * H + slot] = mx;
        s.slot_width[(int64_t)m * H + slot] = (int32_t)W;
        st.n_pushed += 1;
        st.row_len = t;
        st.width = (int32_t)W;
        s.state[m] = st;
    }
}

__global__ void sel_push_compressed_kernel(ap_selector s, const float* __restrict__ comp, int64_t comp_stride,
                                           int64_t t) {
    const int m = blockIdx.x;
    ap_map_state st = s.state[m];
    const int64_t W = cdiv64(t, s.block);
    const int H = s.history;
    const int slot = (int)(st.n_pushed % H);
    float* dst = s.ring + ((int64_t)m * H + slot) * s.w_max;
    const float* src = comp + (int64_t)m * comp_stride;
    float mx = 0.f;
    for (int64_t j = threadIdx.x; j < W; j += blockDim.x) {
        const float v = src[j];
        dst[j] = v;
        mx = track_row_max(mx, v, s.status);
    }
    const int old_w = s.slot_width[(int64_t)m * H + slot];
    for (int64_t j = W + threadIdx.x; j < old_w; j += blockDim.x) dst[j] = 0.f;  // keep the row zero beyond W
    mx = cta_max_nonneg(mx);
    if (threadIdx.x == 0) {
        s.slot_xmax[(int64_t)m * H + slot] = mx;
        s.slot_width[(int64_t)m * H + slot] = (int32_t)W;
        st.n_pushed += 1;
        st.row_len = t;
        st.width = (int32_t)W;
        s.state[m] = st;
    }
}

}  // namespace ap

using namespace ap;

extern "C" {

int ap_max_pool(const void* rows, int in_dtype, int64_t n_rows, int64_t row_stride, int64_t t, int32_t b,
                void* out, int out_dtype, int64_t out_stride, void* stream) {
    AP_REQUIRE(b >= 1, AP_EPARAM, "block size must be >= 1");
    AP_REQUIRE(t >= 1, AP_EPARAM, "row must be a non-empty 1-D vector");
    AP_REQUIRE(n_rows >= 0 && n_rows <= 65535, AP_EPARAM, "n_rows out of range");
    AP_REQUIRE(in_dtype == AP_F32 || in_dtype == AP_F64, AP_EPARAM, "rows must be float32 or float64");
    AP_REQUIRE(out_dtype == AP_F32 || out_dtype == AP_F64, AP_EPARAM, "out must be float32 or float64");
    AP_REQUIRE(!(in_dtype == AP_F64 && out_dtype == AP_F32), AP_EPARAM, "float64 rows need float64 output");
    if (n_rows == 0) return AP_OK;
    const int64_t W = cdiv64(t, b);
    cudaStream_t st = as_stream(stream);
    dim3 grid((unsigned)((W + 255) / 256 < 1024 ? (W + 255) / 256 : 1024), (unsigned)n_rows);
    const bool fast = in_dtype == AP_F32 && out_dtype == AP_F32 && b == 16 && (row_stride % 4) == 0 &&
                      (reinterpret_cast<uintptr_t>(rows) % 16) == 0;
    if (fast) {
        max_pool_f32_b16_kernel<<<grid, 256, 0, st>>>((const float*)rows, row_stride, t, (float*)out, out_stride, W);
    } else if (in_dtype == AP_F32 && out_dtype == AP_F32) {
        max_pool_kernel<float, float><<<grid, 256, 0, st>>>((const float*)rows, n_rows, row_stride, t, b,
                                                            (float*)out, out_stride, W);
    } else if (in_dtype == AP_F32) {
        max_pool_kernel<float, double><<<grid, 256, 0, st>>>((const float*)rows, n_rows, row_stride, t, b,
                                                             (double*)out, out_stride, W);
    } else {
        max_pool_kernel<double, double><<<grid, 256, 0, st>>>((const double*)rows, n_rows, row_stride, t, b,
                                                              (double*)out, out_stride, W);
    }
    return launch_status("ap_max_pool");
}

int ap_expand_indices(const int32_t* blocks, int32_t n_blocks, int32_t b, int64_t t, int64_t* tokens,
                      int32_t* n_tokens, int32_t* status, void* stream) {
    AP_REQUIRE(b >= 1, AP_EPARAM, "block size must be >= 1");
    AP_REQUIRE(t >= 1, AP_EPARAM, "original length must be >= 1");
    AP_REQUIRE(n_blocks >= 0, AP_EPARAM, "n_blocks must be >= 0");
    expand_kernel<<<1, 256, 0, as_stream(stream)>>>(blocks, n_blocks, b, t, tokens, n_tokens, status);
    return launch_status("ap_expand_indices");
}

int ap_sel_reset(const ap_selector* s, void* stream) {
    AP_REQUIRE(s && s->n_maps > 0 && s->history >= 1 && s->block >= 1 && s->w_max >= 1, AP_EPARAM,
               "bad selector descriptor");
    int64_t n = (int64_t)s->n_maps * (s->history > 1 ? s->history : 1);
    int64_t words = (int64_t)s->n_maps * ((s->w_max + 31) / 32);
    if (words > n) n = words;
    int blocks = (int)((n + 255) / 256);
    if (blocks > 65535) blocks = 65535;
    sel_reset_kernel<<<blocks, 256, 0, as_stream(stream)>>>(*s);
    return launch_status("ap_sel_reset");
}

int ap_sel_push_rows(const ap_selector* s, const void* rows, int dtype, int64_t row_stride, int64_t t, int mode,
                     void* stream) {
    AP_REQUIRE(s && s->n_maps > 0, AP_EPARAM, "bad selector descriptor");
    AP_REQUIRE(t >= 1, AP_ESTATE, "observed row must be non-empty");
    AP_REQUIRE(mode >= 0 && mode <= 2, AP_EPARAM, "mode must be 0, 1 or 2");
    AP_REQUIRE(cdiv64(t, s->block) <= s->w_max, AP_EPARAM, "row length %lld exceeds w_max*b", (long long)t);
    cudaStream_t st = as_stream(stream);
    if (dtype == AP_F32) {
        const bool fast = mode != 1 && s->block == 16 && (row_stride % 4) == 0 &&
                          (reinterpret_cast<uintptr_t>(rows) % 16) == 0;
        if (fast)
            sel_push_f32_b16_kernel<<<s->n_maps, 256, 0, st>>>(*s, (const float*)rows, row_stride, t);
        else
            sel_push_kernel<float><<<s->n_maps, 256, 0, st>>>(*s, (const float*)rows, row_stride, t, mode);
    } else if (dtype == AP_F64) {
        sel_push_kernel<double><<<s->n_maps, 256, 0, st>>>(*s, (const double*)rows, row_stride, t, mode);
    } else {
        AP_REQUIRE(false, AP_EPARAM, "rows must be float32 or float64");
    }
    return launch_status("ap_sel_push_rows");
}

int ap_sel_push_compressed(const ap_selector* s, const float* comp, int64_t comp_stride, int64_t t, int prefill,
                           void* stream) {
    (void)prefill;  // the counter only moves in ap_sel_step; prefill pushes never call it
    AP_REQUIRE(s && s->n_maps > 0, AP_EPARAM, "bad selector descriptor");
    AP_REQUIRE(t >= 1, AP_ESTATE, "observed row must be non-empty");
    AP_REQUIRE(cdiv64(t, s->block) <= s->w_max, AP_EPARAM, "row length exceeds w_max*b");
    sel_push_compressed_kernel<<<s->n_maps, 256, 0, as_stream(stream)>>>(*s, comp, comp_stride, t);
    return launch_status("ap_sel_push_compressed");
}

}  // extern "C"
