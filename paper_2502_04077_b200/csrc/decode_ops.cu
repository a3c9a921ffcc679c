// Small fused ops of the decode engine around the critical-token path:
// residual-add + RMSNorm, RoPE + KV-cache append, SiLU-gate, sequence advance.
// All launched with programmatic dependent launch: each triggers its dependents at entry and waits
// for its predecessor before touching memory, so the next projection's weight prefetch overlaps.
#include "common.cuh"

namespace ap {

// h = x + residual (if residual), y = h * rsqrt(mean(h^2) + eps) * w.  One CTA per row.
__global__ void __launch_bounds__(256) rmsnorm_kernel(const __nv_bfloat16* __restrict__ x,
                                                      __nv_bfloat16* __restrict__ residual, const __nv_bfloat16* __restrict__ w,
                                                      __nv_bfloat16* __restrict__ y, int D, float eps) {
    __shared__ float red[8];
    pdl_trigger();
    pdl_wait();  // x / residual come from the kernels just before
    const int row = blockIdx.x;
    const __nv_bfloat16* xr = x + (int64_t)row * D;
    __nv_bfloat16* rr = residual ? residual + (int64_t)row * D : nullptr;
    float ss = 0.f;
    // D is a multiple of 8 * 256 for the shapes we serve (4096); fall back to scalar otherwise
    for (int i = threadIdx.x * 8; i < D; i += 256 * 8) {
        uint4 u = *reinterpret_cast<const uint4*>(xr + i);
        __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&u);
        if (rr) {
            uint4 ru = *reinterpret_cast<const uint4*>(rr + i);
            __nv_bfloat162* rp = reinterpret_cast<__nv_bfloat162*>(&ru);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float2 a = __bfloat1622float2(p[k]), b = __bfloat1622float2(rp[k]);
                p[k] = __floats2bfloat162_rn(a.x + b.x, a.y + b.y);
            }
            *reinterpret_cast<uint4*>(rr + i) = u;  // updated residual stream
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float2 a = __bfloat1622float2(p[k]);
            ss += a.x * a.x + a.y * a.y;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) tot += red[k];
    const float inv = rsqrtf(tot / (float)D + eps);
    const __nv_bfloat16* src = rr ? rr + 0 : xr;
    for (int i = threadIdx.x * 8; i < D; i += 256 * 8) {
        uint4 u = *reinterpret_cast<const uint4*>(src + i);
        uint4 wu = *reinterpret_cast<const uint4*>(w + i);
        __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&u);
        __nv_bfloat162* wp = reinterpret_cast<__nv_bfloat162*>(&wu);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float2 a = __bfloat1622float2(p[k]), b = __bfloat1622float2(wp[k]);
            p[k] = __floats2bfloat162_rn(a.x * inv * b.x, a.y * inv * b.y);
        }
        *reinterpret_cast<uint4*>(y + (int64_t)row * D + i) = u;
    }
}

// qkv: [S][(Hq + 2*Hkv) * 128] -> q_out [S][Hq][128] (rotated), K/V cache at position seq_len[s]-1.
// Rotary embedding with rotate-half pairing (i, i+64), theta^(-2i/128).
__global__ void rope_append_kernel(const __nv_bfloat16* __restrict__ qkv, int Hq, int Hkv,
                                   const int32_t* __restrict__ seq_len, __nv_bfloat16* __restrict__ q_out,
                                   __nv_bfloat16* __restrict__ k_cache, __nv_bfloat16* __restrict__ v_cache, int t_max,
                                   float theta) {
    const int s = blockIdx.y;
    const int head = blockIdx.x;  // [0, Hq + 2*Hkv)
    const int i = threadIdx.x;    // 0..63
    pdl_trigger();
    pdl_wait();  // qkv comes from the projection just before
    const int pos = seq_len[s] - 1;
    const __nv_bfloat16* src = qkv + ((int64_t)s * (Hq + 2 * Hkv) + head) * 128;
    float x1 = __bfloat162float(src[i]), x2 = __bfloat162float(src[i + 64]);
    if (head < Hq + Hkv) {
        const float inv_freq = exp2f(-(float)(2 * i) / 128.f * log2f(theta));
        float sn, cs;
        sincosf((float)pos * inv_freq, &sn, &cs);
        const float y1 = x1 * cs - x2 * sn, y2 = x2 * cs + x1 * sn;
        x1 = y1;
        x2 = y2;
    }
    __nv_bfloat16* dst;
    if (head < Hq) {
        dst = q_out + ((int64_t)s * Hq + head) * 128;
    } else if (head < Hq + Hkv) {
        dst = k_cache + (((int64_t)s * Hkv + (head - Hq)) * t_max + pos) * 128;
    } else {
        if (!v_cache) return;  // offload mode: V goes to the paged store + host (ap_v_append)
        dst = v_cache + (((int64_t)s * Hkv + (head - Hq - Hkv)) * t_max + pos) * 128;
    }
    dst[i] = __float2bfloat16_rn(x1);
    dst[i + 64] = __float2bfloat16_rn(x2);
}

// gu: [S][2*F] (gate | up) -> out [S][F] = silu(gate) * up
__global__ void silu_mul_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ out, int F,
                                int64_t n) {
    pdl_trigger();
    pdl_wait();
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = idx / F, f = idx % F;
        const float g = __bfloat162float(gu[s * 2 * F + f]), u = __bfloat162float(gu[s * 2 * F + F + f]);
        out[idx] = __float2bfloat16_rn(g / (1.f + __expf(-g)) * u);
    }
}

// Greedy token of each row of bf16 logits [rows][n] (torch.argmax semantics: ties -> lowest index).
// grid (chunks, rows): each CTA reduces a chunk to a packed key (orderable value << 32 | ~index),
// merged per row with a 64-bit atomicMax; the row's last CTA decodes it and resets the workspace.
__global__ void __launch_bounds__(256) argmax_rows_kernel(const __nv_bfloat16* __restrict__ logits, int64_t n,
                                                          int64_t chunk, unsigned long long* best, int32_t* done,
                                                          int64_t* tokens) {
    pdl_trigger();
    pdl_wait();
    const int row = blockIdx.y;
    const __nv_bfloat16* x = logits + row * n;
    const int64_t c0 = blockIdx.x * chunk, c1 = c0 + chunk < n ? c0 + chunk : n;
    unsigned long long key = 0;
    auto take = [&](float v, int64_t i) {
        const unsigned long long k = ((unsigned long long)order_key(v) << 32) | (uint32_t)~(uint32_t)i;
        key = k > key ? k : key;
    };
    if ((n & 7) == 0) {  // 16-byte loads (chunk is a multiple of 8)
        for (int64_t i = c0 + threadIdx.x * 8; i < c1; i += 256 * 8) {
            const uint4 u = __ldcs(reinterpret_cast<const uint4*>(x + i));
            const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
            for (int e = 0; e < 8; ++e) take(__bfloat162float(h[e]), i + e);
        }
    } else {
        for (int64_t i = c0 + threadIdx.x; i < c1; i += 256) take(__bfloat162float(x[i]), i);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long k = __shfl_xor_sync(0xffffffffu, key, o);
        key = k > key ? k : key;
    }
    __shared__ unsigned long long s_key[8];
    __shared__ int s_last;
    if ((threadIdx.x & 31) == 0) s_key[threadIdx.x >> 5] = key;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) key = s_key[w] > key ? s_key[w] : key;
        atomicMax(best + row, key);
        __threadfence();
        s_last = atomicAdd(done + row, 1) == (int)gridDim.x - 1;
        if (s_last) {
            const unsigned long long k = atomicExch(best + row, 0ull);
            tokens[row] = (int64_t)(uint32_t)~(uint32_t)(k & 0xffffffffu);
            done[row] = 0;
        }
    }
}

__global__ void advance_kernel(int32_t* seq_len, int n, int by) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) seq_len[i] += by;
}

// grid (chunks, n): sequence s copies embedding row tokens[s] in 16-byte pieces; CTA (0, s) also advances
// seq_len[s].  Launched with programmatic dependent launch: the next step's first projection may start
// streaming its weights while this runs.
__global__ void advance_embed_kernel(int32_t* seq_len, int by, const uint4* __restrict__ embed,
                                     const int64_t* __restrict__ tokens, uint4* __restrict__ out, int hidden16) {
    pdl_trigger();
    pdl_wait();  // the token comes from the previous step's argmax
    const int s = blockIdx.y;
    if (blockIdx.x == 0 && threadIdx.x == 0) seq_len[s] += by;
    const int64_t tok = tokens[s];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < hidden16; i += gridDim.x * blockDim.x)
        out[(int64_t)s * hidden16 + i] = embed[tok * hidden16 + i];
}

}  // namespace ap

using namespace ap;

extern "C" {

int ap_rmsnorm(const void* x, void* residual, const void* weight, void* y, int32_t rows, int32_t dim, float eps,
               void* stream) {
    AP_REQUIRE(dim % 8 == 0, AP_EPARAM, "dim must be a multiple of 8");
    launch_ex(rmsnorm_kernel, dim3(rows), dim3(256), 0, as_stream(stream), 1, (const __nv_bfloat16*)x,
              (__nv_bfloat16*)residual, (const __nv_bfloat16*)weight, (__nv_bfloat16*)y, (int)dim, eps);
    return launch_status("ap_rmsnorm");
}

int ap_rope_append(const void* qkv, int32_t n_seq, int32_t n_q_heads, int32_t n_kv_heads, const int32_t* seq_len,
                   void* q_out, void* k_cache, void* v_cache, int32_t t_max, float theta, void* stream) {
    dim3 grid(n_q_heads + 2 * n_kv_heads, n_seq);
    launch_ex(rope_append_kernel, grid, dim3(64), 0, as_stream(stream), 1, (const __nv_bfloat16*)qkv, (int)n_q_heads,
              (int)n_kv_heads, seq_len, (__nv_bfloat16*)q_out, (__nv_bfloat16*)k_cache, (__nv_bfloat16*)v_cache,
              (int)t_max, theta);
    return launch_status("ap_rope_append");
}

int ap_silu_mul(const void* gate_up, void* out, int32_t rows, int32_t ffn, void* stream) {
    const int64_t n = (int64_t)rows * ffn;
    int blocks = (int)((n + 255) / 256);
    if (blocks > 4096) blocks = 4096;
    launch_ex(silu_mul_kernel, dim3(blocks), dim3(256), 0, as_stream(stream), 1, (const __nv_bfloat16*)gate_up,
              (__nv_bfloat16*)out, (int)ffn, n);
    return launch_status("ap_silu_mul");
}

int64_t ap_argmax_workspace_bytes(int32_t rows) { return rows > 0 ? (int64_t)rows * 12 : -1; }

int ap_argmax_rows(const void* logits, int32_t rows, int64_t n, void* workspace, int64_t workspace_bytes,
                   int64_t* tokens, void* stream) {
    AP_REQUIRE(logits && tokens && rows > 0 && n > 0 && n < (1ll << 32), AP_EPARAM, "bad argmax operands");
    AP_REQUIRE(workspace && workspace_bytes >= (int64_t)rows * 12, AP_EPARAM, "argmax workspace too small");
    const int sms = ap_device_sm_count();
    int64_t chunks = 2 * (int64_t)sms / rows;
    const int64_t max_chunks = (n + 2047) / 2048;
    if (chunks > max_chunks) chunks = max_chunks;
    if (chunks < 1) chunks = 1;
    int64_t chunk = (n + chunks - 1) / chunks;
    chunk = (chunk + 7) / 8 * 8;
    chunks = (n + chunk - 1) / chunk;
    auto* best = (unsigned long long*)workspace;
    auto* done = (int32_t*)((char*)workspace + (int64_t)rows * 8);
    launch_ex(argmax_rows_kernel, dim3((unsigned)chunks, rows), dim3(256), 0, as_stream(stream), 1,
              (const __nv_bfloat16*)logits, n, chunk, best, done, tokens);
    return launch_status("ap_argmax_rows");
}

int ap_advance(int32_t* seq_len, int32_t n, int32_t by, void* stream) {
    advance_kernel<<<(n + 127) / 128, 128, 0, as_stream(stream)>>>(seq_len, n, by);
    return launch_status("ap_advance");
}

int ap_advance_embed(int32_t* seq_len, int32_t n, int32_t by, const void* embed, const int64_t* tokens, void* out,
                     int32_t hidden, void* stream) {
    AP_REQUIRE(seq_len && embed && tokens && out && n >= 1 && n <= 65535, AP_EPARAM, "bad advance_embed operands");
    AP_REQUIRE(hidden > 0 && hidden % 8 == 0, AP_EPARAM, "hidden must be a multiple of 8 (16-byte rows)");
    const int hidden16 = hidden / 8;
    const int chunks = (hidden16 + 127) / 128 < 8 ? (hidden16 + 127) / 128 : 8;
    launch_ex(advance_embed_kernel, dim3(chunks, n), dim3(128), 0, as_stream(stream), 1, seq_len, by,
              (const uint4*)embed, tokens, (uint4*)out, hidden16);
    return launch_status("ap_advance_embed");
}

}  // extern "C"
