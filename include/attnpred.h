/*
 * attnpred.h — C-ABI of libattnpred.so, the B200 (sm_100a) implementation of
 * AttentionPredictor's decode-time critical-token path.
 *
 * The reference (Python package `attncast`, /root/reference/pkg/src/attncast)
 * has no FFI of its own: its boundary is the Python module API of
 * attncast.compress / attncast.predictor / attncast.selector.  Each entry point
 * below names the reference function it replaces (file:line); the Python
 * package `paper_2502_04077_b200` binds these through ctypes and re-exposes
 * the reference names, signatures and exceptions (INTEGRATION.md shows the
 * binding a maintainer would add on the reference side).
 *
 * Conventions
 *  - Every pointer argument is DEVICE memory unless marked [host].
 *  - Every call is stream-ordered on `stream` (a cudaStream_t, may be NULL),
 *    does not allocate, does not synchronise, and is CUDA-graph capturable
 *    (ap_set_weights included: it issues a memcpy node + one kernel).
 *  - Return value: synchronous argument/shape check (AP_OK or AP_E*).
 *  - Data-dependent failures (non-finite input, out-of-range block id) are
 *    written by the kernels into a caller-provided device status word
 *    (`int32_t* status`, 0 = ok, else an AP_E* code) which the host inspects
 *    when it next synchronises.
 */
#ifndef ATTNPRED_H
#define ATTNPRED_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes → Python exceptions (paper_2502_04077_b200/_lib.py) */
#define AP_OK        0
#define AP_EPARAM    1  /* ParameterError */
#define AP_ECONFIG   2  /* ConfigError    */
#define AP_ESTATE    3  /* StateError     */
#define AP_ENUMERIC  4  /* NumericError   */
#define AP_ECUDA     5  /* DeviceError    */
#define AP_EFORMAT   6  /* FormatError     (trace container: magic / version / short header) */
#define AP_ECORRUPT  7  /* CorruptionError (trace container: truncation, length prefix, trailing bytes) */
#define AP_EVALID    8  /* ValidationError (trace header fields, row invariants) */
#define AP_EIO       9  /* OSError         (open / read / write failures) */

/* element types */
#define AP_F32   0
#define AP_F64   1
#define AP_BF16  2

/* predictor arithmetic (DESIGN.md §Predictor precision) */
#define AP_PREC_FP32    0  /* SIMT fp32 FMA, no tensor cores (tolerance rtol 1e-3) */
#define AP_PREC_F16X3   1  /* tcgen05, fp16 hi/lo split with exact power-of-2 scaling:
                              3 MMAs per tap, ~22-bit operands (rtol 1e-3; default) */
#define AP_PREC_F16     2  /* tcgen05, one scaled fp16 MMA per tap (rtol 2e-2) */

#define AP_PARAM_COUNT 4833 /* predictor.py:36-40 */

int ap_version(void);
/* [host] human-readable text of the last synchronous error in this thread */
const char* ap_last_error(void);
/* [host] number of SMs of the current device (grid sizing in callers) */
int ap_device_sm_count(void);
/* [host] keep n SMs free of the persistent GEMV and calibration grids (their grids shrink to
 * ap_sm_budget() = SMs - n) so a selector step on a side stream (ap_sel_step_grid with n CTAs) runs
 * beside them; 0 (default) = every SM. */
int ap_set_sm_reserve(int n);
int ap_sm_budget(void);

/* ---------------------------------------------------------------------------
 * Predictor weights — predictor.py:45-98 (PredictorWeights), APW1 order
 * w1(16,1,3,3) b1(16) w2(32,16,3,3) b2(32) w3(32) b3().
 * Installs one weight set (4833 fp32, device) for every later predictor call
 * ("one weight set serves every (layer, head)", predictor.py:10-13;
 * "weights immutable during inference").  Copies into constant
 * memory and packs the bf16 hi/lo tcgen05 B-operand tiles.
 * ------------------------------------------------------------------------- */
int ap_set_weights(const float* weights4833, void* stream);

/* ---------------------------------------------------------------------------
 * compress.max_pool — compress.py:28-40, batched over rows.
 * rows: n_rows rows of t elements (in_dtype), row i at rows + i*row_stride
 * (elements).  out: ceil(t/b) values per row (out_dtype), stride out_stride.
 * Zero-pads the tail block, per-block max; NaN propagates like numpy.
 * ------------------------------------------------------------------------- */
int ap_max_pool(const void* rows, int in_dtype, int64_t n_rows, int64_t row_stride, int64_t t,
                int32_t b, void* out, int out_dtype, int64_t out_stride, void* stream);

/* compress.expand_indices — compress.py:43-57.  Writes the token ids of the
 * given blocks (each block's range clipped to t) in block order, and the
 * count into *n_tokens.  Out-of-range block → *status = AP_EPARAM. */
int ap_expand_indices(const int32_t* blocks, int32_t n_blocks, int32_t b, int64_t t,
                      int64_t* tokens, int32_t* n_tokens, int32_t* status, void* stream);

/* selector.topk — selector.py:73-81, batched.  For each of n_rows rows of n
 * values (AP_F32 or AP_F64): the k largest, ties to the lower index, -0.0 ==
 * +0.0; ids written in ASCENDING order (set semantics), count in out_count. */
int ap_topk(const void* values, int dtype, int64_t n_rows, int64_t row_stride, int32_t n, int32_t k,
            int32_t* out_ids, int64_t out_stride, int32_t* out_count, int32_t* status, void* stream);

/* predictor.forward — predictor.py:185-216 on explicit H x W grids (fp32,
 * rows row_pitch floats apart (multiple of 4, >= W), grid i at
 * grids + i*grid_stride, 16-byte aligned).  out: W fp32 per grid.
 * rscratch: n_grids*grid_stride fp32 workspace (per-row contributions). */
int ap_predict_forward(const float* grids, int32_t n_grids, int32_t H, int32_t W, int32_t row_pitch,
                       int64_t grid_stride, float* out, int64_t out_stride, float* rscratch, int precision,
                       int32_t* status, void* stream);

/* ---------------------------------------------------------------------------
 * Batched, device-resident selector: one map per (sequence, layer, q-head).
 * Replaces selector.init_state / selector.step (selector.py:61-70,91-154) for
 * n_maps maps at once.  All buffers are caller-owned device memory.
 * ------------------------------------------------------------------------- */
typedef struct ap_map_state {
    int64_t n_pushed;  /* rows pushed into the ring so far (prefill + decode) */
    int64_t r_pushed;  /* n_pushed when the r-map was last brought up to date; -1 = never */
    int64_t row_len;   /* t of the newest pushed row */
    int64_t counter;   /* selector step counter (selector.py:112,126,153) */
    int64_t mid_clip;  /* t used to clip the current middle blocks (selector.py:145) */
    int32_t width;     /* W of the newest row = ceil(row_len / b) */
    int32_t r_width;   /* W when the r-map was last brought up to date */
    int32_t n_mid;     /* number of middle blocks currently selected */
    int32_t r_wgen;    /* forecaster weight generation the r-map was built with (ap_set_weights bumps it) */
    int32_t tie_n;     /* exact-boundary guard at the last update: 0 = no ambiguity, n > 0 = n near-tie
                        * candidates re-scored in fp64, -n = n candidates exceeded the guard capacity */
    uint32_t prev_kth; /* order key of the k-th score at the last update (0 = none): the next update's top-k
                        * first looks for its boundary in a narrow band around it */
} ap_map_state;

typedef struct ap_selector {
    int32_t n_maps;
    int32_t history;          /* H   (SelectorConfig.history)            */
    int32_t block;            /* b   (SelectorConfig.block_size)         */
    int32_t w_max;            /* ring / r-map row pitch in blocks (multiple of 4) */
    int32_t k_mid;            /* SelectorConfig.middle_blocks           */
    int32_t sink;             /* SelectorConfig.sink_tokens             */
    int32_t local;            /* SelectorConfig.local_tokens            */
    int32_t calib_period;     /* M   (SelectorConfig.calibration_period) */
    int32_t update_interval;  /* SelectorConfig.update_interval         */
    int32_t pad_;
    float* ring;              /* [n_maps][H][w_max] compressed history rows        */
    float* rmap;              /* [n_maps][H][w_max] per-row predictor contributions */
    double* rsum;             /* [n_maps][w_max] running sum of rmap over the H slots */
    int32_t* slot_width;      /* [n_maps][H] width of the row stored in each slot   */
    float* slot_xmax;         /* [n_maps][H] max |x| of the row stored in each slot */
    ap_map_state* state;      /* [n_maps]                                           */
    float* scores;            /* [n_maps][w_max] last forecast (selector.py:133)    */
    int32_t* mid_blocks;      /* [n_maps][k_mid] middle block ids, ascending        */
    uint32_t* mid_mask;       /* [n_maps][ceil(w_max/32)] bitmask of middle blocks  */
    int32_t* status;          /* [1] device status word                             */
    int32_t* tie_ws;          /* exact-boundary guard workspace, ap_sel_tie_ws_bytes(n_maps) bytes, zeroed
                               * once before first use; NULL disables the guard                         */
    const int32_t* k_map;     /* [n_maps] per-map middle-block budget (budget allocation across layers /
                               * heads: selector.py:47-50 evaluated per map), each <= k_mid (the pitch of
                               * mid_blocks); NULL = k_mid for every map                                  */
    int32_t* fused_done;      /* [n_maps] zeroed once: with it, ap_sel_step runs forecast + top-k (+ guard)
                               * as ONE launch (each map selected by the CTA that finishes its last
                               * chunk; the count returns to 0 by the end of every step); NULL = separate
                               * top-k launch                                                             */
} ap_selector;

/* Zero the state of every map (selector.init_state with no prefill rows). */
int ap_sel_reset(const ap_selector* s, void* stream);

/* Compress one t-length attention row per map and append it to the history
 * ring (selector.py:112-120).  rows: map i's row at rows + i*row_stride.
 * t: row length, the same for all maps (host scalar).
 * mode 0 = prefill push (selector.init_state, selector.py:61-70: no masking,
 *          counter untouched);
 * mode 1 = decode push: the row is the DENSE row; on calibration steps
 *          (counter % M == 0) it is stored as is, otherwise it is first masked
 *          to the previous selection (evaluation.py:109-112 observed row:
 *          dense values at sink ∪ local ∪ middle, zeros elsewhere);
 * mode 2 = decode push of an already-observed row (stored as given). */
int ap_sel_push_rows(const ap_selector* s, const void* rows, int dtype, int64_t row_stride, int64_t t,
                     int mode, void* stream);

/* Append already-compressed rows (width W each, fp32) — used by the fused
 * attention kernels' outputs and by tests. Same counter semantics as mode 2
 * (or mode 0 when prefill != 0). */
int ap_sel_push_compressed(const ap_selector* s, const float* comp, int64_t comp_stride, int64_t t,
                           int prefill, void* stream);

/* One selector.step tail (selector.py:122-154) for every map: when
 * counter % update_interval == 0 and k_mid > 0, bring the r-map up to date
 * (incrementally: only the history rows whose 3x3 receptive field changed),
 * forecast the next compressed row, mask the sink/local covering blocks
 * (selector.py:134-142), take top-min(K, available) (selector.py:143-145)
 * into mid_blocks / mid_mask; then counter += 1.
 * Exact-boundary guard (s->tie_ws != NULL, precisions FP32 / F16X3): blocks
 * within band = rel * max(|tau|, floor * max|score|) of the k-th forecast tau
 * are, when the boundary among them is ambiguous, re-scored in fp64 from the
 * history window and ordered like selector.py:80, so the ids equal the
 * float64 reference's (per-map outcome in ap_map_state.tie_n). */
int ap_sel_step(const ap_selector* s, int precision, void* stream);
/* ap_sel_step with the persistent forecaster grid capped at grid_ctas CTAs (0 = one per SM) — for a
 * selector step that runs on a few reserved SMs beside other kernels (ap_set_sm_reserve). */
int ap_sel_step_grid(const ap_selector* s, int precision, int grid_ctas, void* stream);

/* Bytes of the guard workspace for n_maps maps (zero it once before first use). */
int64_t ap_sel_tie_ws_bytes(int32_t n_maps);
/* [host] cumulative guard counters of a workspace: [maps over capacity, maps re-scored,
 * candidates re-scored].  Synchronous copy. */
int ap_sel_tie_stats(const int32_t* tie_ws, int32_t* host_out3);
/* [host] guard switch and band (defaults: on, rel 2^-15, floor 2^-5; env ATTNPRED_TIE_GUARD /
 * ATTNPRED_TIE_REL / ATTNPRED_TIE_FLOOR).  Applies to later ap_sel_step calls (graphs keep the
 * values they were captured with). */
int ap_sel_set_tie_guard(int enabled, float rel, float floor_frac);
/* [host] the guard band of the single-MMA fp16 forecaster (AP_PREC_F16; default rel 0 = no guard,
 * env ATTNPRED_TIE_F16_REL / ATTNPRED_TIE_F16_FLOOR). */
int ap_sel_set_tie_guard_f16(float rel, float floor_frac);

/* Number of persistent CTAs the predictor kernels use (for reporting). */
int ap_sel_grid_ctas(int precision);

/* ---------------------------------------------------------------------------
 * Decode attention for one layer (kernel 4).  No reference implementation
 * exists; the math follows attntap/model.py:70-74 and the
 * selection structure selector.py:122-149.  head_dim 128, bf16 q/K/V,
 * 16-token blocks; K/V cache laid out [seq][kv_head][t_max][128].
 * seq_len[s] = number of keys the current query attends (t, incl. itself).
 * Workspaces: partial = n_seq*n_q_heads*n_splits*130 floats;
 * bmax = n_seq*n_q_heads*w_max floats, initialised to -inf once;
 * counters = 2*n_seq*n_q_heads int32, zeroed once (split counters, then calibration LSE-ready epochs).  The split-K partials are
 * merged by the last CTA of each (sequence, head group) to finish — one
 * launch per call, no separate combine kernel.
 * ------------------------------------------------------------------------- */
typedef struct ap_attn_layer {
    int32_t n_seq, n_q_heads, n_kv_heads, head_dim, t_max, n_splits, block, w_max;
    const void* q;          /* bf16 [n_seq][n_q_heads][128]           */
    const void* k_cache;    /* bf16 [n_seq][n_kv_heads][t_max][128]   */
    const void* v_cache;    /* bf16 [n_seq][n_kv_heads][t_max][128]   */
    const int32_t* seq_len; /* [n_seq]                                */
    void* out;              /* bf16 [n_seq][n_q_heads][128]           */
    float* lse;             /* [n_seq][n_q_heads] log2-domain LSE, may be NULL */
    float* partial;
    float* bmax;
    int32_t* counters;      /* [2][n_seq][n_q_heads] zeroed once; split counters, calibration epochs */
} ap_attn_layer;

/* Dense decode attention over keys [0, t) (with_v = 1: output + LSE, the
 * full-attention comparator and the first decode step) and/or the
 * calibration pass (emit = 1): every block's max logit -> the map's
 * compressed dense row exp(blockmax - LSE) = max_pool(softmax row, b)
 * appended to the selector ring (selector.py:112-120).  K-only when
 * with_v = 0.  map(s, h) = s*maps_per_seq + map_base + h/group. */
/* Kernel of the K-only calibration pass (ap_attn_dense with with_v == 0): 1 = TMA + tcgen05
 * (default), 0 = the SIMT dense kernel.  Returns the previous mode.  Same outputs either way. */
int ap_attn_set_calib_kernel(int mode);
int ap_attn_dense(const ap_attn_layer* a, int with_v, const ap_selector* sel, int32_t map_base,
                  int32_t maps_per_seq, int32_t group, int emit, void* stream);

/* Sparse decode attention over the map's current selection (sink ∪ local ∪
 * middle blocks, selector.py:122-149), gathering only those 16-token
 * blocks.  emit = 1 appends the observed compressed row (sparse_renorm:
 * exp(blockmax - LSE_S) on touched blocks, 0 elsewhere) to the ring. */
int ap_attn_sparse(const ap_attn_layer* a, const ap_selector* sel, int32_t map_base, int32_t maps_per_seq,
                   int32_t group, int emit, void* stream);
/* L2 warm-up for the next ap_attn_sparse of the same layer: prefetches (evict_last) the K/V blocks
 * that pass will gather, except the block holding the newest token.  Meant for a side stream
 * beside the layer's qkv projection; no results, no ordering requirement. */
int ap_attn_sparse_prefetch(const ap_attn_layer* a, const ap_selector* sel, int32_t map_base, int32_t maps_per_seq,
                            int32_t group, void* stream);

/* ---------------------------------------------------------------------------
 * Cross-token prefetch (kernel 5) — the real counterpart of the cross_token
 * schedule the reference only models (prefetchsim.py:126-151).  K stays
 * resident (calibration reads all of K); V lives in pinned, mapped host
 * memory.  Per (layer, sequence, KV head) "vmap" the device keeps V pages
 * [sink blocks | recent ring | k_cap middle pages]; vmap =
 * (layer*n_seq + s)*n_kv_heads + h.  Requires KV-group selection
 * (one selector map per KV head).
 * ------------------------------------------------------------------------- */
typedef struct ap_vpages {
    int32_t k_cap, sink_pages, recent_pages, pad_;
    int64_t host_t_max;
    void* pages;            /* bf16 [n_vmaps][sink+recent+k_cap][16][128]            */
    const void* host_v;     /* bf16 pinned+mapped [n_vmaps][host_t_max][128]         */
    int32_t* mid_page;      /* [n_vmaps][k_cap] page of each current middle block    */
    int32_t* old_blocks;    /* [n_vmaps][k_cap] resident middle blocks (sorted)      */
    int32_t* old_pages;     /* [n_vmaps][k_cap]                                      */
    int32_t* old_n;         /* [n_vmaps]                                             */
    int64_t* bytes_copied;  /* [1] running count of host->device bytes (may be NULL) */
} ap_vpages;

/* After ap_sel_step predicted the next step's middle blocks: for every map of
 * `layer`, keep the pages of blocks still selected and gather the new ones
 * from host V (16-byte zero-copy loads).  Launch per layer on a side stream. */
int ap_prefetch(const ap_selector* sel, const ap_vpages* vp, int32_t layer, int32_t n_seq, int32_t n_kv_heads,
                int32_t maps_per_seq, void* stream);
/* Write the step's V row (from qkv) to the paged store and through to host V. */
int ap_v_append(const void* qkv, int32_t n_q_heads, int32_t n_kv_heads, const int32_t* seq_len, const ap_vpages* vp,
                int32_t layer, int32_t n_seq, void* stream);
/* Fill the sink pages and recent ring of every vmap from host V (prompt length t). */
int ap_v_pages_init(const ap_vpages* vp, int64_t t, int64_t n_vmaps, void* stream);
/* ap_attn_sparse with V read from the paged store of `layer` (offload mode). */
int ap_attn_sparse_paged(const ap_attn_layer* a, const ap_selector* sel, int32_t map_base, int32_t maps_per_seq,
                         int32_t group, int emit, const ap_vpages* vp, int32_t layer, void* stream);

/* ---------------------------------------------------------------------------
 * .att1 attention-trace container (reference: trace.py:9-25 layout,
 * TraceHeader.validate 55-72, AttentionTrace.validate 112-168, write_trace
 * 182-212, read_trace 215-291).  Host code: the reader memory-maps a file (or
 * borrows a caller buffer) and addresses any (layer, head, step) row by offset,
 * so golden traces stream straight into device staging buffers for replay; the
 * writer streams rows in file order and produces byte-identical output.
 * Error messages name the location the way the reference does.
 * ------------------------------------------------------------------------- */
typedef struct ap_trace_header {
    int32_t num_layers, num_heads, prefill_len, num_decode_steps;
    int32_t has_qk, head_dim, first_step_offset, pad_;
} ap_trace_header;
typedef struct ap_trace ap_trace;                /* opaque reader */
typedef struct ap_trace_writer ap_trace_writer;  /* opaque writer */

/* TraceHeader.validate (trace.py:55-72): AP_EVALID on a field violation. */
int ap_trace_check_header(const ap_trace_header* h);
/* Row invariants of AttentionTrace.validate (trace.py:138-150): finite, >= 0, float64 sum within
 * 1e-4 of 1; AP_EVALID naming (layer, head, step). */
int ap_trace_check_row(const float* row, int64_t len, int32_t layer, int32_t head, int32_t step);
/* Total container bytes the header declares (header + rows + q/k blocks). */
int64_t ap_trace_nbytes(const ap_trace_header* h);
/* Open a reader over a file (memory-mapped) or over caller bytes (borrowed; keep them alive).
 * Parses the header (AP_EFORMAT: short header, bad magic, bad version; AP_EVALID: fields). */
int ap_trace_open(const char* path, ap_trace** out);
int ap_trace_open_memory(const void* data, int64_t nbytes, ap_trace** out);
void ap_trace_close(ap_trace* t);
int ap_trace_get_header(const ap_trace* t, ap_trace_header* out);
/* Everything read_trace + validate check: every length prefix, truncation (AP_ECORRUPT naming
 * the row), trailing bytes, and per-row invariants (finite, >= 0, sums to 1 within 1e-4:
 * AP_EVALID).  Rows are addressed by offset, so the other readers do not need this first. */
int ap_trace_validate(const ap_trace* t);
/* Rows of (layer, head) for steps [step_lo, step_hi): step s -> dst + (s - step_lo) * dst_stride
 * floats, zero-filled up to pad_to floats (pad_to <= dst_stride; 0 = no padding). */
int ap_trace_read_rows(const ap_trace* t, int32_t layer, int32_t head, int32_t step_lo, int32_t step_hi,
                       float* dst, int64_t dst_stride, int64_t pad_to);
/* Row of `step` for every (layer, head): map m = layer * num_heads + head -> dst + m * dst_stride,
 * zero-filled up to pad_to floats (the staging layout of ap_sel_push_rows). */
int ap_trace_gather_step(const ap_trace* t, int32_t step, float* dst, int64_t dst_stride, int64_t pad_to);
/* q/k blocks of (layer, head) (has_qk): queries [rows_per_head][head_dim], keys [total_len][head_dim]. */
int ap_trace_read_qk(const ap_trace* t, int32_t layer, int32_t head, float* queries, float* keys);

/* Streaming writer: rows in file order (layer-major, head, step oldest first), then (has_qk) one
 * q/k pair per (layer, head) in the same order.  path NULL = in-memory (ap_trace_writer_bytes).
 * append_row validates the row (length AP_EVALID, invariants AP_EVALID naming the location). */
int ap_trace_writer_open(const char* path, const ap_trace_header* h, ap_trace_writer** out);
int ap_trace_writer_append_row(ap_trace_writer* w, const float* row, int64_t len);
int ap_trace_writer_append_qk(ap_trace_writer* w, const float* queries, const float* keys);
/* AP_EVALID if rows / q-k blocks are missing; *nbytes = bytes written. */
int ap_trace_writer_finish(ap_trace_writer* w, int64_t* nbytes);
int ap_trace_writer_bytes(const ap_trace_writer* w, const void** data, int64_t* nbytes);
void ap_trace_writer_free(ap_trace_writer* w);

/* ---------------------------------------------------------------------------
 * Decode-engine helpers around the path (not reference functions: the
 * reference has no model; these exist so a whole LLaMA-shape decode step runs
 * from one CUDA graph).  bf16 tensors, row-major.
 * ------------------------------------------------------------------------- */
/* residual (if non-NULL) += x; y = rmsnorm(residual or x) * weight */
int ap_rmsnorm(const void* x, void* residual, const void* weight, void* y, int32_t rows, int32_t dim, float eps,
               void* stream);
/* qkv [n_seq][(Hq+2Hkv)*128] -> rotated q_out [n_seq][Hq][128]; rotated k and v appended to the
 * caches at position seq_len[s]-1 */
int ap_rope_append(const void* qkv, int32_t n_seq, int32_t n_q_heads, int32_t n_kv_heads, const int32_t* seq_len,
                   void* q_out, void* k_cache, void* v_cache, int32_t t_max, float theta, void* stream);
/* out [rows][ffn] = silu(gate_up[:, :ffn]) * gate_up[:, ffn:] */
int ap_silu_mul(const void* gate_up, void* out, int32_t rows, int32_t ffn, void* stream);
/* tokens[r] = argmax of bf16 logits row r ([rows][n] row-major; torch.argmax semantics, ties to the lowest
 * index).  workspace: ap_argmax_workspace_bytes(rows) bytes, zeroed once, self-resetting. */
int64_t ap_argmax_workspace_bytes(int32_t rows);
int ap_argmax_rows(const void* logits, int32_t rows, int64_t n, void* workspace, int64_t workspace_bytes,
                   int64_t* tokens, void* stream);
/* seq_len[i] += by */
int ap_advance(int32_t* seq_len, int32_t n, int32_t by, void* stream);
/* The start of a decode step in one launch: seq_len[i] += by for i < n, and out[s][:] = embed[tokens[s]][:]
 * (bf16 rows of `hidden` elements, s < n) — ap_advance plus the embedding lookup. */
int ap_advance_embed(int32_t* seq_len, int32_t n, int32_t by, const void* embed, const int64_t* tokens, void* out,
                     int32_t hidden, void* stream);

/* Batch-1..4 bf16 GEMV y[s] = W x[s] (W [N][K] row-major, K % 8 == 0, fp32 accumulate), HBM-streaming.
 * rows_per_warp: ignored (ABI slot of an earlier kernel).  flags: bit 0 = RMSNORM prologue (h = x [+ residual], written to residual_out
 * when non-NULL (must not alias); x = rmsnorm(h) * ln_w, the arithmetic of ap_rmsnorm);
 * bits 1-2 = epilogue: 0 store y [s][N],
 * 1 SILU (W = [gate; up], y [s][N/2] = silu(gate) * up, as ap_silu_mul), 2 ARGMAX (greedy token of
 * each row into tokens[s] (int64), ties to the lowest index, logits also stored when y != NULL;
 * arg_workspace = 4 u64 + 1 int32, zeroed once, self-resetting). */
int ap_gemv(const void* W, const void* x, void* y, int32_t N, int32_t K, int32_t n_seq, int32_t rows_per_warp,
            int32_t flags, const void* residual, void* residual_out, const void* ln_w, float eps,
            void* arg_workspace, void* tokens, void* stream);
/* Fused qkv projection + rotary embedding + KV append for batch-1..4 decode: y = W x (W [(Hq+2Hkv)*128][K],
 * optional RMSNORM prologue as ap_gemv flag bit 0), y stored as ap_gemv would, then for position
 * seq_len[s]-1 the arithmetic of ap_rope_append on the bf16 projection output: rotated q -> q_out,
 * rotated k and v appended to the caches (v_cache NULL: V only in y, for the offload path). */
int ap_gemv_qkv_rope(const void* W, const void* x, void* y, int32_t n_q_heads, int32_t n_kv_heads, int32_t K,
                     int32_t n_seq, int32_t flags, const void* residual, void* residual_out, const void* ln_w, float eps,
                     const int32_t* seq_len, void* q_out, void* k_cache, void* v_cache, int32_t t_max, float theta,
                     void* stream);

/* Batch-5..16 bf16 GEMM y[s][n] = sum_k x[s][k] W[n][k] (W [N][K], x [n_seq][K], y [n_seq][N], all
 * row-major; fp32 accumulate) on tcgen05 tensor cores, TMA-fed, one persistent wave over the SMs.
 * K % 256 == 0, n_seq in 1..16, N <= 524288.  workspace: ap_gemm_tc_workspace_bytes(N, K, n_seq) bytes,
 * zeroed once (self-resetting per-tile counters, then fp32 partials of row tiles split across CTAs); one
 * workspace of the largest size serves GEMMs of every shape on a stream; the sum over
 * splits runs in a fixed order, so results are run-to-run deterministic. */
int64_t ap_gemm_tc_workspace_bytes(int32_t N, int32_t K, int32_t n_seq);
int ap_gemm_tc(const void* W, const void* x, void* y, int32_t N, int32_t K, int32_t n_seq, void* workspace,
               int64_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Forecaster training (not on the decode path).
 * ------------------------------------------------------------------------- */
/* predictor.backward (predictor.py:219-251) for n_samples equal-shape samples: grids [n][H][W] and
 * targets [n][W] fp64, contiguous; weights: 4833 fp64 in the APW1 order.  Accumulates (+=) the SUM over
 * samples of each sample's gradient into grads[4833] and of its loss into *loss_sum (the reference's
 * per-batch accumulation, predictor.py:371-377).  fp64 arithmetic like the reference; every reduction
 * runs in a fixed order, so results are run-to-run deterministic.
 * workspace: ap_train_workspace_bytes(n, H, W) bytes (activations and gradients, 768 B per pixel). */
int64_t ap_train_workspace_bytes(int32_t n_samples, int32_t H, int32_t W);
int ap_train_backward(const double* grids, const double* targets, int32_t n_samples, int32_t H, int32_t W,
                      const double* weights, double* grads, double* loss_sum, void* workspace,
                      int64_t workspace_bytes, void* stream);
/* Adam of predictor.train (predictor.py:381-391) in fp64 with numpy's rounding: g = grad_sum / batch,
 * m = b1 m + (1-b1) g, v = b2 v + (1-b2) g g, w -= lr (m / (1-b1^step)) / (sqrt(v / (1-b2^step)) + eps). */
int ap_adam_step(double* weights, double* m, double* v, const double* grad_sum, int32_t n_params, double batch,
                 double lr, double beta1, double beta2, double eps, int64_t step, void* stream);
/* predictor.forward (predictor.py:185-216) in fp64 — the reference's arithmetic type — for n_grids
 * equal-shape grids [n][H][W] (contiguous fp64) with fp64 weights (4833, APW1 order): out[n*out_stride + w].
 * The default of the reference-compatible `predictor.forward`; uses the conv/head kernels of
 * ap_train_backward, so a forward used as a training target gives an exactly zero residual
 * (reference test_predictor.py:64-70).  workspace: ap_forward_f64_workspace_bytes(n, H, W). */
int64_t ap_forward_f64_workspace_bytes(int32_t n_grids, int32_t H, int32_t W);
int ap_predict_forward_f64(const double* grids, int32_t n_grids, int32_t H, int32_t W, const double* weights,
                           double* out, int64_t out_stride, void* workspace, int64_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ATTNPRED_H */
