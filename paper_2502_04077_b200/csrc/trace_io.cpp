// .att1 attention-trace container: reader (memory-mapped or borrowed bytes, random access by
// offset) and streaming writer.  Host code, part of libattnpred.so.
//
// Reference: attncast/trace.py — byte layout (9-25), header struct "<4sHIIIIBIi" (40-42),
// TraceHeader.validate (55-72), AttentionTrace.validate (112-168), write_trace (182-212),
// read_trace (215-291).  Error classes and messages follow the reference so callers that match
// on them keep working (FormatError / CorruptionError / ValidationError).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/attnpred.h"

namespace ap {
void set_last_error(const char* fmt, ...);
}

namespace {

constexpr int64_t kHeaderSize = 31;  // 4 magic + 2 version + 4*4 + 1 flag + 4 head_dim + 4 offset
constexpr uint16_t kVersion = 1;
constexpr double kRowSumTol = 1e-4;  // ROW_SUM_TOL (trace.py:43)

#define FAIL(code, ...)                     \
    do {                                    \
        ::ap::set_last_error(__VA_ARGS__);  \
        return (code);                      \
    } while (0)

uint32_t rd_u32(const uint8_t* p) { return (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24; }
void wr_u32(uint8_t* p, uint32_t v) {
    p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24);
}

// Geometry of a validated header (all sizes in bytes unless noted).
struct Geometry {
    int64_t rows_per_head, total_len, block, rows_bytes, nbytes;
    static Geometry of(const ap_trace_header& h) {
        Geometry g;
        g.rows_per_head = (int64_t)h.num_decode_steps - h.first_step_offset + 1;
        g.total_len = (int64_t)h.prefill_len + h.num_decode_steps;
        const int64_t R = g.rows_per_head, o = h.first_step_offset, D = h.num_decode_steps;
        const int64_t sum_steps = (o + D) * R / 2;  // sum over s in [o, D]; (o + D) * R is always even
        g.block = 4 * R + 4 * (R * h.prefill_len + sum_steps);
        const int64_t heads = (int64_t)h.num_layers * h.num_heads;
        g.rows_bytes = heads * g.block;
        g.nbytes = kHeaderSize + g.rows_bytes + (h.has_qk ? heads * (R + g.total_len) * h.head_dim * 4 : 0);
        return g;
    }
    // offset of the length prefix of (layer, head, step)
    int64_t row_offset(const ap_trace_header& h, int layer, int head, int step) const {
        const int64_t k = (int64_t)step - h.first_step_offset;  // rows before it in the head's block
        const int64_t before = 4 * k + 4 * (k * h.prefill_len + k * h.first_step_offset + k * (k - 1) / 2);
        return kHeaderSize + ((int64_t)layer * h.num_heads + head) * block + before;
    }
    int64_t qk_offset(const ap_trace_header& h, int layer, int head) const {
        return kHeaderSize + rows_bytes +
               ((int64_t)layer * h.num_heads + head) * (rows_per_head + total_len) * h.head_dim * 4;
    }
};

int check_header(const ap_trace_header& h) {
    if (h.num_layers < 1 || h.num_heads < 1) FAIL(AP_EVALID, "trace needs at least one layer and head");
    if (h.prefill_len < 1) FAIL(AP_EVALID, "prefill_len must be >= 1");
    if (h.num_decode_steps < 0) FAIL(AP_EVALID, "num_decode_steps must be >= 0");
    if (h.first_step_offset > 0) FAIL(AP_EVALID, "first_step_offset must be <= 0");
    if ((int64_t)h.prefill_len + h.first_step_offset < 1)
        FAIL(AP_EVALID, "first_step_offset reaches before the first prompt token");
    if (h.has_qk && h.head_dim < 1) FAIL(AP_EVALID, "has_qk traces must declare head_dim >= 1");
    if (!h.has_qk && h.head_dim != 0) FAIL(AP_EVALID, "head_dim must be 0 when q/k tensors are absent");
    return AP_OK;
}

// Row invariants of AttentionTrace.validate (trace.py:138-150); sum in float64 like np.sum(dtype=f64).
int check_row(const float* row, int64_t len, int layer, int head, int step) {
    double total = 0.0;
    for (int64_t i = 0; i < len; ++i) {
        const float v = row[i];
        if (!std::isfinite(v) || v < 0.f)
            FAIL(AP_EVALID, "(layer %d, head %d, step %d): scores must be finite and non-negative", layer, head, step);
        total += (double)v;
    }
    if (std::fabs(total - 1.0) > kRowSumTol)
        FAIL(AP_EVALID, "(layer %d, head %d, step %d): row sums to %.6f, not 1", layer, head, step, total);
    return AP_OK;
}

}  // namespace

struct ap_trace {
    const uint8_t* data = nullptr;
    int64_t size = 0;
    bool mapped = false;
    ap_trace_header h{};
    Geometry g{};
};

struct ap_trace_writer {
    ap_trace_header h{};
    Geometry g{};
    FILE* fh = nullptr;
    std::vector<uint8_t> mem;
    int64_t written = 0;
    int64_t row_index = 0;  // rows appended so far (file order)
    int64_t qk_index = 0;
    bool failed = false;
};

namespace {

int parse_header(ap_trace* t) {
    if (t->size < kHeaderSize) FAIL(AP_EFORMAT, "stream shorter than a trace header");
    const uint8_t* p = t->data;
    if (std::memcmp(p, "ATT1", 4) != 0)
        FAIL(AP_EFORMAT, "bad magic b'%c%c%c%c', expected b'ATT1'", p[0], p[1], p[2], p[3]);
    const uint16_t version = (uint16_t)(p[4] | p[5] << 8);
    if (version != kVersion) FAIL(AP_EFORMAT, "unsupported version %u", (unsigned)version);
    const uint32_t nl = rd_u32(p + 6), nh = rd_u32(p + 10), pl = rd_u32(p + 14), nd = rd_u32(p + 18);
    const uint32_t hd = rd_u32(p + 23);
    const int32_t off = (int32_t)rd_u32(p + 27);
    if (nl > INT32_MAX || nh > INT32_MAX || pl > INT32_MAX || nd > INT32_MAX || hd > INT32_MAX)
        FAIL(AP_EVALID, "trace header field out of range");
    ap_trace_header& h = t->h;
    h.num_layers = (int32_t)nl; h.num_heads = (int32_t)nh; h.prefill_len = (int32_t)pl;
    h.num_decode_steps = (int32_t)nd; h.has_qk = p[22] ? 1 : 0; h.head_dim = (int32_t)hd;
    h.first_step_offset = off; h.pad_ = 0;
    const int rc = check_header(h);
    if (rc != AP_OK) return rc;
    t->g = Geometry::of(h);
    return AP_OK;
}

// Structural read of one row: length prefix and payload must be present and consistent.
int row_at(const ap_trace* t, int layer, int head, int step, const float** row, int64_t* len) {
    const int64_t want = (int64_t)t->h.prefill_len + step;
    const int64_t off = t->g.row_offset(t->h, layer, head, step);
    if (off + 4 > t->size)
        FAIL(AP_ECORRUPT, "truncated before row length at (layer %d, head %d, step %d)", layer, head, step);
    const uint32_t n = rd_u32(t->data + off);
    if ((int64_t)n != want)
        FAIL(AP_ECORRUPT, "row length %u != %lld at (layer %d, head %d, step %d)", n, (long long)want, layer, head,
             step);
    if (off + 4 + 4 * want > t->size)
        FAIL(AP_ECORRUPT, "truncated mid-row at (layer %d, head %d, step %d)", layer, head, step);
    *row = reinterpret_cast<const float*>(t->data + off + 4);  // little-endian host, 4-byte payload
    *len = want;
    return AP_OK;
}

void copy_row(const float* src, int64_t len, float* dst, int64_t pad_to) {
    std::memcpy(dst, src, (size_t)len * 4);  // payload may be unaligned: memcpy
    for (int64_t i = len; i < pad_to; ++i) dst[i] = 0.f;
}

int bad_handle(const void* p) {
    if (!p) FAIL(AP_EPARAM, "null trace handle");
    return AP_OK;
}

int write_bytes(ap_trace_writer* w, const void* src, int64_t n) {
    if (w->fh) {
        if (std::fwrite(src, 1, (size_t)n, w->fh) != (size_t)n) {
            w->failed = true;
            FAIL(AP_EIO, "trace write failed: %s", std::strerror(errno));
        }
    } else {
        const uint8_t* b = static_cast<const uint8_t*>(src);
        w->mem.insert(w->mem.end(), b, b + n);
    }
    w->written += n;
    return AP_OK;
}

}  // namespace

extern "C" {

int ap_trace_check_header(const ap_trace_header* h) {
    if (!h) FAIL(AP_EPARAM, "null header");
    return check_header(*h);
}

int ap_trace_check_row(const float* row, int64_t len, int32_t layer, int32_t head, int32_t step) {
    if (len < 0 || (len > 0 && !row)) FAIL(AP_EPARAM, "bad row");
    return check_row(row, len, layer, head, step);
}

int64_t ap_trace_nbytes(const ap_trace_header* h) {
    if (!h || check_header(*h) != AP_OK) return -1;
    return Geometry::of(*h).nbytes;
}

int ap_trace_open(const char* path, ap_trace** out) {
    if (!path || !out) FAIL(AP_EPARAM, "null path or output handle");
    *out = nullptr;
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) FAIL(AP_EIO, "%s: %s", path, std::strerror(errno));
    struct stat st;
    if (::fstat(fd, &st) != 0) {
        ::close(fd);
        FAIL(AP_EIO, "%s: %s", path, std::strerror(errno));
    }
    auto* t = new (std::nothrow) ap_trace;
    if (!t) {
        ::close(fd);
        FAIL(AP_EIO, "out of host memory");
    }
    t->size = (int64_t)st.st_size;
    if (t->size > 0) {
        void* m = ::mmap(nullptr, (size_t)t->size, PROT_READ, MAP_PRIVATE, fd, 0);
        if (m == MAP_FAILED) {
            ::close(fd);
            delete t;
            FAIL(AP_EIO, "%s: mmap: %s", path, std::strerror(errno));
        }
        t->data = static_cast<const uint8_t*>(m);
        t->mapped = true;
    }
    ::close(fd);
    const int rc = parse_header(t);
    if (rc != AP_OK) {
        ap_trace_close(t);
        return rc;
    }
    *out = t;
    return AP_OK;
}

int ap_trace_open_memory(const void* data, int64_t nbytes, ap_trace** out) {
    if (!out || (nbytes > 0 && !data) || nbytes < 0) FAIL(AP_EPARAM, "bad buffer");
    *out = nullptr;
    auto* t = new (std::nothrow) ap_trace;
    if (!t) FAIL(AP_EIO, "out of host memory");
    t->data = static_cast<const uint8_t*>(data);
    t->size = nbytes;
    const int rc = parse_header(t);
    if (rc != AP_OK) {
        delete t;
        return rc;
    }
    *out = t;
    return AP_OK;
}

void ap_trace_close(ap_trace* t) {
    if (!t) return;
    if (t->mapped && t->data) ::munmap(const_cast<uint8_t*>(t->data), (size_t)t->size);
    delete t;
}

int ap_trace_get_header(const ap_trace* t, ap_trace_header* out) {
    if (bad_handle(t) || !out) FAIL(AP_EPARAM, "null trace handle or output");
    *out = t->h;
    return AP_OK;
}

int ap_trace_validate(const ap_trace* t) {
    if (int rc = bad_handle(t)) return rc;
    const ap_trace_header& h = t->h;
    for (int l = 0; l < h.num_layers; ++l)
        for (int hh = 0; hh < h.num_heads; ++hh)
            for (int s = h.first_step_offset; s <= h.num_decode_steps; ++s) {
                const float* row;
                int64_t len;
                if (int rc = row_at(t, l, hh, s, &row, &len)) return rc;
            }
    if (h.has_qk) {
        const int64_t q_bytes = t->g.rows_per_head * h.head_dim * 4, k_bytes = t->g.total_len * h.head_dim * 4;
        for (int l = 0; l < h.num_layers; ++l)
            for (int hh = 0; hh < h.num_heads; ++hh) {
                const int64_t off = t->g.qk_offset(h, l, hh);
                if (off + q_bytes > t->size) FAIL(AP_ECORRUPT, "truncated query block at (layer %d, head %d)", l, hh);
                if (off + q_bytes + k_bytes > t->size)
                    FAIL(AP_ECORRUPT, "truncated key block at (layer %d, head %d)", l, hh);
            }
    }
    if (t->size > t->g.nbytes) FAIL(AP_ECORRUPT, "trailing bytes after the declared trace content");
    // row invariants (AttentionTrace.validate runs after the structural read)
    std::vector<float> buf;
    for (int l = 0; l < h.num_layers; ++l)
        for (int hh = 0; hh < h.num_heads; ++hh)
            for (int s = h.first_step_offset; s <= h.num_decode_steps; ++s) {
                const float* row;
                int64_t len;
                row_at(t, l, hh, s, &row, &len);
                buf.resize((size_t)len);
                std::memcpy(buf.data(), row, (size_t)len * 4);
                if (int rc = check_row(buf.data(), len, l, hh, s)) return rc;
            }
    return AP_OK;
}

int ap_trace_read_rows(const ap_trace* t, int32_t layer, int32_t head, int32_t step_lo, int32_t step_hi,
                       float* dst, int64_t dst_stride, int64_t pad_to) {
    if (int rc = bad_handle(t)) return rc;
    const ap_trace_header& h = t->h;
    if (layer < 0 || layer >= h.num_layers || head < 0 || head >= h.num_heads)
        FAIL(AP_EPARAM, "(layer %d, head %d) out of range", layer, head);
    if (step_lo < h.first_step_offset || step_hi > h.num_decode_steps + 1 || step_lo > step_hi)
        FAIL(AP_EPARAM, "steps [%d, %d) outside the stored range [%d, %d]", step_lo, step_hi, h.first_step_offset,
             h.num_decode_steps);
    if (step_hi > step_lo && !dst) FAIL(AP_EPARAM, "null destination");
    const int64_t longest = (int64_t)h.prefill_len + step_hi - 1;
    if (pad_to > dst_stride || (step_hi > step_lo && dst_stride < longest))
        FAIL(AP_EPARAM, "dst_stride %lld too small for rows of %lld floats", (long long)dst_stride, (long long)longest);
    for (int s = step_lo; s < step_hi; ++s) {
        const float* row;
        int64_t len;
        if (int rc = row_at(t, layer, head, s, &row, &len)) return rc;
        copy_row(row, len, dst + (int64_t)(s - step_lo) * dst_stride, pad_to);
    }
    return AP_OK;
}

int ap_trace_gather_step(const ap_trace* t, int32_t step, float* dst, int64_t dst_stride, int64_t pad_to) {
    if (int rc = bad_handle(t)) return rc;
    const ap_trace_header& h = t->h;
    if (step < h.first_step_offset || step > h.num_decode_steps)
        FAIL(AP_EPARAM, "step %d outside the stored range [%d, %d]", step, h.first_step_offset, h.num_decode_steps);
    const int64_t len = (int64_t)h.prefill_len + step;
    if (!dst || dst_stride < len || pad_to > dst_stride)
        FAIL(AP_EPARAM, "dst_stride %lld too small for rows of %lld floats", (long long)dst_stride, (long long)len);
    for (int l = 0; l < h.num_layers; ++l)
        for (int hh = 0; hh < h.num_heads; ++hh) {
            const float* row;
            int64_t n;
            if (int rc = row_at(t, l, hh, step, &row, &n)) return rc;
            copy_row(row, n, dst + ((int64_t)l * h.num_heads + hh) * dst_stride, pad_to);
        }
    return AP_OK;
}

int ap_trace_read_qk(const ap_trace* t, int32_t layer, int32_t head, float* queries, float* keys) {
    if (int rc = bad_handle(t)) return rc;
    const ap_trace_header& h = t->h;
    if (!h.has_qk) FAIL(AP_EPARAM, "trace carries no query/key tensors");
    if (layer < 0 || layer >= h.num_layers || head < 0 || head >= h.num_heads)
        FAIL(AP_EPARAM, "(layer %d, head %d) out of range", layer, head);
    const int64_t q_bytes = t->g.rows_per_head * h.head_dim * 4, k_bytes = t->g.total_len * h.head_dim * 4;
    const int64_t off = t->g.qk_offset(h, layer, head);
    if (off + q_bytes > t->size) FAIL(AP_ECORRUPT, "truncated query block at (layer %d, head %d)", layer, head);
    if (off + q_bytes + k_bytes > t->size) FAIL(AP_ECORRUPT, "truncated key block at (layer %d, head %d)", layer, head);
    if (queries) std::memcpy(queries, t->data + off, (size_t)q_bytes);
    if (keys) std::memcpy(keys, t->data + off + q_bytes, (size_t)k_bytes);
    return AP_OK;
}

int ap_trace_writer_open(const char* path, const ap_trace_header* h, ap_trace_writer** out) {
    if (!h || !out) FAIL(AP_EPARAM, "null header or output handle");
    *out = nullptr;
    if (int rc = check_header(*h)) return rc;
    auto* w = new (std::nothrow) ap_trace_writer;
    if (!w) FAIL(AP_EIO, "out of host memory");
    w->h = *h;
    w->h.has_qk = h->has_qk ? 1 : 0;
    w->g = Geometry::of(w->h);
    if (path) {
        w->fh = std::fopen(path, "wb");
        if (!w->fh) {
            delete w;
            FAIL(AP_EIO, "%s: %s", path, std::strerror(errno));
        }
    } else {
        w->mem.reserve((size_t)w->g.nbytes);
    }
    uint8_t hdr[kHeaderSize];
    std::memcpy(hdr, "ATT1", 4);
    hdr[4] = (uint8_t)kVersion; hdr[5] = (uint8_t)(kVersion >> 8);
    wr_u32(hdr + 6, (uint32_t)w->h.num_layers); wr_u32(hdr + 10, (uint32_t)w->h.num_heads);
    wr_u32(hdr + 14, (uint32_t)w->h.prefill_len); wr_u32(hdr + 18, (uint32_t)w->h.num_decode_steps);
    hdr[22] = (uint8_t)w->h.has_qk;
    wr_u32(hdr + 23, (uint32_t)w->h.head_dim); wr_u32(hdr + 27, (uint32_t)w->h.first_step_offset);
    if (int rc = write_bytes(w, hdr, kHeaderSize)) {
        ap_trace_writer_free(w);
        return rc;
    }
    *out = w;
    return AP_OK;
}

int ap_trace_writer_append_row(ap_trace_writer* w, const float* row, int64_t len) {
    if (int rc = bad_handle(w)) return rc;
    const ap_trace_header& h = w->h;
    const int64_t total = (int64_t)h.num_layers * h.num_heads * w->g.rows_per_head;
    if (w->row_index >= total) FAIL(AP_ESTATE, "every row of the trace was already written");
    const int64_t per_layer = (int64_t)h.num_heads * w->g.rows_per_head;
    const int layer = (int)(w->row_index / per_layer);
    const int head = (int)(w->row_index % per_layer / w->g.rows_per_head);
    const int step = (int)(w->row_index % w->g.rows_per_head) + h.first_step_offset;
    const int64_t want = (int64_t)h.prefill_len + step;
    if (len != want)
        FAIL(AP_EVALID, "(layer %d, head %d, step %d): length %lld != %lld", layer, head, step, (long long)len,
             (long long)want);
    if (len > 0 && !row) FAIL(AP_EPARAM, "null row");
    if (int rc = check_row(row, len, layer, head, step)) return rc;
    uint8_t n[4];
    wr_u32(n, (uint32_t)len);
    if (int rc = write_bytes(w, n, 4)) return rc;
    if (int rc = write_bytes(w, row, 4 * len)) return rc;
    w->row_index += 1;
    return AP_OK;
}

int ap_trace_writer_append_qk(ap_trace_writer* w, const float* queries, const float* keys) {
    if (int rc = bad_handle(w)) return rc;
    const ap_trace_header& h = w->h;
    if (!h.has_qk) FAIL(AP_ESTATE, "trace declared without query/key tensors");
    if (w->row_index < (int64_t)h.num_layers * h.num_heads * w->g.rows_per_head)
        FAIL(AP_ESTATE, "query/key blocks follow every row");
    if (w->qk_index >= (int64_t)h.num_layers * h.num_heads) FAIL(AP_ESTATE, "every q/k block was already written");
    if (!queries || !keys) FAIL(AP_EPARAM, "null query or key block");
    if (int rc = write_bytes(w, queries, w->g.rows_per_head * h.head_dim * 4)) return rc;
    if (int rc = write_bytes(w, keys, w->g.total_len * h.head_dim * 4)) return rc;
    w->qk_index += 1;
    return AP_OK;
}

int ap_trace_writer_finish(ap_trace_writer* w, int64_t* nbytes) {
    if (int rc = bad_handle(w)) return rc;
    const ap_trace_header& h = w->h;
    const int64_t rows = (int64_t)h.num_layers * h.num_heads * w->g.rows_per_head;
    if (w->row_index < rows) FAIL(AP_EVALID, "trace incomplete: %lld of %lld rows written", (long long)w->row_index,
                                   (long long)rows);
    if (h.has_qk && w->qk_index < (int64_t)h.num_layers * h.num_heads)
        FAIL(AP_EVALID, "q/k blocks must cover every layer and head");
    if (w->fh) {
        const bool ok = std::fflush(w->fh) == 0 && !w->failed;
        std::fclose(w->fh);
        w->fh = nullptr;
        if (!ok) FAIL(AP_EIO, "trace write failed");
    }
    if (nbytes) *nbytes = w->written;
    return AP_OK;
}

int ap_trace_writer_bytes(const ap_trace_writer* w, const void** data, int64_t* nbytes) {
    if (int rc = bad_handle(w)) return rc;
    if (!data || !nbytes) FAIL(AP_EPARAM, "null output");
    *data = w->mem.data();
    *nbytes = (int64_t)w->mem.size();
    return AP_OK;
}

void ap_trace_writer_free(ap_trace_writer* w) {
    if (!w) return;
    if (w->fh) std::fclose(w->fh);
    delete w;
}

}  // extern "C"
