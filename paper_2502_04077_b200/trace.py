"""Attention trace data model and the ``.att1`` container — drop-in for ``attncast.trace``.

Same names, dataclasses, signatures and exceptions as the reference module
(reference: pkg/src/attncast/trace.py: layout 9-25, TraceHeader 46-87,
AttentionTrace 90-179, write_trace 182-212, read_trace 215-291, file/bytes
helpers 294-311).  The byte work is native (``csrc/trace_io.cpp`` behind the
``ap_trace_*`` C-ABI): header parsing, row addressing by offset, structural and
row-invariant validation, and serialisation.  Python keeps only the object
model and the structural checks of in-memory traces.

Beyond the reference, :class:`TraceReader` memory-maps a trace and hands out
any (layer, head, step) row without reading the rest — ``gather_step`` fills
the ``[maps][row]`` staging layout that ``BatchedSelector.push_rows`` takes, so
golden traces replay through the device path (``replay_on_device``).
"""

from __future__ import annotations

import ctypes
import io
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ValidationError

MAGIC = b"ATT1"
VERSION = 1
HEADER_SIZE = 31  # 4 magic + 2 version + 4 x u32 + u8 flag + u32 head_dim + i32 offset
ROW_SUM_TOL = 1e-4
FILE_EXTENSION = ".att1"

__all__ = ["MAGIC", "VERSION", "HEADER_SIZE", "ROW_SUM_TOL", "FILE_EXTENSION", "TraceHeader", "AttentionTrace",
           "write_trace", "read_trace", "write_trace_file", "read_trace_file", "trace_to_bytes",
           "trace_from_bytes", "TraceReader"]


@dataclass
class TraceHeader:
    num_layers: int
    num_heads: int
    prefill_len: int
    num_decode_steps: int
    has_qk: bool = False
    head_dim: int = 0
    first_step_offset: int = 0

    def _c(self) -> _lib.TraceHeaderC:
        big = (1 << 31) - 1
        for v in (self.num_layers, self.num_heads, self.prefill_len, self.num_decode_steps, self.head_dim):
            if not -big <= int(v) <= big:
                raise ValidationError("trace header field out of range")
        return _lib.TraceHeaderC(int(self.num_layers), int(self.num_heads), int(self.prefill_len),
                                 int(self.num_decode_steps), 1 if self.has_qk else 0, int(self.head_dim),
                                 int(self.first_step_offset), 0)

    @classmethod
    def _from_c(cls, h: _lib.TraceHeaderC) -> "TraceHeader":
        return cls(h.num_layers, h.num_heads, h.prefill_len, h.num_decode_steps, bool(h.has_qk), h.head_dim,
                   h.first_step_offset)

    def validate(self) -> None:
        """TraceHeader.validate (trace.py:55-72), native."""
        c = self._c()
        _lib.check(_lib.fn("ap_trace_check_header")(ctypes.byref(c)), "trace header")

    @property
    def steps(self) -> range:
        """Stored step indices, oldest first."""
        return range(self.first_step_offset, self.num_decode_steps + 1)

    @property
    def rows_per_head(self) -> int:
        return self.num_decode_steps - self.first_step_offset + 1

    @property
    def total_len(self) -> int:
        """Context length after the last decode step."""
        return self.prefill_len + self.num_decode_steps

    def row_len(self, step: int) -> int:
        return self.prefill_len + step


@dataclass
class AttentionTrace:
    header: TraceHeader
    rows: list  # rows[layer][head][k] float32 row of step header.steps[k]
    queries: list = field(default_factory=list)  # [layer][head] (rows_per_head, head_dim)
    keys: list = field(default_factory=list)     # [layer][head] (total_len, head_dim)

    def row(self, layer: int, head: int, step: int) -> np.ndarray:
        return self.rows[layer][head][step - self.header.first_step_offset]

    def query(self, layer: int, head: int, step: int) -> np.ndarray:
        return self.queries[layer][head][step - self.header.first_step_offset]

    def head_keys(self, layer: int, head: int) -> np.ndarray:
        return self.keys[layer][head]

    def validate(self) -> None:
        """AttentionTrace.validate (trace.py:112-168): structure here, row values natively."""
        h = self.header
        h.validate()
        if len(self.rows) != h.num_layers:
            raise ValidationError("row block count does not match num_layers")
        check_row = _lib.fn("ap_trace_check_row")
        for layer, per_layer in enumerate(self.rows):
            if len(per_layer) != h.num_heads:
                raise ValidationError(f"layer {layer}: head count mismatch")
            for head, per_head in enumerate(per_layer):
                if len(per_head) != h.rows_per_head:
                    raise ValidationError(f"(layer {layer}, head {head}): expected "
                                          f"{h.rows_per_head} rows, found {len(per_head)}")
                for k, row in enumerate(per_head):
                    step = h.first_step_offset + k
                    if not isinstance(row, np.ndarray) or row.dtype != np.float32 or row.ndim != 1:
                        raise ValidationError(f"(layer {layer}, head {head}, step {step}): rows must be 1-D float32")
                    if len(row) != h.row_len(step):
                        raise ValidationError(f"(layer {layer}, head {head}, step {step}): length "
                                              f"{len(row)} != {h.row_len(step)}")
                    r = np.ascontiguousarray(row)
                    _lib.check(check_row(r.ctypes.data, r.size, layer, head, step), "trace row")
        if h.has_qk:
            if len(self.queries) != h.num_layers or len(self.keys) != h.num_layers:
                raise ValidationError("q/k blocks must cover every layer")
            for layer in range(h.num_layers):
                if len(self.queries[layer]) != h.num_heads or len(self.keys[layer]) != h.num_heads:
                    raise ValidationError(f"layer {layer}: q/k blocks must cover every head")
                for head in range(h.num_heads):
                    q, k = self.queries[layer][head], self.keys[layer][head]
                    if q.shape != (h.rows_per_head, h.head_dim):
                        raise ValidationError(f"(layer {layer}, head {head}): query block shape {q.shape}")
                    if k.shape != (h.total_len, h.head_dim):
                        raise ValidationError(f"(layer {layer}, head {head}): key block shape {k.shape}")

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, AttentionTrace):
            return NotImplemented
        if self.header != other.header:
            return False
        for mine, theirs in zip(self.rows, other.rows):
            for rows_a, rows_b in zip(mine, theirs):
                if len(rows_a) != len(rows_b):
                    return False
                if not all(np.array_equal(a, b) for a, b in zip(rows_a, rows_b)):
                    return False
        if self.header.has_qk:
            for blk_a, blk_b in ((self.queries, other.queries), (self.keys, other.keys)):
                for mine, theirs in zip(blk_a, blk_b):
                    if not all(np.array_equal(a, b) for a, b in zip(mine, theirs)):
                        return False
        return True


# ---------------------------------------------------------------- native reader / writer
class TraceReader:
    """Native reader over a file (memory-mapped) or bytes; rows addressed by offset."""

    def __init__(self, source):
        self._buf = None
        handle = ctypes.c_void_p()
        if isinstance(source, (bytes, bytearray, memoryview)):
            self._buf = ctypes.create_string_buffer(bytes(source), len(source)) if len(source) else None
            rc = _lib.fn("ap_trace_open_memory")(self._buf, len(source), ctypes.byref(handle))
        else:
            rc = _lib.fn("ap_trace_open")(os.fsencode(os.fspath(source)), ctypes.byref(handle))
        _lib.check(rc, "trace open")
        self._h = handle
        c = _lib.TraceHeaderC()
        _lib.check(_lib.fn("ap_trace_get_header")(self._h, ctypes.byref(c)), "trace header")
        self.header = TraceHeader._from_c(c)

    def close(self):
        if getattr(self, "_h", None):
            _lib.fn("ap_trace_close")(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        self.close()

    def validate(self) -> None:
        """Structure (length prefixes, truncation, trailing bytes) and row invariants."""
        _lib.check(_lib.fn("ap_trace_validate")(self._h), "trace")

    def read_rows(self, layer: int, head: int, step_lo: int | None = None, step_hi: int | None = None,
                  pad_to: int | None = None) -> np.ndarray:
        """Rows of steps [step_lo, step_hi) as a float32 [n, width] array, zero-padded to pad_to
        (default: the longest row)."""
        h = self.header
        lo = h.first_step_offset if step_lo is None else step_lo
        hi = h.num_decode_steps + 1 if step_hi is None else step_hi
        width = max(pad_to or 0, h.prefill_len + hi - 1, 1)
        out = np.zeros((max(hi - lo, 0), width), dtype=np.float32)
        _lib.check(_lib.fn("ap_trace_read_rows")(self._h, layer, head, lo, hi, out.ctypes.data, width, width),
                   "trace rows")
        return out

    def gather_step(self, step: int, pad_to: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
        """Row of `step` for every (layer, head) as [num_layers * num_heads, width] float32."""
        h = self.header
        width = max(pad_to or 0, h.row_len(step))
        if out is None:
            out = np.zeros((h.num_layers * h.num_heads, width), dtype=np.float32)
        if out.dtype != np.float32 or not out.flags.c_contiguous or out.shape[0] < h.num_layers * h.num_heads:
            raise ValueError("out must be a C-contiguous float32 [maps, width] array")
        _lib.check(_lib.fn("ap_trace_gather_step")(self._h, step, out.ctypes.data, out.shape[1], out.shape[1]),
                   "trace step")
        return out

    def read_qk(self, layer: int, head: int) -> tuple[np.ndarray, np.ndarray]:
        h = self.header
        q = np.empty((h.rows_per_head, h.head_dim), dtype=np.float32)
        k = np.empty((h.total_len, h.head_dim), dtype=np.float32)
        _lib.check(_lib.fn("ap_trace_read_qk")(self._h, layer, head, q.ctypes.data, k.ctypes.data), "trace q/k")
        return q, k

    def to_trace(self) -> AttentionTrace:
        h = self.header
        rows = []
        for layer in range(h.num_layers):
            per_layer = []
            for head in range(h.num_heads):
                blk = self.read_rows(layer, head)
                per_layer.append([blk[k, : h.row_len(s)].copy() for k, s in enumerate(h.steps)])
            rows.append(per_layer)
        queries, keys = [], []
        if h.has_qk:
            for layer in range(h.num_layers):
                qs, ks = zip(*(self.read_qk(layer, head) for head in range(h.num_heads)))
                queries.append(list(qs))
                keys.append(list(ks))
        return AttentionTrace(header=h, rows=rows, queries=queries, keys=keys)


def _serialise(trace: AttentionTrace, path: str | None) -> tuple[int, bytes | None]:
    trace.validate()
    h = trace.header
    c = h._c()
    w = ctypes.c_void_p()
    _lib.check(_lib.fn("ap_trace_writer_open")(None if path is None else os.fsencode(path), ctypes.byref(c),
                                               ctypes.byref(w)), "trace writer")
    try:
        append = _lib.fn("ap_trace_writer_append_row")
        for per_layer in trace.rows:
            for per_head in per_layer:
                for row in per_head:
                    r = np.ascontiguousarray(row, dtype="<f4")
                    _lib.check(append(w, r.ctypes.data, r.size), "trace row")
        if h.has_qk:
            append_qk = _lib.fn("ap_trace_writer_append_qk")
            for layer in range(h.num_layers):
                for head in range(h.num_heads):
                    q = np.ascontiguousarray(trace.queries[layer][head], dtype="<f4")
                    k = np.ascontiguousarray(trace.keys[layer][head], dtype="<f4")
                    _lib.check(append_qk(w, q.ctypes.data, k.ctypes.data), "trace q/k")
        n = ctypes.c_int64()
        _lib.check(_lib.fn("ap_trace_writer_finish")(w, ctypes.byref(n)), "trace writer")
        data = None
        if path is None:
            p, m = ctypes.c_void_p(), ctypes.c_int64()
            _lib.check(_lib.fn("ap_trace_writer_bytes")(w, ctypes.byref(p), ctypes.byref(m)), "trace writer")
            data = ctypes.string_at(p, m.value)
        return n.value, data
    finally:
        _lib.fn("ap_trace_writer_free")(w)


def write_trace(trace: AttentionTrace, destination) -> int:
    """Serialise a validated trace into a binary sink; returns bytes written (trace.py:182-212)."""
    n, data = _serialise(trace, None)
    destination.write(data)
    return n


def read_trace(source) -> AttentionTrace:
    """Inverse of write_trace; validates invariants on load (trace.py:215-291)."""
    data = source.read()
    with TraceReader(data) as r:
        r.validate()
        return r.to_trace()


def write_trace_file(trace: AttentionTrace, path) -> int:
    n, _ = _serialise(trace, os.fspath(path))
    return n


def read_trace_file(path) -> AttentionTrace:
    with TraceReader(path) as r:
        r.validate()
        return r.to_trace()


def trace_to_bytes(trace: AttentionTrace) -> bytes:
    buf = io.BytesIO()
    write_trace(trace, buf)
    return buf.getvalue()


def trace_from_bytes(data: bytes) -> AttentionTrace:
    return read_trace(io.BytesIO(data))
