"""Chunked binary trace I/O (drop-in for ``pkg/src/xstrace/traceio.py``),
columnar and native.

``read_trace_columnar`` decodes XSTRACE1 chunks (docs/trace-format.md:20-50)
with the native decoder in ``csrc/xs_ingest.cu`` on a thread pool (one chunk
per task, the GIL released inside the C call), straight into the columns the
device pipeline consumes; ``read_trace`` wraps it for the reference's
Event-object API.  ``write_trace`` produces the reference's exact bytes
(deterministic chunking, per-chunk string tables in first-use order) with
vectorised numpy encoding.  Errors are the reference's classes and messages.
"""

from __future__ import annotations

import ctypes as C
import os
import struct
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
from typing import Optional, Union

import numpy as np

from . import _lib
from .columnar import ColumnarTrace
from .model import ProcessMeta, Trace, require_valid

MAGIC = b"XSTRACE1"
VERSION = 1
DEFAULT_CHUNK_LIMIT = 20 * 2**20
MIN_CHUNK_LIMIT = 4096
_HEADER = struct.Struct("<8sHQII")
_U32 = struct.Struct("<I")


class TraceFormatError(ValueError):
    """Bad magic, version, or undecodable payload (traceio.py:44-45)."""


class TruncatedTraceError(ValueError):
    """A chunk index named by meta.bin is missing (traceio.py:48-49)."""


class IncompleteTraceError(ValueError):
    """meta.bin absent: the writer never completed this directory (traceio.py:52-53)."""


class XsChunkInfo(C.Structure):
    _fields_ = [("clock_domain", C.c_int64), ("chunk_index", C.c_int32), ("n_records", C.c_int32),
                ("n_strings", C.c_int32), ("version", C.c_int32), ("records_offset", C.c_int64)]


# -- meta.bin ---------------------------------------------------------------------
class _Reader:
    def __init__(self, buf: bytes, context: str):
        self.buf, self.pos, self.context = buf, 0, context

    def take(self, n: int) -> bytes:
        if self.pos + n > len(self.buf):
            raise TraceFormatError(f"format error: {self.context} truncated at byte {self.pos}")
        out = self.buf[self.pos: self.pos + n]
        self.pos += n
        return out

    def unpack(self, st: struct.Struct):
        return st.unpack(self.take(st.size))

    def string(self) -> str:
        (n,) = self.unpack(_U32)
        try:
            return self.take(n).decode("utf-8")
        except UnicodeDecodeError as exc:
            raise TraceFormatError(f"format error: bad utf-8 in {self.context}") from exc


def _check_header(magic, version, index, context, expect_index):
    if magic != MAGIC:
        raise TraceFormatError(f"format error: bad magic {magic!r} in {context}")
    if version != VERSION:
        raise TraceFormatError(f"format error: unsupported version {version} in {context}")
    if expect_index is not None and index != expect_index:
        raise TraceFormatError(f"format error: {context} declares chunk index {index}, expected {expect_index}")


def _read_meta(source: Path):
    meta_path = source / "meta.bin"
    if not meta_path.exists():
        raise IncompleteTraceError(f"incomplete trace: {source} has no meta.bin")
    r = _Reader(meta_path.read_bytes(), "meta.bin")
    magic, version, clock_domain, chunk_count, process_count = r.unpack(_HEADER)
    _check_header(magic, version, chunk_count, "meta.bin", None)
    processes = []
    for _ in range(process_count):
        (pid,) = r.unpack(struct.Struct("<q"))
        name = r.string()
        values = []
        for fmt in ("<q", "<Q", "<Q"):
            (flag,) = r.unpack(struct.Struct("<B"))
            if flag == 1:
                values.append(r.unpack(struct.Struct(fmt))[0])
            elif flag == 0:
                values.append(None)
            else:
                raise TraceFormatError(f"format error: bad optional flag {flag} in meta.bin")
        processes.append(ProcessMeta(pid, name, values[0], values[1], values[2]))
    return clock_domain, chunk_count, processes


# -- chunks -------------------------------------------------------------------------
def _chunk_header(lib, buf: np.ndarray, context: str, index: int, clock_domain: int):
    info = XsChunkInfo()
    err = C.create_string_buffer(256)
    ctx = context.encode()
    st = lib.xs_chunk_info(buf.ctypes.data, buf.size, ctx, C.byref(info), None, None, err, 256)
    if st == 2:
        raise TraceFormatError(f"format error: bad magic {bytes(buf[:8])!r} in {context}")
    if st != 0:
        raise TraceFormatError(err.value.decode())
    _check_header(MAGIC, info.version, info.chunk_index, context, index)
    if info.clock_domain != clock_domain:
        raise TraceFormatError(f"format error: {context} clock domain {info.clock_domain} != {clock_domain}")
    off = np.zeros(max(info.n_strings, 1), np.int64)
    ln = np.zeros(max(info.n_strings, 1), np.int64)
    lib.xs_chunk_info(buf.ctypes.data, buf.size, ctx, C.byref(info), off.ctypes.data, ln.ctypes.data, err, 256)
    strings = []
    for o, n in zip(off[: info.n_strings].tolist(), ln[: info.n_strings].tolist()):
        try:
            strings.append(buf[o: o + n].tobytes().decode("utf-8"))
        except UnicodeDecodeError as exc:
            raise TraceFormatError(f"format error: bad utf-8 in {context}") from exc
    return info, strings


def read_trace_columnar(source: Union[str, os.PathLike], workers: Optional[int] = None) -> ColumnarTrace:
    """Load a trace directory straight into a ColumnarTrace, rows in
    Event.sort_key order exactly like read_trace (traceio.py:243-275)."""
    source = Path(source)
    clock_domain, chunk_count, processes = _read_meta(source)
    lib = _lib.load()
    bufs, heads = [], []
    for index in range(chunk_count):
        path = source / f"trace.{index}.bin"
        if not path.exists():
            raise TruncatedTraceError(f"truncated trace: {source} is missing chunk {index}")
        buf = np.fromfile(path, dtype=np.uint8)
        bufs.append(buf)
        heads.append(_chunk_header(lib, buf, path.name, index, clock_domain))
    names = sorted(set().union(*[set(s) for _, s in heads])) if heads else []
    rank = {s: i for i, s in enumerate(names)}
    counts = [h[0].n_records for h in heads]
    base = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64) if counts else np.zeros(1, np.int64)
    n = int(base[-1])
    cols = {"pid": np.empty(n, np.int64), "tid": np.empty(n, np.int64), "cat": np.empty(n, np.uint8),
            "name": np.empty(n, np.int32), "start": np.empty(n, np.int64), "dur": np.empty(n, np.int64),
            "corr": np.empty(n, np.int64), "has_corr": np.empty(n, np.uint8)}

    def decode(k):
        info, strings = heads[k]
        nmap = np.array([rank[s] for s in strings] or [0], np.int32)
        b = int(base[k])
        err = C.create_string_buffer(256)

        def at(a):
            return a.ctypes.data + b * a.itemsize

        st = lib.xs_chunk_decode(bufs[k].ctypes.data, bufs[k].size, f"trace.{k}.bin".encode(), C.byref(info),
                                 nmap.ctypes.data, at(cols["pid"]), at(cols["tid"]), at(cols["cat"]),
                                 at(cols["name"]), at(cols["start"]), at(cols["dur"]), at(cols["corr"]),
                                 at(cols["has_corr"]), err, 256)
        return None if st == 0 else err.value.decode()

    w = workers or min(len(bufs), os.cpu_count() or 1)
    if w > 1 and len(bufs) > 1:
        with ThreadPoolExecutor(w) as pool:
            errs = list(pool.map(decode, range(len(bufs))))
    else:
        errs = [decode(k) for k in range(len(bufs))]
    for e in errs:
        if e is not None:
            raise TraceFormatError(e)
    # rows in Event.sort_key order (start, end, category, pid, tid, name, corr or -1), stable
    keys = _sort_keys(cols)
    if n > 1 and not _is_sorted(keys):
        order = np.lexsort(tuple(reversed(keys)))
        cols = {k: v[order] for k, v in cols.items()}
    return ColumnarTrace.from_arrays(clock_domain, cols["start"], cols["dur"], cols["pid"], cols["tid"], cols["cat"],
                                     cols["name"], names, cols["corr"], cols["has_corr"], tuple(processes))


def _sort_keys(cols):
    return (cols["start"], cols["start"] + cols["dur"], cols["cat"], cols["pid"], cols["tid"], cols["name"],
            np.where(cols["has_corr"] == 1, cols["corr"], -1))


def _is_sorted(keys) -> bool:
    """Lexicographic non-decreasing check over consecutive rows."""
    undecided = np.ones(keys[0].shape[0] - 1, bool)
    for k in keys:
        a, b = k[:-1], k[1:]
        if np.any(undecided & (a > b)):
            return False
        undecided &= a == b
        if not undecided.any():
            break
    return True


def read_trace(source: Union[str, os.PathLike]) -> Trace:
    """Load a trace directory; inverse of write_trace up to stable ordering."""
    ct = read_trace_columnar(source)
    return ct.to_trace()


# -- writer -------------------------------------------------------------------------
def _record_sizes(has_corr: np.ndarray) -> np.ndarray:
    return 42 + 8 * has_corr.astype(np.int64)  # traceio.record_size (traceio.py:80-82)


def _chunk_bounds(rs: np.ndarray, name: np.ndarray, name_cost: np.ndarray, limit: int) -> list:
    """Row ranges of the chunks _ChunkBuilder would flush (traceio.py:85-114,
    145-160): a chunk grows while header + string table + records fits the
    limit; a record that does not fit starts the next chunk (the first record
    of a chunk always stays)."""
    n = rs.shape[0]
    pre = np.concatenate([[0], np.cumsum(rs)])
    occ = {int(k): np.nonzero(name == k)[0] for k in np.unique(name)} if n else {}
    bounds, i0 = [], 0
    while i0 < n:
        firsts = []
        for k, idx in occ.items():
            j = np.searchsorted(idx, i0)
            if j < idx.size:
                firsts.append((int(idx[j]), int(name_cost[k])))

        def size_through(j):  # chunk bytes holding rows [i0, j]
            return _HEADER.size + 4 + int(pre[j + 1] - pre[i0]) + sum(c for f, c in firsts if f <= j)

        lo, hi = i0, n - 1  # largest j with size_through(j) <= limit (at least i0)
        if size_through(hi) <= limit:
            j = hi
        else:
            while lo < hi:
                mid = (lo + hi + 1) // 2
                if size_through(mid) <= limit:
                    lo = mid
                else:
                    hi = mid - 1
            j = lo
        bounds.append((i0, j + 1))
        i0 = j + 1
    return bounds


def _encode_chunk(ct: ColumnarTrace, order: np.ndarray, a: int, b: int, index: int) -> bytes:
    rows = order[a:b]
    name = ct.name[rows]
    _, first = np.unique(name, return_index=True)
    local_names = name[np.sort(first)]  # first-use order
    lidx = np.zeros(max(len(ct.names), 1), np.int64)
    lidx[local_names] = np.arange(local_names.size)
    has = ct.has_corr[rows].astype(np.int64)
    rs = 42 + 8 * has
    off = np.concatenate([[0], np.cumsum(rs)[:-1]]).astype(np.int64)
    out = np.zeros(int(rs.sum()), np.uint8)

    def put(at, values, dtype):
        v = np.ascontiguousarray(values.astype(dtype)).view(np.uint8).reshape(values.shape[0], -1)
        w = v.shape[1]
        out[(off[:, None] + at + np.arange(w)).reshape(-1)] = v.reshape(-1)

    put(0, rs - 4, "<u4")
    put(4, ct.pids[ct.pid[rows]], "<i8")
    put(12, ct.group_tid[ct.tid[rows]], "<i8")
    put(20, ct.cat[rows], "u1")
    put(21, lidx[name], "<u4")
    put(25, ct.start[rows], "<i8")
    put(33, ct.dur[rows], "<i8")
    put(41, has, "u1")
    sel = np.nonzero(has)[0]
    if sel.size:
        v = np.ascontiguousarray(ct.corr[rows][sel].astype("<i8")).view(np.uint8).reshape(-1, 8)
        out[(off[sel][:, None] + 42 + np.arange(8)).reshape(-1)] = v.reshape(-1)
    table = b"".join(_U32.pack(len(s)) + s for s in (ct.names[k].encode("utf-8") for k in local_names.tolist()))
    return (_HEADER.pack(MAGIC, VERSION, ct.clock_domain, index, b - a) + _U32.pack(local_names.size) + table
            + out.tobytes())


def _encode_meta(clock_domain, processes, chunk_count: int) -> bytes:
    out = bytearray(_HEADER.pack(MAGIC, VERSION, clock_domain, chunk_count, len(processes)))
    for meta in sorted(processes, key=lambda m: m.pid):
        raw = meta.name.encode("utf-8")
        out += struct.pack("<q", meta.pid) + _U32.pack(len(raw)) + raw
        for value, fmt in ((meta.parent, "<q"), (meta.fork_ns, "<Q"), (meta.join_ns, "<Q")):
            out += b"\x00" if value is None else b"\x01" + struct.pack(fmt, value)
    return bytes(out)


def write_trace(trace, sink: Union[str, os.PathLike], chunk_limit_bytes: int = DEFAULT_CHUNK_LIMIT) -> int:
    """Serialize ``trace`` (a Trace or ColumnarTrace) into directory ``sink``;
    returns the chunk count (traceio.py:137-166), byte-identical to the
    reference writer."""
    if chunk_limit_bytes < MIN_CHUNK_LIMIT:
        raise ValueError(f"chunk_limit_bytes must be >= {MIN_CHUNK_LIMIT}, got {chunk_limit_bytes}")
    require_valid(trace)
    return _write_unchecked(trace, sink, chunk_limit_bytes)


def _write_unchecked(trace, sink, chunk_limit_bytes: int = DEFAULT_CHUNK_LIMIT) -> int:
    """write_trace after validation (the encoder alone; host-only)."""
    ct = trace if isinstance(trace, ColumnarTrace) else ColumnarTrace.from_trace(trace)
    sink = Path(sink)
    sink.mkdir(parents=True, exist_ok=True)
    n = ct.n
    if n:
        cols = {"start": ct.start, "dur": ct.dur, "cat": ct.cat, "pid": ct.pids[ct.pid], "tid": ct.group_tid[ct.tid],
                "name": ct.name, "corr": ct.corr, "has_corr": ct.has_corr}
        order = np.lexsort(tuple(reversed(_sort_keys(cols))))
        name_cost = np.array([4 + len(s.encode("utf-8")) for s in ct.names], np.int64)
        bounds = _chunk_bounds(_record_sizes(ct.has_corr[order]), ct.name[order], name_cost, chunk_limit_bytes)
    else:
        order, bounds = np.zeros(0, np.int64), []
    for index, (a, b) in enumerate(bounds):
        (sink / f"trace.{index}.bin").write_bytes(_encode_chunk(ct, order, a, b, index))
    (sink / "meta.bin").write_bytes(_encode_meta(ct.clock_domain, ct.processes, len(bounds)))
    return len(bounds)
