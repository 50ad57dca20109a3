"""Device session: uploads columnar traces and drives the C ABI.

PyTorch is used only for device memory and the current CUDA stream; all
analysis runs in ``libxstrace_b200.so`` (hand-written sm_100a kernels).
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .columnar import ColumnarTrace

_engines: dict = {}
_lock = threading.Lock()


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("xstrace-b200 needs a CUDA device (B200); none is visible")
    return torch


def packed_ptrs(lay, dblock, a: int = 0) -> dict:
    """Device addresses of row ``a`` of every packed column (and of the start
    base of row a's 256-row block) in a device copy of the whole packed block."""
    base = dblock.data_ptr()
    p = {k: base + lay.offsets[k] + a * lay.widths[k] for k in ("start", "dur", "pid", "tid", "name", "corr", "catf")}
    p["start_base"] = base + lay.offsets["start_base"] + (a // 256) * 8
    for k in ("exc_row", "exc_val", "exc_col"):  # (the whole table: xs_unpack skips rows outside the range)
        p[k] = base + lay.offsets[k]
    return p


def unpack_into(eng, lay, ptrs: dict, a: int, b: int, dst, stream=None) -> None:
    """xs_unpack rows [a, b) of a packed trace (``ptrs``: device addresses of
    row a of each packed column, see packed_ptrs) into the wide device
    columns of ``dst`` (rows from 0)."""
    torch = _torch()
    w = lay.widths
    pk = _lib.XsPacked()
    pk.n, pk.row0 = b - a, a
    for k in ("start", "start_base", "dur", "pid", "tid", "name", "corr", "catf"):
        setattr(pk, k, ptrs[k])
    pk.start_w, pk.dur_w, pk.pid_w, pk.tid_w, pk.name_w, pk.corr_w = (w["start"], w["dur"], w["pid"], w["tid"],
                                                                      w["name"], w["corr"])
    pk.n_exc = lay.n_exc
    pk.exc_row, pk.exc_val, pk.exc_col = ptrs["exc_row"], ptrs["exc_val"], ptrs["exc_col"]
    s = torch.cuda.current_stream(eng.device) if stream is None else stream
    eng.check(eng.lib.xs_unpack(eng.ctx, C.byref(pk), dst.start.data_ptr(), dst.dur.data_ptr(), dst.pid.data_ptr(),
                                dst.tid.data_ptr(), dst.cat.data_ptr(), dst.name.data_ptr(), dst.corr.data_ptr(),
                                dst.has_corr.data_ptr(), C.c_void_p(s.cuda_stream)), "xs_unpack")


class DeviceTrace:
    """Columns of a ColumnarTrace resident in device memory.

    A pinned trace (ColumnarTrace.pinned) keeps its own device copy.  An
    ordinary host trace is staged through the engine's page-locked block and
    its device columns live in the engine's staging buffers: such a
    DeviceTrace is valid until the next ordinary-trace DeviceTrace on the same
    device (the public entry points use one at a time; to keep several
    resident at once, pin the traces)."""

    def __init__(self, ct: ColumnarTrace, device: int = 0, non_blocking: bool = False):
        torch = _torch()
        dev = torch.device("cuda", device)
        self.ct = ct
        self.device = device

        pinned = ct._pinned or {}
        block = pinned.get("_block")
        lay = pinned.get("_packed")
        staged = None
        if not pinned and ct.n:
            # ordinary host columns: the native builder packs them into the
            # engine's page-locked staging block (host threads), then the
            # packed path below uploads it in one DMA
            staged = get(device).stage_packed(ct)
            if staged is not None:
                lay, block, pinned = staged
        if lay is not None:  # packed pinned block: one DMA of ~16 B/event, widened by xs_unpack
            # the device staging (packed block + wide columns) is kept with the
            # pinned trace and refilled by every DeviceTrace of it: the content
            # is the same trace, and repeated calls skip ~10 tensor allocations
            # (staged traces: one grow-only set per engine, capacity-sized)
            n = ct.n
            cache = pinned.get("_dev_cache")
            need = (lay.total, n)
            if cache is None or cache[0] != device or (staged is not None and (cache[5][0] < need[0] or
                                                                               cache[5][1] < need[1])):
                cap = (max(need[0], int(need[0] * 1.25)), max(n, int(n * 1.25))) if staged is not None else need
                dblock = torch.empty(max(cap[0], 16), dtype=torch.uint8, device=dev)
                m = max(cap[1], 1)
                spec = (("start", torch.int64, 8), ("dur", torch.int64, 8), ("corr", torch.int64, 8),
                        ("pid", torch.int32, 4), ("tid", torch.int32, 4), ("name", torch.int32, 4),
                        ("cat", torch.uint8, 1), ("has_corr", torch.uint8, 1))
                # every column starts 16-byte aligned: size the block as the
                # sum of the ROUNDED column sizes (38*m would be short by up to
                # 7*15 bytes of padding)
                wide = torch.empty(sum((m * w + 15) // 16 * 16 for _, _, w in spec), dtype=torch.uint8, device=dev)
                cols = {}
                off = 0
                for k, dt, w in spec:
                    cols[k] = wide[off:off + m * w].view(dt)
                    assert cols[k].numel() == m, (k, cols[k].numel(), m)
                    off += (m * w + 15) // 16 * 16
                for k, dt in (("group_pid", torch.int32), ("pid_has_meta", torch.uint8)):
                    cols[k] = torch.zeros(1, dtype=dt, device=dev)  # (empty table; else a view, per call)
                cache = (device, dblock, wide, cols, None, cap)
                pinned["_dev_cache"] = cache
            _, dblock, self._wide, cols, _, _ = cache
            self._dblock = dblock
            ptrs = packed_ptrs(lay, dblock)
            nb = max(lay.total, 16)
            dblock[:nb].copy_(block[:nb], non_blocking=True)
            if staged is not None:
                get(device).staged_upload_done()
            for k, t in cols.items():
                if k in ("group_pid", "pid_has_meta"):
                    o, nbk = lay.offsets[k], lay.nbytes[k]
                    t = dblock[o:o + nbk].view(t.dtype) if nbk else t
                else:
                    t = t[:max(n, 1)]
                setattr(self, k, t)
            if n:
                unpack_into(get(device), lay, ptrs, 0, n, self)
            return
        if block is not None:  # one pinned block (ColumnarTrace.pinned): one DMA, device views
            dblock = block.to(dev, non_blocking=True)
            self._dblock = dblock
            for k, o in zip(ColumnarTrace._COLUMNS, pinned["_offsets"]):
                a = getattr(ct, k)
                if a.size == 0:
                    setattr(self, k, torch.zeros(1, dtype=_TORCH[a.dtype.type], device=dev))
                else:
                    setattr(self, k, dblock[o:o + a.nbytes].view(_TORCH[a.dtype.type]))
            return

        def up(key, dtype):
            t = pinned.get(key)
            a = getattr(ct, key)
            if a.size == 0:
                return torch.zeros(1, dtype=_TORCH[dtype], device=dev)
            if t is not None and t.dtype == _TORCH[dtype]:  # page-locked: asynchronous DMA
                return t.to(dev, non_blocking=True)
            a = np.ascontiguousarray(a, dtype=dtype)
            return torch.from_numpy(a).to(dev, non_blocking=non_blocking)

        self.start = up("start", np.int64)
        self.dur = up("dur", np.int64)
        self.pid = up("pid", np.int32)
        self.tid = up("tid", np.int32)
        self.cat = up("cat", np.uint8)
        self.name = up("name", np.int32)
        self.corr = up("corr", np.int64)
        self.has_corr = up("has_corr", np.uint8)
        self.group_pid = up("group_pid", np.int32)
        self.pid_has_meta = up("pid_has_meta", np.uint8)

    @classmethod
    def from_tensors(cls, ct: ColumnarTrace, tensors: dict, device: int = 0) -> "DeviceTrace":
        obj = cls.__new__(cls)
        obj.ct = ct
        obj.device = device
        for k, v in tensors.items():
            setattr(obj, k, v)
        return obj

    def h2d_bytes(self) -> int:
        return sum(int(t.numel() * t.element_size()) for t in
                   (self.start, self.dur, self.pid, self.tid, self.cat, self.name, self.corr, self.has_corr,
                    self.group_pid, self.pid_has_meta))

    def struct(self, start=None, dur=None) -> _lib.XsEvents:
        ct = self.ct
        s = self.start if start is None else start
        d = self.dur if dur is None else dur
        return _lib.XsEvents(ct.n, s.data_ptr(), d.data_ptr(), self.pid.data_ptr(), self.tid.data_ptr(),
                             self.cat.data_ptr(), self.name.data_ptr(), self.corr.data_ptr(),
                             self.has_corr.data_ptr(), ct.n_pids, ct.n_groups, len(ct.names), 0,
                             self.group_pid.data_ptr(), self.pid_has_meta.data_ptr())


_TORCH = {}


def _init_torch_types():
    import torch

    _TORCH.update({np.int64: torch.int64, np.int32: torch.int32, np.uint8: torch.uint8})


def torch_dtype(np_dtype):
    """torch dtype of a numpy column dtype (int64 / int32 / uint8)."""
    _torch()
    if not _TORCH:
        _init_torch_types()
    return _TORCH[np.dtype(np_dtype).type]


class XsError(RuntimeError):
    def __init__(self, status: int, message: str):
        self.status = status
        super().__init__(message)


@dataclass
class OverlapRaw:
    cell_pid: np.ndarray
    cell_node: np.ndarray
    cell_mask: np.ndarray
    cell_ns: np.ndarray
    node_parent: np.ndarray
    node_name: np.ndarray
    span_lo: np.ndarray
    span_hi: np.ndarray
    tracked: np.ndarray
    has_events: np.ndarray


@dataclass
class CorrectRaw:
    start: object  # device tensor
    dur: object
    removed: np.ndarray     # [n_pids, 4]
    shortfall: np.ndarray   # [n_pids, 4]
    original_total: int
    corrected_total: int
    n_sites: int
    n_slabs: int


class Engine:
    """One C-ABI context per device (workspace reused across calls)."""

    def __init__(self, device: int = 0):
        _torch()
        if not _TORCH:
            _init_torch_types()
        self.lib = _lib.load()
        self.device = device
        self._prof_cache = None
        self.fetched_bytes = 0  # D2H bytes of overlap results read back (bench accounting)
        h = C.c_void_p()
        st = self.lib.xs_ctx_create(device, C.byref(h))
        if st != 0:
            raise RuntimeError(f"xs_ctx_create failed: {self.lib.xs_status_str(st).decode()}")
        self.ctx = h

    def __del__(self):
        try:
            if getattr(self, "ctx", None):
                self.lib.xs_ctx_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass

    # -- helpers ---------------------------------------------------------------
    def stream(self):
        torch = _torch()
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def check(self, st: int, what: str):
        if st != 0:
            msg = self.lib.xs_last_error(self.ctx).decode(errors="replace")
            raise XsError(st, f"{what}: {self.lib.xs_status_str(st).decode()} {msg}".strip())

    def stage_packed(self, ct: ColumnarTrace):
        """Pack host columns into this engine's page-locked staging block
        (native builder, host threads).  Returns (layout, block tensor, the
        staging state dict that keeps the device buffers) or None when the
        trace is not packable.  The block is reused by the next call once the
        DMA recorded by staged_upload_done has finished."""
        from .columnar import pack_native

        torch = _torch()
        st = self.__dict__.setdefault("_staging", {})
        ev = st.get("event")
        if ev is not None:
            ev.synchronize()  # the previous upload out of the block is done

        def alloc(nbytes):
            blk = st.get("block")
            if blk is None or blk.numel() < nbytes:
                blk = torch.empty(max(nbytes, int(nbytes * 1.25)), dtype=torch.uint8, pin_memory=True)
                st["block"] = blk
            return blk.numpy()[:nbytes]

        got = pack_native(ct, alloc)
        if got is None:
            return None
        lay, _ = got
        return lay, st["block"], st

    def staged_upload_done(self) -> None:
        torch = _torch()
        st = self._staging
        ev = st.get("event") or torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        st["event"] = ev

    def launches(self) -> int:
        return int(self.lib.xs_launch_count(self.ctx))

    # -- entry points ------------------------------------------------------------
    def validate(self, dt: DeviceTrace) -> int:
        ev = dt.struct()
        bad = C.c_int64(0)
        self.check(self.lib.xs_validate(self.ctx, C.byref(ev), C.byref(bad), self.stream()), "xs_validate")
        return int(bad.value)

    def overlap(self, dt: DeviceTrace, attribution: int, start=None, dur=None) -> OverlapRaw:
        ev = dt.struct(start, dur)
        self.check(self.lib.xs_overlap(self.ctx, C.byref(ev), attribution, self.stream()), "xs_overlap")
        return self.fetch_overlap()

    def overlap_info(self) -> tuple:
        """(n_cells, n_nodes, n_pids) of the last overlap result (host-side, no copy)."""
        info = _lib.XsOverlapInfo()
        self.check(self.lib.xs_overlap_info(self.ctx, C.byref(info)), "xs_overlap_info")
        return int(info.n_cells), int(info.n_nodes), int(info.n_pids)

    def fetch_overlap(self) -> OverlapRaw:
        info = _lib.XsOverlapInfo()
        self.check(self.lib.xs_overlap_info(self.ctx, C.byref(info)), "xs_overlap_info")
        nc, nn, np_ = int(info.n_cells), int(info.n_nodes), int(info.n_pids)
        # one page-locked block (torch's caching host allocator: reused once
        # the arrays of an earlier result are dropped) so the copy runs at
        # DMA rate instead of through pageable staging; the arrays keep it alive
        shapes = ((nc, np.int32), (nc, np.int32), (nc, np.int32), (nc, np.int64), (nn, np.int32), (nn, np.int32),
                  (np_, np.int64), (np_, np.int64), (np_, np.int64), (np_, np.uint8))
        offs, total = [], 0
        for m, dt in shapes:
            offs.append(total)
            total += (m * np.dtype(dt).itemsize + 15) // 16 * 16
        raw = _torch().empty(max(total, 16), dtype=_torch().uint8, pin_memory=True).numpy()
        r = OverlapRaw(*[raw[o:o + m * np.dtype(dt).itemsize].view(dt) for o, (m, dt) in zip(offs, shapes)])

        def p(a):
            return a.ctypes.data if a.size else None

        self.check(self.lib.xs_overlap_fetch(self.ctx, p(r.cell_pid), p(r.cell_node), p(r.cell_mask), p(r.cell_ns),
                                             p(r.node_parent), p(r.node_name), p(r.span_lo), p(r.span_hi),
                                             p(r.tracked), p(r.has_events), self.stream()), "xs_overlap_fetch")
        self.fetched_bytes += sum(a.nbytes for a in (r.cell_pid, r.cell_node, r.cell_mask, r.cell_ns, r.node_parent,
                                                     r.node_name, r.span_lo, r.span_hi, r.tracked, r.has_events))
        return r

    def _profile(self, dt: DeviceTrace, scaled):
        # the per-name tables stay resident for the last profile seen (a
        # ScaledProfile is immutable), so repeated calls copy nothing
        hit = self._prof_cache
        if hit is not None and hit[0] is scaled and hit[3] == len(dt.ct.names):
            return hit[1], hit[2]
        prof, keep = self._profile_upload(dt, scaled)
        self._prof_cache = (scaled, prof, keep, len(dt.ct.names))
        return prof, keep

    def _profile_upload(self, dt: DeviceTrace, scaled):
        torch = _torch()
        dev = torch.device("cuda", self.device)
        n_names = max(len(dt.ct.names), 1)
        internal = torch.zeros(n_names, dtype=torch.int64, device=dev)
        has = torch.zeros(n_names, dtype=torch.uint8, device=dev)
        if len(dt.ct.names):
            internal.copy_(torch.from_numpy(np.array(scaled.internal, np.int64)))
            has.copy_(torch.from_numpy(np.array(scaled.has_internal, np.uint8)))
        words = np.array(scaled.words_of(scaled.L) + [int(x) for x in scaled.frac_table()], np.uint64)
        tab = torch.from_numpy(words.view(np.int64)).to(dev)  # [L words | frac rows]
        w = scaled.words
        prof = _lib.XsProfile(w, 0, tab.data_ptr(), (C.c_int64 * 4)(*scaled.whole), tab.data_ptr() + 8 * w,
                              internal.data_ptr(), has.data_ptr())
        return prof, (internal, has, tab)

    def correct(self, dt: DeviceTrace, scaled, analyze_attribution: Optional[int] = None,
                host_out=None, dev_out=None, async_copy: bool = False, carries=None) -> CorrectRaw:
        """xs_correct, or xs_analyze when analyze_attribution is given.  With
        ``host_out`` = (start, dur) host int64 buffers (pinned for overlap)
        the corrected columns are also copied there, overlapped with the
        overlap pass (xs_analyze_to_host)."""
        torch = _torch()
        dev = torch.device("cuda", self.device)
        n = max(dt.ct.n, 1)
        if dev_out is not None:  # caller-owned (async_copy: must outlive the copy, see host_copy_wait)
            out_s, out_d = dev_out
        else:
            out_s = torch.empty(n, dtype=torch.int64, device=dev)
            out_d = torch.empty(n, dtype=torch.int64, device=dev)
        ev = dt.struct()
        prof, keep = self._profile(dt, scaled)
        if carries is not None:  # window carries (xs_profile_t.residue_in / span_end_in), per pid of the call
            residue, span_end = carries
            t_res = torch.from_numpy(np.ascontiguousarray(residue, np.uint64).view(np.int64)).to(dev)
            t_end = torch.from_numpy(np.ascontiguousarray(span_end, np.int64)).to(dev)
            prof = _lib.XsProfile.from_buffer_copy(prof)
            prof.residue_in, prof.span_end_in = t_res.data_ptr(), t_end.data_ptr()
            keep = (keep, t_res, t_end)
        bad = C.c_int64(-1)
        if analyze_attribution is None:
            st = self.lib.xs_correct(self.ctx, C.byref(ev), C.byref(prof), out_s.data_ptr(), out_d.data_ptr(),
                                     C.byref(bad), self.stream())
        elif host_out is not None:
            fn = self.lib.xs_analyze_to_host_async if async_copy else self.lib.xs_analyze_to_host
            st = fn(self.ctx, C.byref(ev), C.byref(prof), analyze_attribution,
                                             out_s.data_ptr(), out_d.data_ptr(), _host_ptr(host_out[0]),
                                             _host_ptr(host_out[1]), C.byref(bad), self.stream())
        else:
            st = self.lib.xs_analyze(self.ctx, C.byref(ev), C.byref(prof), analyze_attribution, out_s.data_ptr(),
                                     out_d.data_ptr(), C.byref(bad), self.stream())
        if st == _lib.XS_UNCALIBRATED:
            raise UncalibratedEvent(int(bad.value))
        self.check(st, "xs_correct")
        P = dt.ct.n_pids
        removed = np.zeros(max(P, 1) * 4, np.int64)
        shortfall = np.zeros(max(P, 1) * 4, np.int64)
        info = _lib.XsCorrectInfo()
        self.check(self.lib.xs_correct_report(self.ctx, C.byref(info), removed.ctypes.data, shortfall.ctypes.data,
                                              self.stream()), "xs_correct_report")
        del keep  # (the report read-back has synchronised the call's stream)
        return CorrectRaw(out_s[: dt.ct.n], out_d[: dt.ct.n], removed[: P * 4].reshape(P, 4),
                          shortfall[: P * 4].reshape(P, 4), int(info.original_total), int(info.corrected_total),
                          int(info.n_sites), int(info.n_slabs))

    def host_copy_wait(self) -> None:
        """Wait for every corrected-column copy of correct(async_copy=True)."""
        self.check(self.lib.xs_host_copy_wait(self.ctx), "xs_host_copy_wait")

    def remap(self, pid_idx: np.ndarray, values: np.ndarray) -> np.ndarray:
        torch = _torch()
        dev = torch.device("cuda", self.device)
        if len(values) == 0:
            return np.zeros(0, np.int64)
        p = torch.from_numpy(np.ascontiguousarray(pid_idx, np.int32)).to(dev)
        v = torch.from_numpy(np.ascontiguousarray(values, np.int64)).to(dev)
        out = torch.empty_like(v)
        self.check(self.lib.xs_remap(self.ctx, len(values), p.data_ptr(), v.data_ptr(), out.data_ptr(),
                                     self.stream()), "xs_remap")
        return out.cpu().numpy()

    def transition_sites(self, dt: DeviceTrace, pair_mask: int):
        ev = dt.struct()
        n = C.c_int64(0)
        self.check(self.lib.xs_transition_sites(self.ctx, C.byref(ev), pair_mask, C.byref(n), self.stream()),
                   "xs_transition_sites")
        k = int(n.value)
        pair = np.zeros(max(k, 1), np.int32)
        event = np.zeros(max(k, 1), np.int64)
        self.check(self.lib.xs_transition_fetch(self.ctx, pair.ctypes.data, event.ctypes.data, self.stream()),
                   "xs_transition_fetch")
        return pair[:k], event[:k]


    def union(self, dt: DeviceTrace, category: int, per_pid: bool):
        """(union ns per pid or [trace-wide], span lo, span hi)."""
        ev = dt.struct()
        out = np.zeros(max(dt.ct.n_pids if per_pid else 1, 1), np.int64)
        lo, hi = C.c_int64(0), C.c_int64(0)
        self.check(self.lib.xs_union(self.ctx, C.byref(ev), int(category), 1 if per_pid else 0, out.ctypes.data,
                                     C.byref(lo), C.byref(hi), self.stream()), "xs_union")
        return out, int(lo.value), int(hi.value)

    def utilization(self, dt: DeviceTrace, period_ns: int, intervals: bool = False):
        """(utilized periods, span lo, span hi[, union interval lo/hi arrays])."""
        ev = dt.struct()
        util, nint, lo, hi = C.c_int64(0), C.c_int64(0), C.c_int64(0), C.c_int64(0)
        self.check(self.lib.xs_utilization(self.ctx, C.byref(ev), int(period_ns), C.byref(util), C.byref(nint),
                                           C.byref(lo), C.byref(hi), self.stream()), "xs_utilization")
        res = (int(util.value), int(lo.value), int(hi.value))
        if not intervals:
            return res
        k = int(nint.value)
        ilo = np.zeros(max(k, 1), np.int64)
        ihi = np.zeros(max(k, 1), np.int64)
        if k:
            self.check(self.lib.xs_union_intervals_fetch(self.ctx, ilo.ctypes.data, ihi.ctypes.data, self.stream()),
                       "xs_union_intervals_fetch")
        return res + (ilo[:k], ihi[:k])


def _host_ptr(a) -> int:
    """Address of a host int64 buffer: a numpy array or a CPU torch tensor."""
    if isinstance(a, np.ndarray):
        assert a.dtype == np.int64 and a.flags.c_contiguous
        return a.ctypes.data
    assert a.device.type == "cpu" and a.is_contiguous()
    return a.data_ptr()


class UncalibratedEvent(Exception):
    def __init__(self, index: int):
        self.index = index
        super().__init__(index)


_aux: dict = {}


def get_aux(device: int, k: int) -> Engine:
    """The k-th extra context on a device (k >= 1; k = 0 is get(device)):
    concurrent analyses each need their own workspace and graphs."""
    if k == 0:
        return get(device)
    with _lock:
        eng = _aux.get((device, k))
        if eng is None:
            eng = Engine(device)
            _aux[(device, k)] = eng
        return eng


def _destroy_all() -> None:
    """Free every context's workspace at interpreter exit (the workspace is
    owned by the context: compute-sanitizer's leak check sees it released)."""
    with _lock:
        for eng in list(_engines.values()) + list(_aux.values()):
            try:
                if eng.ctx:
                    eng.lib.xs_ctx_destroy(eng.ctx)
                    eng.ctx = None
            except Exception:
                pass


import atexit  # noqa: E402

atexit.register(_destroy_all)


def get(device: int = 0) -> Engine:
    with _lock:
        eng = _engines.get(device)
        if eng is None:
            eng = Engine(device)
            _engines[device] = eng
        return eng


def validate(trace) -> list:
    """validate_trace: device flag first, reference-style list on the error path."""
    from .model import format_violations, meta_violations

    if meta_violations(trace.processes):
        return format_violations(trace)
    ct = trace if isinstance(trace, ColumnarTrace) else ColumnarTrace.from_trace(trace)
    eng = get()
    dt = DeviceTrace(ct, eng.device)
    try:
        bad = eng.validate(dt)
    except XsError as exc:
        if exc.status == _lib.XS_INVALID_TRACE:
            bad = 1
        else:
            raise
    if bad == 0:
        return []
    src = trace if not isinstance(trace, ColumnarTrace) else ct.to_trace()
    return format_violations(src)
