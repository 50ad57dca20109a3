"""Vectorised synthetic workloads (test and bench infrastructure, not product).

Reproduces the *shape* of the reference generator (``_build_pid`` /
``_instrument_pid``, synth.py:246-375) with numpy so
that 1M-1B event traces build in seconds: a loop of operations (inference /
simulation / backprop) around BACKEND / SIMULATOR calls, ACCEL_API calls
launching kernels on one in-order GPU stream, one ambient HIGH_LEVEL event
per process, and an instrumented twin with a book-keeping slab inserted at
every hook site (InsertionMap, _timeline.py:70-81).  The random streams
differ from CPython's ``random`` (not needed: parity runs the oracle on
*these* traces).

With constant integer overheads the instrumented twin corrects back to the
uninstrumented trace exactly (correction closure): a size-independent parity
property for the 100M-1B configurations.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from .calibration import CalibrationProfile
from .columnar import ColumnarTrace
from .model import ProcessMeta

OPERATION, HIGH_LEVEL, BACKEND, SIMULATOR, ACCEL_API, GPU = range(6)
MAIN_TID, GPU_TID = 0, 1000

# (op name, level, calls, apis_per_call) -- synth.py:748-768
DDPG_PHASES = (("inference", BACKEND, 3, 2), ("simulation", SIMULATOR, 5, 0), ("backprop", BACKEND, 2, 4))
DUR = dict(glue=(1500, 2500), backend=(20000, 60000), simulator=(50000, 150000), api=(5000, 15000),
           api_gap=(1000, 3000), kernel=(10000, 40000))
LAUNCH_DELAY = 500
KERNEL_PROB = 0.7
EXACT = dict(annotation=4000, transition=1000, api_interception=1500, launch=3000, memcpy=1000)
API_NAMES = ("launch", "memcpy")  # sorted(api_internal)


def exact_profile() -> CalibrationProfile:
    return CalibrationProfile(Fraction(EXACT["annotation"]), Fraction(EXACT["transition"]),
                              Fraction(EXACT["api_interception"]),
                              {"launch": Fraction(EXACT["launch"]), "memcpy": Fraction(EXACT["memcpy"])})


def events_per_iteration(phases=DDPG_PHASES) -> float:
    return sum(1 + calls + calls * apis * (1 + KERNEL_PROB) for _, _, calls, apis in phases)


@dataclass
class Block:
    start: np.ndarray
    end: np.ndarray
    cat: int
    tid: int
    names: tuple          # candidate names
    name_sel: np.ndarray  # index into names per event
    corr: np.ndarray = None
    has_corr: np.ndarray = None


@dataclass
class PidTimeline:
    blocks: list
    site_anchor: np.ndarray
    site_amount: np.ndarray


def _u(rng, key, size):
    lo, hi = DUR[key]
    return rng.integers(lo, hi + 1, size=size, dtype=np.int64)


def build_pid(rng: np.random.Generator, iterations: int, phases=DDPG_PHASES, outer_op: str = None,
              second_tid_ops: bool = False) -> PidTimeline:
    """One process' uninstrumented timeline (vectorised _build_pid).

    ``outer_op`` wraps each iteration's phases in one more OPERATION (depth 2);
    ``second_tid_ops`` mirrors every phase op on tid 1 (cross-tid paths).
    """
    it = iterations
    keys = ["glue"]  # iteration glue
    marks = {}       # marker -> number of increments before it
    for ph, (op, level, calls, apis) in enumerate(phases):
        marks[("op_start", ph)] = len(keys)
        keys.append("glue")
        for c in range(calls):
            marks[("call_start", ph, c)] = len(keys)
            if level == BACKEND and apis > 0:
                keys.append("api_gap")
                for a in range(apis):
                    marks[("api_start", ph, c, a)] = len(keys)
                    keys.append("api")
                    marks[("api_end", ph, c, a)] = len(keys)
                    keys.append("api_gap")
            else:
                keys.append("backend" if level == BACKEND else "simulator")
            marks[("call_end", ph, c)] = len(keys)
            keys.append("glue")
        marks[("op_end", ph)] = len(keys)
    K = len(keys)
    inc = np.empty((it, K), np.int64)
    for j, key in enumerate(keys):
        inc[:, j] = _u(rng, key, it)
    csum = np.cumsum(inc.reshape(-1)).reshape(it, K)
    # time after k increments of iteration i: csum[i, k-1]
    T = {m: csum[:, k - 1] for m, k in marks.items()}

    blocks = []
    s_anchor, s_amount = [], []
    ann = EXACT["annotation"]
    zeros = np.zeros(it, np.int64)

    def ann_sites(s, e):
        s_anchor.extend([s, e])
        s_amount.extend([np.full(len(s), ann // 2, np.int64), np.full(len(s), ann - ann // 2, np.int64)])

    for ph, (op, level, calls, apis) in enumerate(phases):
        os_, oe = T[("op_start", ph)], T[("op_end", ph)]
        blocks.append(Block(os_, oe, OPERATION, MAIN_TID, (op,), zeros))
        ann_sites(os_, oe)
        if second_tid_ops:
            blocks.append(Block(os_, oe, OPERATION, 1, (op,), zeros))
            ann_sites(os_, oe)
        call_name = f"{op}_{'backend' if level == BACKEND else 'sim'}"
        for c in range(calls):
            cs, ce = T[("call_start", ph, c)], T[("call_end", ph, c)]
            blocks.append(Block(cs, ce, level, MAIN_TID, (call_name,), zeros))
            s_anchor.append(cs)
            s_amount.append(np.full(it, EXACT["transition"], np.int64))
    if outer_op:
        os_, oe = T[("op_start", 0)], T[("op_end", len(phases) - 1)]
        blocks.append(Block(os_, oe, OPERATION, MAIN_TID, (outer_op,), zeros))
        ann_sites(os_, oe)
    api_s = [T[m] for m in marks if m[0] == "api_start"]
    api_e = [T[("api_end",) + m[1:]] for m in marks if m[0] == "api_start"]
    cursor = 0
    if api_s:
        A_s = np.stack(api_s, axis=1).reshape(-1)  # program order within each iteration
        A_e = np.stack(api_e, axis=1).reshape(-1)
        na = A_s.shape[0]
        sel = rng.integers(0, 2, size=na)
        has_k = rng.random(na) < KERNEL_PROB
        nk = int(has_k.sum())
        corr = np.zeros(na, np.int64)
        corr[has_k] = np.arange(1, nk + 1)
        # in-order stream: E_i = max(a_i, E_{i-1}) + d_i  (running max of a_j - S_{j-1})
        a = A_s[has_k] + LAUNCH_DELAY
        kd = _u(rng, "kernel", nk)
        S = np.cumsum(kd)
        E = S + np.maximum.accumulate(a - (S - kd))
        kstart = E - kd
        blocks.append(Block(A_s, A_e, ACCEL_API, MAIN_TID, API_NAMES, sel, corr, has_k.astype(np.uint8)))
        s_anchor.extend([A_s, A_s])
        s_amount.extend([np.full(na, EXACT["api_interception"], np.int64),
                         np.where(sel == 0, EXACT["launch"], EXACT["memcpy"]).astype(np.int64)])
        blocks.append(Block(kstart, E, GPU, GPU_TID, ("kernel",), np.zeros(nk, np.int64), corr[has_k],
                            np.ones(nk, np.uint8)))
        cursor = int(E[-1]) if nk else 0
    if it:
        end = max(int(csum[-1, -1]), cursor) + int(_u(rng, "glue", 1)[0])
        blocks.append(Block(np.array([0], np.int64), np.array([end], np.int64), HIGH_LEVEL, MAIN_TID, ("script",),
                            np.zeros(1, np.int64)))
    return PidTimeline(blocks, np.concatenate(s_anchor) if s_anchor else np.zeros(0, np.int64),
                       np.concatenate(s_amount) if s_amount else np.zeros(0, np.int64))


def instrument(tl: PidTimeline, start: np.ndarray, dur: np.ndarray, cat: np.ndarray) -> tuple:
    """InsertionMap (_timeline.py:70-81): x -> x + slabs anchored strictly before x."""
    order = np.argsort(tl.site_anchor, kind="stable")
    anchors = tl.site_anchor[order]
    pref = np.concatenate([[0], np.cumsum(tl.site_amount[order])])

    def imap(x):
        return x + pref[np.searchsorted(anchors, x, side="left")]

    s2 = imap(start)
    e2 = imap(start + dur)
    return s2, np.where(cat == GPU, dur, e2 - s2)


def _pid_columns(tl: PidTimeline, name_rank: dict) -> tuple:
    """Concatenate one pid's blocks: (start, dur, cat, tid value, global name rank, corr, has_corr)."""
    bl = tl.blocks
    start = np.concatenate([b.start for b in bl])
    end = np.concatenate([b.end for b in bl])
    cat = np.concatenate([np.full(b.start.shape[0], b.cat, np.uint8) for b in bl])
    tid = np.concatenate([np.full(b.start.shape[0], b.tid, np.int64) for b in bl])
    name = np.concatenate([np.asarray([name_rank[x] for x in b.names], np.int32)[b.name_sel] for b in bl])
    corr = np.concatenate([b.corr if b.corr is not None else np.zeros(b.start.shape[0], np.int64) for b in bl])
    hasc = np.concatenate([b.has_corr if b.has_corr is not None else np.zeros(b.start.shape[0], np.uint8)
                           for b in bl])
    return start, end - start, cat, tid, name, corr, hasc


def ddpg_names(outer_op: str = None, phases=DDPG_PHASES) -> list:
    names = {"kernel", "script", *API_NAMES}
    for op, level, _, _ in phases:
        names.add(op)
        names.add(f"{op}_{'backend' if level == BACKEND else 'sim'}")
    if outer_op:
        names.add(outer_op)
    return sorted(names)


def assemble(parts: list, names: list, metas: list, clock_domain: int = 1) -> ColumnarTrace:
    """Per-pid column tuples (pid value, start, dur, cat, tid value, name rank,
    corr, has_corr), pids ascending, rows already in the wanted order ->
    ColumnarTrace, interning (pid, tid) groups per pid (no global sort)."""
    pids = np.array(sorted({p[0] for p in parts} | {m.pid for m in metas}), np.int64)
    pidx = {int(v): i for i, v in enumerate(pids.tolist())}
    g_pid, g_tid, tid_cols, pid_cols = [], [], [], []
    for p in sorted(parts, key=lambda x: x[0]):
        tids = p[4]
        uniq, inv = np.unique(tids, return_inverse=True)
        base = len(g_pid)
        g_pid.extend([pidx[p[0]]] * len(uniq))
        g_tid.extend(uniq.tolist())
        tid_cols.append((inv.reshape(-1) + base).astype(np.int32))
        pid_cols.append(np.full(tids.shape[0], pidx[p[0]], np.int32))
    parts = sorted(parts, key=lambda x: x[0])

    def cat_(k, dt):
        return np.ascontiguousarray(np.concatenate([q[k] for q in parts]) if parts else np.zeros(0, dt), dtype=dt)

    return ColumnarTrace(clock_domain, cat_(1, np.int64), cat_(2, np.int64),
                         np.concatenate(pid_cols) if parts else np.zeros(0, np.int32),
                         np.concatenate(tid_cols) if parts else np.zeros(0, np.int32),
                         cat_(3, np.uint8), cat_(5, np.int32), cat_(6, np.int64), cat_(7, np.uint8), pids,
                         np.array(g_pid, np.int32), np.array(g_tid, np.int64), list(names), tuple(metas))


def _ddpg_pid(args):
    seed, pid, iterations, outer_op, second_tid_ops, processes, want = args
    names = ddpg_names(outer_op)
    rank = {n: i for i, n in enumerate(names)}
    tl = build_pid(np.random.default_rng([seed, pid]), iterations, outer_op=outer_op, second_tid_ops=second_tid_ops)
    start, dur, cat, tid, name, corr, hasc = _pid_columns(tl, rank)
    order = np.lexsort((dur, start))  # one row order for both twins
    out = {}
    for inst in want:
        s, d = instrument(tl, start, dur, cat) if inst else (start, dur)
        lo, hi = (int(s.min()), int((s + d).max())) if s.size else (0, 0)
        if pid == 1 or processes == 1:
            meta = ProcessMeta(pid, "ddpg_root" if processes > 1 else "ddpg")
        else:
            meta = ProcessMeta(pid, f"ddpg_worker_{pid - 2}", parent=1, fork_ns=lo, join_ns=hi)
        out[inst] = ((pid, s[order], d[order], cat[order], tid[order], name[order], corr[order], hasc[order]), meta)
    return out


def _map(fn, jobs, workers: int):
    if workers and workers > 1 and len(jobs) > 1:
        import multiprocessing as mp
        import sys
        # fork is cheapest, but forking a process that already holds a CUDA
        # context (and its helper threads) can abort the child: spawn then
        torch = sys.modules.get("torch")
        cuda_up = torch is not None and torch.cuda.is_initialized()
        with mp.get_context("spawn" if cuda_up else "fork").Pool(min(workers, len(jobs))) as pool:
            return pool.map(fn, jobs, chunksize=1)
    return [fn(j) for j in jobs]


def ddpg_trace(iterations: int, processes: int = 1, seed: int = 1234, outer_op: str = None,
               second_tid_ops: bool = False, both: bool = False, workers: int = 0, first_pid: int = 1):
    """DDPG-style trace (configs 1-2: iterations=27027 -> ~1M events).

    Returns the instrumented ColumnarTrace, or (uninstrumented, instrumented)
    when ``both``.  Rows are ordered by (pid, start, dur) like read_trace.
    ``workers`` > 1 builds the pids in a process pool (configs 3-4).
    """
    want = (False, True) if both else (True,)
    pids = range(first_pid, first_pid + processes)
    jobs = [(seed, pid, iterations, outer_op, second_tid_ops, processes, want) for pid in pids]
    res = _map(_ddpg_pid, jobs, workers)
    names = ddpg_names(outer_op)
    out = [assemble([r[inst][0] for r in res], names, [r[inst][1] for r in res]) for inst in want]
    return (out[0], out[1]) if both else out[0]


# ---------------------------------------------------------------------------
# Config 3: multi-process, multi-phase, nested

CONFIG3_ITERS_PER_1M = 24510  # ~1.0M events per pid with outer_op + second_tid_ops


def config3_trace(processes: int = 100, events_per_pid: int = 1_000_000, seed: int = 1234, both: bool = False,
                  workers: int = 0, first_pid: int = 1):
    """Config 3: ``processes`` pids x ~``events_per_pid`` events, an outer
    per-iteration op around the three phase ops (depth 2), every phase op
    mirrored on a second tid (cross-tid path merge), all six categories."""
    iters = max(1, round(events_per_pid * CONFIG3_ITERS_PER_1M / 1_000_000))
    return ddpg_trace(iters, processes=processes, seed=seed, outer_op="iteration", second_tid_ops=True, both=both,
                      workers=workers, first_pid=first_pid)


# ---------------------------------------------------------------------------
# Config 5: adversarial

ADV_API_NAMES = ("launch", "memcpy", "sync")


def adversarial_profile() -> CalibrationProfile:
    """Fractional calibration for config 5 (exercises quantize_amounts' drift)."""
    return CalibrationProfile(Fraction(12345, 7), Fraction(1000, 3), Fraction(3001, 2),
                              {"launch": Fraction(5999, 2), "memcpy": Fraction(1000), "sync": Fraction(7, 3)})


def _adv_pid(args):
    """One adversarial process: recursive ops to ``depth`` on tid 0, shallow
    ops on tids 1-3, heavily overlapping CPU events, ``streams`` GPU streams of
    long concurrent kernels, 1% zero-duration events, 10% duplicate
    correlation ids, timestamps on a coarse grid (many equal endpoints)."""
    seed, pid, n, depth, streams = args
    rng = np.random.default_rng([seed, pid, 5])
    gran = 64
    T = max(n, 16) * 2000
    n_deep = max(1, int(0.03 * n))
    n_sh = max(3, int(0.03 * n)) // 3 * 3
    n_gpu = max(1, int(0.22 * n))
    n_dup = n_gpu // 10
    n_api = n_gpu + n_dup + n_gpu // 10
    n_cpu = max(0, n - n_deep - n_sh - n_gpu - n_api - 1)
    S, D, C, TID, NM, CO, HC = [], [], [], [], [], [], []
    names = adversarial_names(depth)
    rank = {x: i for i, x in enumerate(names)}

    def add(s, d, cat, tid, name, corr=None, hasc=None):
        k = s.shape[0]
        S.append(s.astype(np.int64))
        D.append(d.astype(np.int64))
        C.append(np.full(k, cat, np.uint8))
        TID.append(np.broadcast_to(np.asarray(tid, np.int64), (k,)).copy())
        NM.append(np.broadcast_to(np.asarray(name, np.int32), (k,)).copy())
        CO.append(np.zeros(k, np.int64) if corr is None else corr.astype(np.int64))
        HC.append(np.zeros(k, np.uint8) if hasc is None else hasc.astype(np.uint8))

    # deep recursive ops on tid 0: a reflecting random walk over the depth
    t = np.sort(rng.integers(0, T, 2 * n_deep)) // gran * gran
    coin = rng.random(2 * n_deep).tolist()
    pick = rng.integers(0, 3, 2 * n_deep).tolist()
    stack, ops_s, ops_e, ops_n = [], [], [], []
    pushes = n_deep
    tl = t.tolist()
    for i in range(2 * n_deep):
        d = len(stack)
        push = pushes > 0 and (d == 0 or (d < depth and coin[i] < 0.5))
        if push:
            parent = stack[-1][1] if stack else -1
            nm = parent if (parent >= 0 and pick[i] == 0 and coin[i] < 0.1) else rank[f"L{d % 6}_{pick[i]}"]
            stack.append((tl[i], nm))
            pushes -= 1
        else:
            s0, nm = stack.pop()
            ops_s.append(s0)
            ops_e.append(tl[i])
            ops_n.append(nm)
    ops_s, ops_e = np.array(ops_s, np.int64), np.array(ops_e, np.int64)
    add(ops_s, ops_e - ops_s, OPERATION, 0, np.array(ops_n, np.int32))
    # shallow ops on tids 1..3 (depth <= 2; some names shared with tid 0)
    for tid in (1, 2, 3):
        m = n_sh // 3
        tt = np.sort(rng.integers(0, T, 2 * m)) // gran * gran
        a, b = tt[0::2], tt[1::2]
        nm = np.where(rng.random(m) < 0.3, rank["L0_0"], rank[f"sh{tid}"]).astype(np.int32)
        add(a, b - a, OPERATION, tid, nm)
        kid = rng.random(m) < 0.5
        ca = (a + (b - a) // 4)[kid] // gran * gran
        cb = np.maximum(ca, (b - (b - a) // 4)[kid] // gran * gran)
        add(ca, cb - ca, OPERATION, tid, rank["inner"])
    # ambient HIGH_LEVEL
    add(np.array([0]), np.array([T + 4 * gran]), HIGH_LEVEL, 0, rank["script"])
    # CPU events, heavy-tailed durations, all four CPU tids
    cs = rng.integers(0, T, n_cpu) // gran * gran
    cd = np.minimum((rng.pareto(1.5, n_cpu) + 1) * 2000, T / 10).astype(np.int64) // gran * gran
    ccat = np.where(rng.random(n_cpu) < 0.5, BACKEND, SIMULATOR)
    ctid = rng.integers(0, 4, n_cpu)
    for cat in (BACKEND, SIMULATOR):
        sel = ccat == cat
        add(cs[sel], cd[sel], cat, ctid[sel], rank["backend_call" if cat == BACKEND else "sim_step"])
    # ACCEL_API: ids 1..n_gpu, n_dup duplicate ids, some without correlation
    as_ = rng.integers(0, T, n_api) // gran * gran
    ad = rng.integers(1, 200, n_api) * gran
    acorr = np.zeros(n_api, np.int64)
    ahas = np.zeros(n_api, np.uint8)
    acorr[:n_gpu] = np.arange(1, n_gpu + 1)
    acorr[n_gpu:n_gpu + n_dup] = rng.integers(1, n_gpu + 1, n_dup)
    ahas[:n_gpu + n_dup] = 1
    aname = np.array([rank[x] for x in ADV_API_NAMES], np.int32)[rng.integers(0, 3, n_api)]
    add(as_, ad, ACCEL_API, rng.integers(0, 4, n_api), aname, acorr, ahas)
    # GPU: long concurrent kernels on `streams` streams
    Dk = int(min(T // 2, 10_000 * T // max(n_gpu, 1)))
    gs = rng.integers(0, T, n_gpu) // gran * gran
    gd = (rng.random(n_gpu) * Dk + Dk // 2).astype(np.int64) // gran * gran
    add(gs, gd, GPU, 1000 + rng.integers(0, streams, n_gpu), rank["kernel"], np.arange(1, n_gpu + 1),
        np.ones(n_gpu, np.uint8))
    start, dur, cat = np.concatenate(S), np.concatenate(D), np.concatenate(C)
    tid, name, corr, hasc = np.concatenate(TID), np.concatenate(NM), np.concatenate(CO), np.concatenate(HC)
    # 1% zero-duration resource events
    res = np.nonzero(cat != OPERATION)[0]
    zero = res[rng.random(res.shape[0]) < 0.01]
    dur[zero] = 0
    order = np.lexsort((dur, start))
    lo, hi = int(start.min()), int((start + dur).max())
    meta = ProcessMeta(pid, f"adv_{pid}", parent=None if pid == 1 else 1, fork_ns=None if pid == 1 else lo,
                       join_ns=None if pid == 1 else hi)
    return (pid, start[order], dur[order], cat[order], tid[order], name[order], corr[order], hasc[order]), meta


def adversarial_names(depth: int = 64) -> list:
    names = {"script", "backend_call", "sim_step", "kernel", "inner", *ADV_API_NAMES}
    names.update(f"L{d}_{k}" for d in range(6) for k in range(3))
    names.update(f"sh{t}" for t in (1, 2, 3))
    return sorted(names)


def zipf_sizes(total: int, pids: int, s: float) -> list:
    w = np.arange(1, pids + 1, dtype=np.float64) ** -s
    sizes = np.floor(w / w.sum() * total).astype(np.int64)
    sizes[0] += total - int(sizes.sum())
    return [max(32, int(x)) for x in sizes]


def adversarial_trace(n_events: int = 10_000_000, pids: int = 64, seed: int = 1234, zipf: float = 1.5,
                      depth: int = 64, streams: int = 256, workers: int = 0, only=None) -> ColumnarTrace:
    """Config 5: ``n_events`` over ``pids`` processes with Zipf(``zipf``)
    sizes (s=1.5 puts ~42% of the events in the largest pid at 64 pids),
    recursive ops to ``depth``, ``streams`` concurrent GPU streams, 1%
    zero-duration events, 10% duplicate correlation ids.  ``only``: pid
    values (1-based) to generate -- exactly those processes of the full trace."""
    sizes = zipf_sizes(n_events, pids, zipf)
    keep = range(pids) if only is None else [p - 1 for p in only]
    res = _map(_adv_pid, [(seed, p + 1, sizes[p], depth, streams) for p in keep], workers)
    return assemble([r[0] for r in res], adversarial_names(depth), [r[1] for r in res])


# ---------------------------------------------------------------------------
# Device generator (csrc/xs_synth.cu, test/bench infrastructure)

_SYN_NAMES = ("kernel", "script", "launch", "memcpy", "inference", "inference_backend", "simulation",
              "simulation_sim", "backprop", "backprop_backend")


@dataclass
class DeviceSynth:
    """Both twins of a generated trace resident on the device: ``cols[twin]``
    (twin "un" / "inst") maps column names to device tensors; ``meta`` holds
    the tables (pids, (pid, tid) groups, names, processes) of each twin."""

    meta: dict
    cols: dict
    n: int

    def columnar(self, twin: str = "inst") -> ColumnarTrace:
        """The twin as an ordinary host ColumnarTrace (copies the columns)."""
        c = self.cols[twin]
        m = self.meta[twin]
        return ColumnarTrace(1, c["start"].cpu().numpy(), c["dur"].cpu().numpy(), c["pid"].cpu().numpy(),
                             c["tid"].cpu().numpy(), c["cat"].cpu().numpy(), c["name"].cpu().numpy(),
                             c["corr"].cpu().numpy(), c["has_corr"].cpu().numpy(), m["pids"], m["group_pid"],
                             m["group_tid"], m["names"], m["processes"], m["pid_has_meta"])

    def device_trace(self, twin: str = "inst", device: int = 0):
        """A DeviceTrace over the resident columns (no host copy): the host
        trace object only carries the tables and the row count."""
        from . import _engine
        m = self.meta[twin]
        z64 = np.broadcast_to(np.int64(0), (self.n,))
        z32 = np.broadcast_to(np.int32(0), (self.n,))
        z8 = np.broadcast_to(np.uint8(0), (self.n,))
        ct = ColumnarTrace(1, z64, z64, z32, z32, z8, z32, z64, z8, m["pids"], m["group_pid"], m["group_tid"],
                           m["names"], m["processes"], m["pid_has_meta"])
        return _engine.DeviceTrace.from_tensors(ct, dict(self.cols[twin], group_pid=m["group_pid_dev"],
                                                         pid_has_meta=m["pid_has_meta_dev"]), device)


def device_ddpg_trace(iterations: int, processes: int = 1, seed: int = 1234, outer_op: str = None,
                      second_tid_ops: bool = False, first_pid: int = 1, device: int = 0) -> DeviceSynth:
    """The DDPG-style workload (ddpg_trace / config3_trace shape: the same
    phases, durations, kernel probability, in-order stream, outer op and tid-1
    mirrors) generated on the device in both twins (xs_synth_plan /
    xs_synth_generate); instrumented with the exact profile's amounts, so
    correct_trace(inst, exact_profile()) == un bit for bit."""
    import ctypes as C

    import torch

    from . import _engine, _lib

    eng = _engine.get(device)
    dev = torch.device("cuda", device)
    names = ddpg_names(outer_op)
    rank = {x: i for i, x in enumerate(names)}
    sym = [rank[x] for x in _SYN_NAMES] + [rank[outer_op] if outer_op else 0]
    names_dev = torch.tensor(sym, dtype=torch.int32, device=dev)
    ann = EXACT["annotation"]
    spec = _lib.XsSynthSpec(iterations, seed, processes, 1 if outer_op else 0,
                            1 if second_tid_ops else 0, first_pid, ann // 2, ann - ann // 2, EXACT["transition"],
                            EXACT["api_interception"], EXACT["launch"], EXACT["memcpy"], names_dev.data_ptr())
    n = C.c_int64(0)
    eng.check(eng.lib.xs_synth_plan(eng.ctx, C.byref(spec), C.byref(n), eng.stream()), "xs_synth_plan")
    n = int(n.value)
    t = {k: torch.empty(n, dtype=dt, device=dev) for k, dt in
         (("su", torch.int64), ("du", torch.int64), ("si", torch.int64), ("di", torch.int64), ("pid", torch.int32),
          ("tid", torch.int32), ("cat", torch.uint8), ("name", torch.int32), ("corr", torch.int64),
          ("has_corr", torch.uint8))}
    span = torch.empty(2 * processes, dtype=torch.int64, device=dev)
    eng.check(eng.lib.xs_synth_generate(eng.ctx, C.byref(spec), *(t[k].data_ptr() for k in (
        "su", "du", "si", "di", "pid", "tid", "cat", "name", "corr", "has_corr")), span.data_ptr(), eng.stream()),
        "xs_synth_generate")
    ends = span.cpu().numpy().reshape(processes, 2)
    del names_dev
    pids = np.arange(first_pid, first_pid + processes, dtype=np.int64)
    tids = [0, 1, GPU_TID] if second_tid_ops else [0, GPU_TID]
    group_pid = np.repeat(np.arange(processes, dtype=np.int32), len(tids))
    group_tid = np.tile(np.array(tids, np.int64), processes)
    shared = {"pids": pids, "group_pid": group_pid, "group_tid": group_tid, "names": names,
              "pid_has_meta": np.ones(processes, np.uint8),
              "group_pid_dev": torch.from_numpy(group_pid).to(dev),
              "pid_has_meta_dev": torch.ones(processes, dtype=torch.uint8, device=dev)}
    meta = {}
    for twin, col in (("un", 0), ("inst", 1)):
        procs = []
        for k, pv in enumerate(pids.tolist()):
            if pv == 1 or processes == 1:
                procs.append(ProcessMeta(pv, "ddpg_root" if processes > 1 else "ddpg"))
            else:
                procs.append(ProcessMeta(pv, f"ddpg_worker_{pv - 2}", parent=1, fork_ns=0,
                                         join_ns=int(ends[k, col])))
        meta[twin] = dict(shared, processes=tuple(procs))
    common = {k: t[k] for k in ("pid", "tid", "cat", "name", "corr", "has_corr")}
    cols = {"un": dict(common, start=t["su"], dur=t["du"]), "inst": dict(common, start=t["si"], dur=t["di"])}
    return DeviceSynth(meta, cols, n)
