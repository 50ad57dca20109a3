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


def ddpg_trace(iterations: int, processes: int = 1, seed: int = 1234, outer_op: str = None,
               second_tid_ops: bool = False, both: bool = False):
    """DDPG-style trace (configs 1-2: iterations=27027 -> ~1M events).

    Returns the instrumented ColumnarTrace, or (uninstrumented, instrumented)
    when ``both``.  Rows are ordered by (pid, start, dur) like read_trace.
    """
    per = {False: [], True: []}
    metas = {False: [], True: []}
    names_all = set()
    for pid in range(1, processes + 1):
        tl = build_pid(np.random.default_rng([seed, pid]), iterations, outer_op=outer_op,
                       second_tid_ops=second_tid_ops)
        start = np.concatenate([b.start for b in tl.blocks])
        end = np.concatenate([b.end for b in tl.blocks])
        dur = end - start
        cat = np.concatenate([np.full(b.start.shape[0], b.cat, np.uint8) for b in tl.blocks])
        tid = np.concatenate([np.full(b.start.shape[0], b.tid, np.int64) for b in tl.blocks])
        name_s = np.concatenate([np.asarray(b.names, dtype=object)[b.name_sel] for b in tl.blocks])
        corr = np.concatenate([b.corr if b.corr is not None else np.zeros(b.start.shape[0], np.int64)
                               for b in tl.blocks])
        hasc = np.concatenate([b.has_corr if b.has_corr is not None else np.zeros(b.start.shape[0], np.uint8)
                               for b in tl.blocks])
        for b in tl.blocks:
            names_all.update(b.names)
        order = np.lexsort((dur, start))  # one row order for both twins
        for inst in (False, True):
            s, d = instrument(tl, start, dur, cat) if inst else (start, dur)
            per[inst].append((pid, s[order], d[order], cat[order], tid[order], name_s[order], corr[order],
                              hasc[order]))
            lo, hi = (int(s.min()), int((s + d).max())) if s.size else (0, 0)
            if pid == 1 or processes == 1:
                metas[inst].append(ProcessMeta(pid, "ddpg_root" if processes > 1 else "ddpg"))
            else:
                metas[inst].append(ProcessMeta(pid, f"ddpg_worker_{pid - 2}", parent=1, fork_ns=lo, join_ns=hi))
    names = sorted(names_all)
    rank = {n: i for i, n in enumerate(names)}
    out = []
    for inst in (False, True):
        parts = per[inst]
        cols = [np.concatenate([p[k] for p in parts]) for k in range(1, 8)]
        pidv = np.concatenate([np.full(p[1].shape[0], p[0], np.int64) for p in parts])
        uniq, inv = np.unique(cols[4], return_inverse=True)
        name = np.array([rank[x] for x in uniq.tolist()], np.int32)[inv.reshape(-1)]
        out.append(ColumnarTrace.from_arrays(1, cols[0], cols[1], pidv, cols[3], cols[2], name, names, cols[5],
                                             cols[6], tuple(metas[inst])))
    return (out[0], out[1]) if both else out[1]
