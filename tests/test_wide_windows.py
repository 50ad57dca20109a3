"""Host logic of the wide-process time windows (_split.wide_cuts /
window_trace, used by compute_overlap for a process whose span needs more
than 59 bits): the windowed overlap -- each window through the C oracle, the
window breakdowns merged like overlap._merge_windows -- equals the oracle on
the whole process, for the 2^62-wide reference golden case and for random
traces cut into many windows (WIDE_BITS lowered)."""

import numpy as np
import pytest

import oracle
from golden_util import dec_trace, load
from paper_2102_04285_b200 import _split, synth
from paper_2102_04285_b200.columnar import ColumnarTrace


def _windowed(ct, attr, bits=None, monkeypatch=None):
    if bits is not None:
        monkeypatch.setattr(_split, "WIDE_BITS", bits)
    rows_by_pid = _split.pid_rows(ct)
    cells, spans, tracked = {}, {}, {}
    for p in range(ct.n_pids):
        if rows_by_pid[p].size == 0:
            continue
        sub, _ = _split.sub_trace(ct, [p], rows_by_pid)
        cuts = _split.wide_cuts(sub)
        bounds = [None] + cuts + [None]
        nwin = 0
        for a, b in zip(bounds[:-1], bounds[1:]):
            win = _split.window_trace(sub, a, b)
            if win.n == 0:
                continue
            nwin += 1
            if a is not None:  # clipped intervals stay inside the window
                assert (win.start >= a).all() or ((win.cat == 0) | (win.dur == 0))[win.start < a].all()
            c, s, u = oracle.overlap(win, attr)
            for k, v in c.items():
                cells[k] = cells.get(k, 0) + v
            for pid, (lo, hi) in s.items():
                tracked[pid] = tracked.get(pid, 0) + (hi - lo) - u[pid]
                spans[pid] = (min(spans[pid][0], lo), max(spans[pid][1], hi)) if pid in spans else (lo, hi)
    untracked = {pid: (hi - lo) - tracked[pid] for pid, (lo, hi) in spans.items()}
    return cells, spans, untracked


def test_wide_golden_case_windows_equal_whole():
    case = [c for c in load("edge_cases.json.gz") if c["name"] == "single_pid_span_2e62"][0]
    ct = ColumnarTrace.from_trace(dec_trace(case["trace"]))
    assert _split.wide_pids(ct) == [0]
    sub, _ = _split.sub_trace(ct, [0], _split.pid_rows(ct))
    cuts = _split.wide_cuts(sub)
    assert len(cuts) >= 16  # 2^62 + 2^60 in windows of < 2^59 ns
    bounds = [int(sub.start.min())] + cuts + [int((sub.start + sub.dur).max())]
    assert max(b - a for a, b in zip(bounds[:-1], bounds[1:])) < 1 << _split.WIDE_BITS
    for attr in (0, 1):
        assert _windowed(ct, attr) == oracle.overlap(ct, attr)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("attr", [0, 1])
def test_many_windows_equal_whole(seed, attr, monkeypatch):
    ct = synth.ddpg_trace(200, processes=2, seed=seed)
    whole = oracle.overlap(ct, attr)
    # windows a few operations long: dozens of cuts per process
    bits = int(ct.dur[ct.cat == 0].max()).bit_length() + 2
    got = _windowed(ct, attr, bits=bits, monkeypatch=monkeypatch)
    assert got == whole


def test_forbidden_ranges_keep_ops_and_launchers_whole(monkeypatch):
    ct = synth.ddpg_trace(200, processes=1, seed=3)
    monkeypatch.setattr(_split, "WIDE_BITS", int(ct.dur[ct.cat == 0].max()).bit_length() + 2)
    cuts = _split.wide_cuts(ct)
    assert cuts
    op = ct.cat == 0
    s, e = ct.start[op], ct.start[op] + ct.dur[op]
    for c in cuts:
        assert not ((s < c) & (c < e)).any()
    api = (ct.cat == 4) & (ct.has_corr == 1)
    gpu = (ct.cat == 5) & (ct.has_corr == 1)
    first = {}
    for c_, st in sorted(zip(ct.corr[api].tolist(), ct.start[api].tolist())):
        first.setdefault(c_, st)
    for c_, st in zip(ct.corr[gpu].tolist(), ct.start[gpu].tolist()):
        a, b = min(first[c_], st), max(first[c_], st)
        for c in cuts:
            assert not (a < c <= b)


def test_too_wide_operation_is_an_error(monkeypatch):
    monkeypatch.setattr(_split, "WIDE_BITS", 12)
    ct = synth.ddpg_trace(30, processes=1, seed=1, outer_op="outer")  # one op around everything
    with pytest.raises(ValueError):
        _split.wide_cuts(ct)
