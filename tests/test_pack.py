"""Packed upload format (include/xstrace_b200.h xs_packed_t): host packing
chooses the narrowest exact width per column and round-trips bit for bit
through the host restatement of xs_unpack (columnar.unpack_block); the CUDA
widening is checked against the same columns in tests/test_gpu_pack.py."""

import numpy as np
import pytest

from paper_2102_04285_b200 import synth
from paper_2102_04285_b200.columnar import ColumnarTrace, pack_block, unpack_block

COLS = ("start", "dur", "pid", "tid", "cat", "name", "corr", "has_corr")


def _variants():
    base = synth.adversarial_trace(20_000, pids=5)
    yield "adversarial", base, {}
    n = base.n
    rng = np.random.default_rng(3)
    yield "negative_dur", base, {"dur": np.where(rng.random(n) < 0.01, -5, base.dur)}
    yield "wide_start", base, {"start": base.start + np.where(np.arange(n) % 977 == 0, 1 << 40, 0)}
    yield "corr_64", base, {"corr": base.corr + (1 << 33)}
    yield "dur_64", base, {"dur": base.dur + (1 << 32)}
    yield "int64_extremes", base, {"start": np.where(np.arange(n) % 300 == 7, np.iinfo(np.int64).min,
                                                     base.start),
                                   "dur": np.where(np.arange(n) % 500 == 9, np.iinfo(np.int64).max, base.dur)}


def _replace(ct, cols):
    import dataclasses
    return dataclasses.replace(ct, **{k: np.ascontiguousarray(v, np.int64) for k, v in cols.items()}, _source=None)


def _roundtrip(ct):
    lay, raw = pack_block(ct)
    for a, b in ((0, ct.n), (0, min(ct.n, 1)), (257, min(ct.n, 5000)), (ct.n // 3, ct.n)):
        if a > b:
            continue
        u = unpack_block(raw, lay, a, b)
        for k in COLS:
            assert u[k].dtype == getattr(ct, k).dtype or k in ("cat", "has_corr")
            assert np.array_equal(u[k], getattr(ct, k)[a:b]), k
    return lay


def test_pack_roundtrip_and_widths():
    widths = {}
    for name, base, cols in _variants():
        ct = _replace(base, cols) if cols else base
        widths[name] = _roundtrip(ct).widths
    assert widths["adversarial"]["start"] == 4 and widths["adversarial"]["dur"] == 4
    # a few misfits go to the exception table; a column of them takes 64 bits
    assert widths["negative_dur"]["dur"] == 4 and widths["wide_start"]["start"] == 4
    assert widths["dur_64"]["dur"] == 8 and widths["corr_64"]["corr"] == 8
    assert widths["int64_extremes"]["start"] == 8 and widths["int64_extremes"]["dur"] == 4
    for name, base, cols in _variants():
        ct = _replace(base, cols) if cols else base
        lay, _ = pack_block(ct)
        assert (lay.n_exc > 0) == (name in ("negative_dur", "wide_start", "int64_extremes")), name


def test_pack_index_widths_and_small_traces():
    names = [f"n{i:05d}" for i in range(70_000)]
    n = 1000
    rng = np.random.default_rng(0)
    ct = ColumnarTrace.from_arrays(0, np.sort(rng.integers(0, 10**9, n)), rng.integers(0, 100, n),
                                   rng.integers(0, 300, n), rng.integers(0, 5, n), np.full(n, 1, np.uint8),
                                   rng.integers(0, len(names), n), names)
    lay = _roundtrip(ct)
    assert lay.widths["pid"] == 2 and lay.widths["name"] == 4 and lay.widths["tid"] == 2
    for m in (0, 1, 255, 256, 257):
        sub = ColumnarTrace.from_arrays(0, np.arange(m) * 7, np.ones(m), np.ones(m), np.ones(m),
                                        np.zeros(m, np.uint8), np.zeros(m), ["a"])
        lay, raw = pack_block(sub)
        u = unpack_block(raw, lay)
        assert all(np.array_equal(u[k], getattr(sub, k)) for k in COLS)


def test_pack_refuses_unrepresentable_category():
    ct = synth.ddpg_trace(20)
    import dataclasses
    bad = dataclasses.replace(ct, cat=np.where(np.arange(ct.n) == 3, 200, ct.cat).astype(np.uint8), _source=None)
    assert pack_block(bad) is None


def test_exception_table_sorted_and_adjacent():
    """The pipelined path uploads the exception table as one byte range:
    rows, values, columns are adjacent in the block and sorted by row."""
    import dataclasses

    ct = synth.adversarial_trace(20_000, pids=5)
    n = ct.n
    bad = dataclasses.replace(ct, dur=np.where(np.arange(n) % 101 == 5, -1, ct.dur).astype(np.int64),
                              corr=np.where(np.arange(n) % 131 == 3, 1 << 40, ct.corr).astype(np.int64),
                              _source=None)
    lay, raw = pack_block(bad)
    assert lay.n_exc > 0
    o = lay.offsets
    assert o["exc_val"] == o["exc_row"] + (lay.nbytes["exc_row"] + 15) // 16 * 16
    assert o["exc_col"] == o["exc_val"] + (lay.nbytes["exc_val"] + 15) // 16 * 16
    rows = raw[o["exc_row"]:o["exc_row"] + lay.nbytes["exc_row"]].view(np.int64)
    assert np.all(np.diff(rows) >= 0)


def _native_equal(ct, threads):
    from paper_2102_04285_b200.columnar import pack_native
    ref = pack_block(ct)
    got = pack_native(ct, n_threads=threads)
    if ref is None:
        assert got is None
        return
    (l1, r1), (l2, r2) = ref, got
    assert l1.offsets == l2.offsets and l1.nbytes == l2.nbytes and l1.widths == l2.widths
    assert l1.total == l2.total and l1.n_exc == l2.n_exc
    assert np.array_equal(r1, r2)


def test_native_pack_matches_numpy_builder():
    """xs_pack_plan / xs_pack_fill (host threads) write the same bytes as the
    numpy builder, for every thread count (the row partition and the
    per-thread exception slots must not change the block)."""
    import os

    from paper_2102_04285_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        import pytest
        pytest.skip("library not built")
    for name, base, cols in _variants():
        ct = _replace(base, cols) if cols else base
        for threads in (1, 3, 8):
            _native_equal(ct, threads)
    for m in (0, 1, 255, 256, 257, 70_000):
        sub = ColumnarTrace.from_arrays(0, np.arange(m) * 7, np.ones(m), np.ones(m), np.ones(m),
                                        np.zeros(m, np.uint8), np.zeros(m), ["a"])
        _native_equal(sub, 4)
    import dataclasses
    ct = synth.ddpg_trace(20)
    _native_equal(dataclasses.replace(ct, cat=np.where(np.arange(ct.n) == 3, 200, ct.cat).astype(np.uint8),
                                      _source=None), 2)


@pytest.mark.timeout(300)
def test_native_pack_concurrent_callers():
    """Several host threads packing at once (analyze_columnar_pipelined packs
    each worker's next batch concurrently): the shared worker pool takes one
    pass at a time -- no hang, no corrupted blocks."""
    import threading

    from paper_2102_04285_b200.columnar import pack_native
    from paper_2102_04285_b200.correction import _pid_batches, _row_slice

    ct = synth.config3_trace(processes=9, events_per_pid=150_000, workers=4)
    parts = _pid_batches(ct, 9)
    want = {}
    for k, (a, b) in enumerate(parts):
        lay, blk = pack_block(_row_slice(ct, a, b))
        want[k] = bytes(np.frombuffer(blk, np.uint8)[: lay.total]) if not isinstance(blk, np.ndarray) else \
            bytes(blk[: lay.total])
    bad = []

    def work(w):
        for _ in range(4):
            for k, (a, b) in enumerate(parts):
                if k % 3 == w:
                    lay, blk = pack_native(_row_slice(ct, a, b), None, n_threads=3)
                    if bytes(blk[: lay.total]) != want[k]:
                        bad.append(k)

    ths = [threading.Thread(target=work, args=(w,)) for w in range(3)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not bad
