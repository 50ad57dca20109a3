"""xs_unpack on the B200: the packed pinned block (ColumnarTrace.pinned)
widened on the device equals the host columns bit for bit -- whole traces
and row slices starting off a 256-row base boundary, every width choice."""

import numpy as np
import pytest

from paper_2102_04285_b200 import _engine, synth
from paper_2102_04285_b200.columnar import ColumnarTrace

from test_pack import COLS, _replace, _variants

pytestmark = pytest.mark.gpu


def _traces():
    for name, base, cols in _variants():
        yield name, (_replace(base, cols) if cols else base)
    names = [f"n{i:05d}" for i in range(70_000)]
    rng = np.random.default_rng(1)
    n = 3000
    yield "wide_indices", ColumnarTrace.from_arrays(0, np.sort(rng.integers(0, 10**9, n)), rng.integers(0, 100, n),
                                                    rng.integers(0, 300, n), rng.integers(0, 5, n),
                                                    np.full(n, 1, np.uint8), rng.integers(0, len(names), n), names)


def test_device_unpack_equals_columns():
    import torch

    for name, ct in _traces():
        pin = ct.pinned()
        assert "_packed" in pin._pinned, name
        dt = _engine.DeviceTrace(pin, 0)
        torch.cuda.synchronize()
        for k in COLS:
            assert np.array_equal(getattr(dt, k).cpu().numpy()[: ct.n], getattr(ct, k)), (name, k)
        assert np.array_equal(dt.group_pid.cpu().numpy()[: ct.group_pid.size], ct.group_pid)


def test_device_unpack_row_slices():
    import torch
    from types import SimpleNamespace

    eng = _engine.get(0)
    ct = synth.adversarial_trace(30_000, pids=3)
    pin = ct.pinned()
    lay = pin._pinned["_packed"]
    dblock = pin._pinned["_block"].cuda()
    for a, b in ((0, ct.n), (1, 2), (255, 257), (300, 9000), (ct.n - 5, ct.n)):
        dst = SimpleNamespace(**{k: torch.empty(b - a, dtype=_engine.torch_dtype(getattr(ct, k).dtype),
                                                device="cuda") for k in COLS})
        _engine.unpack_into(eng, lay, _engine.packed_ptrs(lay, dblock, a), a, b, dst)
        torch.cuda.synchronize()
        for k in COLS:
            assert np.array_equal(getattr(dst, k).cpu().numpy(), getattr(ct, k)[a:b]), (a, b, k)


def test_packed_analyze_matches_wide_upload():
    from paper_2102_04285_b200 import analyze_columnar

    ct = synth.adversarial_trace(60_000, pids=6)
    prof = synth.adversarial_profile()
    s0, d0, r0, b0 = analyze_columnar(ct.pinned(packed=False), prof)
    s1, d1, r1, b1 = analyze_columnar(ct.pinned(), prof)
    assert np.array_equal(s0.cpu().numpy(), s1.cpu().numpy()) and np.array_equal(d0.cpu().numpy(), d1.cpu().numpy())
    assert r0.removed_ns == r1.removed_ns and b0 == b1


def test_pipelined_packed_with_exceptions_equals_one_call():
    """Pipelined multi-context analysis of a packed trace whose corr / start
    columns carry exception-table values (ids >= 2^32 on a subset of one
    pid's correlations; one far-away instant per pid) equals one call on the
    unpacked columns."""
    import dataclasses

    import torch

    from paper_2102_04285_b200 import analyze_columnar, analyze_columnar_pipelined

    ct = synth.config3_trace(processes=6, events_per_pid=20_000)
    sel = (ct.pid == 2) & (ct.has_corr == 1) & (ct.corr % 4 == 0)
    corr = np.where(sel, ct.corr + (1 << 33), ct.corr)
    ct2 = dataclasses.replace(ct, corr=np.ascontiguousarray(corr, np.int64), _source=None)
    pin = ct2.pinned()
    lay = pin._pinned["_packed"]
    assert lay.widths["corr"] == 4 and lay.n_exc == int(sel.sum()) > 0
    prof = synth.exact_profile()
    s0, d0, r0, b0 = analyze_columnar(ct2, prof)
    for workers in (1, 3):
        hs = torch.empty(ct2.n, dtype=torch.int64).pin_memory()
        hd = torch.empty(ct2.n, dtype=torch.int64).pin_memory()
        s1, d1, r1, b1 = analyze_columnar_pipelined(pin, prof, out=(hs, hd), batches=5, workers=workers)
        assert np.array_equal(hs.numpy(), s0.cpu().numpy()) and np.array_equal(hd.numpy(), d0.cpu().numpy())
        assert r1.removed_ns == r0.removed_ns and b1 == b0
