"""A medium analyze (correction + overlap) for compute-sanitizer: a 2-process
DDPG trace (~55k events: chunks with wide key ranges, so the local-bin sorts
take the s2 > 0 paths) and a 64-process adversarial trace (hashed cells, deep
paths), both checked against the C oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2102_04285_b200 import analyze_columnar, synth  # noqa: E402
from paper_2102_04285_b200.columnar import ColumnarTrace  # noqa: E402


def check(ct, prof):
    for _ in range(2):  # eager, then captured
        s, d, rep, bd = analyze_columnar(ct, prof)
    os_, od, orep, _ = oracle.correct(ct, prof)
    assert np.array_equal(s.cpu().numpy(), os_) and np.array_equal(d.cpu().numpy(), od)
    cor = ColumnarTrace(ct.clock_domain, os_, od, ct.pid, ct.tid, ct.cat, ct.name, ct.corr, ct.has_corr, ct.pids,
                        ct.group_pid, ct.group_tid, ct.names, ct.processes, ct.pid_has_meta)
    cells, spans, untracked = oracle.overlap(cor, 0)
    ours = {(k.pid, k.path, frozenset(int(c) for c in k.categories)): v for k, v in bd.cells.items()}
    assert ours == cells and bd.spans == spans and bd.untracked == untracked
    print("ok", ct.n, len(ours))


if __name__ == "__main__":  # (the generators may spawn worker processes)
    check(synth.ddpg_trace(1500, processes=2), synth.exact_profile())
    check(synth.adversarial_trace(100_000, pids=64, workers=1), synth.adversarial_profile())
