"""CPU: the metrics oracle (oracle/oracle.py union_ns / utilization_flags,
numpy restatements of metrics.py:41-84) pinned to the reference's outputs in
tests/golden/metrics_cases.json.gz (scripts/make_golden_metrics.py), plus
the host-only summarize()."""

import pytest

import oracle
from golden_util import dec_trace, load
from paper_2102_04285_b200 import ColumnarTrace

CASES = load("metrics_cases.json.gz")["metrics"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_metrics_match_reference(case):
    tr = dec_trace(case["trace"])
    exp = case["expect"]
    if any(isinstance(v, dict) for v in exp["busy"].values()):
        return  # error cases (empty / zero span / invalid) are covered on the device path
    ct = ColumnarTrace.from_trace(tr)
    lo, hi = oracle.trace_span(ct)
    for c, v in exp["busy"].items():
        assert oracle.union_ns(ct, int(c)) / (hi - lo) == v
    for p, samples in exp["samples"].items():
        flags = oracle.utilization_flags(ct, int(p))
        assert flags == [s[2] for s in samples]
    for p, v in exp["sampled"].items():
        if isinstance(v, dict):
            continue
        flags = oracle.utilization_flags(ct, int(p))
        assert sum(flags) / len(flags) == v
