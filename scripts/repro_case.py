"""Run one golden correction case through analyze (debug helper)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from golden_util import dec_profile, dec_trace, load  # noqa: E402

from paper_2102_04285_b200.columnar import ColumnarTrace  # noqa: E402
from paper_2102_04285_b200.correction import analyze_columnar  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "random_0"
case = [c for c in load("correction_cases.json.gz") if c["name"] == name][0]
trace = dec_trace(case["trace"])
prof = dec_profile(case["profile"])
s, d, rep, bd = analyze_columnar(ColumnarTrace.from_trace(trace), prof)
print("ok", s.cpu().numpy().tolist() == case["expect"]["start"])
