#!/usr/bin/env python3
"""tests/golden/ladder_profile_noisy1234_2000.txt: the fractional profile
SURVEY.md 8(d) names for config 2 --
build_profile(generate_calibration_ladder(preset_noisy(seed=1234, iterations=2000)))
-- produced by the REFERENCE (oracle/_ref, built by oracle/build_ref.sh) and
stored in its own text format (calibration.py:173-220).  The GPU box has no
/root/reference, so the full-scale parity tests read this file."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

from xstrace.calibration import build_profile  # noqa: E402
from xstrace.synth import generate_calibration_ladder, preset_noisy  # noqa: E402

prof = build_profile(generate_calibration_ladder(preset_noisy(seed=1234, iterations=2000)).values())
with open(os.path.join(ROOT, "tests", "golden", "ladder_profile_noisy1234_2000.txt"), "w") as fh:
    fh.write(prof.to_text())
print(prof.to_text())
