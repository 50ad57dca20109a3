"""Time the device generator (xs_synth) on the config-4 scale: 1000
processes x 24510 iterations of the config-3 shape (~1B events, both twins
resident in HBM).  Prints events, seconds, and a closure check on one
sampled process (the instrumented twin corrects back to the uninstrumented
one through the device pipeline)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2102_04285_b200 import _engine, synth  # noqa: E402

pids = int(os.environ.get("XS_PIDS", "1000"))
torch.cuda.init()
synth.device_ddpg_trace(10, processes=2, outer_op="iteration", second_tid_ops=True)  # (warm: module load)
torch.cuda.synchronize()
t0 = time.perf_counter()
g = synth.device_ddpg_trace(synth.CONFIG3_ITERS_PER_1M, processes=pids, outer_op="iteration", second_tid_ops=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
# closure on one sampled process (a 1M-event slice: pid-contiguous rows)
pid = torch.tensor(0, device="cuda")
rows = torch.nonzero(g.cols["un"]["pid"] == 7).flatten()
a, b = int(rows[0]), int(rows[-1]) + 1
sub = synth.DeviceSynth(g.meta, {tw: {k: v[a:b] for k, v in c.items()} for tw, c in g.cols.items()}, b - a)
un = sub.columnar("un")
eng = _engine.get(0)
raw = eng.correct(sub.device_trace("inst"), synth.exact_profile().scaled(un.names), analyze_attribution=0)
ok = bool(np.array_equal(raw.start.cpu().numpy(), un.start) and np.array_equal(raw.dur.cpu().numpy(), un.dur))
print(json.dumps({"events": g.n, "processes": pids, "generate_s": round(dt, 3),
                  "events_per_s": round(g.n / dt, 1), "closure_exact_pid7": ok,
                  "hbm_gb_both_twins": round(g.n * 54 / 1e9, 1)}))
