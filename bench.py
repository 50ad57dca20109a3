#!/usr/bin/env python3
"""Benchmark: trace events/sec analysed (overlap + correction) on B200.

Workload (BASELINE.json configs[1]): a synthetic DDPG-style instrumented trace
of ~1M events per GPU (3 operation scopes; Python/C/CUDA-API/GPU-kernel
categories) corrected with the calibrated integer profile {annotation 4000,
transition 1000, api_interception 1500, launch 3000, memcpy 1000}; one step is
the ``xstrace analyze --profile`` path: correct_trace + compute_overlap of the
corrected trace (cli.py:168-171), one ``xs_analyze`` device call.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 runs under torch.distributed.run, one process per GPU; each rank analyses
its own ~1M-event process (weak scaling) and the per-rank overlap histograms
are merged with an NCCL all-reduce keyed by a global path table.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ITERATIONS = 27027  # ~1M events per process
METRIC = "trace events/sec analysed (overlap+correction)"
UNIT = "events/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--iterations", type=int, default=ITERATIONS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5],
                    help="BASELINE.json config: 2 (default, the metric's workload), 3 (100M events, 100 pids, "
                         "nested), 4 (1B events, 1000 pids, strong-scaled over the ranks), 5 (adversarial 10M)")
    ap.add_argument("--events", type=int, default=0, help="events per GPU for --config 3/5 (default 100M / 10M)")
    ap.add_argument("--device-gen", action="store_true",
                    help="--config 4: generate the trace on the device (xs_synth: ~1B events in ~4 s) instead of "
                         "the host generator (~200 s); the reference arm always uses the host generator")
    ap.add_argument("--ref-budget", type=float, default=120.0,
                    help="--impl reference: stop the timed steps once this many seconds are spent")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


WORKLOADS = {
    2: "config2: DDPG-style instrumented trace, ~1M events/GPU, 3 operation scopes, integer calibrated profile; "
       "step = correct_trace + compute_overlap(corrected)",
    3: "config3: multi-process multi-phase DDPG-style instrumented trace, 1M events per pid, outer op around 3 "
       "phase ops (depth 2), ops on 2 tids, 6 categories, integer calibrated profile; step = correct_trace + "
       "compute_overlap(corrected)",
    4: "config4: 1000 processes x 1M events (config-3 shape: outer op around 3 phase ops, ops on 2 tids, 6 "
       "categories) = 1B events, integer calibrated profile, strong-scaled: contiguous pid blocks per rank, each "
       "rank's share resident in HBM in batches of <=100 processes (one xs_analyze per batch), NCCL sparse merge of "
       "every batch's Breakdown inside the step",
    5: "config5: adversarial trace, 64 Zipf(1.5)-sized pids, recursive ops to depth 64, 256 GPU streams of long "
       "concurrent kernels, 1% zero-duration, 10% duplicate correlation ids, fractional calibrated profile; "
       "step = correct_trace + compute_overlap(corrected)",
}


def make_workload(args, rank: int):
    """(instrumented trace, uninstrumented twin or None, profile) for this rank's shard."""
    from paper_2102_04285_b200 import synth
    workers = os.cpu_count() or 1
    if args.config == 2:
        un, inst = make_trace(args.iterations, rank, both=True)
        return inst, un, synth.exact_profile()
    if args.config == 3:
        ev = args.events or 100_000_000
        procs = max(1, ev // 1_000_000)
        un, inst = synth.config3_trace(processes=procs, events_per_pid=ev // procs, both=True, workers=workers,
                                       first_pid=rank * procs + 1)
        return inst, un, synth.exact_profile()
    ev = args.events or 10_000_000
    return synth.adversarial_trace(ev, pids=64, seed=1234 + rank, workers=workers), None, \
        synth.adversarial_profile()


def make_trace(iterations: int, rank: int, both: bool = False):
    """Rank r analyses process r+1 (distinct seed): a weak-scaling shard."""
    from paper_2102_04285_b200 import synth
    from paper_2102_04285_b200.columnar import ColumnarTrace
    from paper_2102_04285_b200.model import ProcessMeta

    out = synth.ddpg_trace(iterations, processes=1, seed=1234 + rank, both=both)
    if rank:
        out = tuple(ColumnarTrace(ct.clock_domain, ct.start, ct.dur, ct.pid, ct.tid, ct.cat, ct.name, ct.corr,
                                  ct.has_corr, ct.pids + rank, ct.group_pid, ct.group_tid, ct.names,
                                  tuple(ProcessMeta(m.pid + rank, m.name, m.parent, m.fork_ns, m.join_ns)
                                        for m in ct.processes), ct.pid_has_meta)
                    for ct in (out if both else (out,)))
        if not both:
            out = out[0]
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def stage_bytes(stage: str, n: int, nnz: int, ns: int, nrec: int) -> float:
    """Algorithmic DRAM bytes of one occurrence of a stage as implemented
    (DESIGN.md section 3): the bytes its kernels must read and write once --
    n events, nnz nonzero-duration events, ns hook sites, nrec transition
    records.  The endpoint keys are 8 bytes (pid | t_rel | 4-bit code: the
    4-byte payload of SURVEY 8(d)'s canonical 12-byte record lives in the
    code bits); record sorts are bucketed (histogram read of the key, one
    scatter pass and one in-bucket pass over (key, value))."""
    if stage == "pass1_validate_spans":  # start, dur, pid, tid, cat, has_corr, name
        return 30.0 * n
    if stage == "endpoint_keygen":      # k_bk_hist: start, dur, pid, cat -> bucket counts
        return 21.0 * n
    if stage == "endpoint_sort":        # k_bk_scatter: the same reads, 2 keys written per nonzero event
        return 21.0 * n + 16.0 * nnz
    if stage == "sweep_scan_hist":      # k_bk_sweep: one read of the 2 sorted keys per nonzero event
        return 16.0 * nnz
    if stage == "site_sort":            # count + generate (35 B/event) + (k8,v4) site records: write 13,
        return 35.0 * n + 69.0 * ns     # histogram 8, scatter 24, in-bucket 24
    if stage == "transition_sort":      # record generation (21 B/event) + (k8,v4) records: write 12,
        return 21.0 * n + 68.0 * nrec   # histogram 8, scatter 24, in-bucket 24
    if stage == "remap":                # start, dur, pid, cat in; start', dur' out
        return 37.0 * n
    if stage == "quantize_scan":        # site key 8, slot 4, owner 4, subkind 1, amount 8
        return 25.0 * ns
    if stage == "removal_scan":         # site key, slot, amount, subkind + extents (a, len, E)
        return 45.0 * ns
    return 0.0


def transition_records(ct) -> int:
    """Records of the correction's transition pass (H -> B, H -> S): two
    endpoints per nonzero HIGH_LEVEL event, one query per BACKEND/SIMULATOR."""
    return int(2 * np.count_nonzero((ct.cat == 1) & (ct.dur > 0)) + np.count_nonzero((ct.cat == 2) | (ct.cat == 3)))


def traffic_from_profiles(stage: str, config: int):
    """ncu DRAM bytes per launch of the stage's kernel, from this config's
    capture (profiles/ncu_traffic_c<config>.json), else None."""
    p = os.path.join(ROOT, "profiles", f"ncu_traffic_c{config}.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    return d.get(stage)


def pid_sample(ct, budget_events: int):
    """Sub-trace of the smallest pids whose events total <= budget (per-pid
    results are independent: overlap.py:126, correction.py:132)."""
    counts = np.bincount(ct.pid, minlength=ct.n_pids)
    keep, tot = [], 0
    for p in np.argsort(counts, kind="stable"):
        if counts[p] == 0:
            continue
        if tot + counts[p] > budget_events and keep:
            break
        keep.append(int(p))
        tot += int(counts[p])
    return (ct.select_pids(keep) if len(keep) < ct.n_pids else ct), keep


def oracle_sample_check(ct, profile, out_s, out_d, bd, budget=1_500_000):
    """Config 5: the measured step's corrected columns and cells vs the oracle
    on a bounded sample of pids."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    from paper_2102_04285_b200.columnar import ColumnarTrace
    sub, keep = pid_sample(ct, budget)
    rows = np.isin(ct.pid, np.asarray(keep, np.int32))
    s, d, _, _ = oracle.correct(sub, profile)
    ok = bool(np.array_equal(out_s[rows], s) and np.array_equal(out_d[rows], d))
    cor = ColumnarTrace(sub.clock_domain, s, d, sub.pid, sub.tid, sub.cat, sub.name, sub.corr, sub.has_corr,
                        sub.pids, sub.group_pid, sub.group_tid, sub.names, sub.processes, sub.pid_has_meta)
    cells, spans, untracked = oracle.overlap(cor, 0)
    pv = {int(ct.pids[p]) for p in keep}
    ours = {(k.pid, k.path, frozenset(int(c) for c in k.categories)): v for k, v in bd.cells.items() if k.pid in pv}
    ok = ok and ours == cells and {p: bd.spans[p] for p in pv} == spans and \
        {p: bd.untracked[p] for p in pv} == untracked
    return ok, f"{len(keep)} of {ct.n_pids} pids, {sub.n} events: corrected columns + cells/spans/untracked"


def cpu_baseline_port(ct, profile, seconds: float):
    """The C restatement (oracle/) of correct_trace + compute_overlap(corrected):
    the reference algorithm, compiled, one thread, on a bounded sample of pids
    (the whole trace at config 2)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    from paper_2102_04285_b200.columnar import ColumnarTrace
    full_n = ct.n
    ct, _ = pid_sample(ct, 2_000_000)

    t0 = time.perf_counter()
    runs = 0
    while True:
        s, d, _rep, _ = oracle.correct(ct, profile)
        ct2 = ColumnarTrace(ct.clock_domain, s, d, ct.pid, ct.tid, ct.cat, ct.name, ct.corr, ct.has_corr, ct.pids,
                            ct.group_pid, ct.group_tid, ct.names, ct.processes, ct.pid_has_meta)
        oracle.overlap(ct2, 0)
        runs += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    what = "full" if ct.n == full_n else f"pid sample of the {full_n}-event"
    return {"value": runs * ct.n / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{runs} x {ct.n}-event {what} trace, oracle/xs_oracle.c correct+overlap, {dt:.1f}s"}


# ---------------------------------------------------------------------------
def _analyze_e2e(ct, profile, out, pipelined):
    from paper_2102_04285_b200 import analyze_columnar, analyze_columnar_pipelined
    if pipelined:
        return analyze_columnar_pipelined(ct, profile, out=out)
    return analyze_columnar(ct, profile, out=out)


def settle_clocks(dev, ms: float = 200.0):
    """~ms of dense GPU work before the warm-up steps: a config-2 step is ~1 ms,
    so the first timed steps would otherwise run while the SM clock is still
    ramping up from idle (not a measurement of the path; no analysis runs)."""
    import torch
    a = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    while (time.perf_counter() - t0) * 1e3 < ms:
        for _ in range(8):
            a = (a @ a).clamp_(-1, 1)
        torch.cuda.synchronize()
    del a


def first_calls(ct_pin, profile, out, pipelined, k: int = 3):
    """Wall time of this process's first k analysis calls on the bench trace
    (public API, pinned host columns): the first pays context creation,
    workspace allocation and an eager run, the second captures the pipeline
    graphs, later calls replay them."""
    import torch
    ms = []
    for _ in range(k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _analyze_e2e(ct_pin, profile, out, pipelined)
        ms.append(round((time.perf_counter() - t0) * 1e3, 3))
    return ms


def time_e2e(fn, flush, steps):
    import torch
    ms = []
    res = None
    for _ in range(steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = fn()
        ms.append((time.perf_counter() - t0) * 1e3)
    return float(np.median(ms)), res


def trace_api_e2e(ct, profile, reps: int = 2):
    """The reference's own call sequence through the drop-in API, from a
    Trace of Python Event objects: correct_trace(trace, profile) then
    compute_overlap(corrected) (cli.py:168-171).  Returns (median ms, phases)."""
    from paper_2102_04285_b200 import compute_overlap, correct_trace
    trace = ct.to_trace()
    ms, last = [], None
    for _ in range(reps + 1):
        t0 = time.perf_counter()
        corrected, _rep = correct_trace(trace, profile)
        t1 = time.perf_counter()
        bd = compute_overlap(corrected)
        _ = len(bd.cells)
        t2 = time.perf_counter()
        ms.append((t2 - t0) * 1e3)
        last = {"correct_trace_ms": round((t1 - t0) * 1e3, 1), "compute_overlap_ms": round((t2 - t1) * 1e3, 1)}
    return float(np.median(ms[1:])), last


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    from paper_2102_04285_b200 import _engine
    from paper_2102_04285_b200.distributed import merge_breakdown_raw

    ct, un, profile = make_workload(args, rank)
    n = ct.n
    pipelined = ct.n_pids >= 8  # many processes: upload the next pid batch while analysing this one
    # the caller's trace columns in page-locked host memory (the e2e input)
    ct_pin = ct.pinned(packed=False)
    out_s = torch.empty(n, dtype=torch.int64).pin_memory()
    out_d = torch.empty(n, dtype=torch.int64).pin_memory()
    first_ms = first_calls(ct_pin, profile, (out_s, out_d), pipelined)

    scaled = profile.scaled(ct.names)
    eng = _engine.get(local)
    dt_dev = _engine.DeviceTrace(ct_pin, local)
    nnz = int((ct.dur > 0).sum())
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def step_device():
        raw = eng.correct(dt_dev, scaled, analyze_attribution=0)
        merged = None
        if world > 1:
            merged = merge_breakdown_raw(ct, eng.fetch_overlap(), dev)
        return raw, merged

    clocks = ClockSampler(local).__enter__()  # sampled across warmup + timed steps
    settle_clocks(dev)
    for _ in range(max(args.warmup, 1)):
        flush.fill_(1.0)  # (the same L2 state as the timed steps)
        step_device()  # (results dropped: every call gets the same output buffers, as in the timed loop)
    torch.cuda.synchronize()
    launches0 = eng.launches()
    times = []
    stream = torch.cuda.current_stream(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush between steps
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step_device()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    clocks.__exit__(None, None, None)
    launches = eng.launches() - launches0
    import ctypes as C
    from paper_2102_04285_b200 import _lib
    info = _lib.XsCorrectInfo()  # sites of the timed call (before any other analysis on this context)
    eng.lib.xs_correct_report(eng.ctx, C.byref(info), None, None, eng.stream())
    ns_sites = int(info.n_sites)
    # per-stage device times come from a separate pass: the timing events
    # themselves must not sit inside the timed region
    eng.lib.xs_profile_enable(eng.ctx, 1)
    for _ in range(args.steps):
        flush.fill_(1.0)
        step_device()
    torch.cuda.synchronize()
    ms_arr = np.zeros(32)
    calls_arr = np.zeros(32, np.int64)
    nst = eng.lib.xs_profile_read(eng.ctx, ms_arr.ctypes.data, calls_arr.ctypes.data, 32)
    eng.lib.xs_profile_enable(eng.ctx, 0)
    stage_names = [eng.lib.xs_profile_stage_name(i).decode() for i in range(nst)]
    total_ms = float(np.sum(times))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    total_events = n * world
    value = total_events / (ms_per_step / 1e3)

    # e2e (headline) through the public API: the trace's columns sit in
    # page-locked host memory; every step uploads them (38 B/event), analyses,
    # reads the corrected columns back into pinned buffers and decodes the
    # Breakdown (spans/untracked; the cells dict is built on first access)
    h2d = int(ct_pin._pinned["_block"].numel())

    def step_e2e(src):
        f0 = eng.fetched_bytes
        _, _, _, bd = _analyze_e2e(src, profile, (out_s, out_d), pipelined)
        d2h = 16 * n + (eng.fetched_bytes - f0) + 8 * 4 * ct.n_pids * 2  # columns + overlap arrays + report
        return d2h, bd

    e2e_steps = max(3, args.steps // 2)
    step_e2e(ct_pin)
    e2e_step, (d2h, bd) = time_e2e(lambda: step_e2e(ct_pin), flush, e2e_steps)
    # the same from ordinary (pageable) numpy columns: the native builder packs
    # them into page-locked staging inside every step (16 B/event on the wire)
    step_e2e(ct)
    np_step, _ = time_e2e(lambda: step_e2e(ct), flush, e2e_steps)
    if world > 1:
        t = torch.tensor([e2e_step, np_step], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_step, np_step = (float(x) for x in t.tolist())
    api = None
    if args.config == 2 and world == 1:
        api_ms, phases = trace_api_e2e(ct, profile)
        api = {"value": round(n / (api_ms / 1e3), 1), "unit": UNIT, "ms_per_step": round(api_ms, 1),
               "path": "correct_trace(Trace of Event objects) + compute_overlap(corrected Trace), the "
                       "reference's call sequence (cli.py:168-171) through the drop-in API", **phases}

    # correctness of the measured result: closure against the uninstrumented
    # twin (configs 2/3), or the oracle on a bounded sample of pids (config 5)
    check = {}
    if un is not None:
        check["closure_exact"] = bool(np.array_equal(out_s.numpy(), un.start) and np.array_equal(out_d.numpy(), un.dur))
    else:
        check["oracle_sample_exact"], check["oracle_sample"] = oracle_sample_check(ct, profile, out_s.numpy(),
                                                                                   out_d.numpy(), bd)

    # roofline for the dominant stage
    peak, peak_kind = load_peaks()
    nrec = transition_records(ct)
    stages = {}
    for i, nm in enumerate(stage_names):
        if calls_arr[i]:
            stages[nm] = {"ms_total": round(float(ms_arr[i]), 4), "occurrences": int(calls_arr[i]),
                          "ms_avg": round(float(ms_arr[i]) / int(calls_arr[i]), 5)}
    # roofline of the dominant kernel: among the stages that are one main
    # kernel per occurrence (so ncu's per-launch DRAM bytes map onto them),
    # the one with the largest share of the step; every modeled stage is
    # listed in stage_rooflines
    single = ("sweep_scan_hist", "endpoint_keygen", "endpoint_sort", "pass1_validate_spans", "quantize_scan",
              "removal_scan", "remap")
    modeled = [k for k in stages if stage_bytes(k, n, nnz, ns_sites, nrec) > 0]

    def roof_of(k):
        algo = stage_bytes(k, n, nnz, ns_sites, nrec)
        achieved = algo / (stages[k]["ms_avg"] / 1e3) / 1e9
        return {"kernel": k, "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": round(achieved / peak, 4), "algorithmic_bytes_per_launch": algo,
                "traffic": traffic_from_profiles(k, args.config),
                "share_of_step": round(stages[k]["ms_total"] / total_ms, 3) if total_ms else None}

    cands = [k for k in modeled if k in single] or modeled
    dom = max(cands, key=lambda k: stages[k]["ms_total"]) if cands else None
    roof = roof_of(dom) if dom else None
    stage_roofs = {k: {f: roof_of(k)[f] for f in ("achieved", "frac", "traffic")} for k in modeled}
    pipe_bytes = sum(stage_bytes(k, n, nnz, ns_sites, nrec) * v["occurrences"]
                     for k, v in stages.items()) / args.steps
    s_per_ev = ns_sites / max(n, 1)
    survey_b = 325 + 45 + s_per_ev * 400 + 32  # B_ov (P=5) + B_corr (P_s=6)
    pipeline = {"model_bytes_per_event": round(pipe_bytes / n, 1),
                "achieved_GBps": round(pipe_bytes / (ms_per_step / 1e3) / 1e9, 1),
                "frac": round(pipe_bytes / (ms_per_step / 1e3) / 1e9 / peak, 4),
                "survey_model_bytes_per_event": round(survey_b, 1),
                "survey_model_GBps": round(survey_b * n / (ms_per_step / 1e3) / 1e9, 1),
                "survey_model_frac": round(survey_b * n / (ms_per_step / 1e3) / 1e9 / peak, 4),
                "compulsory_bytes_per_event": 45 + 21}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_port(ct, profile, args.cpu_seconds)
        cpu["cores_available"] = os.cpu_count()

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "step_ms": [round(t, 4) for t in times],
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config],
                       "events_per_gpu": n, "pids_per_gpu": ct.n_pids, "events_total": total_events,
                       "attribution": "instant",
                       "l2": f"flushed (256 MB write) between timed steps; inputs {h2d / 1e6:.0f} MB/GPU",
                       "parallelism": f"pid-sharded x{world}" + (", NCCL all-reduce histogram merge" if world > 1
                                                                   else "")},
            "e2e": {"value": round(total_events / (e2e_step / 1e3), 1), "unit": UNIT,
                    "ms_per_step": round(e2e_step, 3),
                    "api": ("analyze_columnar_pipelined (9 pid batches over 3 contexts; one call when a pid dominates)"
                            if pipelined else "analyze_columnar"),
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(d2h),
                    "path": "the trace's columns in page-locked host memory (ColumnarTrace.pinned(packed=False)) -> "
                            "H2D of every column inside the step -> xs_analyze_to_host (corrected columns D2H "
                            "overlapped with the overlap pass) -> D2H cell arrays -> Breakdown (spans/untracked "
                            "decoded; the cells dict of OverlapKeys is built on first access)"},
            "e2e_from_numpy": {"value": round(total_events / (np_step / 1e3), 1), "unit": UNIT,
                               "ms_per_step": round(np_step, 3),
                               "path": "ordinary numpy columns: native host packing into page-locked staging "
                                       "(xs_pack_plan/xs_pack_fill, host threads) + one DMA of the packed block "
                                       "inside every step, then as e2e"},
            "e2e_trace_api": api,
            "first_calls_ms": first_ms,
            "gpu_launches": int(launches / args.steps),
            "roofline": roof, "stage_rooflines": stage_roofs, "pipeline_roofline": pipeline, "stages_ms": stages,
            "sites": ns_sites, "transition_records": nrec,
            "cpu_baseline": cpu, "clocks": clocks.summary(), **check,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
def _ref_sample(config: int, worker: int, iterations: int, events: int):
    """Worker w's input: the identical bench trace (config 2), or one process
    of the identical config-3 / config-5 trace (same seeds: those pids' events
    are exactly the bench trace's)."""
    from paper_2102_04285_b200 import synth
    if config == 2:
        return make_trace(iterations, 0), synth.exact_profile(), "the identical config-2 trace (whole)"
    if config in (3, 4):
        return (synth.config3_trace(processes=1, events_per_pid=1_000_000, first_pid=worker + 1),
                synth.exact_profile(), f"pid {worker + 1} of the identical config-{config} trace")
    ev = events or 10_000_000
    sizes = synth.zipf_sizes(ev, 64, 1.5)
    small = [p + 1 for p in sorted(range(64), key=lambda p: -sizes[p]) if sizes[p] <= 300_000]
    pid = small[worker % len(small)]
    return (synth.adversarial_trace(ev, pids=64, only=[pid]), synth.adversarial_profile(),
            f"pid {pid} of the identical config-5 trace")


def _ref_worker(args):
    """One host core: build the reference's own Trace of Event objects
    (untimed), then time correct_trace + compute_overlap(corrected) through
    the unmodified reference package (oracle/_ref, native Cython sweep)."""
    config, worker, iterations, events, warmup, steps, barrier, stop, budget = args
    ref = os.path.join(ROOT, "oracle", "_ref")
    sys.path.insert(0, ref)
    from xstrace import model as RM
    from xstrace.calibration import CalibrationProfile as RP
    from xstrace.correction import correct_trace as ref_correct
    from xstrace.overlap import HAVE_NATIVE_SWEEP, compute_overlap as ref_overlap

    ct, p, what = _ref_sample(config, worker, iterations, events)
    cats = [RM.Category(c) for c in range(6)]
    names = ct.names
    events_ = [RM.Event(int(ct.pids[pp]), int(ct.group_tid[g]), cats[c], names[nm], s, d, k if h else None)
               for pp, g, c, nm, s, d, k, h in zip(ct.pid.tolist(), ct.tid.tolist(), ct.cat.tolist(),
                                                   ct.name.tolist(), ct.start.tolist(), ct.dur.tolist(),
                                                   ct.corr.tolist(), ct.has_corr.tolist())]
    trace = RM.Trace(ct.clock_domain, events_, [RM.ProcessMeta(m.pid, m.name, m.parent, m.fork_ns, m.join_ns)
                                                for m in ct.processes])
    prof = RP(p.annotation_ns, p.transition_ns, p.api_interception_ns, dict(p.api_internal_ns))

    def step():
        out, _ = ref_correct(trace, prof)
        ref_overlap(out)

    for _ in range(warmup):
        step()
    spans = []
    t_begin = None
    for _ in range(steps):
        barrier.wait()  # every worker runs the same number of steps
        if stop.value:
            break
        t0 = time.perf_counter()
        t_begin = t_begin or t0
        step()
        t1 = time.perf_counter()
        spans.append((t0, t1))
        if worker == 0 and (t1 - t_begin) + (t1 - t0) > budget:
            stop.value = 1  # (set before the next barrier: every worker sees it)
    return ct.n, spans, what, HAVE_NATIVE_SWEEP


def run_reference(args):
    """The reference's own CPU implementation of the path on all host cores,
    on the same workload: one worker process per core, each analysing its
    own copy of the identical bench trace (config 2; configs 3 / 5: one of
    the identical trace's processes each) through the unmodified reference
    package; throughput = all events analysed / wall time of the common timed
    phase.  A step is ~10-30 s of CPU work, so warm-up is capped at one step
    and the timed steps stop once ~--ref-budget seconds are spent."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    ref = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref, "xstrace")):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (run oracle/build_ref.sh)"}))
        return
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    ctx = mp.get_context("fork")
    mgr = ctx.Manager()
    barrier = mgr.Barrier(cores)
    stop = mgr.Value("i", 0)
    warm = min(max(args.warmup, 0), 1)
    with ctx.Pool(cores) as pool:
        res = pool.map(_ref_worker, [(args.config, w, args.iterations, args.events, warm, args.steps, barrier, stop,
                                      args.ref_budget) for w in range(cores)], chunksize=1)
    steps_run = min(len(r[1]) for r in res)
    total = sum(r[0] * steps_run for r in res)
    wall = max(r[1][steps_run - 1][1] for r in res) - min(r[1][0][0] for r in res)
    value = total / wall
    step_s = sorted(b - a for r in res for a, b in r[1][:steps_run])
    single = res[0][0] / step_s[len(step_s) // 2]
    sample = (f"{cores} worker processes x {res[0][2]} ({res[0][0]} events each), reference xstrace "
              f"correct_trace + compute_overlap, native sweep={res[0][3]}, {steps_run} timed step(s) after {warm} "
              f"warm-up")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": steps_run, "steps_requested": args.steps, "warmup": warm, "warmup_requested": args.warmup,
        "ms_per_step": round(wall / steps_run * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "events_per_step": sum(r[0] for r in res),
                   "same_config": args.config == 2,
                   "same_trace": "every worker analyses the identical bench trace" if args.config == 2 else
                   "every worker analyses one process of the identical bench trace"},
        "single_process_events_per_s": round(single, 1),
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def run_config4(args):
    """Config 4: the fixed 1B-event trace strong-scaled over the ranks.  Rank r
    owns a contiguous block of the (equal-sized) processes, generated from the
    per-pid seeds (so the trace is identical for every N) and kept resident in
    HBM in batches of <= 100 processes; a step analyses every batch
    (xs_analyze: correct_trace + compute_overlap(corrected)) and merges all
    batches of all ranks into one Breakdown (NCCL sparse merge) -- the merge
    is inside the timed region."""
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    from paper_2102_04285_b200 import _engine, synth
    from paper_2102_04285_b200.distributed import merge_breakdown_parts

    total = args.events or 1_000_000_000
    n_pids = max(1, total // 1_000_000)
    lo = rank * n_pids // world
    hi = (rank + 1) * n_pids // world
    eng = _engine.get(local)
    prof = synth.exact_profile()
    batches = []
    gen_s = 0.0
    for a in range(lo, hi, 100):
        t0 = time.time()
        if args.device_gen:  # both twins generated in HBM; the instrumented one is analysed in place
            g = synth.device_ddpg_trace(synth.CONFIG3_ITERS_PER_1M, processes=min(100, hi - a), first_pid=a + 1,
                                        outer_op="iteration", second_tid_ops=True, device=local)
            torch.cuda.synchronize()
            dt = g.device_trace("inst", local)
            ct = dt.ct
            del g.cols["un"]
            keep = g  # (owns the columns)
        else:
            ct = synth.config3_trace(processes=min(100, hi - a), events_per_pid=1_000_000, first_pid=a + 1,
                                     workers=os.cpu_count())
            keep = ct.pinned()  # (a pinned trace keeps its own device copy: batches never alias)
            dt = _engine.DeviceTrace(keep, local)
        gen_s += time.time() - t0
        batches.append((ct, dt, prof.scaled(ct.names), keep))
    n_local = sum(b[0].n for b in batches)

    def step():
        parts = []
        for ct, dt, sc, _ in batches:
            eng.correct(dt, sc, analyze_attribution=0)
            parts.append((ct, eng.fetch_overlap()))
        return merge_breakdown_parts(parts, dev)

    clocks = ClockSampler(local).__enter__()
    for _ in range(max(args.warmup, 1)):
        bd = step()
    stream = torch.cuda.current_stream(dev)
    launches0 = eng.launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        bd = step()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    clocks.__exit__(None, None, None)
    launches = eng.launches() - launches0
    tot = torch.tensor([float(np.sum(times)), float(n_local)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = tot.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = tot.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        total_ms, events = float(mx[0].item()), int(sm[1].item())
    else:
        total_ms, events = float(tot[0].item()), n_local
    ms_per_step = total_ms / args.steps
    # every process: cells + untracked = span (conservation); the merged result holds every pid
    conserve = all(sum(v for k, v in bd.cells.items() if k.pid == p) + bd.untracked[p] == h - l
                   for p, (l, h) in list(bd.spans.items())[:50])
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": round(events / (ms_per_step / 1e3), 1), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3),
            "step_ms": [round(t, 3) for t in times], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": WORKLOADS[4], "events_total": events, "pids": n_pids,
                       "batches_per_rank": len(batches), "l2": "inputs 38 GB/rank > L2",
                       "parallelism": f"contiguous pid blocks x{world}, NCCL sparse merge"},
            "gpu_launches": int(launches / args.steps), "merged_pids": len(bd.spans), "conservation": conserve,
            "generation_s_rank0": round(gen_s, 1),
            "generator": "device (xs_synth)" if args.device_gen else "host (synth.config3_trace)",
            "clocks": clocks.summary()}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.config == 4:
        run_config4(a)
    else:
        run_ours(a)
