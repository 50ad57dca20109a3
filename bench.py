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
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 5],
                    help="BASELINE.json config: 2 (default, the metric's workload), 3 (100M events, 100 pids, "
                         "nested), 5 (adversarial 10M)")
    ap.add_argument("--events", type=int, default=0, help="events per GPU for --config 3/5 (default 100M / 10M)")
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


def stage_bytes(stage: str, n: int, nnz: int, ns: int, key_bits_main: int, key_bits_site: int) -> float:
    """Algorithmic DRAM bytes of one occurrence of a stage ('Roofline')."""
    def passes(bits):
        return max(1, -(-bits // 8))
    if stage == "endpoint_sort":   # keys-only onesweep over 2n keys: 1 histogram read + P x (read+write)
        return 2 * n * (8 + 16 * passes(key_bits_main))
    if stage == "sweep_scan_hist":  # one read of the sorted nonzero endpoints
        return 2 * nnz * 8
    if stage == "endpoint_keygen":  # read start/dur/pid/cat/has_corr, write 2 keys
        return n * (8 + 8 + 4 + 1 + 1) + 2 * n * 8
    if stage == "site_sort":        # two (key8,val4) pair sorts over the sites + generation
        return 2 * ns * (8 + 24 * passes(key_bits_site)) + n * 21
    if stage == "remap":            # read start/dur/pid/cat, write start'/dur'
        return n * (8 + 8 + 4 + 1) + n * 16
    if stage == "quantize_scan":
        return ns * (8 + 4 + 4 + 1 + 8)
    if stage == "removal_scan":
        return ns * (8 + 4 + 8 + 1) + ns * 24
    if stage == "pass1_validate_spans":
        return n * (8 + 8 + 4 + 4 + 1 + 1 + 4)
    if stage == "transition_sort":  # two (key8,val4) pair sorts over ~0.3n records (B/S queries + H endpoints)
        return 0.0
    return 0.0


def traffic_from_profiles(stage: str):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
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
def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    from paper_2102_04285_b200 import _engine, synth
    from paper_2102_04285_b200.distributed import merge_breakdown_raw
    from paper_2102_04285_b200.overlap import decode_breakdown

    ct, un, profile = make_workload(args, rank)
    scaled = profile.scaled(ct.names)
    eng = _engine.get(local)
    dt_dev = _engine.DeviceTrace(ct, local)
    n = ct.n
    nnz = int((ct.dur > 0).sum())
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def step_device():
        raw = eng.correct(dt_dev, scaled, analyze_attribution=0)
        merged = None
        if world > 1:
            merged = merge_breakdown_raw(ct, eng.fetch_overlap(), dev)
        return raw, merged

    clocks = ClockSampler(local).__enter__()  # sampled across warmup + timed steps
    for _ in range(max(args.warmup, 1)):
        raw, _ = step_device()
    torch.cuda.synchronize()
    launches0 = eng.launches()
    times = []
    stream = torch.cuda.current_stream(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush between steps (inputs 37 MB < L2)
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

    # end-to-end through the public API (analyze_columnar) with host buffers:
    # the user's columns in pinned memory, uploaded every step, the corrected
    # columns read back into pinned buffers, the Breakdown decoded on the host
    from paper_2102_04285_b200 import analyze_columnar
    ct_host = ct.pinned()
    out_s = torch.empty(n, dtype=torch.int64).pin_memory()
    out_d = torch.empty(n, dtype=torch.int64).pin_memory()
    h2d = int(ct_host._pinned["_block"].numel())  # the one pinned block uploaded per step

    from paper_2102_04285_b200 import analyze_columnar_pipelined
    pipelined = ct.n_pids >= 8  # many processes: upload the next pid batch while analysing this one

    def step_e2e():
        f0 = eng.fetched_bytes
        if pipelined:
            s_, d_, rep, bd = analyze_columnar_pipelined(ct_host, profile, out=(out_s, out_d))
        else:
            s_, d_, rep, bd = analyze_columnar(ct_host, profile, out=(out_s, out_d))
        d2h = 16 * n + (eng.fetched_bytes - f0) + 8 * 4 * ct.n_pids * 2  # columns + overlap arrays + report
        return d2h, bd

    for _ in range(2):
        step_e2e()
    e2e_ms = []
    d2h = 0
    for _ in range(max(3, args.steps // 2)):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d2h, bd = step_e2e()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_step = float(np.median(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e_step], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_step = float(t.item())

    # correctness of the measured step: closure against the uninstrumented twin
    # (configs 2/3), or the oracle on a bounded sample of pids (config 5)
    check = {}
    if un is not None:
        check["closure_exact"] = bool(np.array_equal(out_s.numpy(), un.start) and np.array_equal(out_d.numpy(), un.dur))
    else:
        check["oracle_sample_exact"], check["oracle_sample"] = oracle_sample_check(ct, profile, out_s.numpy(),
                                                                                   out_d.numpy(), bd)

    # roofline for the dominant stage
    peak, peak_kind = load_peaks()
    tb = int(max(1, int((ct.start + ct.dur).max() - ct.start.min())).bit_length())
    key_bits_main = tb + 4 + max(0, (ct.n_pids - 1).bit_length())
    key_bits_site = tb + 3 + max(0, (ct.n_pids - 1).bit_length())
    stages = {}
    for i, nm in enumerate(stage_names):
        if calls_arr[i]:
            stages[nm] = {"ms_total": round(float(ms_arr[i]), 4), "occurrences": int(calls_arr[i]),
                          "ms_avg": round(float(ms_arr[i]) / int(calls_arr[i]), 5)}
    import ctypes as C
    from paper_2102_04285_b200 import _lib
    info = _lib.XsCorrectInfo()
    eng.lib.xs_correct_report(eng.ctx, C.byref(info), None, None, eng.stream())
    ns_sites = int(info.n_sites)
    # roofline of the dominant kernel: among the stages that are one main
    # kernel per occurrence (so ncu's per-launch DRAM bytes map onto them),
    # the one with the largest share of the step; every modeled stage is
    # listed in stage_rooflines
    single = ("sweep_scan_hist", "endpoint_keygen", "endpoint_sort", "pass1_validate_spans", "quantize_scan",
              "removal_scan", "remap")
    modeled = [k for k in stages if stage_bytes(k, n, nnz, ns_sites, key_bits_main, key_bits_site) > 0]

    def roof_of(k):
        algo = stage_bytes(k, n, nnz, ns_sites, key_bits_main, key_bits_site)
        achieved = algo / (stages[k]["ms_avg"] / 1e3) / 1e9
        return {"kernel": k, "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": round(achieved / peak, 4), "algorithmic_bytes_per_launch": algo,
                "traffic": traffic_from_profiles(k),
                "share_of_step": round(stages[k]["ms_total"] / total_ms, 3) if total_ms else None}

    cands = [k for k in modeled if k in single] or modeled
    dom = max(cands, key=lambda k: stages[k]["ms_total"]) if cands else None
    roof = roof_of(dom) if dom else None
    stage_roofs = {k: {f: roof_of(k)[f] for f in ("achieved", "frac", "traffic")} for k in modeled}
    pipe_bytes = sum(stage_bytes(k, n, nnz, ns_sites, key_bits_main, key_bits_site) * v["occurrences"]
                     for k, v in stages.items()) / args.steps
    pipeline = {"model_bytes_per_event": round(pipe_bytes / n, 1),
                "achieved_GBps": round(pipe_bytes / (ms_per_step / 1e3) / 1e9, 1),
                "compulsory_bytes_per_event": 45 + 21}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_port(ct, profile, args.cpu_seconds)
        cpu["cores_available"] = os.cpu_count()

    in_mb = h2d / 1e6
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "step_ms": [round(t, 4) for t in times], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config],
                       "events_per_gpu": n, "pids_per_gpu": ct.n_pids, "events_total": total_events,
                       "attribution": "instant",
                       "l2": f"flushed (256 MB write) between timed steps; inputs {in_mb:.0f} MB/GPU",
                       "parallelism": f"pid-sharded x{world}" + (", NCCL all-reduce histogram merge" if world > 1
                                                                   else "")},
            "e2e": {"value": round(total_events / (e2e_step / 1e3), 1), "unit": UNIT, "ms_per_step": round(e2e_step, 3),
                    "api": ("analyze_columnar_pipelined (9 pid batches over 3 contexts; one call when a pid dominates)" if pipelined
                            else "analyze_columnar"),
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(d2h),
                    "path": "analyze_columnar(pinned host columns): H2D -> xs_analyze_to_host (corrected columns D2H "
                            "overlapped with the overlap pass) -> D2H cell arrays -> Breakdown (spans/untracked "
                            "decoded; the cells dict of OverlapKeys is built on first access)"},
            "gpu_launches": int(launches / args.steps),
            "roofline": roof, "stage_rooflines": stage_roofs, "pipeline_roofline": pipeline, "stages_ms": stages,
            "cpu_baseline": cpu, "clocks": clocks.summary(), **check,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
def _ref_sample(config: int, worker: int, iterations: int, events: int):
    """Worker w's bounded sample of the bench workload (distinct seeds/pids)."""
    from paper_2102_04285_b200 import synth
    if config == 2:  # 1/10 of the 1M-event trace
        return make_trace(max(1, iterations // 10), worker), synth.exact_profile(), "1/10 of the config-2 trace"
    if config == 3:  # one 100k-event pid of config 3
        return (synth.config3_trace(processes=1, events_per_pid=100_000, first_pid=worker + 1),
                synth.exact_profile(), "one 100k-event config-3 pid")
    n = max(64 * 32, (events or 10_000_000) // 100)
    return (synth.adversarial_trace(n, pids=64, seed=1234 + worker), synth.adversarial_profile(),
            f"1/100 of the config-5 trace ({n} events, 64 pids)")


def _ref_worker(args):
    """One host core: build the reference's own Trace of Event objects
    (untimed), then time correct_trace + compute_overlap(corrected) through
    the unmodified reference package (oracle/_ref, native Cython sweep)."""
    config, worker, iterations, events, warmup, steps, barrier = args
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
    barrier.wait()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    t1 = time.perf_counter()
    return ct.n * steps, t0, t1, what, HAVE_NATIVE_SWEEP, ct.n


def run_reference(args):
    """The reference's own CPU implementation of the path on all host cores:
    one worker process per core, each analysing its own bounded sample of the
    workload through the unmodified reference package; throughput = all
    events / wall time of the common timed phase."""
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
    with ctx.Pool(cores) as pool:
        res = pool.map(_ref_worker, [(args.config, w, args.iterations, args.events, max(args.warmup, 1), args.steps,
                                      barrier) for w in range(cores)], chunksize=1)
    total = sum(r[0] for r in res)
    wall = max(r[2] for r in res) - min(r[1] for r in res)
    value = total / wall
    per_step_events = sum(r[5] for r in res)
    sample = (f"{cores} worker processes x {res[0][3]} ({res[0][5]} events each), reference xstrace "
              f"correct_trace + compute_overlap, native sweep={res[0][4]}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(wall / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "events_per_step": per_step_events},
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
