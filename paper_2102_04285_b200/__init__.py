"""xstrace-b200: B200-native trace-analysis hot path of RL-Scope (arXiv 2102.04285).

Drop-in for the reference package's hot path (``xstrace.compute_overlap``,
``xstrace.correct_trace``, ``xstrace.count_transitions`` and the data model
they take).  Host code is Python; the analysis runs in hand-written sm_100a
CUDA kernels behind the C ABI in ``include/xstrace_b200.h``.
"""

from .calibration import CalibrationProfile, HOOK_KINDS
from .columnar import ColumnarTrace
from .correction import (
    CorrectionReport,
    UncalibratedHookError,
    analyze_columnar,
    analyze_columnar_pipelined,
    correct_trace,
    correct_trace_columnar,
    correction_bias,
)
from .model import (
    Category,
    Event,
    InvalidTraceError,
    ProcessMeta,
    Trace,
    Violation,
    pid_spans,
    require_valid,
    traces_equal,
    validate_trace,
)
from .metrics import (
    ReportRow,
    UtilizationSample,
    busy_fraction,
    sampled_utilization,
    summarize,
    utilization_samples,
)
from .traceio import (
    IncompleteTraceError,
    TraceFormatError,
    TruncatedTraceError,
    read_trace,
    read_trace_columnar,
    write_trace,
)
from .procview import ProcessNode, ProcessTree, build_process_tree, render_tree, to_dot
from .overlap import (
    Attribution,
    Breakdown,
    OverlapKey,
    TransitionCounts,
    TRANSITION_PAIRS,
    WRAPPER_PAIRS,
    compute_overlap,
    compute_overlap_columnar,
    count_transitions,
    sweep_pid,
    transition_sites,
)

__version__ = "0.1.0"

__all__ = [
    "analyze_columnar_pipelined",
    "IncompleteTraceError",
    "TraceFormatError",
    "TruncatedTraceError",
    "read_trace",
    "read_trace_columnar",
    "write_trace",
    "ProcessNode",
    "ProcessTree",
    "ReportRow",
    "UtilizationSample",
    "build_process_tree",
    "busy_fraction",
    "render_tree",
    "sampled_utilization",
    "summarize",
    "sweep_pid",
    "to_dot",
    "utilization_samples",
    "Attribution",
    "Breakdown",
    "CalibrationProfile",
    "Category",
    "ColumnarTrace",
    "CorrectionReport",
    "Event",
    "HOOK_KINDS",
    "InvalidTraceError",
    "OverlapKey",
    "ProcessMeta",
    "TRANSITION_PAIRS",
    "Trace",
    "TransitionCounts",
    "UncalibratedHookError",
    "Violation",
    "WRAPPER_PAIRS",
    "analyze_columnar",
    "compute_overlap",
    "compute_overlap_columnar",
    "correct_trace",
    "correct_trace_columnar",
    "correction_bias",
    "count_transitions",
    "pid_spans",
    "require_valid",
    "traces_equal",
    "transition_sites",
    "validate_trace",
]
