"""B200-native packed-jobs runtime for triples-mode GPU sharing (arXiv 2410.22254).

Drop-in surface (same names and semantics as the reference ``trilaunch``):
triples core, plan/dealing/workload I/O, ``run_plan`` -> ``RunReport``.
``run_plan(..., backend="packed")`` runs every slot pinned to a GPU as one
lane of a per-GPU packed runtime (``libtlk.so``, hand-written sm_100a
kernels) instead of one time-sliced process per task.
"""

from .core import (
    DEFAULT_ENV_NAMES,
    CpuOversubscribed,
    EnvNames,
    NodeSpec,
    NoGpu,
    NonPositiveField,
    SlotBinding,
    TripleError,
    TripleSpec,
    Verdict,
    assign_gpu,
    expand_slots,
    render_env,
    validate_triple,
)
from .executor import RunReport, TaskResult, classify_failure, run_plan
from .plan import (
    LaunchPlan,
    PlanSummary,
    TaskDef,
    build_plan,
    emit_script,
    load_workload,
    plan_summary,
)

__version__ = "0.1.0"
