"""DualPath KV-Cache loading on B200 (arXiv 2602.21548), B200-native.

Drop-in for the reference's ``pdsim`` Python module
(/root/reference/proj/python/pdsim/__init__.py): the same names
(``ClusterConfig``, ``Round``, ``Trajectory``, ``synthesize``, ``load_trace``,
``save_trace``, ``simulate``, ``ConfigError``, ``SimulationError``), backed by
the B200 engine's own C++ planner, plus the GPU executor that moves the KV
bytes the scheduler's decisions imply (``ExecOptions``, ``build_exec_plan``,
``EngineRuntime``, ``run_step_all``) and ``plan`` (every planner option, with
the decision log and per-request plan).

The product path is native only: importing this package loads the in-tree
``_core`` extension and ``libdualpath.so`` (sm_100a kernels); if they are
missing the import fails loudly -- there is no CPU fallback.
"""

import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))

# The executor waits on device counters with stream memory operations
# (cuStreamWaitValue32) on some streams while other streams of the same GPU
# produce the awaited data; streams multiplexed onto one hardware queue would
# serialise behind such a wait.  Give every stream its own queue (must be set
# before the CUDA context exists).
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

try:
    from . import _core
except ImportError as exc:  # pragma: no cover - exercised only on broken builds
    raise ImportError(
        "paper_2602_21548_b200: native extension not built "
        f"({exc}); run `python -c 'import __graft_entry__ as g; g.build()'`"
    ) from exc

from ._core import (  # noqa: E402
    ABI_VERSION,
    ClusterConfig,
    ConfigError,
    EngineRuntime,
    ExecOptions,
    ExecPlan,
    FullBlockFile,
    FullBlockTrie,
    Round,
    SimulationError,
    StepResult,
    Trajectory,
    blocks_for,
    build_forward_batch,
    estimate_attention_time,
    QuotaInfeasibleError,
    build_exec_plan,
    context_before,
    derive_variant,
    extend_with_synthetic_round,
    load_balance_ratio,
    load_trace,
    plan,
    poisson_arrivals,
    run_step_all,
    run_live,
    save_trace,
    session_chain,
    schedule_de_groups,
    schedule_de_within_group,
    schedule_pe_fetch,
    select_read_path,
    simulate,
    synthesize,
)

LIBDUALPATH = _os.path.join(_HERE, "libdualpath.so")

__all__ = [
    "ABI_VERSION",
    "ClusterConfig",
    "ConfigError",
    "EngineRuntime",
    "ExecOptions",
    "ExecPlan",
    "FullBlockFile",
    "FullBlockTrie",
    "LIBDUALPATH",
    "Round",
    "SimulationError",
    "StepResult",
    "Trajectory",
    "QuotaInfeasibleError",
    "blocks_for",
    "build_forward_batch",
    "estimate_attention_time",
    "build_exec_plan",
    "context_before",
    "derive_variant",
    "extend_with_synthetic_round",
    "load_balance_ratio",
    "load_trace",
    "plan",
    "poisson_arrivals",
    "run_step_all",
    "run_live",
    "save_trace",
    "session_chain",
    "schedule_de_groups",
    "schedule_de_within_group",
    "schedule_pe_fetch",
    "select_read_path",
    "simulate",
    "synthesize",
]
