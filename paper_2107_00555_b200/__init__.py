"""paper_2107_00555_b200 — B200-native map-execution backend for the
data-centric Python DSL of arXiv 2107.00555 (reference: ``sdfgkit``).

Drop-in for the reference executor (pkg/src/sdfgkit/interp.py:139):

    from sdfgkit import frontend                  # the reference frontend
    import paper_2107_00555_b200 as b2
    g, _ = frontend.compile_source(src)
    out = b2.interpret(g, b2.ExecContext(bindings={"N": 2000, "TSTEPS": 100})
                          .bind_inputs({"A": A, "B": B}))

Graphs may also be given as schema-v1 JSON (pkg/src/sdfgkit/serialize.py).
"""

from .machine import (  # noqa: F401
    Counters, ExecContext, GpuExecutor, InterpOptions, InterpreterError, OutOfBoundsError,
    get_executor, interpret, run_twice_determinism,
)
from .plan import PlanError  # noqa: F401
from .runtime import BackendUnavailable  # noqa: F401
from . import sdfg  # noqa: F401
from . import validate  # noqa: F401  (validate.validate(g): ir.validate restated)
from .dist import ProcessGrid  # noqa: F401
from .distribution import (  # noqa: F401
    distribute, distribute_elementwise, distribution_pipeline, expand_matmul_distributed,
    remove_redundant_comm,
)
from .simrun import CollectiveOrderError, DeadlockError, RankSim, SimError, sim_run  # noqa: F401
from .expansions import (  # noqa: F401
    b200_registry, install as install_expansions, patched_cpu_registry,
)

__all__ = [
    "interpret", "ExecContext", "InterpOptions", "Counters", "InterpreterError",
    "OutOfBoundsError", "GpuExecutor", "get_executor", "PlanError", "BackendUnavailable", "sdfg",
    "run_twice_determinism", "validate", "ProcessGrid", "distribute", "distribute_elementwise",
    "distribution_pipeline", "expand_matmul_distributed", "remove_redundant_comm", "sim_run",
    "RankSim", "DeadlockError", "SimError", "CollectiveOrderError", "b200_registry",
    "install_expansions", "patched_cpu_registry",
]
