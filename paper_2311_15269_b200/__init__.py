"""B200-native rebuild of Tessel's schedule-search hot path (arXiv 2311.15269).

Drop-in for the reference package ``repsched``'s search API
(placement -> repetend construction -> completion): the module names mirror
the reference (placement, schedule, repetend, solver, completion, _core) and
every decide probe and candidate evaluation runs on sm_100a kernels through
the C ABI in include/tessel_b200.h.  There is no CPU fallback.
"""

__version__ = "0.1.0"

from . import placement, schedule  # noqa: F401  (pure data model, importable without a GPU)


def __getattr__(name):
    # compute modules load the native library lazily
    if name in ("repetend", "solver", "completion", "engine", "_core", "_native", "workloads",
                "parallel", "to_search", "extension", "validate", "emitter", "simulator"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
