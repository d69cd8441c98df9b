"""B200-native search-step engine for Chameleon / ReLeASE (arXiv 1905.12799).

Drop-in replacement for the data-parallel search step of the reference
``knobtuner`` package: the module-level functions its driver imports by name
(driver.py:12-23) — ``predict``, ``run_sa_round``, ``adaptive_sample`` (and
their helpers) — with identical signatures and results, running on
hand-written sm_100a kernels in ``lib/libknobtuner_b200.so`` (C ABI:
``include/knobtuner_b200.h``).  There is no CPU fallback: without the library
or a CUDA device every engine call raises ``EngineUnavailable``.

``install()`` rebinds those names inside an importable reference package so
its unchanged driver and CLI run on the B200.
"""

from . import errors, report, tune
from ._lib import EngineUnavailable, engine
from .agent import Agent, AgentHyperparams, init_agent, run_search_round, run_search_rows
from .cost_model import BoostParams, CostModel, Tree, device_forest, fit, predict, predict_rows
from .landscape import SyntheticBackend, SyntheticLandscape, batch_runtimes, best_runtime, runtimes_rows, synthetic_runtime, true_fitness
from .sa import SAParams, run_sa_round, run_sa_rows
from .sampler import (
    KNEE_CONSTANT,
    ClusteringResult,
    VisitedSet,
    adaptive_sample,
    adaptive_sample_rows,
    kmeans,
    knee_scan,
    mode_config,
    round_to_config,
)
from .space import Configuration, DesignSpace, KnobDef, grid, pack, space_from_dict, unpack
from .trajectory import Trajectory

__version__ = "0.1.0"

__all__ = [
    "Agent", "AgentHyperparams", "init_agent", "run_search_round", "run_search_rows",
    "ClusteringResult", "Configuration", "CostModel", "DesignSpace", "EngineUnavailable", "KNEE_CONSTANT", "KnobDef",
    "BoostParams", "SAParams", "SyntheticBackend", "SyntheticLandscape", "Trajectory", "Tree", "VisitedSet", "adaptive_sample",
    "adaptive_sample_rows", "batch_runtimes", "best_runtime", "device_forest", "engine", "errors", "fit", "grid", "install",
    "kmeans", "knee_scan", "mode_config", "pack", "predict", "predict_rows", "round_to_config", "run_sa_round",
    "run_sa_rows", "runtimes_rows", "space_from_dict", "synthetic_runtime", "true_fitness", "unpack",
]


def install() -> dict:
    """Route an importable reference ``knobtuner`` through this engine.

    Rebinds the names the reference's driver/agent/sa modules imported at load
    time (driver.py:12-23, agent.py:22, sa.py:21) and adopts its exception
    classes.  Returns the replaced originals so callers can restore them.
    """
    import importlib

    kt = importlib.import_module("knobtuner")
    mods = {name: importlib.import_module(f"knobtuner.{name}") for name in
            ("driver", "agent", "sa", "sampler", "cost_model", "backends", "errors", "report")}
    errors.adopt(mods["errors"])
    patches = [
        (mods["driver"], "predict", predict), (mods["driver"], "run_sa_round", run_sa_round),
        (mods["driver"], "fit", fit), (mods["driver"], "_top_unvisited", tune.top_unvisited),
        (mods["report"], "per_step_best", report.per_step_best),
        (mods["report"], "convergence_steps_for_round", report.convergence_steps_for_round),
        (mods["report"], "pca_project", report.pca_project),
        (mods["driver"], "adaptive_sample", adaptive_sample), (mods["driver"], "run_search_round", run_search_round),
        (mods["agent"], "predict", predict),
        (mods["sa"], "predict", predict), (kt, "predict", predict), (kt, "run_sa_round", run_sa_round),
        (kt, "adaptive_sample", adaptive_sample), (kt, "run_search_round", run_search_round),
    ]
    saved = {}
    for mod, name, fn in patches:
        saved[(mod.__name__, name)] = getattr(mod, name)
        setattr(mod, name, fn)
    return saved
