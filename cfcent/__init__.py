"""Import-name shim: ``import cfcent`` resolves to the B200 package
``paper_1607_02955_b200`` so code (and the reference's own unit tests,
``pkg/tests``) written against the reference package ``cfcent``
(pkg/src/cfcent/__init__.py:1-99) runs unchanged on the device path.

The submodules the reference tests import (``cfcent.solver``,
``cfcent.graph``, ``cfcent.generators``, ``cfcent.resistance``,
``cfcent.centrality``, ``cfcent.errors``) are the product modules
themselves.  Names of the reference that solve no Laplacian system and are
out of scope for this build (shortest-path closeness, the
degree asymptotic, the evaluation/noise experiments, edge-list parsing)
exist so imports succeed, and raise ``NotImplementedError`` when called.
"""

from __future__ import annotations

import sys as _sys

import paper_1607_02955_b200 as _p
from paper_1607_02955_b200 import *  # noqa: F401,F403
from paper_1607_02955_b200 import __all__ as _all
from paper_1607_02955_b200 import (centrality, errors, generators, graph,  # noqa: F401
                                   resistance, solver)

for _m in ("centrality", "errors", "generators", "graph", "resistance", "solver"):
    _sys.modules[f"{__name__}.{_m}"] = getattr(_p, _m)

__version__ = _p.__version__


def _out_of_scope(name: str):
    def f(*args, **kwargs):
        raise NotImplementedError(
            f"cfcent.{name} is outside the B200 hot path (SURVEY.md §2/§8: it solves no "
            "Laplacian system); use the reference package for it")
    f.__name__ = name
    f.__qualname__ = name
    return f


_OUT_OF_SCOPE = ("sp_closeness", "degree_asymptotic", "load_edge_list", "insert_noise_edges",
                 "compare_rankings", "degree_correlation_experiment", "max_relative_error",
                 "noise_resilience", "rank_inversions", "relative_std_dev", "spearman")
for _n in _OUT_OF_SCOPE:
    globals()[_n] = _out_of_scope(_n)


class RankComparison:  # evaluation.py result type (out of scope)
    def __init__(self, *a, **k):
        raise NotImplementedError("cfcent.RankComparison is outside the B200 hot path")


__all__ = list(_all) + list(_OUT_OF_SCOPE) + ["RankComparison"]
