"""B200-native (sm_100a, fp64) steady-state solver for the spatial hypercube
queueing model with heterogeneous service rates (arXiv 2603.03019).

The product is the C-ABI library ``libhq.so`` (include/hq.h) built from
``csrc/``; ``hq`` is its thin ctypes binding.  Build with
``python -m paper_2603_03019_b200.build``.
"""
from . import hq  # noqa: F401
from .hq import Solver, hq_create, hq_destroy, hq_error_string, hq_measures, hq_solve, hq_stats  # noqa: F401

__all__ = ["hq", "Solver", "hq_create", "hq_solve", "hq_measures", "hq_destroy", "hq_error_string", "hq_stats"]
