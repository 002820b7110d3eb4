"""B200-native HALLaR (cuHALLaR, arXiv 2505.13719) behind the lrsdp API.

The solver lives in ``libcuhallar.so`` (C-ABI, include/cuhallar.h): a
persistent cooperative sm_100a kernel runs the whole augmented-Lagrangian /
HLR / ADAP-AIPP / ADAP-FISTA / Lanczos solve on device.  This package is the
thin host-side mirror of the reference operator/solver interface.
"""
from .api import (  # noqa: F401
    CapacityError, CudaError, GaussPrSpec, Graph, InputError, McSpec, NumericalError, PrSpec, SdpInstance, SolveReport,
    SolverConfig, TraceEvent, build_theta_instance, gen_gauss_phase_retrieval, gen_matrix_completion, gen_phase_retrieval,
    graph_from_edges, load_graph, make_cycle, make_hypercube, make_petersen,
    matcomp_constraint_count, matcomp_from_samples, shard_export, solve, solve_rank, solve_sharded, version,
    LIB_PATH,
)
