"""B200-native F2M (fractional 2-matching) GDP solver — arXiv:2011.08170, rebuilt for sm_100a.

Drop-in for the reference's Python package `f2m` (/root/reference/proj/python/f2m): the same
names, keyword arguments, defaults and exception types, backed by hand-written sm_100a CUDA
kernels behind the C ABI in include/f2m_gpu.h (libf2m_gpu.so). There is no CPU fallback:
importing fails loudly if the extension is not built, and compute calls raise DeviceError
without a CUDA device.

    import paper_2011_08170_b200 as f2m
    inst = f2m.generate_instance(100000, seed=1)
    result = f2m.full_solve(inst, k=10)
"""
import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))

try:
    from . import _f2m  # noqa: F401  (loads libf2m.so and libf2m_gpu.so from this directory)
except ImportError as _e:  # pragma: no cover - exercised only on a broken build
    raise ImportError(
        "paper_2011_08170_b200: native extension not built (run `python -c 'import __graft_entry__ as g; g.build()'` "
        f"or `make -C {_HERE}`): {_e}") from _e

from ._f2m import (  # noqa: E402
    DegenerateExtraction,
    DeviceError,
    DistanceMode,
    DualState,
    Graph,
    Infeasible,
    Instance,
    ParseError,
    PrimalSolution,
    SolveFailed,
    TooLarge,
    adjusted_length,
    brute_force_f2m,
    build_knn_graph,
    classify_edges,
    device_info,
    dual_objective,
    extract_primal,
    full_solve,
    full_solve_arrays,
    full_solve_device,
    full_solve_graph,
    gauss_seidel_sweep,
    generate_clustered_instance,
    generate_instance,
    graph_from_edges,
    jacobi_sweep,
    jacobi_sweeps,
    kernel_launch_count,
    last_sweep_kernel,
    last_sweep_kernel_desc,
    load_tsplib,
    make_initial_state,
    node_update_delta,
    parse_tsplib,
    serialize_tsplib,
    set_device,
    solve_duals,
    solve_zero_component,
    validate_graph,
    verify_solution,
    write_lp,
    write_solution,
)

# The reference package's public names (python/f2m/__init__.py) come first.
__all__ = [
    "DegenerateExtraction", "DistanceMode", "DualState", "Graph", "Infeasible", "Instance",
    "ParseError", "PrimalSolution", "SolveFailed", "TooLarge", "adjusted_length",
    "brute_force_f2m", "build_knn_graph", "dual_objective", "extract_primal", "full_solve",
    "generate_instance", "load_tsplib", "node_update_delta", "parse_tsplib", "serialize_tsplib",
    "solve_duals", "validate_graph", "verify_solution", "write_lp",
    # B200 extensions
    "DeviceError", "classify_edges", "device_info", "full_solve_arrays", "full_solve_device",
    "full_solve_graph", "gauss_seidel_sweep", "generate_clustered_instance", "graph_from_edges",
    "jacobi_sweep", "jacobi_sweeps", "kernel_launch_count", "last_sweep_kernel", "last_sweep_kernel_desc",
    "make_initial_state", "set_device", "solve_zero_component", "write_solution",
]

__version__ = "0.1.0"

NATIVE_LIBRARIES = tuple(_os.path.join(_HERE, n) for n in ("libf2m_gpu.so", "libf2m.so"))
