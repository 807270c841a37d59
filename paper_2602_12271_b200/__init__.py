"""B200-native tiled MonarchAttention (MonarchRT, arXiv 2602.12271).

Drop-in for the hot path of the reference package ``monarchbench``:
``solve`` / ``solve_tiled`` / ``attention_output`` with the same layout types,
plus the batched CUDA operator ``monarch_attention`` over (B, H, N, d)
tensors.  All arithmetic runs in the in-tree sm_100a library
``libmonarch_b200.so`` through its C ABI (include/monarch_b200.h).
"""

from .layout import (
    AXES,
    AxisDigit,
    BlockConfig,
    LayoutError,
    LayoutPermutation,
    Lowered,
    TilePlan,
    TokenOrdering,
    VideoShape,
    aligned_config,
    build_permutation,
    config_from_sizes,
    enumerate_aligned_configs,
    flatten_index,
    generalized_ordering,
    lower_chunked,
    lower_square,
    make_tile_plan,
    phi_ordering,
    rho_ordering,
)

__all__ = [
    "AXES", "AxisDigit", "BlockConfig", "LayoutError", "LayoutPermutation", "Lowered", "TilePlan",
    "TokenOrdering", "VideoShape", "aligned_config", "build_permutation", "config_from_sizes",
    "enumerate_aligned_configs", "flatten_index", "generalized_ordering", "lower_chunked",
    "lower_square", "make_tile_plan", "phi_ordering", "rho_ordering",
    "AttentionProblem", "SolverConfig", "SolverError", "SolverTrace", "MonarchFactors",
    "TiledMonarchFactors", "FactorError", "ShapeError", "solve", "solve_tiled",
    "attention_output", "monarch_attention", "monarch_attention_host",
    "load_problem", "save_problem", "TensorFileError", "load_qkv", "FrameKVCache", "Rollout", "rollout_chunks",
    "save_factors", "load_factors", "densify", "densify_tiled", "approx_attention_matrix", "objective",
    "identity_factors", "frobenius_mse",
]


def __getattr__(name):
    # torch-dependent API is imported lazily so the layout mirror stays importable alone
    if name in ("AttentionProblem", "SolverConfig", "SolverTrace", "MonarchFactors",
                "TiledMonarchFactors", "FactorError", "ShapeError", "solve", "solve_tiled",
                "attention_output"):
        from . import solver
        return getattr(solver, name)
    if name in ("SolverError", "monarch_attention", "monarch_attention_host"):
        from . import ops
        return getattr(ops, name)
    if name in ("load_problem", "save_problem", "TensorFileError", "load_qkv", "FrameKVCache", "Rollout",
                "rollout_chunks"):
        from . import rollout
        return getattr(rollout, name)
    if name in ("save_factors", "load_factors", "densify", "densify_tiled", "approx_attention_matrix", "objective",
                "identity_factors", "frobenius_mse"):
        from . import verify
        return getattr(verify, name)
    raise AttributeError(name)
