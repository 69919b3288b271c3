"""B200-native temporal multilinear sieve (arXiv 2001.07158 hot path).

Python mirror of the reference's tsieve C++ API for the temporal-sieve path;
all compute runs in libtsv.so (hand-written sm_100a CUDA) through the C-ABI
in include/tsv.h.  The C++ drop-in (same headers as the reference) and the
``tsieve`` CLI live under ``cpp/``.
"""
from .graph import (LoadResult, MotifQuery, TemporalGraph, VertexColoring,  # noqa: F401
                    load_graph, restrict_to, save_colors, save_graph)
from .sieve import (EDGE_MODELS, AnchorSpec, DeviceShades, SieveConfig,  # noqa: F401
                    SieveOutcome, ShadeAssignment, build_shades, eval_points_device, eval_temporal_sieve,
                    false_negative_bound, finalize, xor_combine_device)

__all__ = [
    "TemporalGraph", "VertexColoring", "MotifQuery", "LoadResult", "load_graph", "restrict_to",
    "save_graph", "save_colors", "SieveConfig", "ShadeAssignment", "AnchorSpec", "SieveOutcome",
    "build_shades", "eval_temporal_sieve", "false_negative_bound", "DeviceShades",
    "eval_points_device", "xor_combine_device", "finalize", "EDGE_MODELS",
]
