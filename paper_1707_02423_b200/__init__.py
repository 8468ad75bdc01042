"""B200-native IsoRank CFG-pair similarity (drop-in for sasscfg's ISO path).

Public surface mirrors ``pkg/src/sasscfg/__init__.py:41-54`` for the hot
path: ``isorank_align``, ``isorank_distance``, ``measure_distance``,
``pairwise``, ``minmax_scale``, ``export_heatmap_csv``, the flat measures
(``euclidean``, ``manhattan``, ``minkowski``, ``jaccard``, ``cosine``) plus
the types they use; ``nearest`` and ``isorank_pairs`` are new batched entry
points; ``matrices_from_listings`` / ``load_corpus_matrices`` build the
matrices natively from listings and profiles (``loader.py``).
"""

import importlib

from .errors import (BadK, BadOrder, BadTarget, CorpusError, DegenerateInput, DeviceError, DimMismatch,
                     DuplicateKernel, EmptyGraph, ListingSyntaxError, ProfileSyntaxError, SasscfgError,
                     UnresolvedLabel)

# Names that need libcfgsim.so resolve on first use (PEP 562), so host-only
# modules (synth, packing, workload, errors) import without loading the GPU
# library — the CPU reference arm of bench.py relies on that.  Any product
# call still loads the library and raises ImportError if it is missing.
_LAZY = {
    "matrix": ("GLOBAL", "INTERPOLATED", "RAW_COUNTS", "ROW_STOCHASTIC", "TransitionMatrix", "interpolate_to",
               "normalize_pair"),
    "corpus": ("DeviceCorpus",),
    "packing": ("pack",),
    "loader": ("load_corpus_matrices", "load_manifest", "matrices_from_listings"),
    "similarity": ("AlignmentResult", "MeasureId", "PairwiseMatrix", "cosine", "euclidean", "export_heatmap_csv",
                   "isorank_align", "isorank_distance", "isorank_pairs", "jaccard", "manhattan", "measure_distance",
                   "minkowski", "minmax_scale", "nearest", "pairwise", "pairwise_all"),
}
_WHERE = {name: mod for mod, names in _LAZY.items() for name in names}


def __getattr__(name):
    mod = _WHERE.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    value = getattr(importlib.import_module(f".{mod}", __name__), name)
    globals()[name] = value
    return value


def __dir__():
    return sorted(set(globals()) | set(_WHERE))


__version__ = "0.1.0"

__all__ = [
    "AlignmentResult", "BadK", "BadOrder", "BadTarget", "DegenerateInput", "DeviceCorpus", "DeviceError",
    "DimMismatch", "DuplicateKernel", "EmptyGraph", "GLOBAL", "INTERPOLATED", "MeasureId",
    "PairwiseMatrix", "RAW_COUNTS", "ROW_STOCHASTIC", "SasscfgError", "TransitionMatrix",
    "export_heatmap_csv", "interpolate_to", "isorank_align", "isorank_distance", "isorank_pairs",
    "measure_distance", "minmax_scale", "nearest", "normalize_pair", "pack", "pairwise", "pairwise_all",
    "euclidean", "manhattan", "minkowski", "jaccard", "cosine",
    "CorpusError", "ListingSyntaxError", "ProfileSyntaxError", "UnresolvedLabel",
    "load_corpus_matrices", "load_manifest", "matrices_from_listings",
]
