"""B200-native IsoRank CFG-pair similarity (drop-in for sasscfg's ISO path).

Public surface mirrors ``pkg/src/sasscfg/__init__.py:41-54`` for the hot
path: ``isorank_align``, ``isorank_distance``, ``measure_distance``,
``pairwise``, ``minmax_scale``, ``export_heatmap_csv``, the flat measures
(``euclidean``, ``manhattan``, ``minkowski``, ``jaccard``, ``cosine``) plus
the types they use; ``nearest`` and ``isorank_pairs`` are new batched entry
points; ``matrices_from_listings`` / ``load_corpus_matrices`` build the
matrices natively from listings and profiles (``loader.py``).
"""

from .errors import (BadOrder, BadTarget, CorpusError, DegenerateInput, DeviceError, DimMismatch,
                     DuplicateKernel, EmptyGraph, ListingSyntaxError, ProfileSyntaxError, SasscfgError,
                     UnresolvedLabel)
from .matrix import (GLOBAL, INTERPOLATED, RAW_COUNTS, ROW_STOCHASTIC, TransitionMatrix, interpolate_to,
                     normalize_pair)
from .corpus import DeviceCorpus, pack
from .loader import load_corpus_matrices, load_manifest, matrices_from_listings
from .similarity import (AlignmentResult, MeasureId, PairwiseMatrix, cosine, euclidean, export_heatmap_csv,
                         isorank_align, isorank_distance, isorank_pairs, jaccard, manhattan, measure_distance,
                         minkowski, minmax_scale, nearest, pairwise)

__version__ = "0.1.0"

__all__ = [
    "AlignmentResult", "BadOrder", "BadTarget", "DegenerateInput", "DeviceCorpus", "DeviceError",
    "DimMismatch", "DuplicateKernel", "EmptyGraph", "GLOBAL", "INTERPOLATED", "MeasureId",
    "PairwiseMatrix", "RAW_COUNTS", "ROW_STOCHASTIC", "SasscfgError", "TransitionMatrix",
    "export_heatmap_csv", "interpolate_to", "isorank_align", "isorank_distance", "isorank_pairs",
    "measure_distance", "minmax_scale", "nearest", "normalize_pair", "pack", "pairwise",
    "euclidean", "manhattan", "minkowski", "jaccard", "cosine",
    "CorpusError", "ListingSyntaxError", "ProfileSyntaxError", "UnresolvedLabel",
    "load_corpus_matrices", "load_manifest", "matrices_from_listings",
]
