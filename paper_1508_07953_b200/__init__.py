"""B200-native RIANN per-frame ANN-field query (drop-in for the reference
``riann`` package's hot path: process_frame / stream_fields / riann_query).

Hand-written sm_100a CUDA kernels behind a C ABI (include/riann_b200.h),
bound with ctypes.  Results are bit-identical to the reference's numpy
implementation (indices, float64 distances, FrameStats).  There is no CPU
fallback: without the built library or a B200 the compute calls raise.
"""

from ._native import current_device, set_device
from .annf import ANNF_MAGIC, ANNF_VERSION, AnnfStream, AnnfWriter, read_annf, stream_to_annf
from .engine import AnnField, FrameStats, frame_units, grid_shape, init_field, process_frame, stream_fields
from .errors import DimensionError, FormatError, ModelCapacityError, RiannError
from .evaluation import CoherencyStats, coherency_stats, exact_nn, exact_nn_batch, field_exact_oracle
from .model import DEFAULT_REF_CAP, ReferenceModel, compute_sorted_lists
from .patches import (
    EUCLIDEAN,
    EuclideanMetric,
    Metric,
    Patch,
    PatchGrid,
    distance,
    extract_patches,
    get_metric,
    normalize_patch,
    normalize_rows,
    register_metric,
)
from .shards import ShardedTables, shard_model
from .search import QueryResult, SearchParams, query_rng_key, riann_query, riann_query_batch, ring_candidates
from .modelio import MODEL_MAGIC, MODEL_VERSION, deserialize_model, load_model, model_memory_bytes, save_model, serialize_model
from .transforms import EffectTable, apply_effect, reconstruct_frame, reconstruction_error, reconstruction_table

__version__ = "0.1.0"

__all__ = [
    "ANNF_MAGIC",
    "ANNF_VERSION",
    "AnnField",
    "AnnfStream",
    "AnnfWriter",
    "EffectTable",
    "apply_effect",
    "read_annf",
    "reconstruct_frame",
    "reconstruction_error",
    "reconstruction_table",
    "stream_to_annf",
    "CoherencyStats",
    "coherency_stats",
    "MODEL_MAGIC",
    "MODEL_VERSION",
    "deserialize_model",
    "load_model",
    "model_memory_bytes",
    "save_model",
    "serialize_model",
    "DEFAULT_REF_CAP",
    "DimensionError",
    "EUCLIDEAN",
    "EuclideanMetric",
    "FormatError",
    "FrameStats",
    "Metric",
    "ModelCapacityError",
    "Patch",
    "PatchGrid",
    "QueryResult",
    "ReferenceModel",
    "RiannError",
    "SearchParams",
    "compute_sorted_lists",
    "current_device",
    "distance",
    "exact_nn",
    "exact_nn_batch",
    "extract_patches",
    "field_exact_oracle",
    "shard_model",
    "ShardedTables",
    "frame_units",
    "get_metric",
    "grid_shape",
    "init_field",
    "normalize_patch",
    "normalize_rows",
    "process_frame",
    "query_rng_key",
    "register_metric",
    "riann_query",
    "riann_query_batch",
    "ring_candidates",
    "set_device",
    "stream_fields",
    "__version__",
]
