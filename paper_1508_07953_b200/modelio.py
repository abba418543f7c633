"""RIAN model container (reference model.py:398-461).

    "RIAN" | <HIHHBB version, n, patch_w, patch_h, channels, metric_id
    refs (n, dim) <f4 | sorted_dist (n, n) <f4 | sorted_idx (n, n) <u4

Bytes are identical to the reference's serialize_model (tests/golden).  For a
model whose sorted tables were built on the GPU (K3), ``save_model`` streams
them to the file in row chunks straight from HBM (34 GB at n = 65,536 never
has to exist in host memory as float64, unlike the reference), and
``load_model`` maps the file: the tables are uploaded from the page cache the
first time the model is made resident, with no table rebuild.
"""

from __future__ import annotations

import struct

import numpy as np

from .errors import FormatError
from .model import ReferenceModel

MODEL_MAGIC = b"RIAN"
MODEL_VERSION = 1
_HEADER = "<HIHHBB"  # version, n, patch_w, patch_h, channels, metric_id
_HEADER_LEN = 4 + struct.calcsize(_HEADER)


def model_memory_bytes(n: int, dim: int) -> int:
    """Serialized footprint of a model of the given size (model.py:459-461)."""
    return 4 * (n * dim + 2 * n * n)


def _header(model) -> bytes:
    pw, ph = model.patch_size
    return MODEL_MAGIC + struct.pack(_HEADER, MODEL_VERSION, model.n, int(pw), int(ph), int(model.channels),
                                     int(model.metric_id))


def _chunks(model, rows_per_chunk):
    """(float32 dist rows, int32 idx rows) chunks of the sorted tables: host
    tables when the model has them, else downloaded from the GPU."""
    n = model.n
    own = isinstance(model, ReferenceModel)
    host = (not own) or model.has_host_tables
    for r0 in range(0, n, rows_per_chunk):
        r1 = min(n, r0 + rows_per_chunk)
        if host:
            yield np.asarray(model.sorted_dist[r0:r1]), np.asarray(model.sorted_idx[r0:r1])
        else:
            yield model.table_rows(r0, r1 - r0)


def _write(model, fh, rows_per_chunk=None) -> None:
    n = model.n
    rows_per_chunk = rows_per_chunk or max(1, (256 << 20) // max(1, 8 * n))
    fh.write(_header(model))
    fh.write(np.ascontiguousarray(model.refs, dtype="<f4").tobytes())
    # sorted_dist block, then sorted_idx block (two passes over the rows)
    for sd, _ in _chunks(model, rows_per_chunk):
        fh.write(np.ascontiguousarray(sd, dtype="<f4").tobytes())
    for _, si in _chunks(model, rows_per_chunk):
        fh.write(np.ascontiguousarray(si, dtype="<u4").tobytes())


def serialize_model(model) -> bytes:
    """Encode a model in the RIAN container (model.py:398-411)."""
    import io

    buf = io.BytesIO()
    _write(model, buf)
    return buf.getvalue()


def _parse_header(data) -> tuple:
    if len(data) < _HEADER_LEN:
        raise FormatError("model file truncated inside the header")
    if bytes(data[:4]) != MODEL_MAGIC:
        raise FormatError(f"bad magic {bytes(data[:4])!r}, expected {MODEL_MAGIC!r}")
    version, n, pw, ph, channels, metric_id = struct.unpack(_HEADER, bytes(data[4:_HEADER_LEN]))
    if version != MODEL_VERSION:
        raise FormatError(f"unsupported model version {version}")
    return n, pw, ph, channels, metric_id


def _check_length(total, n, dim):
    expected = _HEADER_LEN + 4 * (n * dim + 2 * n * n)
    if total != expected:
        raise FormatError(f"model payload length {total} does not match header "
                          f"(n={n}, dim={dim} requires {expected} bytes)")


def deserialize_model(data: bytes) -> ReferenceModel:
    """Decode a RIAN container (model.py:414-446): refs float32, sorted_dist
    float64 (float32-exact values), sorted_idx int32, as the reference returns."""
    n, pw, ph, channels, metric_id = _parse_header(data)
    dim = pw * ph * channels
    _check_length(len(data), n, dim)
    off = _HEADER_LEN
    refs = np.frombuffer(data, dtype="<f4", count=n * dim, offset=off).reshape(n, dim)
    off += 4 * n * dim
    dist = np.frombuffer(data, dtype="<f4", count=n * n, offset=off).reshape(n, n)
    off += 4 * n * n
    idx = np.frombuffer(data, dtype="<u4", count=n * n, offset=off).reshape(n, n)
    return ReferenceModel(refs.astype(np.float32), dist.astype(np.float64), idx.astype(np.int32), (pw, ph),
                          channels=channels, metric_id=metric_id)


def save_model(path, model) -> None:
    """Write a model (GPU-built tables stream from HBM in row chunks)."""
    with open(path, "wb") as fh:
        _write(model, fh)


def load_model(path) -> ReferenceModel:
    """Map a RIAN file: refs are read, the tables stay memory-mapped (float32
    distances, uint32 indices viewed as int32) until the model is uploaded."""
    with open(path, "rb") as fh:
        head = fh.read(_HEADER_LEN)
        fh.seek(0, 2)
        total = fh.tell()
    n, pw, ph, channels, metric_id = _parse_header(head)
    dim = pw * ph * channels
    _check_length(total, n, dim)
    off = _HEADER_LEN
    refs = np.array(np.memmap(path, dtype="<f4", mode="r", offset=off, shape=(n, dim)), dtype=np.float32)
    off += 4 * n * dim
    dist = np.memmap(path, dtype="<f4", mode="r", offset=off, shape=(n, n))
    off += 4 * n * n
    idx = np.memmap(path, dtype="<i4", mode="r", offset=off, shape=(n, n))  # indices < 2^31: same bits
    return ReferenceModel(refs, dist, idx, (pw, ph), channels=channels, metric_id=metric_id)
