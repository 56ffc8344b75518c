"""On-disk weight / index vectors in the reference's flat binary layout (M/storage.py:29-91).

Layout (unchanged, so files interoperate with ``megores.storage``): an 8-byte little-endian
unsigned element count, then the little-endian payload -- float32 or float64 weights (the
width is recovered from the file size) or int64 indices.

B200 additions: ``load_weights(..., device="cuda")`` reads the payload straight into a pinned
host buffer and uploads it asynchronously, returning a device-resident WeightVector ready for
the resamplers; ``save_indices`` accepts CUDA tensors.  CSV writers mirror M/storage.py:59-99.
"""

from __future__ import annotations

import csv
import os
import struct

import numpy as np

from . import _device as D
from .weights import WeightVector

_COUNT = struct.Struct("<Q")
_WEIGHT_DTYPES = {4: ("<f4", "single"), 8: ("<f8", "double")}


def _payload(path, what: str):
    size = os.path.getsize(path)
    if size < _COUNT.size:
        raise ValueError(f"{path}: truncated {what} file")
    with open(path, "rb") as fh:
        (count,) = _COUNT.unpack(fh.read(_COUNT.size))
    return count, size - _COUNT.size


def _write(path, count: int, data: np.ndarray) -> None:
    with open(path, "wb") as fh:
        fh.write(_COUNT.pack(count))
        data.tofile(fh)


def save_weights(path, w) -> None:
    """Weights of a WeightVector (host or device) in float32/float64 by its precision."""
    values = w.values.detach().cpu().numpy() if D.is_tensor(w.values) else np.asarray(w.values)
    dt = "<f4" if w.precision == "single" else "<f8"
    _write(path, len(values), np.ascontiguousarray(values, dtype=dt))


def load_weights(path, device=None) -> WeightVector:
    """Read a weight file; precision follows the element width.  ``device``: keep on host
    (None) or upload to a CUDA device through a pinned staging buffer."""
    count, body = _payload(path, "weight")
    if count == 0 or body % count:
        raise ValueError(f"{path}: payload of {body} bytes does not fit {count} elements")
    width = body // count
    if width not in _WEIGHT_DTYPES:
        raise ValueError(f"{path}: unsupported element width {width}")
    dt, precision = _WEIGHT_DTYPES[width]
    if device is None:
        return WeightVector(np.fromfile(path, dtype=dt, count=count, offset=_COUNT.size), precision)
    t = D.torch()
    host = t.empty(count, dtype=t.float32 if width == 4 else t.float64).pin_memory()
    with open(path, "rb") as fh:
        fh.seek(_COUNT.size)
        fh.readinto(memoryview(host.numpy()).cast("B"))
    return WeightVector(host.to(device, non_blocking=True), precision)


def save_indices(path, indices) -> None:
    """int64 index vector (ancestors, offspring counts); numpy or CUDA tensor."""
    if D.is_tensor(indices):
        indices = indices.detach().cpu().numpy()
    _write(path, len(indices), np.ascontiguousarray(indices, dtype="<i8"))


def load_indices(path) -> np.ndarray:
    count, body = _payload(path, "index")
    if body != 8 * count:
        raise ValueError(f"{path}: payload does not match header length {count}")
    return np.fromfile(path, dtype="<i8", count=count, offset=_COUNT.size).astype(np.int64)


def save_weights_csv(path, w) -> None:
    values = w.values.detach().cpu().numpy() if D.is_tensor(w.values) else np.asarray(w.values)
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(("index", "weight"))
        out.writerows((k, repr(float(v))) for k, v in enumerate(values))


def save_indices_csv(path, indices, column="value") -> None:
    if D.is_tensor(indices):
        indices = indices.detach().cpu().numpy()
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow((column,))
        out.writerows((int(v),) for v in indices)


def save_trajectory_csv(path, truth, observations) -> None:
    truth = np.asarray(truth, dtype=np.float64)
    observations = np.asarray(observations, dtype=np.float64)
    if truth.shape != observations.shape:
        raise ValueError("truth and observations must have equal length")
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(("t", "truth", "observation"))
        out.writerows((k + 1, repr(float(x)), repr(float(z))) for k, (x, z) in enumerate(zip(truth, observations)))
