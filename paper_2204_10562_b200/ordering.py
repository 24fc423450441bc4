"""Device ordering by recursive minimum cuts (reference ordering.py:23-113).

Both entry points run the deterministic Stoer-Wagner procedure on the GPU
(k_rdo / k_min_cut in csrc/prm.cu): one warp per recursion-tree node, the
cluster's contracted weight matrix in shared memory, warp-shuffle arg-max
with the reference's tie rules (largest adjacency, then smallest GPU id).
"""

from dataclasses import dataclass
from typing import Dict, Optional, Sequence, Tuple

import numpy as np

from . import _device
from .model import ClusterGraph, ValidationError, check_numeric_range, validate_cluster


@dataclass(frozen=True)
class DeviceOrdering:
    """A permutation v_1..v_V of the cluster's GPUs with its rank map."""
    order: Tuple[int, ...]
    rank: Dict[int, int]


def _ordering_packed(cluster: ClusterGraph) -> _device.Packed:
    ids = tuple(sorted(cluster.gpu_ids))
    pos = {g: k for k, g in enumerate(ids)}
    V = len(ids)
    bw = np.zeros((V, V))
    for (a, b), w in cluster.bandwidth.items():
        bw[pos[a], pos[b]] = bw[pos[b], pos[a]] = w
    one = np.ones(1)
    zero = np.zeros(1)
    return _device.Packed(ids, one, one, zero, zero, zero, bw)


def _check(cluster: ClusterGraph) -> None:
    for (a, b), v in cluster.bandwidth.items():
        if not (1e-100 <= v <= 1e100):
            raise ValidationError(f"bandwidth ({a},{b}) = {v!r} outside the supported range [1e-100, 1e100]")


def rdo(cluster: ClusterGraph) -> DeviceOrdering:
    """ordering.py:94-113 on the GPU."""
    _check(cluster)
    packed = _ordering_packed(cluster)
    db = _device.DeviceBatch([(packed, 1, 0, None)], capture_events=False)
    db.run("rdo")
    order = db.d_iin[db.n_ib:].cpu().numpy()
    ids = packed.ids
    out = tuple(ids[int(k)] for k in order[:packed.V])
    return DeviceOrdering(order=out, rank={v: k + 1 for k, v in enumerate(out)})


def global_min_cut(cluster: ClusterGraph, vertices: Optional[Sequence[int]] = None
                   ) -> Tuple[Tuple[int, ...], Tuple[int, ...], float]:
    """ordering.py:30-91 on the GPU: (side_a, side_b, weight), side_a holding the smallest id."""
    verts = sorted(vertices) if vertices is not None else sorted(cluster.gpu_ids)
    if len(verts) < 2:
        raise ValidationError("min cut needs at least 2 vertices")
    known = set(cluster.gpu_ids)
    for v in verts:
        if v not in known:
            raise ValidationError(f"vertex {v} is not a GPU of the cluster")
    _check(cluster)
    packed = _ordering_packed(cluster)
    pos = {g: k for k, g in enumerate(packed.ids)}
    db = _device.DeviceBatch([(packed, 1, 0, None)], capture_events=False)
    in_a, w = db.min_cut(0, [pos[v] for v in verts])
    side_a = tuple(v for v, f in zip(verts, in_a) if f)
    side_b = tuple(v for v, f in zip(verts, in_a) if not f)
    return side_a, side_b, w


__all__ = ["DeviceOrdering", "rdo", "global_min_cut", "validate_cluster", "check_numeric_range"]
