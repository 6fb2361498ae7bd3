"""Shared test helpers."""
import numpy as np


def node_rows(pm):
    """Per node, the global point ids of its rows in the product's tree order
    (leaf sets in leaf-id order; an internal node groups its rows by child,
    where the reference keeps one ascending index set, geometry.hpp:38)."""
    ints, _ = pm.nodes()
    perm = pm.perm()
    begin = np.zeros(len(ints), dtype=np.int64)
    pos = 0
    for i in range(len(ints)):
        if ints[i, 2] < 0:
            begin[i] = pos
            pos += ints[i, 3]
    for i in range(len(ints) - 1, -1, -1):
        if ints[i, 2] >= 0:
            begin[i] = begin[ints[i, 2]]
    return lambda nd: perm[begin[nd]: begin[nd] + ints[nd, 3]]
