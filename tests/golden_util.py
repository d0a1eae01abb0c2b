"""Loading helpers for the reference-generated fixtures in tests/golden/."""

from __future__ import annotations

import functools
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=1)
def cases():
    with open(os.path.join(GOLDEN, "golden_cases.json")) as f:
        return json.load(f)["cases"]


@functools.lru_cache(maxsize=1)
def data():
    return dict(np.load(os.path.join(GOLDEN, "golden_data.npz")))


def case(name):
    for c in cases():
        if c["name"] == name:
            return c
    raise KeyError(name)


def names(kind, store=None):
    return [c["name"] for c in cases() if c["kind"] == kind
            and (store is None or c.get("store") == store)]


def grown(box6, g):
    b = np.asarray(box6, np.int64).copy()
    b[:3] -= np.asarray(g, np.int64)
    b[3:] += np.asarray(g, np.int64)
    return b


def seg_digest(rows13):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(rows13, np.int64)).astype("<i8").tobytes()).hexdigest()


def fab_digest(bits_arr):
    return hashlib.sha256(np.ascontiguousarray(bits_arr.ravel(order="F")).tobytes()).hexdigest()


def stats_dict(arr):
    """golden stats rows [src, dst, messages, bytes] -> {(s, d): (m, b)}."""
    return {(int(r[0]), int(r[1])): (int(r[2]), int(r[3])) for r in np.asarray(arr).reshape(-1, 4)}


def scale_boxes(n, b):
    out = []
    for z in range(0, n, b):
        for y in range(0, n, b):
            for x in range(0, n, b):
                out.append([x, y, z, x + b - 1, y + b - 1, z + b - 1])
    return np.asarray(out, np.int64)
