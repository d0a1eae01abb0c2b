"""Deterministic synthetic inputs shared by the oracle, the golden-fixture
generator and the parity tests (test infrastructure only).

Valid cell (i, j, k, c) of a field over the index "domain" box D gets
``splitmix64(seed ^ lin)`` with ``lin = ((c*E2 + (k-D.lo2))*E1 + (j-D.lo1))*E0
+ (i-D.lo0)`` (E = extents of D), as proposed in SURVEY.md section 8(d) /
BASELINE.md "CPU baseline plan".  float64 values are ``(x >> 11) * 2**-53``;
float32 values are ``(x >> 40) * 2**-24``.  Ghost cells hold a signalling-NaN
poison (0x7FF40000DEADBEEF for float64 as in core/config.py:21 of the
reference; 0x7F80DEAD for float32) so that any copy that goes through
floating-point arithmetic, or touches a cell it should not, is visible when
comparing raw bits.
"""

from __future__ import annotations

import numpy as np

SEED = 20261017
POISON64 = np.uint64(0x7FF40000DEADBEEF)
POISON32 = np.uint32(0x7F80DEAD)

_M1 = np.uint64(0x9E3779B97F4A7C15)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)


def splitmix64(x):
    x = np.asarray(x, np.uint64)
    with np.errstate(over="ignore"):
        z = x + _M1
        z = (z ^ (z >> np.uint64(30))) * _M2
        z = (z ^ (z >> np.uint64(27))) * _M3
    return z ^ (z >> np.uint64(31))


def value_bits(lin, seed, itemsize):
    h = splitmix64(np.uint64(seed) ^ np.asarray(lin, np.uint64))
    if itemsize == 8:
        return (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return ((h >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)).astype(np.float32)


def fill_fab(arr, fab_lo, valid_lo, valid_hi, domain_lo, domain_hi, seed=SEED,
             ghost_tag=None):
    """Fill an F-order (nx, ny, nz, nc) array over a storage box starting at
    ``fab_lo``: hash values on the valid box, poison elsewhere.  All vectors
    are 3-long (padded).  With ``ghost_tag`` (an int, e.g. the fab id) the
    ghost cells get distinct hash values ``splitmix64(seed ^ ~(tag << 40 |
    local_offset))`` instead of poison (used as ParallelCopy sources with
    ``ngrow_src > 0``)."""
    itemsize = arr.dtype.itemsize
    u = arr.view(np.uint64 if itemsize == 8 else np.uint32)
    if ghost_tag is None:
        u[...] = POISON64 if itemsize == 8 else POISON32
    else:
        off = np.arange(arr.size, dtype=np.uint64).reshape(arr.shape, order="F")
        lin = ~((np.uint64(ghost_tag) << np.uint64(40)) | off)
        arr[...] = value_bits(lin, seed, itemsize)
    nx, ny, nz, nc = arr.shape
    E = [int(domain_hi[d]) - int(domain_lo[d]) + 1 for d in range(3)]
    lo = [int(valid_lo[d]) for d in range(3)]
    hi = [int(valid_hi[d]) for d in range(3)]
    i = np.arange(lo[0], hi[0] + 1, dtype=np.int64)
    j = np.arange(lo[1], hi[1] + 1, dtype=np.int64)
    k = np.arange(lo[2], hi[2] + 1, dtype=np.int64)
    c = np.arange(nc, dtype=np.int64)
    lin = ((((c[None, None, None, :] * E[2] + (k[None, None, :, None] - domain_lo[2])) * E[1]
             + (j[None, :, None, None] - domain_lo[1])) * E[0])
           + (i[:, None, None, None] - domain_lo[0]))
    vals = value_bits(lin, seed, itemsize)
    sl = tuple(slice(lo[d] - int(fab_lo[d]), hi[d] - int(fab_lo[d]) + 1) for d in range(3))
    arr[sl] = vals
    return arr


def make_fab(fab_lo, fab_hi, ncomp, dtype, valid_lo, valid_hi, domain_lo, domain_hi,
             seed=SEED, ghost_tag=None):
    shape = tuple(int(fab_hi[d]) - int(fab_lo[d]) + 1 for d in range(3)) + (int(ncomp),)
    arr = np.empty(shape, dtype=dtype, order="F")
    return fill_fab(arr, fab_lo, valid_lo, valid_hi, domain_lo, domain_hi, seed, ghost_tag)


def bits(arr):
    """Raw-bit view for bit-exact comparison (NaN payloads included)."""
    return arr.view(np.uint64 if arr.dtype.itemsize == 8 else np.uint32)
