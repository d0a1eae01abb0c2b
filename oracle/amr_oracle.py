"""CPU ORACLE (test infrastructure only) for the coarse/fine level transfers.

Only ``tests/`` may import it; the product (``paper_2403_12179_b200.amr``)
never does.  numpy restatement of the reference's arithmetic in
``/root/reference/pkg/src/miniamr_core/amr.py``:

* ``interp``        <- ``interp_box``         amr.py:269-314
* ``restrict``      <- ``avg_one`` in ``average_down``  amr.py:251-264
* ``fill_targets``  <- ``_same_level_sources`` + ``_coarse_fill_targets``
                       amr.py:322-352 (box algebra from ghost_oracle)

Parity pinning: ``tests/golden/make_golden_amr.py`` runs the reference
itself (interp_box, average_down, fill_patch) and stores the raw bits of
every fab; ``tests/test_amr_oracle.py`` checks this module against those
fixtures (the interp / restriction cases bit for bit).

Arrays are F-order ``(nx, ny, nz, ncomp)`` over a storage box given as a
padded 6-vector ``[lo0 lo1 lo2 hi0 hi1 hi2]``; ``ratio`` is a 3-vector (1 on
axes >= spacedim).
"""

from __future__ import annotations

import itertools

import numpy as np

from . import ghost_oracle as go


def interp(crse, crse_box, fine, fine_box, region, ratio, linear, spacedim):
    """fine[region] <- interpolation of crse (amr.py:292-314), in place."""
    rlo, rhi = region[:3], region[3:]
    clo, flo = crse_box[:3], fine_box[:3]
    fidx = [np.arange(rlo[d], rhi[d] + 1, dtype=np.int64) for d in range(3)]
    parent = [fi // r for fi, r in zip(fidx, ratio)]
    ploc = [p - c for p, c in zip(parent, clo)]
    nc = crse.shape[3]
    vals = crse[np.ix_(*ploc, np.arange(nc))]
    if linear:
        vals = vals.copy()
        for d in range(spacedim):
            up = list(ploc)
            dn = list(ploc)
            up[d] = ploc[d] + 1
            dn[d] = ploc[d] - 1
            slope = 0.5 * (crse[np.ix_(*up, np.arange(nc))] - crse[np.ix_(*dn, np.arange(nc))])
            off = (np.mod(fidx[d], ratio[d]) + 0.5) / ratio[d] - 0.5
            shape = [1, 1, 1, 1]
            shape[d] = off.size
            vals += slope * off.reshape(shape)
    dst = tuple(slice(rlo[d] - flo[d], rhi[d] - flo[d] + 1) for d in range(3))
    fine[dst] = vals


def restrict(fine, fine_box, valid_box, ratio, spacedim):
    """Mean of the ratio^D children of every coarse cell under valid_box
    (amr.py:251-264); returns the coarse array over coarsen(valid_box)."""
    sl = tuple(slice(valid_box[d] - fine_box[d], valid_box[3 + d] - fine_box[d] + 1) for d in range(3))
    fdat = fine[sl]
    acc = None
    for oz in range(ratio[2]):
        for oy in range(ratio[1]):
            for ox in range(ratio[0]):
                part = fdat[ox::ratio[0], oy::ratio[1], oz::ratio[2]]
                acc = part.copy() if acc is None else acc + part
    rpow = int(np.prod(ratio[:spacedim]))
    return acc / rpow


def _grow(b, g):
    b = np.asarray(b, np.int64).copy()
    b[:3] -= g
    b[3:] += g
    return b


def _meet(a, b):
    return np.concatenate([np.maximum(a[:3], b[:3]), np.minimum(a[3:], b[3:])])


def _shift(b, s):
    s = np.asarray(s, np.int64)
    return np.concatenate([b[:3] + s, b[3:] + s])


def fill_targets(fine_boxes, ngrow, domain, periodic, spacedim):
    """Per fine fab, the ghost boxes with no same-level source
    (amr.py:322-352).  Boxes padded to 3 axes; returns {fab: [box, ...]}."""
    period = [int(domain[3 + d] - domain[d] + 1) for d in range(3)]
    reach = max(period[:spacedim])
    big = _grow(domain, np.array([reach if d < spacedim else 0 for d in range(3)]))
    sources = []
    for b in fine_boxes:
        b = np.asarray(b, np.int64)
        sources.append(b)
        per_axis = []
        for d in range(spacedim):  # comm.py:250-266 against the grown domain
            if not periodic[d]:
                per_axis.append([0])
                continue
            kmin = -((b[3 + d] - big[d]) // period[d])
            kmax = (big[3 + d] - b[d]) // period[d]
            per_axis.append([k * period[d] for k in range(kmin, kmax + 1)])
        for sv in itertools.product(*per_axis):
            if any(v != 0 for v in sv):
                sources.append(_shift(b, list(sv) + [0] * (3 - spacedim)))
    bigc = max(period[:spacedim]) + max(ngrow[:spacedim]) + 1
    clip = np.asarray(domain, np.int64).copy()
    for d in range(spacedim):
        if periodic[d]:
            clip[d] -= bigc
            clip[3 + d] += bigc
    out = {}
    g = np.asarray([ngrow[d] if d < spacedim else 0 for d in range(3)], np.int64)
    for gi, b in enumerate(fine_boxes):
        b = np.asarray(b, np.int64)
        rest = go.box_diff(_grow(b, g), b)
        for s in sources:
            nxt = []
            for r in rest:
                nxt.extend(go.box_diff(r, s))
            rest = nxt
        rest = [_meet(r, clip) for r in rest]
        rest = [r for r in rest if np.all(r[3:] >= r[:3])]
        if rest:
            out[gi] = rest
    return out


def advance(u, u_box, valid_box, coef, spacedim):
    """heat.py:172-189 on valid_box, component 0: returns the new values
    (F-order (nx, ny, nz)) in numpy's operation order."""
    lo = [int(valid_box[d] - u_box[d]) for d in range(3)]
    hi = [int(valid_box[3 + d] - u_box[d]) + 1 for d in range(3)]

    def at(dx, dy, dz):
        return u[lo[0] + dx:hi[0] + dx, lo[1] + dy:hi[1] + dy, lo[2] + dz:hi[2] + dz, 0]

    acc = at(0, 0, 0).copy()
    one = u.dtype.type(coef[0]) if u.dtype == np.float32 else coef[0]
    if spacedim >= 1:
        acc += one * (at(1, 0, 0) - 2.0 * at(0, 0, 0) + at(-1, 0, 0))
    if spacedim >= 2:
        c = u.dtype.type(coef[1]) if u.dtype == np.float32 else coef[1]
        acc += c * (at(0, 1, 0) - 2.0 * at(0, 0, 0) + at(0, -1, 0))
    if spacedim >= 3:
        c = u.dtype.type(coef[2]) if u.dtype == np.float32 else coef[2]
        acc += c * (at(0, 0, 1) - 2.0 * at(0, 0, 0) + at(0, 0, -1))
    return acc
