"""The coarse/fine oracle (oracle/amr_oracle.py) against fixtures produced by
running the reference's interp_box / average_down / fill_patch
(tests/golden/make_golden_amr.py): bit-exact, CPU only."""

from __future__ import annotations

import functools
import json
import os

import numpy as np
import pytest

from oracle import amr_oracle as ao
from oracle import ghost_oracle as go
from oracle import inputs

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=1)
def meta():
    with open(os.path.join(GOLDEN, "golden_amr.json")) as f:
        return json.load(f)


@functools.lru_cache(maxsize=1)
def data():
    return dict(np.load(os.path.join(GOLDEN, "golden_amr.npz")))


def cases(kind):
    return [c for c in meta()["cases"] if c["kind"] == kind]


def names(kind):
    return [c["name"] for c in cases(kind)]


def case(name):
    return next(c for c in meta()["cases"] if c["name"] == name)


def grown(b, g):
    b = np.asarray(b, np.int64).copy()
    b[:3] -= np.asarray(g, np.int64)
    b[3:] += np.asarray(g, np.int64)
    return b


def g3(v, dim):
    return [v if d < dim else 0 for d in range(3)]


def r3(r, dim):
    return [r if d < dim else 1 for d in range(3)]


def poisoned(box, nc, dtype):
    shape = tuple(int(box[3 + d] - box[d] + 1) for d in range(3)) + (nc,)
    a = np.empty(shape, dtype=dtype, order="F")
    inputs.bits(a)[...] = inputs.POISON64 if a.dtype.itemsize == 8 else inputs.POISON32
    return a


def hashed(box, valid, domain, nc, dtype, seed):
    return inputs.make_fab(box[:3], box[3:], nc, dtype, valid[:3], valid[3:], domain[:3], domain[3:], seed)


# ------------------------------------------------------------------ interp

def interp_inputs(c):
    dt = np.dtype(c["dtype"])
    cb = np.asarray(c["crse_box"], np.int64)
    crse = hashed(cb, cb, cb, c["ncomp"], dt, c["seed"])
    fine = poisoned(c["fine_box"], c["ncomp"], dt)
    return crse, fine


@pytest.mark.parametrize("name", names("interp"))
def test_interp_oracle_matches_reference(name):
    c = case(name)
    crse, fine = interp_inputs(c)
    ao.interp(crse, np.asarray(c["crse_box"]), fine, np.asarray(c["fine_box"]), np.asarray(c["region"]),
              r3(c["ratio"], c["dim"]), c["scheme"] == "linear", c["dim"])
    assert np.array_equal(inputs.bits(fine), data()[f"{name}/fine"])


# ------------------------------------------------------------ average_down

def avgdown_expected(c):
    dim, dt, nc, r = c["dim"], np.dtype(c["dtype"]), c["ncomp"], c["ratio"]
    cdom = np.asarray([0, 0, 0] + [e - 1 for e in c["cext"]], np.int64)
    fdom = np.asarray([0, 0, 0] + [(e * rr) - 1 for e, rr in zip(c["cext"], r3(r, dim))], np.int64)
    crse = {gi: hashed(grown(b, g3(c["cngrow"], dim)), np.asarray(b), cdom, nc, dt, meta()["seed_crse"])
            for gi, b in enumerate(c["crse_boxes"])}
    tmp_boxes, tmp = [], {}
    for gi, b in enumerate(c["fine_boxes"]):
        fb = grown(b, g3(c["fngrow"], dim))
        fine = hashed(fb, np.asarray(b), fdom, nc, dt, meta()["seed_fine"])
        tb = np.asarray(b, np.int64).copy()
        tb[:3] //= np.asarray(r3(r, dim))
        tb[3:] //= np.asarray(r3(r, dim))
        tmp_boxes.append(tb)
        tmp[gi] = ao.restrict(fine, fb, np.asarray(b), r3(r, dim), dim)
    # ParallelCopy tmp -> coarse (no geometry), the reference's rank order
    plan = go.plan_parallel_copy(c["crse_boxes"], tmp_boxes, [0] * 3, [0] * 3, None, None,
                                 c["fine_rank"], c["crse_rank"], c["nranks"])
    clo = {gi: grown(b, g3(c["cngrow"], dim))[:3] for gi, b in enumerate(c["crse_boxes"])}
    tlo = {gi: b[:3] for gi, b in enumerate(tmp_boxes)}
    go.execute(plan, tmp, tlo, crse, clo, 0, 0, nc)
    return crse


@pytest.mark.parametrize("name", names("average_down"))
def test_average_down_oracle_matches_reference(name):
    c = case(name)
    crse = avgdown_expected(c)
    for gi, a in crse.items():
        assert np.array_equal(inputs.bits(a), data()[f"{name}/crse{gi}"]), f"coarse fab {gi}"


# -------------------------------------------------------------- fill_patch

def fill_patch_expected(c):
    dim, dt, nc, r = c["dim"], np.dtype(c["dtype"]), c["ncomp"], c["ratio"]
    rr = r3(r, dim)
    per = [bool(p) for p in c["periodic"]]
    cdom = np.asarray([0, 0, 0] + [e - 1 for e in c["cext"]], np.int64)
    fdom = np.asarray([0, 0, 0] + [e * q - 1 for e, q in zip(c["cext"], rr)], np.int64)
    ng = g3(c["fngrow"], dim)
    fboxes = [np.asarray(b, np.int64) for b in c["fine_boxes"]]
    fine = {gi: hashed(grown(b, ng), b, fdom, nc, dt, meta()["seed_fine"]) for gi, b in enumerate(fboxes)}
    flo = {gi: grown(b, ng)[:3] for gi, b in enumerate(fboxes)}
    fperiod = [int(fdom[3 + d] + 1) for d in range(3)]
    cperiod = [int(cdom[3 + d] + 1) for d in range(3)]
    for _ in range(2):  # the generator calls fill_patch twice
        plan = go.plan_fill_boundary(fboxes, ng, per, fperiod, c["fine_rank"], c["nranks"])
        go.execute(plan, fine, flo, fine, flo, 0, 0, nc)
        targets = ao.fill_targets(fboxes, ng, fdom, per, dim)
        if not targets:
            continue
        reach = 1 if c["scheme"] == "linear" else 0
        cboxes = {}
        for gi in sorted(targets):
            b = grown(fboxes[gi], ng)
            b[:3] //= np.asarray(rr)
            b[3:] //= np.asarray(rr)
            cboxes[gi] = grown(b, g3(reach, dim))
        crse = {gi: hashed(np.asarray(b), np.asarray(b), cdom, nc, dt, meta()["seed_crse"])
                for gi, b in enumerate(c["crse_boxes"])}
        order = sorted(targets)
        gplan = go.plan_parallel_copy([cboxes[g] for g in order], c["crse_boxes"], [0] * 3, [0] * 3, per,
                                      cperiod, c["crse_rank"], [c["fine_rank"][g] for g in order], c["nranks"])
        gath = {p: poisoned(cboxes[g], nc, dt) for p, g in enumerate(order)}
        glo = {p: cboxes[g][:3] for p, g in enumerate(order)}
        go.execute(gplan, crse, {gi: np.asarray(b)[:3] for gi, b in enumerate(c["crse_boxes"])}, gath, glo,
                   0, 0, nc)
        for p, gi in enumerate(order):
            for region in targets[gi]:
                ao.interp(gath[p], cboxes[gi], fine[gi], grown(fboxes[gi], ng), region, rr,
                          c["scheme"] == "linear", dim)
    return fine


@pytest.mark.parametrize("name", names("fill_patch"))
def test_fill_patch_oracle_matches_reference(name):
    c = case(name)
    fine = fill_patch_expected(c)
    for gi, a in fine.items():
        assert np.array_equal(inputs.bits(a), data()[f"{name}/fine{gi}"]), f"fine fab {gi}"
    assert c["plan_builds"] == [2] * c["nranks"]  # FillBoundary plan + fill_patch plan
