"""Config reports (paper_2506_14781_b200/reports.py) against the reference's
own analysis.cpp (time_to_residual, residual_curve incl. its bootstrap CI),
built from the reference sources into oracle/_ref (ref_harness.cpp)."""
import ctypes as C
import math
import random

import numpy as np
import pytest

import pyoracle as O
from paper_2506_14781_b200 import instances as I
from paper_2506_14781_b200 import reports as RP

needs_ref = pytest.mark.skipif(not O.ref_available("mt"), reason="oracle/_ref not built")


def P(a):
    return a.ctypes.data_as(C.c_void_p)


class Rec:
    def __init__(self, t, f, feasible, state=None):
        self.sweep_count, self.f, self.feasible, self.state = t, f, feasible, state


def test_mt19937_64_known_answer():
    # the C++ standard's required value: the 10000th output of a
    # default-constructed std::mt19937_64 (seed 5489)
    g = RP.MT19937_64(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042


def test_decode_majority_and_ties():
    copies = [[0, 1, 2], [3, 4]]
    s = np.array([1, -1, 1, -1, 1], dtype=np.int8)
    logical, feasible = RP.decode(copies, s)
    assert list(logical) == [1, -1] and not feasible  # tie -> first copy
    logical, feasible = RP.decode(copies, np.array([1, 1, 1, -1, -1], dtype=np.int8))
    assert list(logical) == [1, -1] and feasible


@needs_ref
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_time_to_residual_matches_reference(seed):
    rng = np.random.default_rng(seed)
    n = 200
    t = np.arange(1, n + 1, dtype=np.int64) * 5
    f = -np.sort(rng.uniform(0, 10, n))[::-1].copy() + rng.normal(0, 0.3, n)
    feas = (rng.random(n) < 0.6).astype(np.int32)
    L = O.ref_lib("mt")
    for e_gs, rho in ((-10.5, 0.01), (-9.0, 0.05), (-20.0, 0.0)):
        out = C.c_int64(0)
        assert L.tgr_time_to_residual(n, P(t), P(f), P(feas), C.c_double(e_gs), 7, C.c_double(rho),
                                      C.byref(out)) == 0
        got = RP.time_to_residual([RP.EnergySample(int(a), float(b), bool(c)) for a, b, c in zip(t, f, feas)],
                                  e_gs, 7, rho)
        assert (got if got is not None else -1) == out.value


@needs_ref
@pytest.mark.parametrize("strict,resamples", [(False, 200), (True, 50), (False, 0)])
def test_residual_curve_matches_reference(strict, resamples):
    pr = I.wishart_planted(6, 0.5, seed=4)
    n_log, cpl, fields = pr.meta["logical"]
    copies = pr.copies
    R, K, n = 5, 9, pr.n
    rng = random.Random(7)
    recs, flat_f, flat_feas, flat_states = [], [], [], []
    t = np.array([(k + 1) * 10 for k in range(K)], dtype=np.int64)
    for r in range(R):
        rr = []
        for k in range(K):
            st = np.array([rng.choice((-1, 1)) for _ in range(n)], dtype=np.int8)
            feasible = rng.random() < 0.5
            if feasible:  # make the chains agree
                for chain in copies:
                    st[list(chain)] = st[chain[0]]
            f = RP.logical_energy(pr.meta["logical"], RP.decode(copies, st)[0]) if feasible else rng.uniform(-5, 5)
            rr.append(Rec(int(t[k]), f, feasible, st))
            flat_f.append(f)
            flat_feas.append(int(feasible))
            flat_states.append(st)
        recs.append(rr)
    e_gs = [pr.meta["planted_energy"] - 0.1 * r for r in range(R)]
    runs = [(recs[r], e_gs[r], r % 3) for r in range(R)]
    curve = RP.residual_curve(runs, copies, pr.meta["logical"], n_log, strict=strict,
                              bootstrap_resamples=resamples, seed=11)
    L = O.ref_lib("mt")
    off = np.cumsum([0] + [len(c) for c in copies]).astype(np.int32)
    chain = np.array([p for c in copies for p in c], dtype=np.int32)
    lci = np.array([c[0] for c in cpl], dtype=np.int32)
    lcj = np.array([c[1] for c in cpl], dtype=np.int32)
    lw = np.array([c[2] for c in cpl], dtype=np.float64)
    lh = np.array(fields, dtype=np.float64)
    ff = np.array(flat_f, dtype=np.float64)
    fe = np.array(flat_feas, dtype=np.int32)
    ss = np.ascontiguousarray(np.stack(flat_states).astype(np.int8))
    eg = np.array(e_gs, dtype=np.float64)
    ids = np.array([r % 3 for r in range(R)], dtype=np.int32)
    ot = np.zeros(K, dtype=np.int64)
    orho = np.zeros(K)
    oci = np.zeros(K)
    if resamples == 0:
        pytest.skip("the reference takes percentiles of an empty bootstrap (undefined)")
    rc = L.tgr_residual_curve(R, K, n, P(t), P(ff), P(fe), P(ss), P(eg), P(ids), n_log, P(off), P(chain),
                              len(cpl), P(lci), P(lcj), P(lw), P(lh), int(strict), resamples,
                              C.c_uint64(11), P(ot), P(orho), P(oci))
    assert rc == 0
    for k in range(K):
        pt = curve.points[k]
        assert pt.t == ot[k]
        if math.isnan(orho[k]):
            assert math.isnan(pt.rho_e)
        else:
            assert pt.rho_e == orho[k]
            assert pt.ci95 == oci[k]
    assert curve.trials == R and curve.instances == 3
