"""Decoded-sample histogram and KL curve (analysis.cpp:215-241; decode
constraints.cpp:149-162; kl_divergence oracle.cpp:178-195).
Golden curves come from the reference's own kl_curve over its run_2dpt
(tools/gen_golden_kl.py -> tests/golden/kl.json, config 1: K10 +-1 sparsified to
20 physical spins, 8x8 grid); the C port replays them on the CPU, the B200
engine decodes, histograms and evaluates KL on the device every round (GPU)."""
import json
import os

import numpy as np
import pytest

import pyoracle as O
from paper_2506_14781_b200.instances import Problem

FIX = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "kl.json")))
CASES = FIX["cases"]
IDS = [f"seed{c['seed']}-{'discard' if c['discard'] else 'all'}" for c in CASES]


def physical():
    i = FIX["instance"]
    return Problem(i["n"], np.array(i["ci"], np.int32), np.array(i["cj"], np.int32),
                   np.array(i["cw"]), np.array(i["fields"]), np.array(i["pa"], np.int32),
                   np.array(i["pb"], np.int32))


def logical():
    i = FIX["logical"]
    return Problem(i["n"], np.array(i["ci"], np.int32), np.array(i["cj"], np.int32),
                   np.array(i["cw"]), np.array(i["fields"]), np.zeros(0, np.int32),
                   np.zeros(0, np.int32))


def golden_kl(c):
    return np.array([np.nan if x is None else x for x in c["kl"]])


@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_port_replays_reference_kl_curve(c):
    t, smp, kl = O.kl_curve(physical(), FIX["betas"], FIX["penalties"], c["total_sweeps"], c["sps"],
                            c["seed"], logical(), FIX["copies"], FIX["beta_kl"], c["discard"])
    assert smp.tolist() == c["samples"]
    np.testing.assert_array_equal(kl, golden_kl(c))
    assert t.tolist() == [k * c["sps"] for k in range(1, len(t) + 1)]


def test_port_boltzmann_normalised():
    p = O.enumerate_boltzmann(logical(), FIX["beta_kl"])
    assert p.shape == (1024,) and abs(p.sum() - 1.0) < 1e-12 and p.min() > 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_engine_kl_curve_matches_reference(c):
    from paper_2506_14781_b200.api import RunConfig, Schedule, run_2dpt_kl
    pts = run_2dpt_kl(physical(), Schedule(FIX["betas"], FIX["penalties"]),
                      RunConfig(total_sweeps=c["total_sweeps"], sweeps_per_swap=c["sps"], seed=c["seed"]),
                      logical(), FIX["copies"], FIX["beta_kl"], c["discard"])
    assert [p.samples for p in pts] == c["samples"]          # decode + histogram: exact
    # KL: device log vs glibc log and a tree-ordered sum -> FP64 rounding level
    np.testing.assert_allclose([p.kl for p in pts], golden_kl(c), rtol=1e-11, atol=1e-15)
    assert pts[-1].t == c["total_sweeps"]
    assert pts[-1].iid_reference == pytest.approx(1023 / (2.0 * c["samples"][-1]))


@pytest.mark.gpu
def test_engine_batched_kl_curves():
    # C1-style many-chain curves: every seed is one instance of a batch, each with its own
    # device histogram; instance b must equal the single run with seed b
    from paper_2506_14781_b200.api import Engine, RunConfig, Schedule, run_2dpt_batch
    want = {c["seed"]: c for c in CASES if not c["discard"]}
    seeds = sorted(want)
    pr = physical()
    with Engine(0) as eng:
        eng.set_kl_decoder(logical(), FIX["copies"], FIX["beta_kl"], False)
        run_2dpt_batch([pr] * len(seeds), [Schedule(FIX["betas"], FIX["penalties"])] * len(seeds),
                       RunConfig(total_sweeps=1500, store_states=False, digest=False), seeds,
                       engine=eng, sink=lambda *a: 0)
        for b, sd in enumerate(seeds):
            pts = eng.kl_curve(b, 1500)
            assert [p.samples for p in pts] == want[sd]["samples"]
            np.testing.assert_allclose([p.kl for p in pts], golden_kl(want[sd]), rtol=1e-11, atol=1e-15)


@pytest.mark.gpu
def test_engine_kl_decoder_errors():
    from paper_2506_14781_b200.api import Engine, RunConfig
    from paper_2506_14781_b200.instances import ConfigError
    with Engine(0) as eng:
        eng.set_problem(physical())
        eng.set_schedule(FIX["betas"], FIX["penalties"])
        eng.set_kl_decoder(logical(), FIX["copies"], FIX["beta_kl"])
        with pytest.raises(ConfigError, match="SLOT"):
            eng.run(RunConfig(total_sweeps=10, engine="plane"), None, flags=0)
        with pytest.raises(ConfigError):
            eng.set_kl_decoder(logical(), [[0]] * 9 + [[]], FIX["beta_kl"])  # a spin without copies
        eng.clear_kl_decoder()
        eng.run(RunConfig(total_sweeps=10, engine="plane"), None, flags=0)  # plane again without it
