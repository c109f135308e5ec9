"""The C-ABI library (include/tempergrid_b200.h): loads on a CPU-only host,
exports every declared entry point, fails loudly without a GPU, and its
host-side helpers (canonical order, swap replay) agree with the oracle."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import pyoracle as O
from paper_2506_14781_b200 import _lib
from paper_2506_14781_b200 import instances as I

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "tempergrid_b200.h")).read()
    return sorted(set(re.findall(r"\b(tg_[a-z0-9_]+)\s*\(", text)) - {"tg_sink_fn"})


def test_header_declares_what_the_binding_uses():
    assert set(_lib.EXPORTED) == set(declared_symbols())


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for sym in declared_symbols():
        assert hasattr(L, sym), sym
    assert L.tg_abi_version() == 1


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = _lib.lib()
    h = C.c_void_p()
    rc = L.tg_create(0, C.byref(h))
    assert rc == _lib.TG_ERR_CUDA
    buf = C.create_string_buffer(256)
    L.tg_last_error(None, buf, 256)
    assert b"CUDA" in buf.value or b"device" in buf.value


@pytest.mark.parametrize("mk", [lambda: I.k10_pm1(1), lambda: I.bipartite_3regular(256, seed=5),
                                lambda: I.wishart_planted(8, 0.5, seed=1), I.five_node_complete])
def test_canonical_order_native_python_and_port_agree(mk):
    pr = mk()
    a = I.canonical_order_native(pr)
    b = I.canonical_order_py(pr)
    c = O.canonical_order(pr)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[0], c[0])
    assert a[2] == b[2] == c[2]
    # a proper colouring: no edge inside a colour class
    col = a[1]
    for x, y in list(zip(pr.ci, pr.cj)) + list(zip(pr.pa, pr.pb)):
        assert col[x] != col[y]


def test_canonical_instances_are_fixed_points():
    for pr in (I.k10_pm1(1), I.bipartite_3regular(128, seed=2)):
        order = I.canonical_order(pr)[0]
        np.testing.assert_array_equal(order, np.arange(pr.n))


def swap_round_py(I_, J_, betas, pens, rnd, seed, base, f, g, slot_state):
    """Single-process restatement of one swap phase (engine.cpp:148-187)."""
    even = 1 if rnd % 2 == 0 else 0
    direction = 1 if ((rnd - 1) // 2) % 2 == 0 else -1
    dp = (J_ > 1) and (I_ == 1 or direction == 1)
    db = (I_ > 1) and (J_ == 1 or (J_ > 1 and direction != 1))
    sseed = O.derive_seed(seed, 2, 0)
    k = 0
    acc = []
    if dp:
        for i in range(I_):
            for p in range(even, J_ - 1, 2):
                a, b = i * J_ + p, i * J_ + p + 1
                x = betas[i] * (pens[p + 1] - pens[p]) * (g[slot_state[b]] - g[slot_state[a]])
                u = (O.stream_bits(sseed, base + k) >> 11) * 2.0 ** -53
                k += 1
                if x >= 0 or u < np.exp(x):
                    slot_state[a], slot_state[b] = slot_state[b], slot_state[a]
                    acc.append(("p", i * (J_ - 1) + p))
    elif db:
        for j in range(J_):
            for bb in range(even, I_ - 1, 2):
                a, b = bb * J_ + j, (bb + 1) * J_ + j
                ea = f[slot_state[a]] + pens[j] * g[slot_state[a]]
                eb = f[slot_state[b]] + pens[j] * g[slot_state[b]]
                x = (betas[bb + 1] - betas[bb]) * (eb - ea)
                u = (O.stream_bits(sseed, base + k) >> 11) * 2.0 ** -53
                k += 1
                if x >= 0 or u < np.exp(x):
                    slot_state[a], slot_state[b] = slot_state[b], slot_state[a]
                    acc.append(("b", bb * J_ + j))
    return k, acc


def test_host_swap_replay_matches_restatement():
    L = _lib.lib()
    rng = np.random.default_rng(3)
    betas = np.array([0.2, 0.5, 1.0, 2.0])
    pens = np.array([0.0, 0.5, 1.0])
    R = 12
    ss_lib = np.arange(R, dtype=np.int32)
    ss_py = list(range(R))
    ap = np.zeros(4 * 2, np.int64)
    ab = np.zeros(3 * 3, np.int64)
    base = 0
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    for rnd in range(1, 40):
        f = rng.normal(size=R) * 3
        g = 4.0 * rng.integers(0, 4, size=R)
        rc = L.tg_swap_phase_host(4, P(betas), 3, P(pens), rnd, 0, 11, base, P(f), P(g), P(ss_lib),
                                  P(ap), P(ab))
        assert rc == 0
        k, _ = swap_round_py(4, 3, betas, pens, rnd, 11, base, f, g, ss_py)
        base += k
        assert list(ss_lib) == ss_py
