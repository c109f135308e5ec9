"""The oracle's bit-plane decisions are drawn lazily, MSB first
(oracle/tg_oracle.c plane_less): check that they equal the full 53-bit
uniform compared with T (u = U53 * 2^-53 < T), including thresholds at and
next to the grid points K * 2^-53 where only the last planes decide."""
import ctypes as C

import numpy as np

import pyoracle as O


def test_lazy_plane_decision_equals_full_uniform():
    L = O.port_lib()
    L.tgo_plane_less.restype = C.c_int
    L.tgo_plane_less.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32, C.c_int, C.c_double]
    rng = np.random.default_rng(7)
    pkey = O.port_lib().tgo_derive(11, 8, 0)
    n_cases = 0
    for _ in range(3000):
        grp = int(rng.integers(0, 64))
        lane = int(rng.integers(0, 32))
        t = int(rng.integers(0, 1 << 40))
        site = int(rng.integers(0, 1 << 20))
        u53 = O.port_lib().tgo_plane(pkey, grp, t, site, lane)
        u = u53 * 2.0 ** -53
        # random thresholds, and thresholds within a few ulps of u itself
        cands = [float(rng.random()), float(rng.random()) ** 8, 0.0, 1.0, 2.0, 1e-300,
                 u, np.nextafter(u, 0.0), np.nextafter(u, 1.0), (u53 + 1) * 2.0 ** -53,
                 max(u53 - 1, 0) * 2.0 ** -53]
        for T in cands:
            assert L.tgo_plane_less(pkey, grp, t, site, lane, T) == int(u < T), (grp, lane, t, site, T)
            n_cases += 1
    assert n_cases == 33000
