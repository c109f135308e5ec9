"""The reference-side binding (integration/engine_b200.cpp): the reference's
own run_2dpt and run_2dpt_b200 (the B200 engine through the C ABI) must emit
byte-identical trace_to_jsonl text (engine.cpp:272-313) -- every round's f, g,
feasibility, RLE target state and cumulative acceptance rates -- when both
consume Philox draws (oracle/_ref/libtgref_shim.so, built against the
reference headers and the Philox shadow rng.hpp)."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2506_14781_b200 import instances as I

HERE = os.path.dirname(os.path.abspath(__file__))
SHIM = os.path.join(os.path.dirname(HERE), "oracle", "_ref", "libtgref_shim.so")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(SHIM), reason="oracle/_ref shim not built")]


def compare(pr, betas, pens, total, sps, seed, grid=False):
    L = C.CDLL(SHIM)
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    a = [np.ascontiguousarray(x, dtype=t) for x, t in (
        (pr.ci, np.int32), (pr.cj, np.int32), (pr.cw, np.float64), (pr.fields, np.float64),
        (pr.pa, np.int32), (pr.pb, np.int32), (betas, np.float64), (pens, np.float64))]
    cap = 64 << 20
    ref = C.create_string_buffer(cap)
    gpu = C.create_string_buffer(cap)
    err = C.create_string_buffer(512)
    L.tg_shim_compare.restype = C.c_int
    rc = L.tg_shim_compare(pr.n, len(a[0]), P(a[0]), P(a[1]), P(a[2]), P(a[3]), len(a[4]), P(a[4]),
                           P(a[5]), len(a[6]), P(a[6]), len(a[7]), P(a[7]), C.c_int64(total),
                           C.c_int64(sps), C.c_uint64(seed), 1 if grid else 0, ref, cap, gpu, cap,
                           err, 512)
    assert rc == 0, err.value
    return ref.value.decode(), gpu.value.decode()


def test_k10_config1_trace_identical():
    b, p = I.config_schedule("c1")
    ref, gpu = compare(I.k10_pm1(1), b, p, 500, 1, 5)
    assert ref.count("\n") == 500
    assert gpu == ref


def test_five_node_trace_identical():
    f = I.five_node_complete()
    pr = I.to_canonical(I.sparsify(5, list(zip(f.ci.tolist(), f.cj.tolist(), f.cw.tolist())),
                                   f.fields.tolist(), 2, 3))
    ref, gpu = compare(pr, [1.0], [2.0, 4.0, 6.0, 8.0], 20000, 500, 77)  # acceptance.cpp:540-549
    assert gpu == ref


def test_grid_records_identical():
    ref, gpu = compare(I.k10_pm1(3), [0.5, 1.0, 2.0], [0.0, 0.5, 1.0], 60, 2, 9, grid=True)
    assert gpu == ref


def test_errors_map_to_reference_exceptions():
    with pytest.raises(AssertionError, match="strictly increasing"):
        compare(I.k10_pm1(1), [1.0, 0.5], [0.0], 10, 1, 1)


def compare_jcolumn(pr, betas, p_fixed, repeats, total, sps, seed):
    L = C.CDLL(SHIM)
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    a = [np.ascontiguousarray(x, dtype=t) for x, t in (
        (pr.ci, np.int32), (pr.cj, np.int32), (pr.cw, np.float64), (pr.fields, np.float64),
        (pr.pa, np.int32), (pr.pb, np.int32), (betas, np.float64))]
    cap = 16 << 20
    ref = C.create_string_buffer(cap)
    gpu = C.create_string_buffer(cap)
    err = C.create_string_buffer(512)
    L.tg_shim_compare_jcolumn.restype = C.c_int
    rc = L.tg_shim_compare_jcolumn(pr.n, len(a[0]), P(a[0]), P(a[1]), P(a[2]), P(a[3]), len(a[4]),
                                   P(a[4]), P(a[5]), len(a[6]), P(a[6]), C.c_double(p_fixed),
                                   int(repeats), C.c_int64(total), C.c_int64(sps), C.c_uint64(seed),
                                   ref, cap, gpu, cap, err, 512)
    assert rc == 0, err.value
    return ref.value.decode(), gpu.value.decode()


def test_jcolumn_baseline_identical():
    # run_jcolumn_pt (engine.cpp:221-270) vs run_jcolumn_pt_b200, as acceptance.cpp:385-393
    # calls it: the grid schedule's betas, mean penalty, J repeats
    b, p = I.config_schedule("c1")
    ref, gpu = compare_jcolumn(I.k10_pm1(2), b, float(np.mean(p)), len(p), 2000, 2, 7000)
    assert ref.count("\n") == 1001
    assert gpu == ref
