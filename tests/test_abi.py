"""C-ABI library checks that need no GPU (-m "not gpu"): the library builds and
loads, exports every symbol include/fbp.h declares, and validates arguments."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2007_06289_b200 import build
    build.build()
    from paper_2007_06289_b200 import fbp
    return fbp.lib()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "fbp.h")).read()
    return re.findall(r"FBP_API\s+[\w\s\*]+?\b(fbp_\w+)\s*\(", txt)


def test_exports_every_declared_symbol(L):
    syms = header_symbols()
    assert len(syms) == 15, syms
    for s in syms:
        assert hasattr(L, s), s
    from paper_2007_06289_b200 import fbp
    assert sorted(syms) == sorted(fbp.EXPORTED)


def test_status_strings(L):
    for code in range(7):
        assert L.fbp_status_str(code).decode().startswith("FBP_")


def _create(L, n, b, a, max_batch=1, device=0):
    h = ctypes.c_void_p()
    bb = (ctypes.c_double * max(1, len(b)))(*b)
    aa = (ctypes.c_double * max(1, len(a)))(*a)
    st = L.fbp_plan_create(ctypes.byref(h), n, max_batch, len(b), bb, len(a), aa, device)
    return st, h


@pytest.mark.parametrize("n", [0, 1, 3, 6, 100, 16384, -4])
def test_plan_rejects_bad_N(L, n):
    st, h = _create(L, n, [0.1, -0.2, 0.1], [-0.5])
    assert st == 1 and not h.value
    assert "power of two" in L.fbp_last_error().decode()


def test_plan_rejects_unstable_feedback(L):
    # roots of z^2 - 2.5 z + 1 are 2 and 0.5 -> unstable (Schur-Cohn)
    st, h = _create(L, 64, [1.0], [-2.5, 1.0])
    assert st == 3 and not h.value
    st, h = _create(L, 64, [1.0], [-1.0])        # pole on the unit circle
    assert st == 3
    st, h = _create(L, 64, [1.0], [0.3, -1.2, 0.9])  # |k_3| = 0.9 but a step-down |k| >= 1
    assert st in (0, 3, 6)


def test_plan_rejects_bad_orders_and_batch(L):
    assert _create(L, 64, [], [0.1])[0] == 2
    assert _create(L, 64, [0.1] * 9, [0.1])[0] == 2
    assert _create(L, 64, [0.1], [0.01] * 9)[0] == 2
    assert _create(L, 64, [0.1], [-0.5], max_batch=0)[0] == 2
    assert _create(L, 64, [float("nan")], [-0.5])[0] == 2


def test_valid_plan_without_gpu_reports_device(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    st, h = _create(L, 64, [0.12, -0.23, 0.10], [-1.02, 0.0017, 0.0947])
    assert st == 6 and not h.value


def test_calls_reject_null_plan(L):
    assert L.fbp_reconstruct(None, None, None, 1, None) == 2
    assert L.fbp_iir_filter(None, None, None, 1, None) == 2
    assert L.fbp_fht_backproject(None, None, None, 1, ctypes.c_float(1.0), None) == 2
    assert L.fbp_reconstruct_host(None, None, None, 1) == 2
    assert L.fbp_plan_launch_count(None) == -1
    L.fbp_plan_destroy(None)


def test_python_plan_raises_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2007_06289_b200 import Plan, FbpError
    with pytest.raises(FbpError):
        Plan(64, [0.12, -0.23, 0.10], [-1.02, 0.0017, 0.0947])


def test_product_build_reads_no_tuning_environment(L):
    """Developer knobs (FBP_XB, FBP_TAIL, FBP_DBG, ...) exist only in -DFBP_DEV_MASK=1
    builds: the product library contains none of their names."""
    from paper_2007_06289_b200 import fbp
    data = open(fbp._LIB_PATH, "rb").read()
    for name in (b"FBP_XB", b"FBP_TAIL", b"FBP_DBG", b"FBP_PREFETCH", b"FBP_SWEEP_CTAS", b"FBP_SWEEP_SEG",
                 b"FBP_FXA", b"FBP_FXB", b"FBP_VERBOSE"):
        assert name not in data, name
