"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/dtwlb.h declares, validates arguments before touching the device, and
reports ECUDA (never a silent CPU fallback) when no sm_100 device is present."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "dtwlb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:int|void|char)\s*\*?\s*(\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_0811_3301_b200 import build, binding
    build.build()
    return binding.load()


def test_header_declares_the_boundary():
    fns = _header_functions()
    for f in ["lb_envelope", "lb_keogh", "lb_piecewise", "lb_piecewise_sym", "lb_improved", "dtw_band", "nn_search", "nn_merge",
              "dtwlb_last_error", "dtwlb_release_workspace"]:
        assert f in fns, fns


def test_binding_exports_match_header():
    from paper_0811_3301_b200 import binding
    assert sorted(binding.EXPORTS) == _header_functions()


def test_library_exports_every_declared_symbol(lib):
    so = ctypes.CDLL(os.path.join(ROOT, "paper_0811_3301_b200", "libdtwlb.so"))
    for f in _header_functions():
        assert hasattr(so, f), f"libdtwlb.so does not export {f}"


def test_argument_validation_precedes_device(lib):
    from paper_0811_3301_b200.binding import NnOpts
    null = None
    assert lib.lb_envelope(null, 0, 1, null, null, 1, null) == 1          # n < 1
    assert b"n = 0" in lib.dtwlb_last_error()
    assert lib.lb_envelope(null, 8, -1, null, null, 1, null) == 1         # w < 0
    assert lib.lb_keogh(null, null, 1, 1, 8, 3, null, null) == 2          # p = 3 unsupported
    assert lib.lb_piecewise(null, null, 1, 1, 8, 3, null, null) == 2      # p = 3 unsupported
    assert lib.lb_piecewise(null, null, 1, 1, 0, 1, null, null) == 1      # n < 1
    assert lib.lb_piecewise_sym(null, null, null, 1, 1, 8, 1, 3, null, null) == 2   # p = 3 unsupported
    assert lib.lb_piecewise_sym(null, null, null, 1, 1, 8, -1, 1, null, null) == 1  # w < 0
    assert lib.dtw_band(null, null, 8, 2, 3, null, 1, null) == 2          # p = 3 unsupported
    assert lib.dtw_band(null, null, 8, 2, 5, null, 1, null) == 2          # p = 5 unsupported
    assert lib.dtw_band(null, null, 8, 2, 4, null, 1, null) == 1          # p = 4 (DTW_4) ok: NULL -> EINVAL
    assert lib.nn_search(null, 1, null, 4, 8, 1, 4, 1, null, null, None, None, null) == 2   # p = 4: dtw_band only
    assert lib.dtw_band(null, null, 8, 2, 0, null, 1, null) == 1          # p = 0 (inf) ok, NULL pointers
    assert lib.nn_search(null, 1, null, 4, 8, 1, 0, 1, null, null, None, None, null) == 2   # p = inf
    assert lib.nn_search(null, 1, null, 0, 8, 1, 1, 1, null, null, None, None, null) == 1   # N = 0
    assert lib.nn_search(null, 1, null, 4, 8, 1, 1, 5, null, null, None, None, null) == 1   # k > N
    assert lib.nn_search(null, 1, null, 4, 8, 1, 1, 0, null, null, None, None, null) == 1   # k < 1
    assert lib.nn_search(null, 1, null, 4, 8, 1, 2, 1, null, null, None, None, null) == 1   # NULL pointers
    assert lib.nn_search(null, 0, null, 4, 8, 1, 2, 1, null, null, None, None, null) == 0   # Q == 0: no-op
    assert lib.lb_envelope(null, 8, 1, null, null, 0, null) == 0          # count == 0: no-op
    assert lib.nn_merge(null, null, 0, 1, 1, null, null, null) == 1       # G < 1


def test_no_device_means_ecuda_not_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    buf = (ctypes.c_float * 64)()
    a = ctypes.addressof(buf)
    st = lib.lb_envelope(ctypes.c_void_p(a), 8, 1, ctypes.c_void_p(a + 64), ctypes.c_void_p(a + 128), 2, None)
    assert st == 4, st                                                    # DTWLB_ECUDA
    assert b"device" in lib.dtwlb_last_error().lower()


def test_communicator_bootstrap_without_device(lib):
    """dtwlb_get_unique_id needs no GPU (NCCL builds the id from the host); dtwlb_comm_init
    validates its arguments, then reports ECUDA without an sm_100 device -- never a fallback."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    buf = ctypes.create_string_buffer(128)
    st = lib.dtwlb_get_unique_id(buf)
    assert st in (0, 5), st                                       # OK, or ENCCL if NCCL is absent
    h = ctypes.c_void_p()
    assert lib.dtwlb_comm_init(buf, 2, 2, ctypes.byref(h)) == 1   # rank outside [0, nranks)
    assert lib.dtwlb_comm_init(None, 1, 0, ctypes.byref(h)) == 1  # NULL id
    assert lib.dtwlb_comm_init(buf, 1, 0, ctypes.byref(h)) == 4   # no device: ECUDA
    assert lib.dtwlb_comm_destroy(None) == 0
