"""The C-ABI library loads and exports every symbol include/bf.h declares; host-side
validation works without a GPU (no compute calls are made here)."""
import ctypes
import os
import re

import pytest

from helpers import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bf():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1810_11451_b200 as bf
    return bf


def _declared_functions():
    names = set()
    for hdr in ("bf.h", "bf_filter.h", "bf_ofdm.h"):
        src = open(os.path.join(ROOT, "include", hdr)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(bff?_[a-z_]+)\s*\(", src))
    return sorted(names)


def test_header_declares_the_boundary_calls():
    names = _declared_functions()
    for required in ("bf_plan_create", "bf_set_precoders", "bf_apply", "bf_destroy",
                     "bf_status_string"):
        assert required in names


def test_library_exports_every_declared_symbol(bf):
    from paper_1810_11451_b200 import _lib
    L = ctypes.CDLL(_lib.LIB_PATH)
    names = _declared_functions()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) == set(_lib.EXPORTS)


def test_no_oracle_in_product(bf):
    """The product library and package never reference the oracle."""
    so = open(os.path.join(ROOT, "paper_1810_11451_b200", "libbf.so"), "rb").read()
    assert b"bfo_beamform" not in so
    pkg = os.path.join(ROOT, "paper_1810_11451_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in text and "from oracle" not in text, fn
                assert "bf_oracle" not in text, fn


def test_status_strings(bf):
    L = bf.lib()
    for s in bf.Status:
        assert L.bf_status_string(int(s)).decode() == "BF_" + (
            "OK" if s.name == "OK" else "ERR_" + s.name)
    assert L.bf_version() == 1


@pytest.mark.parametrize("dims,expect", [
    ((64, -1, 60, 0), "INVALID_VALUE"),
    ((0, 8, 60, 0), "INVALID_VALUE"),
    ((64, 8, 0, 0), "INVALID_VALUE"),
    ((64, 8, 60, 7), "INVALID_VALUE"),
    ((64, 37, 60, 0), "UNSUPPORTED"),
    ((32, 8, 60, 0), "UNSUPPORTED"),
    ((64, 8, 64, 1), "UNSUPPORTED"),
])
def test_plan_create_validates_before_touching_gpu(bf, dims, expect):
    assert bf.plan_create_status(*dims) == bf.Status[expect]


def test_plan_create_without_device(bf):
    if gpu_available():
        pytest.skip("a GPU is present")
    assert bf.plan_create_status(64, 36, 60, 0) == bf.Status.NO_DEVICE
    assert "no CUDA device" in bf.lib().bf_last_error().decode()


def test_null_plan_calls_are_rejected(bf):
    L = bf.lib()
    assert L.bf_apply(None, None, None, None, 0, None) == bf.Status.INVALID_VALUE
    assert L.bf_set_precoders(None, None, 1, None) == bf.Status.INVALID_VALUE
    assert L.bf_destroy(None) == bf.Status.INVALID_VALUE


def test_filter_plan_validates_before_touching_gpu(bf):
    assert bf.filter_plan_create_status(1024) == bf.Status.UNSUPPORTED
    assert bf.filter_plan_create_status(0) == bf.Status.INVALID_VALUE
    if not gpu_available():
        assert bf.filter_plan_create_status(2048) == bf.Status.NO_DEVICE


def test_batch_and_share_validation_without_gpu(bf):
    """bf_apply_batch / bf_plan_set_sm_share argument checks (host-side, no GPU touched)."""
    import ctypes as ct
    from paper_1810_11451_b200._lib import BatchJob
    L = bf.lib()
    assert L.bf_apply_batch(None, 0, None) == bf.Status.OK                 # empty list: no-op
    assert L.bf_apply_batch(None, 1, None) == bf.Status.INVALID_VALUE      # NULL list
    assert L.bf_apply_batch(None, -1, None) == bf.Status.INVALID_VALUE
    jobs = (BatchJob * 2)()
    assert L.bf_apply_batch(jobs, 2, None) == bf.Status.INVALID_VALUE      # NULL plan
    assert "plan is NULL" in L.bf_last_error().decode()
    assert L.bf_plan_set_sm_share(None, 4) == bf.Status.INVALID_VALUE
    assert ct.sizeof(BatchJob) == 48
