"""The C ABI from plain C99 (examples/bf_demo.c, built by build()): argument checks,
identity beamforming bit-exact through cudaMalloc'd buffers, and the OFDM output stage
(bf_ofdm_*: one active subcarrier -> a complex exponential behind its cyclic prefix), no
Python on the path."""
import os
import subprocess

import pytest

from helpers import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "build", "bf_demo")


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()
    if not os.path.exists(DEMO):
        pytest.skip("gcc unavailable: demo not built")


def test_c_demo_without_gpu_reports_no_device():
    if gpu_available():
        pytest.skip("a GPU is present")
    r = subprocess.run([DEMO], capture_output=True, text=True, timeout=60)
    assert r.returncode == 2, r.stdout + r.stderr
    assert "no CUDA device" in r.stdout


@pytest.mark.gpu
def test_c_demo_on_gpu():
    if not gpu_available():
        pytest.skip("needs a CUDA device")
    r = subprocess.run([DEMO], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bf_demo: ok" in r.stdout
