"""GPU parity of the fused filter stage (libbf.so bff_*) against the fp64 oracle.

Contract (DESIGN.md §2 F3): per signal, max_k |y_gpu[k] - y_ref[k]| <= 1e-5 *
||s||_2 * max_k |DFT(h)[k]|; for the bare FFT, 1e-5 * sqrt(n) * ||x||_2.
"""
import ctypes

import numpy as np
import pytest

import bf_synth as syn
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():   # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import bf_synth.cuda as sync  # noqa: E402
import paper_1810_11451_b200 as bf  # noqa: E402
from paper_1810_11451_b200 import FilterPlan  # noqa: E402

DEV = torch.device("cuda", 0)
NT = oracle.max_threads()
TOL = 1e-5


def run_filter(s, h, inplace=False):
    plan = FilterPlan()
    plan.set_taps(torch.from_numpy(h).to(DEV))
    sd = torch.from_numpy(np.ascontiguousarray(s)).to(DEV)
    y = plan.apply(sd, out=sd if inplace else None)
    torch.cuda.synchronize()
    plan.close()
    return y.cpu().numpy()


def check(y, y_ref, bound, what):
    err = np.abs(y.astype(np.complex128) - y_ref.astype(np.complex128)).max(axis=1)
    rel = err / bound
    assert (rel <= TOL).all(), f"{what}: worst err/bound {rel.max():.3e}"
    return float(rel.max())


def test_fft_matches_oracle_dft():
    x = syn.filter_signals(7, 0, np.arange(6))
    plan = FilterPlan()
    X = plan.fft(torch.from_numpy(x).to(DEV))
    torch.cuda.synchronize()
    X = X.cpu().numpy()
    ref = oracle.dft(x)
    bound = np.sqrt(2048) * np.linalg.norm(x.astype(np.complex128), axis=1)
    worst = check(X, ref, bound, "fft")
    assert worst < 1e-6
    plan.close()


@pytest.mark.parametrize("n_sig", [1, 16, 37])
def test_filter_matches_oracle(n_sig):
    wl = syn.filter_workload("fl0")
    s = syn.filter_signals(wl.seed, 0, np.arange(n_sig))
    h = syn.filter_taps()
    y_ref, bound = oracle.filter_apply(s, h, n_threads=NT)
    y = run_filter(s, h)
    worst = check(y, y_ref, bound, f"filter n_sig={n_sig}")
    assert worst < 1e-6


@pytest.mark.parametrize("kernel", ["warp_tab", "warp", "cta1", "cta2"])
def test_comparison_kernels_match_oracle(kernel, monkeypatch):
    # the non-default kernels BFF_FILTER_KERNEL selects (read at plan creation) — forward
    # FFT and filter, a ragged count of signals (not a multiple of 4 warps / 2 per CTA)
    monkeypatch.setenv("BFF_FILTER_KERNEL", kernel)
    wl = syn.filter_workload("fl0")
    s = syn.filter_signals(wl.seed, 0, np.arange(37))
    h = syn.filter_taps()
    y_ref, bound = oracle.filter_apply(s, h, n_threads=NT)
    assert check(run_filter(s, h), y_ref, bound, f"filter {kernel}") < 1e-6
    plan = FilterPlan()
    X = plan.fft(torch.from_numpy(s[:5]).to(DEV))
    torch.cuda.synchronize()
    plan.close()
    bound = np.sqrt(2048) * np.linalg.norm(s[:5].astype(np.complex128), axis=1)
    assert check(X.cpu().numpy(), oracle.dft(s[:5]), bound, f"fft {kernel}") < 1e-6


def test_filter_equals_circular_convolution():
    s = syn.filter_signals(8, 0, np.arange(4))
    rng = np.random.default_rng(8)
    h = (rng.standard_normal(2048) + 1j * rng.standard_normal(2048)).astype(np.complex64) / 64
    y_ref, bound = oracle.filter_apply(s, h, n_threads=NT, direct=True)
    check(run_filter(s, h), y_ref, bound, "vs direct circular convolution")


def test_identity_and_delay_filters():
    s = syn.filter_signals(9, 0, np.arange(5))
    d = np.zeros(2048, np.complex64); d[0] = 1
    bound = np.linalg.norm(s.astype(np.complex128), axis=1)
    check(run_filter(s, d), s, bound, "identity filter")
    d3 = np.zeros(2048, np.complex64); d3[3] = 1
    check(run_filter(s, d3), np.roll(s, 3, axis=1), bound, "delay by 3")


def test_in_place_and_batch_independence():
    s = syn.filter_signals(10, 0, np.arange(50))
    h = syn.filter_taps()
    a = run_filter(s, h)
    b = run_filter(s, h, inplace=True)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    c = run_filter(s[17:18], h)
    assert np.array_equal(c.view(np.uint32), a[17:18].view(np.uint32))


def test_device_signal_generator_matches_host():
    out = torch.empty((5, 2048), dtype=torch.complex64, device=DEV)
    sync.gen_filter_signals(out, 6, 0, first=1000)
    assert np.array_equal(out.cpu().numpy(), syn.filter_signals(6, 0, np.arange(1000, 1005)))


@pytest.mark.slow
def test_fl1_full_size_sampled():
    wl = syn.filter_workload("fl1")
    s = torch.empty((wl.n_signals, 2048), dtype=torch.complex64, device=DEV)
    sync.gen_filter_signals(s, wl.seed)
    h = syn.filter_taps()
    plan = FilterPlan()
    plan.set_taps(torch.from_numpy(h).to(DEV))
    y = plan.apply(s)
    torch.cuda.synchronize()
    ids = np.array([0, 1, 12345, wl.n_signals - 1])
    y_ref, bound = oracle.filter_apply(syn.filter_signals(wl.seed, 0, ids), h, n_threads=NT)
    check(y[torch.from_numpy(ids).to(DEV)].cpu().numpy(), y_ref, bound, "fl1 sampled")
    assert torch.isfinite(torch.view_as_real(y)).all().item()
    plan.close()


def test_filter_error_paths():
    L = bf.lib()
    plan = FilterPlan()
    s = torch.zeros((2, 2048), dtype=torch.complex64, device=DEV)
    with pytest.raises(bf.BfError) as e:
        plan.apply(s)
    assert e.value.status == bf.Status.NO_PRECODERS
    plan.set_taps(torch.zeros(2048, dtype=torch.complex64, device=DEV))
    big = torch.zeros((3, 2048), dtype=torch.complex64, device=DEV)
    st = L.bff_apply(plan._h, ctypes.c_void_p(big.data_ptr()), ctypes.c_void_p(big.data_ptr() + 16384),
                     2, None)
    assert st == bf.Status.INVALID_VALUE                 # partial overlap
    st = L.bff_apply(plan._h, ctypes.c_void_p(big.data_ptr() + 8), ctypes.c_void_p(s.data_ptr()), 1,
                     None)
    assert st == bf.Status.MISALIGNED
    assert L.bff_apply(plan._h, None, None, 0, None) == bf.Status.OK
    plan.close()


@pytest.mark.parametrize("n_sig", [1, 149, 600])
def test_filter_no_write_outside_y(n_sig):
    """Out-of-bounds write check (compute-sanitizer is closed on this pool): y sits between
    guard bands of a sentinel pattern that must survive; every word of y is written."""
    guard = 2048
    plan = FilterPlan()
    plan.set_taps(torch.from_numpy(syn.filter_taps()).to(DEV))
    s = torch.from_numpy(syn.filter_signals(8, 0, np.arange(n_sig))).to(DEV)
    words = n_sig * 2048 * 2
    buf = torch.full((guard + words + guard,), 0x7FC0DEAD, dtype=torch.int32, device=DEV)
    y = buf[guard:guard + words].view(torch.complex64).view(n_sig, 2048)
    plan.apply(s, out=y)
    torch.cuda.synchronize()
    h = buf.cpu().numpy()
    assert (h[:guard] == 0x7FC0DEAD).all() and (h[guard + words:] == 0x7FC0DEAD).all()
    assert not (h[guard:guard + words] == 0x7FC0DEAD).any()
    plan.close()
