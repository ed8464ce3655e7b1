"""GPU parity of the OFDM output stage (libbf.so bf_ofdm_*, include/bf_ofdm.h) against the
fp64 oracle (oracle/ofdm_oracle.c).

Contract (DESIGN.md §2 O5): per (symbol, antenna), max_t |y_gpu - y_exact| <=
1e-5 * |scale| * (sum_q T_q + sqrt(n) ||X||_2) — the oracle returns that bound.
"""
import numpy as np
import pytest

import bf_synth as syn
import oracle
from helpers import TOL

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():   # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1810_11451_b200 as bf  # noqa: E402
from paper_1810_11451_b200 import OfdmPlan, Plan, Status  # noqa: E402
from paper_1810_11451_b200.ofdm import ofdm_plan_create_status  # noqa: E402

DEV = torch.device("cuda", 0)
NT = oracle.max_threads()


def run(W, S, tags, nb, cp, scale, chunk=0, variant="auto"):
    plan = Plan(W.shape[-1], variant=variant)
    Wd = torch.from_numpy(np.ascontiguousarray(W[None] if W.ndim == 2 else W)).to(DEV)
    plan.set_precoders(Wd)
    op = OfdmPlan(plan, nb, cp=cp, scale=scale)
    if chunk:
        op.set_chunk(chunk)
    Sd = torch.from_numpy(np.ascontiguousarray(S)).to(DEV)
    td = None if tags is None else torch.from_numpy(np.ascontiguousarray(tags)).to(DEV)
    y = op.apply(Sd, td)
    torch.cuda.synchronize()
    out = y.cpu().numpy()
    op.close()
    plan.close()
    return out


def check(y, y_ref, bound, what):
    assert y.shape == y_ref.shape, (y.shape, y_ref.shape)
    assert np.isfinite(y.view(np.float32)).all(), what
    err = np.abs(y.astype(np.complex128) - y_ref.astype(np.complex128)).max(axis=2)
    rel = err / np.where(bound > 0, bound, 1.0)
    assert (rel <= TOL).all(), f"{what}: worst err/bound {rel.max():.3e} at {np.unravel_index(rel.argmax(), rel.shape)}"
    return float(rel.max())


def gaussian(rng, shape, scale=1.0):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64) * np.float32(scale)


@pytest.mark.parametrize("spec", ["1", "0"])
def test_of0_workload_matches_oracle(spec, monkeypatch):
    # nb = 26: the kernel specialised for its half band (the default) and the generic one
    monkeypatch.setenv("BFO_OFDM_SPEC", spec)
    wl = syn.ofdm_workload("of0")
    W, S, tags = syn.ofdm_inputs(wl)
    scale = float(np.float32(1.0 / np.sqrt(wl.n)))
    y_ref, bound = oracle.ofdm(W, S, wl.nb, n=wl.n, cp=wl.cp, scale=scale, group_idx=tags, n_threads=NT)
    y = run(W, S, tags, wl.nb, wl.cp, scale)
    worst = check(y, y_ref, bound, "of0")
    assert worst < 1e-6     # ~2 orders inside the contract (fp32 FFT + the split-precision product)


@pytest.mark.parametrize("variant", ["ffma", "tensor"])
def test_ragged_shapes_gaussian_inputs(variant):
    # odd nb (a block straddles the two halves of the spectrum), no cyclic prefix, f = 7,
    # three precoder groups with random tags, Gaussian fp32 W and S, a chunk size that
    # leaves a ragged last chunk (37 = 9 x 4 + 1)
    rng = np.random.default_rng(11)
    nb, n_sym, f, G = 5, 37, 7, 3
    W = gaussian(rng, (G, 64, f))
    S = gaussian(rng, (n_sym * nb, f, 60))
    tags = rng.integers(0, G, n_sym * nb).astype(np.int32)
    y_ref, bound = oracle.ofdm(W, S, nb, n=2048, cp=0, scale=0.5, group_idx=tags, n_threads=NT)
    y = run(W, S, tags, nb, 0, 0.5, chunk=4, variant=variant)
    assert check(y, y_ref, bound, f"ragged {variant}") < 1e-6


def test_many_signals_per_warp():
    # 600 symbols x 64 antennas = 38 400 signals: every warp of the persistent grid runs
    # many signals (the next signal's fetch overlaps the current transform); nb = 1
    rng = np.random.default_rng(12)
    nb, n_sym, f = 1, 600, 4
    W = gaussian(rng, (64, f))
    S = gaussian(rng, (n_sym * nb, f, 60))
    y_ref, bound = oracle.ofdm(W, S, nb, n=2048, cp=144, scale=1.0, n_threads=NT)
    y = run(W, S, None, nb, 144, 1.0)
    assert check(y, y_ref, bound, "many signals") < 1e-6


@pytest.mark.parametrize("kernel", ["sb", "db", "cpa", "cpa_db"])
def test_each_ifft_kernel_matches_oracle(kernel, monkeypatch):
    # every selectable IFFT kernel (BFO_OFDM_KERNEL, read at plan creation): one buffer per
    # warp (4 warps, 2 CTAs per SM) and two (6 warps, 1 CTA per SM); odd nb, many signals
    # per warp, a ragged signal count (not a multiple of the warps per CTA)
    monkeypatch.setenv("BFO_OFDM_KERNEL", kernel)
    rng = np.random.default_rng(14)
    nb, n_sym, f = 3, 401, 5
    W = gaussian(rng, (64, f))
    S = gaussian(rng, (n_sym * nb, f, 60))
    y_ref, bound = oracle.ofdm(W, S, nb, n=2048, cp=160, scale=0.75, n_threads=NT)
    y = run(W, S, None, nb, 160, 0.75, chunk=100)
    assert check(y, y_ref, bound, f"kernel {kernel}") < 1e-6


def test_maximum_band_and_prefix():
    # nb = 34: 2040 of 2048 bins active (4 zero bins either side of n/2); cp = 2047 (max)
    rng = np.random.default_rng(13)
    nb, n_sym, f = 34, 3, 36
    W = gaussian(rng, (64, f), 0.25)
    S = gaussian(rng, (n_sym * nb, f, 60))
    y_ref, bound = oracle.ofdm(W, S, nb, n=2048, cp=2047, scale=-0.125, n_threads=NT)
    y = run(W, S, None, nb, 2047, -0.125)
    assert check(y, y_ref, bound, "nb 34 cp 2047") < 1e-6


def test_f0_gives_zero_samples():
    S = np.zeros((4 * 26, 0, 60), dtype=np.complex64)
    W = np.zeros((64, 0), dtype=np.complex64)
    plan = Plan(0)
    op = OfdmPlan(plan, 26, cp=144)
    y = op.apply(torch.from_numpy(S).to(DEV))
    torch.cuda.synchronize()
    assert y.shape == (4, 64, 2192)
    assert (y.cpu().numpy() == 0).all()
    del W


def test_chunking_and_ifft_stage_are_bitwise_consistent():
    # the result of a symbol does not depend on the chunk size, and bf_ofdm_apply equals
    # bf_apply followed by bf_ofdm_ifft bit for bit (same kernels)
    wl = syn.ofdm_workload("of0")
    W, S, tags = syn.ofdm_inputs(wl)
    plan = Plan(wl.f)
    plan.set_precoders(torch.from_numpy(W).to(DEV))
    op = OfdmPlan(plan, wl.nb, cp=wl.cp, scale=0.03125)
    Sd, td = torch.from_numpy(S).to(DEV), torch.from_numpy(tags).to(DEV)
    y1 = op.apply(Sd, td)
    op.set_chunk(1)
    y2 = op.apply(Sd, td)
    R = plan.apply(Sd, td)
    y3 = op.ifft(R)
    y4 = op.ifft(R[2 * wl.nb:4 * wl.nb].contiguous())
    torch.cuda.synchronize()
    a, b, c = (t.cpu().numpy().view(np.uint32) for t in (y1, y2, y3))
    assert (a == b).all() and (a == c).all()
    assert (y4.cpu().numpy().view(np.uint32) == a[2:4]).all()


def test_host_argument_errors():
    plan = Plan(8)
    assert ofdm_plan_create_status(plan, 26, n=1024) == Status.UNSUPPORTED
    assert ofdm_plan_create_status(plan, 26, cp=2048) == Status.INVALID_VALUE
    assert ofdm_plan_create_status(plan, 26, cp=-1) == Status.INVALID_VALUE
    assert ofdm_plan_create_status(plan, 35) == Status.INVALID_VALUE     # 2100 > 2048 bins
    assert ofdm_plan_create_status(plan, 0) == Status.INVALID_VALUE
    assert ofdm_plan_create_status(plan, 26, scale=float("inf")) == Status.INVALID_VALUE
    assert ofdm_plan_create_status(Plan(8, layout="planar"), 26) == Status.UNSUPPORTED
    op = OfdmPlan(plan, 2)
    R = torch.zeros((4, 64, 60), dtype=torch.complex64, device=DEV)
    y = torch.zeros((2 * 64 * 2048 + 1,), dtype=torch.complex64, device=DEV)
    from paper_1810_11451_b200.ofdm import _lib
    from paper_1810_11451_b200.plan import _ptr
    import ctypes
    mis = ctypes.c_void_p(y.data_ptr() + 8)
    assert _lib().bf_ofdm_ifft(op._h, _ptr(R), 2, mis, None) == Status.MISALIGNED
    assert _lib().bf_ofdm_ifft(op._h, _ptr(R), -1, _ptr(y), None) == Status.INVALID_VALUE
    assert _lib().bf_ofdm_ifft(op._h, _ptr(R), 0, None, None) == Status.OK     # no-op
    assert _lib().bf_ofdm_ifft(op._h, None, 2, _ptr(y), None) == Status.INVALID_VALUE
    # y overlapping R
    assert _lib().bf_ofdm_ifft(op._h, _ptr(R), 2, _ptr(R), None) == Status.INVALID_VALUE
    with pytest.raises(bf.BfError):
        op.set_chunk(-1)


def test_of1_full_size_sampled():
    # BASELINE-scale workload in the bench's launch configuration (of1: 2^15 symbols, the
    # default 4096-symbol chunks, AUTO -> tensor kernel at f = 36): every 512th symbol (all
    # antennas, 64 symbols, incl. the last one) vs the oracle
    import bf_synth.cuda as sync
    wl = syn.ofdm_workload("of1")
    S = torch.empty((wl.n_blocks, wl.f, wl.b), dtype=torch.complex64, device=DEV)
    sync.gen_symbols(S, wl.seed, 0, wl.f, wl.b, wl.M)
    tags = (torch.arange(wl.n_blocks, device=DEV) % wl.nb).to(torch.int32)
    W = syn.precoders(wl.seed, 0, wl.nb, wl.n_ant, wl.f, "unit_columns")
    scale = float(np.float32(1.0 / np.sqrt(wl.n)))
    plan = Plan(wl.f)
    plan.set_precoders(torch.from_numpy(W).to(DEV))
    op = OfdmPlan(plan, wl.nb, cp=wl.cp, scale=scale)
    y = op.apply(S, tags)
    del S
    ids = np.unique(np.append(np.arange(0, wl.n_sym, 512), wl.n_sym - 1))
    got = y[torch.from_numpy(ids).to(DEV)].cpu().numpy()
    Wp, Sp, tp = syn.ofdm_inputs(wl, ids)
    y_ref, bound = oracle.ofdm(Wp, Sp, wl.nb, n=wl.n, cp=wl.cp, scale=scale, group_idx=tp, n_threads=NT)
    assert check(got, y_ref, bound, "of1 sampled") < 1e-6
    del y
    op.close()
    plan.close()


def test_int16_output_is_the_rounded_fp32_output():
    # BF_OFDM_OUT_I16: sat(rne(y 2^e)) of the fp32 samples, bit for bit, at e = 12 (the
    # bench's), 3 and 22 (mostly saturated); within 2^-(e+1) + the O5 bound of the oracle
    wl = syn.ofdm_workload("of0")
    W, S, tags = syn.ofdm_inputs(wl)
    scale = float(np.float32(1.0 / np.sqrt(wl.n)))
    plan = Plan(wl.f)
    plan.set_precoders(torch.from_numpy(W).to(DEV))
    op = OfdmPlan(plan, wl.nb, cp=wl.cp, scale=scale)
    Sd, td = torch.from_numpy(S).to(DEV), torch.from_numpy(tags).to(DEV)
    y32 = op.apply(Sd, td).cpu().numpy()
    y_ref, bound = oracle.ofdm(W, S, wl.nb, n=wl.n, cp=wl.cp, scale=scale, group_idx=tags, n_threads=NT)
    for e in (12, 3, 22):
        op.set_output("i16", e)
        y16 = op.apply(Sd, td)
        torch.cuda.synchronize()
        assert y16.dtype == torch.int16 and tuple(y16.shape) == (6, 64, 2192, 2)
        got = y16.cpu().numpy()
        comp = np.stack([y32.real, y32.imag], axis=-1).astype(np.float32) * np.float32(2.0 ** e)
        want = np.clip(np.rint(comp), -32768, 32767).astype(np.int16)     # rint: half to even
        assert (got == want).all(), e
        if e == 12:
            assert np.abs(comp).max() < 32767            # no saturation at the bench's exponent
            yq = (got[..., 0].astype(np.float64) + 1j * got[..., 1]) / 2.0 ** e
            err = np.abs(yq - y_ref.astype(np.complex128)).max(axis=2)
            assert (err <= 2.0 ** -(e + 1) * np.sqrt(2) + TOL * bound).all()
        if e == 22:
            assert (np.abs(got) == 32767).any() or (got == -32768).any()
    op.set_output("f32")
    assert op.apply(Sd, td).dtype == torch.complex64
    from paper_1810_11451_b200.ofdm import _lib
    assert _lib().bf_ofdm_plan_set_output(op._h, 2, 0) == Status.INVALID_VALUE
    assert _lib().bf_ofdm_plan_set_output(op._h, 1, 200) == Status.INVALID_VALUE
    op.close()
    plan.close()


def test_int16_output_needs_the_default_kernel(monkeypatch):
    monkeypatch.setenv("BFO_OFDM_KERNEL", "sb")
    plan = Plan(4)
    op = OfdmPlan(plan, 2)
    from paper_1810_11451_b200.ofdm import _lib
    assert _lib().bf_ofdm_plan_set_output(op._h, 1, 12) == Status.UNSUPPORTED
