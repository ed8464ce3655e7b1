"""GPU parity: libbf.so (through the C ABI binding) against the CPU oracle.

Every case uses seeded bf_synth inputs.  Small cases compare every element;
full BASELINE.json sizes run in the bench's launch configuration and compare
sampled blocks (regenerated on the host by block id) plus properties.
Tolerance: |R_gpu - R_ref| <= 1e-5 * T element-wise (BASELINE.json north_star
item 4); bitwise for f = 0 and copy-like W (identity, selection, permutation).
"""
import os

import numpy as np
import pytest

import bf_synth as syn
import oracle
from helpers import TOL, assert_bitwise, assert_parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():   # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import bf_synth.cuda as sync  # noqa: E402
import paper_1810_11451_b200 as bf  # noqa: E402
from paper_1810_11451_b200 import Layout, Plan, Variant  # noqa: E402

DEV = torch.device("cuda", 0)
NT = oracle.max_threads()
VARIANTS = [Variant.FFMA, Variant.TENSOR]


@pytest.fixture(params=VARIANTS, ids=lambda v: v.name.lower())
def variant(request):
    return request.param


def run_plan(W, S, tags=None, layout=Layout.INTERLEAVED, variant=Variant.AUTO):
    """Device run of the numpy inputs; returns R as complex64 numpy [n][64][60]."""
    f = W.shape[-1]
    plan = Plan(f=f, layout=layout, variant=variant)
    if layout == Layout.PLANAR:
        Wd = torch.from_numpy(syn.to_planar(W)).to(DEV)
        Sd = torch.from_numpy(syn.to_planar(S)).to(DEV)
    else:
        Wd = torch.from_numpy(np.ascontiguousarray(W)).to(DEV)
        Sd = torch.from_numpy(np.ascontiguousarray(S)).to(DEV)
    plan.set_precoders(Wd)
    td = None if tags is None else torch.from_numpy(tags).to(DEV)
    R = plan.apply(Sd, td)
    torch.cuda.synchronize()
    R = R.cpu().numpy()
    plan.close()
    return syn.from_planar(R) if layout == Layout.PLANAR else R


# ---------------------------------------------------------------------------
# full-element parity at oracle-friendly sizes
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("layout", [Layout.INTERLEAVED, Layout.PLANAR])
def test_c1_full(layout, variant):
    wl = syn.workload("c1")
    W, S, _ = syn.workload_inputs(wl)
    R_ref, T, _ = oracle.beamform(W, S, n_threads=NT)
    R = run_plan(W, S, layout=layout, variant=variant)
    assert_parity(R, R_ref, T, what="c1")


def test_c2_full(variant):
    wl = syn.workload("c2")
    W, S, _ = syn.workload_inputs(wl)
    R_ref, T, _ = oracle.beamform(W, S, n_threads=NT)
    R = run_plan(W, S, variant=variant)
    worst = assert_parity(R, R_ref, T, what="c2")
    # both paths sit far inside the 1e-5 bound
    assert worst < (1e-6 if variant == Variant.FFMA else 4e-6), worst


@pytest.mark.parametrize("layout", [Layout.INTERLEAVED, Layout.PLANAR])
@pytest.mark.parametrize("f", syn.C3_FLOWS)
def test_c3_every_f_ragged(f, layout, variant):
    """Every f of the sweep at a ragged block count spanning several CTAs' ranges."""
    wl = syn.workload("c3", f)
    ids = np.arange(0, 1237)
    W, S, _ = syn.workload_inputs(wl, ids)
    R_ref, T, _ = oracle.beamform(W, S, n_threads=NT)
    R = run_plan(W, S, layout=layout, variant=variant)
    if f == 0:
        assert not R.view(np.uint32).any()
    assert_parity(R, R_ref, T, what=f"c3 f={f}")


@pytest.mark.parametrize("f", list(range(1, 37)))
def test_every_instantiation(f, variant):
    """Each of the 36 compiled f values (odd K, non-powers of two) against the oracle."""
    W = syn.precoders(99, f, 3, 64, f, "unit_columns")
    S = syn.qam_symbols(99, f, np.arange(41), f, 60, 64)
    tags = syn.subband_tags(99, np.arange(41), 3)
    R_ref, T, _ = oracle.beamform(W, S, tags, n_threads=NT)
    assert_parity(run_plan(W, S, tags, variant=variant), R_ref, T, what=f"f={f}")
    assert_parity(run_plan(W, S, tags, Layout.PLANAR, variant), R_ref, T, what=f"f={f} planar")


def test_grouped_small_full(variant):
    """c4 shape (55 groups, tags) at a size the oracle covers completely."""
    wl = syn.workload("c4")
    ids = np.arange(3001)
    W, S, tags = syn.workload_inputs(wl, ids)
    R_ref, T, _ = oracle.beamform(W, S, tags, n_threads=NT)
    assert_parity(run_plan(W, S, tags, variant=variant), R_ref, T, what="c4 small")


# ---------------------------------------------------------------------------
# exactness fixtures (bitwise)
# ---------------------------------------------------------------------------
def test_f0_is_positive_zero():
    plan = Plan(f=0)
    plan.set_precoders(torch.zeros((1, 64, 0), dtype=torch.complex64, device=DEV))
    R = torch.full((7, 64, 60), float("nan"), dtype=torch.complex64, device=DEV)
    plan.apply(torch.zeros((7, 0, 60), dtype=torch.complex64, device=DEV), out=R)
    torch.cuda.synchronize()
    assert not R.cpu().numpy().view(np.uint32).any()


@pytest.mark.parametrize("layout", [Layout.INTERLEAVED, Layout.PLANAR])
@pytest.mark.parametrize("f", [1, 8, 17, 36])
def test_identity_and_selection_bitwise(f, layout, variant):
    S = syn.qam_symbols(5, 0, np.arange(50), f, 60, 64)
    W = np.zeros((2, 64, f), np.complex64)
    W[0, np.arange(f), np.arange(f)] = 1                   # identity [I_f; 0]
    rng = np.random.default_rng(f)
    sigma = rng.integers(0, f, size=64)
    sigma[:f] = rng.permutation(f)
    W[1, np.arange(64), sigma] = 1                          # selection / permutation
    tags = (np.arange(50) % 2).astype(np.int32)
    R = run_plan(W, S, tags, layout, variant)
    R_ref, _, _ = oracle.beamform(W, S, tags)
    assert_bitwise(R, R_ref, "copy-like W vs oracle")
    assert_bitwise(R[0::2, :f], S[0::2], "identity rows")
    assert not R[0::2, f:].view(np.uint32).any()
    assert_bitwise(R[1::2], S[1::2][:, sigma], "selection rows")


def test_gaussian_integers_bitwise_at_full_shape(variant):
    """Integer partial sums < 2^24 are exact in any order: GPU == oracle bitwise."""
    rng = np.random.default_rng(3)
    G, f = 55, 36
    W = (rng.integers(-3, 4, (G, 64, f)) + 1j * rng.integers(-3, 4, (G, 64, f))).astype(np.complex64)
    S = syn.qam_symbols(11, 0, np.arange(500), f, 60, 64, normalised=False)
    tags = syn.subband_tags(3, np.arange(500), G)
    R_ref, _, _ = oracle.beamform(W, S, tags, n_threads=NT)
    assert_bitwise(run_plan(W, S, tags, variant=variant), R_ref, "gaussian integers")


def test_power_of_two_scaling_and_one_real_nonzero(variant):
    wl = syn.workload("c2")
    W, S, _ = syn.workload_inputs(wl, np.arange(64))
    R1 = run_plan(W, S, variant=variant)
    R2 = run_plan((W * np.float32(4.0)).astype(np.complex64), S, variant=variant)
    assert_bitwise(R2, R1 * np.float32(4.0), "2^e scaling")
    f = 12
    rng = np.random.default_rng(2)
    sigma = rng.integers(0, f, size=64)
    Wc = np.zeros((1, 64, f), np.complex64)
    Wc[0, np.arange(64), sigma] = rng.standard_normal(64).astype(np.float32)
    S = syn.qam_symbols(9, 0, np.arange(20), f, 60, 64)
    R_ref, T, _ = oracle.beamform(Wc, S)
    if variant == Variant.FFMA:     # one fused product, correctly rounded
        assert_bitwise(run_plan(Wc, S, variant=variant), R_ref, "one real nonzero per row")
    else:                           # split-precision product: within the contract
        assert_parity(run_plan(Wc, S, variant=variant), R_ref, T, what="one real nonzero")


def test_conjugation_symmetry_bitwise(variant):
    wl = syn.workload("c2")
    W, S, _ = syn.workload_inputs(wl, np.arange(32))
    R = run_plan(W, S, variant=variant)
    Rc = run_plan(np.conj(W), np.conj(S), variant=variant)
    assert_bitwise(Rc, np.conj(R), "conjugation symmetry")


def test_linearity_in_S_and_W(variant):
    wl = syn.workload("c3", 24)
    W, S1, _ = syn.workload_inputs(wl, np.arange(30))
    S2 = syn.qam_symbols(8, 1, np.arange(30), 24, 60, 64)
    W2 = syn.precoders(8, 2, 1, 64, 24, "unit_columns")
    R_ref, T, _ = oracle.beamform(W, S1 + S2, n_threads=NT)
    R = run_plan(W, S1, variant=variant) + run_plan(W, S2, variant=variant)
    assert_parity(R, R_ref, T, tol=2 * TOL, what="linearity in S")
    R_ref, T, _ = oracle.beamform(W + W2, S1, n_threads=NT)
    R = run_plan(W, S1, variant=variant) + run_plan(W2, S1, variant=variant)
    assert_parity(R, R_ref, T, tol=2 * TOL, what="linearity in W")


# ---------------------------------------------------------------------------
# properties: determinism, batch independence, layouts, host path
# ---------------------------------------------------------------------------
def test_determinism_and_batch_independence(variant):
    wl = syn.workload("c4")
    W, S, tags = syn.workload_inputs(wl, np.arange(2000))
    a = run_plan(W, S, tags, variant=variant)
    b = run_plan(W, S, tags, variant=variant)
    assert_bitwise(a, b, "repeat")
    c = run_plan(W, S[701:1300], tags[701:1300], variant=variant)
    assert_bitwise(c, a[701:1300], "sub-batch")
    d = run_plan(W, S[:1], tags[:1], variant=variant)
    assert_bitwise(d, a[:1], "single block")


def test_planar_equals_interleaved_bitwise(variant):
    wl = syn.workload("c3", 31)
    W, S, _ = syn.workload_inputs(wl, np.arange(300))
    assert_bitwise(run_plan(W, S, layout=Layout.PLANAR, variant=variant),
                   run_plan(W, S, variant=variant), "layouts")


def test_device_generator_matches_host_generator():
    for wl, planar in ((syn.workload("c4"), False), (syn.workload("c3", 17), True),
                       (syn.workload("c1"), False)):
        ids = np.array([0, 1, 2, 777, wl.n_blocks - 1], dtype=np.int64)
        Sd, td = sync.workload_device(wl, DEV, ids=torch.from_numpy(ids).to(DEV), planar=planar)
        _, S, tags = syn.workload_inputs(wl, ids)
        got = Sd.cpu().numpy()
        assert_bitwise(syn.from_planar(got) if planar else got, S, f"generator {wl.name}")
        if tags is not None:
            assert np.array_equal(td.cpu().numpy(), tags)
    ids = np.arange(5000, 5100, dtype=np.int64)
    m = torch.empty(100, dtype=torch.int32, device=DEV)
    sync.gen_modulations(m, 4, ids=torch.from_numpy(ids).to(DEV))
    assert np.array_equal(m.cpu().numpy(), syn.block_modulations(4, ids))
    S = torch.empty((100, 20, 60), dtype=torch.complex64, device=DEV)
    sync.gen_symbols(S, 4, 3, 20, 60, 0, ids=torch.from_numpy(ids).to(DEV))
    assert_bitwise(S.cpu().numpy(),
                   syn.qam_symbols(4, 3, ids, 20, 60, syn.block_modulations(4, ids)), "mixed QAM")


@pytest.mark.parametrize("tagged", [False, True])
def test_apply_host_equals_apply(tagged, variant):
    wl = syn.workload("c4")
    W, S, tags = syn.workload_inputs(wl, np.arange(5000))
    if not tagged:
        W, tags = W[:1], None
    plan = Plan(f=36, variant=variant)
    plan.set_host_chunk(1024)     # several chunks, ragged tail, all three slots
    plan.set_precoders(torch.from_numpy(W).to(DEV))
    S_h = torch.from_numpy(S).pin_memory()
    t_h = None if tags is None else torch.from_numpy(tags).pin_memory()
    R_h = torch.empty((5000, 64, 60), dtype=torch.complex64).pin_memory()
    plan.apply_host(S_h, t_h, R_h)
    torch.cuda.synchronize()
    Rd = plan.apply(torch.from_numpy(S).to(DEV), None if tags is None else t_h.to(DEV))
    torch.cuda.synchronize()
    assert_bitwise(R_h.numpy(), Rd.cpu().numpy(), "host pipeline")
    plan.close()


# ---------------------------------------------------------------------------
# routing (a3): bit-exact index work
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n,G", [(1, 55), (4095, 55), (4097, 2), (100_003, 55), (70_000, 1024)])
def test_route_is_stable_counting_sort(n, G):
    tags = syn.subband_tags(12, np.arange(n), G)
    plan = Plan(f=4)
    plan.set_precoders(torch.zeros((G, 64, 4), dtype=torch.complex64, device=DEV))
    perm, offs = plan.route(torch.from_numpy(tags).to(DEV))
    torch.cuda.synchronize()
    assert np.array_equal(perm.cpu().numpy(), np.argsort(tags, kind="stable"))
    starts = np.concatenate([[0], np.cumsum(np.bincount(tags, minlength=G))])
    assert np.array_equal(offs.cpu().numpy(), np.concatenate([starts, [n]]))


def test_invalid_tags_are_left_unwritten_and_checked(monkeypatch, variant):
    wl = syn.workload("c4")
    W, S, tags = syn.workload_inputs(wl, np.arange(300))
    tags = tags.copy()
    tags[[5, 17]] = [55, -1]
    plan = Plan(f=36, variant=variant)
    plan.set_precoders(torch.from_numpy(W).to(DEV))
    Sd, td = torch.from_numpy(S).to(DEV), torch.from_numpy(tags).to(DEV)
    R = torch.full((300, 64, 60), 7.0, dtype=torch.complex64, device=DEV)
    plan.apply(Sd, td, out=R)
    torch.cuda.synchronize()
    Rn = R.cpu().numpy()
    assert (Rn[[5, 17]] == 7.0).all()
    ok = np.setdiff1d(np.arange(300), [5, 17])
    R_ref, T, _ = oracle.beamform(W, S[ok], tags[ok], n_threads=NT)
    assert_parity(Rn[ok], R_ref, T, what="valid blocks beside invalid tags")
    monkeypatch.setenv("BF_CHECK", "1")
    with pytest.raises(bf.BfError) as e:
        plan.apply(Sd, td, out=R)
    assert e.value.status == bf.Status.INVALID_VALUE


@pytest.mark.parametrize("layout", [Layout.INTERLEAVED, Layout.INTERLEAVED_I16OUT])
def test_f0_with_tags_honours_invalid_tags(monkeypatch, layout):
    """f = 0 with tags: validly tagged blocks become +0.0, blocks with tags outside
    [0, n_groups) are left unwritten (bf.h), and BF_CHECK=1 reports them."""
    n, G = 77, 3
    plan = Plan(f=0, layout=layout)
    plan.set_precoders(torch.zeros((G, 64, 0), dtype=torch.complex64, device=DEV))
    tags = (np.arange(n) % G).astype(np.int32)
    tags[[4, 50]] = [G, -2]
    td = torch.from_numpy(tags).to(DEV)
    shape = plan.r_shape(n)
    R = torch.full(shape, 7, dtype=plan.r_dtype, device=DEV)
    plan.apply(torch.zeros((n, 0, 60), dtype=torch.complex64, device=DEV), td, out=R)
    torch.cuda.synchronize()
    Rn = R.cpu().numpy().reshape(n, -1)
    assert (Rn[[4, 50]] == 7).all()
    ok = np.setdiff1d(np.arange(n), [4, 50])
    assert not Rn[ok].view(np.uint16 if Rn.dtype.itemsize == 2 else np.uint32).any()
    monkeypatch.setenv("BF_CHECK", "1")
    with pytest.raises(bf.BfError) as e:
        plan.apply(torch.zeros((n, 0, 60), dtype=torch.complex64, device=DEV), td, out=R)
    assert e.value.status == bf.Status.INVALID_VALUE
    plan.close()


def test_invalid_tags_with_one_group(variant):
    """One precoder group and tags: the tags are still honoured (bf.h), so a tag other than 0
    leaves its block unwritten — the single-group shortcut applies only to group_idx = NULL.
    Found by tools/stress_tc.py."""
    W = syn.precoders(8, 12, 1, 64, 12, "unit_columns")
    S = syn.qam_symbols(8, 12, np.arange(50), 12, 60, 64)
    tags = np.zeros(50, np.int32)
    tags[[3, 40]] = [1, -7]
    plan = Plan(f=12, variant=variant)
    plan.set_precoders(torch.from_numpy(W).to(DEV))
    R = torch.full((50, 64, 60), 7.0, dtype=torch.complex64, device=DEV)
    plan.apply(torch.from_numpy(S).to(DEV), torch.from_numpy(tags).to(DEV), out=R)
    torch.cuda.synchronize()
    Rn = R.cpu().numpy()
    assert (Rn[[3, 40]] == 7.0).all()
    ok = np.setdiff1d(np.arange(50), [3, 40])
    R_ref, T, _ = oracle.beamform(W, S[ok], None, n_threads=NT)
    assert_parity(Rn[ok], R_ref, T, what="one group, valid tags")
    plan.close()


# ---------------------------------------------------------------------------
# error paths of the C ABI
# ---------------------------------------------------------------------------
def test_error_paths():
    L = bf.lib()
    plan = Plan(f=8)
    S = torch.zeros((4, 8, 60), dtype=torch.complex64, device=DEV)
    with pytest.raises(bf.BfError) as e:
        plan.apply(S)
    assert e.value.status == bf.Status.NO_PRECODERS
    plan.set_precoders(torch.zeros((64, 8), dtype=torch.complex64, device=DEV))
    buf = torch.zeros(4 * 8 * 60 * 2 + 2, dtype=torch.float32, device=DEV)
    R = torch.zeros((4, 64, 60), dtype=torch.complex64, device=DEV)
    import ctypes
    st = L.bf_apply(plan._h, ctypes.c_void_p(buf.data_ptr() + 8), None,
                    ctypes.c_void_p(R.data_ptr()), 4, None)
    assert st == bf.Status.MISALIGNED
    big = torch.zeros(4 * 7680 + 4 * 960, dtype=torch.float32, device=DEV)
    st = L.bf_apply(plan._h, ctypes.c_void_p(big.data_ptr()), None,
                    ctypes.c_void_p(big.data_ptr() + 4 * 960 * 4 - 512), 4, None)
    assert st == bf.Status.INVALID_VALUE                     # R overlaps S
    assert L.bf_apply(plan._h, None, None, None, 0, None) == bf.Status.OK   # n = 0 no-op
    assert L.bf_apply(plan._h, None, None, ctypes.c_void_p(R.data_ptr()), -1, None) == \
        bf.Status.INVALID_VALUE
    assert L.bf_set_precoders(plan._h, ctypes.c_void_p(R.data_ptr()), 1025, None) == \
        bf.Status.UNSUPPORTED
    with pytest.raises(ValueError):
        plan.apply(torch.zeros((4, 7, 60), dtype=torch.complex64, device=DEV))
    plan.close()


# ---------------------------------------------------------------------------
# full BASELINE.json sizes in the bench's launch configuration, sampled parity
# ---------------------------------------------------------------------------
def _bound_T(W, S, tags):
    """T = sum_k |w_ik| |s_kj| in fp64 (the tolerance scale) as a matrix product of the
    moduli — the same quantity the oracle's bound output holds, computed faster for the
    large samples below."""
    g = np.zeros(len(S), np.int64) if tags is None else tags.astype(np.int64)
    return np.matmul(np.abs(W.astype(np.complex128))[g], np.abs(S.astype(np.complex128)))


def _check_ids(wl, R_dev, ids, planar=False, chunk=4096):
    worst = 0.0
    for c0 in range(0, len(ids), chunk):
        part = ids[c0:c0 + chunk]
        W, S, tags = syn.workload_inputs(wl, part)
        R_ref, _, _ = oracle.beamform(W, S, tags, n_threads=NT, bound=False)
        got = R_dev[torch.from_numpy(part).to(R_dev.device)].cpu().numpy()
        if planar:
            got = syn.from_planar(got)
        worst = max(worst, assert_parity(got, R_ref, _bound_T(W, S, tags), what=f"{wl.name} sampled"))
    return worst


def _sampled_check(wl, R_dev, n_sample=96, planar=False, seed=0):
    rng = np.random.default_rng(seed)
    n = wl.n_blocks
    ids = np.unique(np.concatenate([[0, 1, n - 2, n - 1], rng.integers(0, n, n_sample)]))
    return _check_ids(wl, R_dev, ids, planar)


@pytest.mark.slow
def test_c4_full_size_sampled(variant):
    """c4 at full size (2^20 blocks, 55 groups) in the bench's launch configuration: every
    16th block (65 536, SURVEY.md §8(d)'s 1/16 sample) plus the first and last against the
    oracle, and every block written."""
    wl = syn.workload("c4")
    W = syn.precoders(wl.seed, wl.sub, wl.n_groups, wl.n_ant, wl.f, wl.w_norm)
    Sd, td = sync.workload_device(wl, DEV)
    plan = Plan(f=36, variant=variant)
    plan.set_precoders(torch.from_numpy(W).to(DEV))
    R = plan.apply(Sd, td)
    torch.cuda.synchronize()
    del Sd
    ids = np.unique(np.concatenate([np.arange(0, wl.n_blocks, 16), [1, wl.n_blocks - 1]]))
    _check_ids(wl, R, ids)
    # property at full size: every block was written (no NaN sentinel survives)
    assert torch.isfinite(torch.view_as_real(R)).all().item()
    plan.close()


@pytest.mark.slow
@pytest.mark.parametrize("f", [1, 7, 16, 36])
@pytest.mark.parametrize("layout", [Layout.INTERLEAVED, Layout.PLANAR])
def test_c3_full_size_sampled(f, layout, variant):
    wl = syn.workload("c3", f)
    planar = layout == Layout.PLANAR
    W = syn.precoders(wl.seed, wl.sub, 1, 64, f, wl.w_norm)
    Sd, _ = sync.workload_device(wl, DEV, planar=planar)
    plan = Plan(f=f, layout=layout, variant=variant)
    plan.set_precoders(torch.from_numpy(syn.to_planar(W) if planar else W).to(DEV))
    R = plan.apply(Sd)
    torch.cuda.synchronize()
    _sampled_check(wl, R, planar=planar)
    plan.close()


@pytest.mark.slow
def test_c5_sampled_chunks(variant):
    """c5: every 64th 4096-block chunk (32 chunks, all 8 cells, per-cell f, mixed modulation,
    55 tagged groups) applied on its own; every 8th block of each against the oracle."""
    wl = syn.workload("c5")
    fc = syn.cell_flows(wl.seed, 8)
    plans = {}
    for chunk in range(0, 2048, 64):
        cell = (chunk // 64 + chunk) % 8                     # spread the sample over the cells
        chunk = chunk + (cell - chunk % 8) % 8
        f = int(fc[cell])
        ids = np.arange(chunk * 4096, (chunk + 1) * 4096, dtype=np.int64)
        W = syn.precoders(wl.seed, cell, 55, 64, f, "none")
        Sd = torch.empty((4096, f, 60), dtype=torch.complex64, device=DEV)
        sync.gen_symbols(Sd, wl.seed, 0, f, 60, 0, first=int(ids[0]))
        td = torch.empty(4096, dtype=torch.int32, device=DEV)
        sync.gen_tags(td, wl.seed, 55, first=int(ids[0]))
        if cell not in plans:
            plans[cell] = Plan(f=f, variant=variant)
            plans[cell].set_precoders(torch.from_numpy(W).to(DEV))
        R = plans[cell].apply(Sd, td)
        torch.cuda.synchronize()
        sel = np.arange(0, 4096, 8)
        S = syn.qam_symbols(wl.seed, 0, ids[sel], f, 60, syn.block_modulations(wl.seed, ids[sel]))
        tags = syn.subband_tags(wl.seed, ids[sel], 55)
        R_ref, _, _ = oracle.beamform(W, S, tags, n_threads=NT, bound=False)
        assert_parity(R[torch.from_numpy(sel).to(DEV)].cpu().numpy(), R_ref, _bound_T(W, S, tags),
                      what=f"c5 chunk {chunk} (cell {cell}, f={f})")
    for p in plans.values():
        p.close()


def test_variants_agree_within_contract():
    """The two kernels differ only by rounding: |R_ffma - R_tc| <= 2e-5 T and equal on copies."""
    wl = syn.workload("c4")
    W, S, tags = syn.workload_inputs(wl, np.arange(900))
    R_ref, T, _ = oracle.beamform(W, S, tags, n_threads=NT)
    a = run_plan(W, S, tags, variant=Variant.FFMA)
    b = run_plan(W, S, tags, variant=Variant.TENSOR)
    assert_parity(a, b, T, tol=2 * TOL, what="ffma vs tensor")
    p = Plan(f=36)
    assert p.variant in (Variant.FFMA, Variant.TENSOR)
    p.set_variant("tensor")
    assert p.variant == Variant.TENSOR
    p.close()


# ---------------------------------------------------------------------------
# fp16 output (BF_LAYOUT_INTERLEAVED_F16OUT)
# ---------------------------------------------------------------------------
def run_f16(W, S, tags, variant):
    plan = Plan(f=W.shape[-1], layout=Layout.INTERLEAVED_F16OUT, variant=variant)
    plan.set_precoders(torch.from_numpy(np.ascontiguousarray(W)).to(DEV))
    R = plan.apply(torch.from_numpy(np.ascontiguousarray(S)).to(DEV),
                   None if tags is None else torch.from_numpy(tags).to(DEV))
    torch.cuda.synchronize()
    plan.close()
    h = R.cpu().numpy().astype(np.float64)
    return h[..., 0] + 1j * h[..., 1]


def test_f16_output_within_contract(variant):
    """|R16 - R_exact| <= sqrt(2) 2^-11 |R_exact| + 1e-5 T (+ fp16 subnormal spacing)."""
    wl = syn.workload("c4")
    W, S, tags = syn.workload_inputs(wl, np.arange(701))
    R_ref, T, _ = oracle.beamform(W, S, tags, n_threads=NT)
    R16 = run_f16(W, S, tags, variant)
    lim = np.sqrt(2) * 2.0 ** -11 * np.abs(R_ref.astype(np.complex128)) + TOL * T + 2.0 ** -24
    err = np.abs(R16 - R_ref.astype(np.complex128))
    assert (err <= lim).all(), (err / lim).max()
    # and it is the fp32 result rounded once: compare with the fp32 path rounded on the host
    R32 = run_plan(W, S, tags, variant=variant)
    expect = R32.real.astype(np.float16).astype(np.float64) + 1j * R32.imag.astype(np.float16).astype(np.float64)
    assert np.array_equal(R16, expect)


@pytest.mark.parametrize("f", [1, 17, 36])
def test_f16_output_identity_is_rounded_copy(f, variant):
    S = syn.qam_symbols(5, 0, np.arange(30), f, 60, 64)
    W = np.zeros((1, 64, f), np.complex64)
    W[0, np.arange(f), np.arange(f)] = 1
    R16 = run_f16(W, S, None, variant)
    exp = S.real.astype(np.float16).astype(np.float64) + 1j * S.imag.astype(np.float16).astype(np.float64)
    assert np.array_equal(R16[:, :f], exp)
    assert not np.any(R16[:, f:])


def test_apply_routed_equals_apply(variant):
    """bf_route on one stream + bf_apply_routed on another == bf_apply, bitwise."""
    wl = syn.workload("c4")
    W, S, tags = syn.workload_inputs(wl, np.arange(1500))
    plan = Plan(f=36, variant=variant)
    plan.set_precoders(torch.from_numpy(W).to(DEV))
    Sd, td = torch.from_numpy(S).to(DEV), torch.from_numpy(tags).to(DEV)
    ref = plan.apply(Sd, td)
    side = torch.cuda.Stream()
    perm = torch.empty(1500, dtype=torch.int32, device=DEV)
    offs = torch.empty(57, dtype=torch.int32, device=DEV)
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        plan.route_into(td, perm, offs)
    torch.cuda.current_stream().wait_stream(side)
    got = plan.apply_routed(Sd, perm, offs)
    untagged = plan.apply_routed(Sd[:10], None, None)
    torch.cuda.synchronize()
    assert_bitwise(got.cpu().numpy(), ref.cpu().numpy(), "routed")
    R_ref, T, _ = oracle.beamform(W[0], S[:10], n_threads=NT)
    assert_parity(untagged.cpu().numpy(), R_ref, T, what="untagged routed")
    plan.close()


def test_sm_share_concurrent_plans_bitwise(variant):
    """bf_plan_set_sm_share: plans of different f on their own streams, each on a share of
    the SMs, running side by side; results equal the default full-grid applies bitwise."""
    shares, fs = [5, 37, 1, 200], [3, 36, 17, 8]
    plans, ins, refs = [], [], []
    for i, (sh, f) in enumerate(zip(shares, fs)):
        W = syn.precoders(41, i, 4, 64, f, "unit_columns")
        S = syn.qam_symbols(41, i, np.arange(2003), f, 60, 16)
        tags = syn.subband_tags(41, np.arange(2003) + i, 4)
        p = Plan(f=f, variant=variant)
        p.set_precoders(torch.from_numpy(W).to(DEV))
        Sd, td = torch.from_numpy(S).to(DEV), torch.from_numpy(tags).to(DEV)
        refs.append(p.apply(Sd, td))
        p.set_sm_share(sh)
        cfg = p.kernel_config(2003)
        sms = torch.cuda.get_device_properties(DEV).multi_processor_count
        assert cfg["grid"] == min(sh, sms) * cfg["ctas_per_sm"]
        plans.append(p)
        ins.append((Sd, td))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in plans]
    outs = []
    for p, (Sd, td), st in zip(plans, ins, streams):
        with torch.cuda.stream(st):
            outs.append(p.apply(Sd, td))
    torch.cuda.synchronize()
    for i, (got, ref) in enumerate(zip(outs, refs)):
        assert_bitwise(got.cpu().numpy(), ref.cpu().numpy(), f"share {shares[i]}")
    W = syn.precoders(41, 0, 4, 64, fs[0], "unit_columns")
    S = syn.qam_symbols(41, 0, np.arange(2003), fs[0], 60, 16)
    R_ref, T, _ = oracle.beamform(W, S, syn.subband_tags(41, np.arange(2003), 4), n_threads=NT)
    assert_parity(outs[0].cpu().numpy(), R_ref, T, what="sm share 5")
    with pytest.raises(bf.BfError):
        plans[0].set_sm_share(-1)
    for p in plans:
        p.close()


@pytest.mark.parametrize("n,G,share", [(1, 1, 0), (3, 55, 0), (7, 5, 3), (150, 55, 0), (301, 1024, 0),
                                       (4096, 55, 146), (4097, 2, 7), (5000, 300, 148)])
def test_cost_balanced_partition_covers_every_block(n, G, share):
    """The tensor kernel splits the group-sorted list over CTAs by tiles + W reloads: every
    valid block is written exactly as by a single-CTA launch (empty groups, one-block groups,
    more CTAs than tiles, many groups)."""
    f = 12
    ids = np.arange(n)
    W = syn.precoders(7, G, G, 64, f, "unit_columns")
    S = syn.qam_symbols(7, G, ids, f, 60, 16)
    tags = syn.subband_tags(7, ids, G)
    if G > 3:
        tags[tags % 3 == 1] = 0          # leave some groups empty, make group 0 large
    Sd, td = torch.from_numpy(S).to(DEV), torch.from_numpy(tags).to(DEV)
    outs = []
    for sh in (share, 1):
        plan = Plan(f=f, variant=Variant.TENSOR)
        plan.set_precoders(torch.from_numpy(W).to(DEV))
        plan.set_sm_share(sh)
        R = torch.full((n, 64, 60), float("nan"), dtype=torch.complex64, device=DEV)
        plan.apply(Sd, td, out=R)
        torch.cuda.synchronize()
        outs.append(R.cpu().numpy())
        plan.close()
    assert np.isfinite(outs[0].view(np.float32)).all()
    assert_bitwise(outs[0], outs[1], f"n={n} G={G} share={share}")
    R_ref, T, _ = oracle.beamform(W, S, tags, n_threads=NT)
    assert_parity(outs[0], R_ref, T, what=f"partition n={n} G={G}")


@pytest.mark.parametrize("layout", [Layout.INTERLEAVED, Layout.PLANAR, Layout.INTERLEAVED_F16OUT,
                                    Layout.INTERLEAVED_I16OUT])
@pytest.mark.parametrize("f", [1, 7, 36])
def test_no_write_outside_R(f, layout, variant):
    """Out-of-bounds write check (compute-sanitizer is closed on this pool): R is a slice of
    a larger buffer whose guard bands hold a sentinel pattern; after tagged and untagged
    applies at ragged sizes the guards are untouched, and every byte of R was written."""
    n, guard = 333, 4096
    W = syn.precoders(11, f, 5, 64, f, "unit_columns")
    S = syn.qam_symbols(11, f, np.arange(n), f, 60, 16)
    tags = syn.subband_tags(11, np.arange(n), 5)
    plan = Plan(f=f, layout=layout, variant=variant)
    Wd = torch.from_numpy(syn.to_planar(W) if layout == Layout.PLANAR else W).to(DEV)
    Sd = torch.from_numpy(syn.to_planar(S) if layout == Layout.PLANAR else S).to(DEV)
    plan.set_precoders(Wd)
    r_words = int(np.prod(plan.r_shape(n))) * torch.empty((), dtype=plan.r_dtype).element_size() // 4
    for td in (None, torch.from_numpy(tags).to(DEV)):
        buf = torch.full((guard + r_words + guard,), 0x7FC0DEAD, dtype=torch.int32, device=DEV)
        R = buf[guard:guard + r_words].view(plan.r_dtype).view(plan.r_shape(n))
        plan.apply(Sd, td, out=R)
        torch.cuda.synchronize()
        h = buf.cpu().numpy()
        assert (h[:guard] == 0x7FC0DEAD).all() and (h[guard + r_words:] == 0x7FC0DEAD).all()
        assert not (h[guard:guard + r_words] == 0x7FC0DEAD).any(), "R not fully written"
    plan.close()


@pytest.mark.parametrize("layout", [Layout.INTERLEAVED, Layout.PLANAR, Layout.INTERLEAVED_F16OUT,
                                    Layout.INTERLEAVED_I16OUT])
def test_apply_batch_equals_routed_applies(layout):
    """bf_apply_batch over 19 jobs (more than one pack of 16): plans of different f, tagged
    and untagged, f = 0, an FFMA-forced plan, an empty job, a plan used twice — bitwise equal
    to the jobs' own bf_apply_routed calls, and within the contract of the oracle."""
    planar = layout == Layout.PLANAR
    specs = [(36, 55, 700), (1, 1, 33), (7, 5, 129), (0, 1, 9), (17, 3, 1), (36, 55, 0),
             (12, 300, 901), (3, 2, 64)] + [(f, 4, 40 + f) for f in (5, 9, 20, 24, 31, 33, 35, 2, 13, 30, 36)]
    plans, jobs, refs, host = {}, [], [], []
    for i, (f, G, n) in enumerate(specs):
        key = (f, G)
        if key not in plans:
            pl = Plan(f=f, layout=layout, variant=Variant.FFMA if (f, G) == (17, 3) else Variant.AUTO)
            W = syn.precoders(21, i, G, 64, f, "unit_columns")
            pl.set_precoders(torch.from_numpy(syn.to_planar(W) if planar else W).to(DEV))
            plans[key] = (pl, W)
        pl, W = plans[key]
        S = syn.qam_symbols(21, 100 + i, np.arange(n), f, 60, 64)
        Sd = torch.from_numpy(syn.to_planar(S) if planar else S).to(DEV)
        perm = offs = None
        tags = None
        if G > 1 and n > 0:
            tags = syn.subband_tags(21, np.arange(n) + 7 * i, G)
            perm, offs = pl.route(torch.from_numpy(tags).to(DEV))
        out = torch.full(pl.r_shape(n), 7.0, dtype=pl.r_dtype, device=DEV)
        # a batch runs AUTO plans on the tensor kernel (AUTO may pick FFMA at small f)
        forced = pl.variant != Variant.TENSOR and (f, G) != (17, 3)
        if forced:
            pl.set_variant(Variant.TENSOR)
        ref = pl.apply_routed(Sd, perm, offs) if n > 0 else out.clone()
        if forced:
            pl.set_variant(Variant.AUTO)
        jobs.append((pl, Sd, perm, offs, out))
        refs.append(ref)
        host.append((W, S, tags))
    torch.cuda.synchronize()
    bf.apply_batch(jobs)
    torch.cuda.synchronize()
    for i, ((_, _, _, _, out), ref) in enumerate(zip(jobs, refs)):
        assert_bitwise(out.cpu().numpy(), ref.cpu().numpy(), f"job {i} {specs[i]}")
    if layout == Layout.INTERLEAVED:
        for i in (0, 2, 6, 12):
            W, S, tags = host[i]
            R_ref, T, _ = oracle.beamform(W, S, tags, n_threads=NT)
            assert_parity(jobs[i][4].cpu().numpy(), R_ref, T, what=f"batch job {i}")
    for pl, _ in plans.values():
        pl.close()


def test_apply_batch_errors():
    a, b = Plan(f=8), Plan(f=8, layout=Layout.PLANAR)
    for pl in (a, b):
        pl.set_precoders(torch.zeros(pl.w_shape(1), dtype=pl.dtype, device=DEV))
    S = torch.zeros(a.s_shape(4), dtype=a.dtype, device=DEV)
    R = torch.empty(a.r_shape(4), dtype=a.dtype, device=DEV)
    Sp = torch.zeros(b.s_shape(4), dtype=b.dtype, device=DEV)
    Rp = torch.empty(b.r_shape(4), dtype=b.dtype, device=DEV)
    with pytest.raises(bf.BfError, match="layout"):
        bf.apply_batch([(a, S, None, None, R), (b, Sp, None, None, Rp)])
    perm = torch.zeros(4, dtype=torch.int32, device=DEV)
    with pytest.raises(bf.BfError, match="job 0"):
        bf.apply_batch([(a, S, perm, None, R)])
    bf.apply_batch([])
    for pl in (a, b):
        pl.close()


@pytest.mark.slow
def test_c5_batched_windows_sampled():
    """c5 in the bench's launch configuration: windows of 8 consecutive 4096-block chunks
    (one per cell), each chunk routed, one bf_apply_batch per window on 146 SMs; sampled
    blocks of every chunk against the oracle."""
    wl = syn.workload("c5")
    fc = syn.cell_flows(wl.seed, 8)
    sms = torch.cuda.get_device_properties(DEV).multi_processor_count
    plans = []
    Ws = []
    for cell in range(8):
        W = syn.precoders(wl.seed, cell, 55, 64, int(fc[cell]), "none")
        pl = Plan(f=int(fc[cell]))
        pl.set_precoders(torch.from_numpy(W).to(DEV))
        pl.set_sm_share(sms - 2)
        plans.append(pl)
        Ws.append(W)
    for w in (0, 97, 255):
        jobs, ids_of = [], []
        for c in range(8 * w, 8 * w + 8):
            f = int(fc[c % 8])
            first = c * 4096
            Sd = torch.empty((4096, f, 60), dtype=torch.complex64, device=DEV)
            sync.gen_symbols(Sd, wl.seed, 0, f, 60, 0, first=first)
            td = torch.empty(4096, dtype=torch.int32, device=DEV)
            sync.gen_tags(td, wl.seed, 55, first=first)
            perm, offs = plans[c % 8].route(td)
            R = torch.empty((4096, 64, 60), dtype=torch.complex64, device=DEV)
            jobs.append((plans[c % 8], Sd, perm, offs, R))
            ids_of.append(np.arange(first, first + 4096, dtype=np.int64))
        bf.apply_batch(jobs)
        torch.cuda.synchronize()
        for (pl, _, _, _, R), ids, c in zip(jobs, ids_of, range(8 * w, 8 * w + 8)):
            sel = np.arange(c % 61, 4096, 61)
            f = pl.f
            S = syn.qam_symbols(wl.seed, 0, ids[sel], f, 60, syn.block_modulations(wl.seed, ids[sel]))
            tags = syn.subband_tags(wl.seed, ids[sel], 55)
            R_ref, T, _ = oracle.beamform(Ws[c % 8], S, tags, n_threads=NT)
            assert_parity(R[torch.from_numpy(sel).to(DEV)].cpu().numpy(), R_ref, T,
                          what=f"c5 window {w} chunk {c} (f={f})")
    for pl in plans:
        pl.close()


def test_apply_batch_in_cuda_graph():
    """bf_apply_batch and bf_route captured into a CUDA graph (as the c5 bench runs them):
    replays reproduce the eager results bitwise, also after the inputs change in place."""
    plans, jobs, eager = [], [], []
    for i, f in enumerate((36, 5, 17)):
        pl = Plan(f=f)
        pl.set_precoders(torch.from_numpy(syn.precoders(51, i, 7, 64, f, "unit_columns")).to(DEV))
        S = torch.from_numpy(syn.qam_symbols(51, i, np.arange(999), f, 60, 64)).to(DEV)
        T = torch.from_numpy(syn.subband_tags(51, np.arange(999) + i, 7)).to(DEV)
        perm = torch.empty(999, dtype=torch.int32, device=DEV)
        offs = torch.empty(9, dtype=torch.int32, device=DEV)
        R = torch.empty((999, 64, 60), dtype=torch.complex64, device=DEV)
        plans.append(pl)
        jobs.append((pl, S, perm, offs, R, T))
    side = torch.cuda.Stream()

    def step():
        for pl, S, perm, offs, R, T in jobs:
            pl.route_into(T, perm, offs)
        bf.apply_batch([(pl, S, perm, offs, R) for pl, S, perm, offs, R, _ in jobs])

    with torch.cuda.stream(side):
        step()
    torch.cuda.synchronize()
    eager = [j[4].clone() for j in jobs]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        step()
    for j in jobs:
        j[4].zero_()
    g.replay()
    torch.cuda.synchronize()
    for j, e in zip(jobs, eager):
        assert_bitwise(j[4].cpu().numpy(), e.cpu().numpy(), "graph replay")
    jobs[1][1].mul_(-1)                      # S of job 1 changes in place: the replay follows
    g.replay()
    torch.cuda.synchronize()
    replayed = jobs[1][4].clone()
    with torch.cuda.stream(side):
        step()
    torch.cuda.synchronize()
    assert_bitwise(replayed.cpu().numpy(), jobs[1][4].cpu().numpy(), "replay after S *= -1")
    assert not torch.equal(replayed, eager[1])
    for pl in plans:
        pl.close()


def test_non_finite_inputs_stay_local(variant):
    """A NaN or Inf in S[n][k][j] makes exactly column j of block n non-finite (for every
    antenna with W[i][k] != 0) and leaves every other element equal to the clean run
    (reading R16: IEEE propagation, no cross-talk).  Non-finite values are
    outside the tensor domain: the tensor kernel recomputes those two blocks with the FFMA
    kernel's arithmetic (its fix-up), so there they equal the clean FFMA run."""
    f = 9
    W = syn.precoders(61, 0, 1, 64, f, "unit_columns")
    S = syn.qam_symbols(61, 0, np.arange(20), f, 60, 16)
    clean = run_plan(W, S, variant=variant)
    clean_ffma = run_plan(W, S, variant=Variant.FFMA)
    bad = S.copy()
    bad[3, 2, 7] = complex(np.nan, 0.0)
    bad[11, 8, 59] = complex(np.inf, 1.0)
    got = run_plan(W, bad, variant=variant)
    want = clean.copy()
    want[[3, 11]] = clean_ffma[[3, 11]]
    mask = np.zeros(got.shape, bool)
    mask[3, :, 7] = True
    mask[11, :, 59] = True
    assert not np.isfinite(got[mask].view(np.float32)).all()
    assert not np.isfinite(got[3, :, 7]).any()
    assert_bitwise(np.where(mask, 0, got), np.where(mask, 0, want), "unaffected elements")
    assert_bitwise(got[[3, 11]], run_plan(W, bad, variant=Variant.FFMA)[[3, 11]], "== FFMA kernel")


# ---------------------------------------------------------------------------
# int16 fronthaul output (BF_LAYOUT_INTERLEAVED_I16OUT)
# ---------------------------------------------------------------------------
def run_i16(W, S, tags, variant, e=None):
    plan = Plan(f=W.shape[-1], layout=Layout.INTERLEAVED_I16OUT, variant=variant)
    if e is not None:
        plan.set_output_exponent(e)
    plan.set_precoders(torch.from_numpy(np.ascontiguousarray(W)).to(DEV))
    R = plan.apply(torch.from_numpy(np.ascontiguousarray(S)).to(DEV),
                   None if tags is None else torch.from_numpy(tags).to(DEV))
    torch.cuda.synchronize()
    plan.close()
    return R.cpu().numpy()


def host_i16(R32, e):
    """sat(rne(R x 2^e)) per component, NaN -> 0 (the layout's definition, bf.h)."""
    out = []
    for comp in (R32.real, R32.imag):
        x = comp.astype(np.float64) * 2.0 ** e
        x = np.where(np.isnan(x), 0.0, np.rint(x))
        out.append(np.clip(x, -32768, 32767).astype(np.int16))
    return np.stack(out, axis=-1)


@pytest.mark.parametrize("e", [None, 3, 20])
def test_i16_output_is_the_fp32_result_rounded_and_saturated(e, variant):
    """R16 equals the same kernel's fp32 result times 2^e, rounded to nearest-even and
    saturated (e = 20 saturates most samples), exactly; the default exponent is 12."""
    wl = syn.workload("c4")
    W, S, tags = syn.workload_inputs(wl, np.arange(501))
    R16 = run_i16(W, S, tags, variant, e)
    R32 = run_plan(W, S, tags, variant=variant)
    assert np.array_equal(R16, host_i16(R32, 12 if e is None else e))
    if e == 20:
        assert (np.abs(R16.astype(np.int32)) >= 32767).mean() > 0.5


@pytest.mark.parametrize("e", [12, 15])
def test_i16_output_against_oracle(e, variant):
    """int16 output at general W against the oracle: off saturation every sample is within
    half an output step of R_exact (2^-(e+1) per component) plus the fp32 contract;
    saturated samples carry the sign of R_exact and the extreme code."""
    wl = syn.workload("c4")
    W, S, tags = syn.workload_inputs(wl, np.arange(1501))
    R16 = run_i16(W, S, tags, variant, e).astype(np.float64)
    R_ref, T, _ = oracle.beamform(W, S, tags, n_threads=NT)
    ref = R_ref.astype(np.complex128)
    big = 32767 * 2.0 ** -e
    for comp, got in ((ref.real, R16[..., 0]), (ref.imag, R16[..., 1])):
        unsat = np.abs(comp) < big - 2.0 ** -e
        err = np.abs(got[unsat] * 2.0 ** -e - comp[unsat])
        assert (err <= 2.0 ** -(e + 1) + TOL * T[unsat] + 1e-12).all(), err.max()
        sat = np.abs(comp) >= big + 2.0 ** -e
        assert (np.abs(got[sat]) >= 32767).all() and (np.sign(got[sat]) == np.sign(comp[sat])).all()
    if e == 15:
        assert (np.abs(R16) >= 32767).any()                 # the saturating branch is exercised


def test_i16_identity_reproduces_integer_samples(variant):
    """Identity W on S holding integers / 2^12: the int16 output is those integers exactly."""
    f = 8
    rng = np.random.default_rng(5)
    S = (rng.integers(-2000, 2000, size=(9, f, 60)) + 1j * rng.integers(-2000, 2000, size=(9, f, 60)))
    S = (S / 4096.0).astype(np.complex64)
    W = np.zeros((1, 64, f), np.complex64)
    W[0, np.arange(f), np.arange(f)] = 1
    R16 = run_i16(W, S, None, variant)
    assert np.array_equal(R16[:, :f, :, 0], np.rint(S.real * 4096).astype(np.int16))
    assert np.array_equal(R16[:, :f, :, 1], np.rint(S.imag * 4096).astype(np.int16))
    assert not R16[:, f:].any()
    p = Plan(f=f, layout=Layout.INTERLEAVED_I16OUT)
    with pytest.raises(bf.BfError):
        p.set_output_exponent(65)
    p.close()


# ---------------------------------------------------------------------------
# every shared-memory configuration of the tensor kernel (TcSmem: double or single W
# buffer, R stage or not, ring depth; int16 direct vs staged), with many group changes
# per CTA (2 SMs), so the single-W-buffer reload path runs for every f that uses it
# ---------------------------------------------------------------------------
def run_shared(W, S, tags, layout, share):
    plan = Plan(f=W.shape[-1], layout=layout, variant=Variant.TENSOR)
    plan.set_sm_share(share)
    conv = syn.to_planar if layout == Layout.PLANAR else np.ascontiguousarray
    plan.set_precoders(torch.from_numpy(conv(W)).to(DEV))
    R = plan.apply(torch.from_numpy(conv(S)).to(DEV), torch.from_numpy(tags).to(DEV))
    torch.cuda.synchronize()
    plan.close()
    R = R.cpu().numpy()
    return syn.from_planar(R) if layout == Layout.PLANAR else R


@pytest.mark.parametrize("f", [3, 12, 13, 20, 25, 26, 27, 31, 33, 36])
def test_smem_configs_with_group_changes(f):
    G, n = 13, 600
    W = syn.precoders(71, f, G, 64, f, "unit_columns")
    S = syn.qam_symbols(71, f, np.arange(n), f, 60, 64)
    tags = syn.subband_tags(71, np.arange(n), G)
    R_ref, T, _ = oracle.beamform(W, S, tags, n_threads=NT)
    R32 = run_shared(W, S, tags, Layout.INTERLEAVED, 2)
    assert_parity(R32, R_ref, T, what=f"f={f} interleaved, 2 SMs")
    assert np.array_equal(R32, run_plan(W, S, tags, variant=Variant.TENSOR)), "partition-dependent"
    assert_parity(run_shared(W, S, tags, Layout.PLANAR, 2), R_ref, T, what=f"f={f} planar, 2 SMs")
    h = run_shared(W, S, tags, Layout.INTERLEAVED_F16OUT, 3).astype(np.float64)
    expect16 = R32.real.astype(np.float16).astype(np.float64) + 1j * R32.imag.astype(np.float16).astype(np.float64)
    assert np.array_equal(h[..., 0] + 1j * h[..., 1], expect16)
    assert np.array_equal(run_shared(W, S, tags, Layout.INTERLEAVED_I16OUT, 3), host_i16(R32, 12))


@pytest.mark.parametrize("layout", [Layout.INTERLEAVED, Layout.PLANAR])
@pytest.mark.parametrize("f", [5, 13, 36])
def test_exact_and_general_groups_interleaved(f, layout):
    """Groups whose W is exactly tf32 (selection: the S1/S2/S3 path, bit-exact) and general
    groups (S1 alternating between two TMEM regions) in one launch, many group changes per CTA
    (2 SMs): every block against the oracle, the selection groups bit for bit."""
    G, n = 6, 2400
    W = syn.precoders(33, f, G, 64, f, "unit_columns")
    for g in (1, 4):                                   # selection precoders: tf32-exact
        W[g] = 0
        W[g][np.arange(64), np.arange(64) % f] = 1 if g == 1 else -2
    S = syn.qam_symbols(33, f, np.arange(n), f, 60, 64)
    tags = syn.subband_tags(33, np.arange(n), G)
    R_ref, T, _ = oracle.beamform(W, S, tags, n_threads=NT)
    R = run_shared(W, S, tags, layout, 2)
    assert_parity(R, R_ref, T, what=f"f={f} exact+general")
    sel = np.isin(tags, [1, 4])
    assert np.array_equal(R[sel], R_ref[sel]), "selection groups must be bit-exact"
