"""GPU accuracy of the tensor-core split-precision path against the oracle.

The QAM inputs of the BASELINE configs hold a handful of distinct magnitudes, so they
exercise only a few bit patterns of the operand splits.  These cases use inputs that do
exercise them: continuous complex-Gaussian fp32 S and W at the c4 shape, the same with a
2^+-20 dynamic range inside each block, adversarial fixtures where every k of a block
holds the same worst-case (s, w) pair (the per-k errors then add coherently;
tests/golden/tc_adversarial.txt, found by tools/tc_emulate.py), and values outside the
tensor domain (|s| or |w| below 2^-40 or from 2^40 up, NaN, Inf), which the kernel must
hand to its FFMA fix-up (bitwise equal to the FFMA kernel).  Tolerance as everywhere:
|R_gpu - R_ref| <= 1e-5 * sum_k |w_ik| |s_kj| per element (BASELINE.json north_star
item 4); each case also asserts the margin DESIGN.md §7's bound gives.
"""
import os
import sys

import numpy as np
import pytest

import bf_synth as syn
import oracle
from helpers import TOL, assert_bitwise, assert_parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():   # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1810_11451_b200 as bf  # noqa: E402
from paper_1810_11451_b200 import Layout, Plan, Variant  # noqa: E402

DEV = torch.device("cuda", 0)
NT = oracle.max_threads()
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "tc_adversarial.txt")
# proven worst case of the tensor path at f <= 36 against the oracle
# (complex modulus): 5.95e-6 T from the split and the tensor core's accumulation (in the
# bit-exact model measured by tools/tc_acc_probe, profiles/r02_tc_acc_model.json), plus
# the oracle's own rounding to fp32 (2^-24 T)
TC_BOUND = 6.1e-6
FFMA_BOUND = 6.2e-6      # sqrt(2) gamma_72 + 2^-24
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import tc_emulate  # noqa: E402  (numpy emulation of the tensor kernel's arithmetic)


def run(W, S, tags=None, variant=Variant.TENSOR, layout=Layout.INTERLEAVED, share=0):
    plan = Plan(f=W.shape[-1], layout=layout, variant=variant)
    if share:
        plan.set_sm_share(share)
    conv = syn.to_planar if layout == Layout.PLANAR else np.ascontiguousarray
    plan.set_precoders(torch.from_numpy(conv(W)).to(DEV))
    R = plan.apply(torch.from_numpy(conv(S)).to(DEV),
                   None if tags is None else torch.from_numpy(tags).to(DEV))
    torch.cuda.synchronize()
    resolved = plan.variant
    plan.close()
    R = R.cpu().numpy()
    if layout == Layout.PLANAR:
        R = syn.from_planar(R)
    return R, resolved


def gaussian_c4(n, exp_spread=0, seed=41):
    W = syn.precoders(seed, 0, 55, 64, 36, "none")
    S = syn.gaussian_symbols(seed, 0, np.arange(n), 36, 60, exp_spread)
    tags = syn.subband_tags(seed, np.arange(n), 55)
    return W, S, tags


@pytest.mark.parametrize("variant", [Variant.TENSOR, Variant.FFMA], ids=["tensor", "ffma"])
@pytest.mark.parametrize("spread", [0, 20], ids=["gauss", "gauss_2e20"])
def test_gaussian_fp32_c4_shape(variant, spread):
    """c4 shape (55 groups of 64 x 36, tagged) with CN(0,1) fp32 S and W (not QAM): every
    element within 1e-5 T and within the proven bound of its kernel."""
    W, S, tags = gaussian_c4(3001, spread)
    R_ref, T, _ = oracle.beamform(W, S, tags, n_threads=NT)
    R, _ = run(W, S, tags, variant)
    worst = assert_parity(R, R_ref, T, what=f"gaussian c4 shape spread={spread}")
    # FFMA: sqrt(2) gamma_72 + 2^-24 ~ 6.1e-6; tensor: TC_BOUND
    assert worst <= (TC_BOUND if variant == Variant.TENSOR else FFMA_BOUND), worst


@pytest.mark.parametrize("layout", [Layout.INTERLEAVED, Layout.PLANAR])
def test_gaussian_fp32_every_f(layout):
    """Gaussian fp32 inputs for every f (tensor kernel, both layouts, ragged n)."""
    for f in (1, 2, 5, 8, 13, 17, 24, 31, 36):
        W = syn.precoders(43, f, 3, 64, f, "none")
        S = syn.gaussian_symbols(43, f, np.arange(257), f, 60, 8)
        tags = syn.subband_tags(43, np.arange(257), 3)
        R_ref, T, _ = oracle.beamform(W, S, tags, n_threads=NT)
        R, _ = run(W, S, tags, layout=layout)
        worst = assert_parity(R, R_ref, T, what=f"gaussian f={f}")
        assert worst <= TC_BOUND, (f, worst)


def adversarial_blocks():
    """(name, sr, si, wr, wi) with [f = 36] vectors per case, from tests/golden/tc_adversarial.txt
    (rows of one pair repeated over k, and full per-k vectors), plus the review's single real
    products (worst cases of the earlier bf16 corrections) and an all-positive embedding."""
    f = 36
    cases, lines = [], [ln for ln in open(GOLDEN) if ln.strip() and not ln.startswith("#")]
    i = 0
    while i < len(lines):
        parts = lines[i].split()
        if parts[0] == "complex":
            v = [np.full(f, np.float32(x)) for x in parts[2:6]]
            cases.append((f"pair{i}", *v))
            i += 1
        else:                                   # "vector": 4 lines of f values follow
            v = [np.array(lines[i + 1 + r].split(), dtype=np.float64).astype(np.float32) for r in range(4)]
            cases.append((f"vector{i}", *v))
            i += 5
    one = lambda x: np.full(f, np.float32(x))  # noqa: E731
    cases.append(("review", one(1.0825167), one(0.0), one(1.0043917), one(0.0)))
    cases.append(("review2", one(1.0112544), one(0.0), one(1.0424854), one(0.0)))
    cases.append(("positive", one(1.9999999), one(1.9999999), one(1.9999998), one(-1.9999998)))
    return cases


def adversarial_inputs():
    cases = adversarial_blocks()
    f = 36
    W = np.empty((len(cases), 64, f), np.complex64)
    S = np.empty((len(cases) * 2, f, 60), np.complex64)
    for g, (_, sr, si, wr, wi) in enumerate(cases):
        W[g] = (wr + 1j * wi)[None, :]
        S[2 * g] = (sr + 1j * si)[:, None]
        S[2 * g + 1] = (-sr + 1j * si)[:, None]            # a second sign pattern per group
    tags = np.repeat(np.arange(len(cases), dtype=np.int32), 2)
    return W, S, tags


def test_adversarial_fixture():
    """Blocks built from the worst cases an emulation search found (errors adding coherently
    over f = 36, the truncating accumulator cutting small addends off large partial sums):
    within 1e-5 T and within DESIGN.md §7's proven bound, for both kernels."""
    W, S, tags = adversarial_inputs()
    assert len(W) >= 8
    R_ref, T, _ = oracle.beamform(W, S, tags, n_threads=NT)
    for variant in (Variant.TENSOR, Variant.FFMA):
        R, _ = run(W, S, tags, variant)
        worst = assert_parity(R, R_ref, T, what=f"adversarial {variant.name}")
        assert worst <= (TC_BOUND if variant == Variant.TENSOR else FFMA_BOUND), (variant, worst)


def test_tensor_kernel_is_the_bit_exact_model():
    """The bound of DESIGN.md §7 rests on a model of the tensor core's accumulation fitted
    with tools/tc_acc_probe.  Here the whole kernel is checked against that model: the
    numpy emulation of its scaling, splits, fp16 terms and MMA order (tools/tc_emulate.py,
    model accumulation) must reproduce the kernel's output bit for bit on every block inside
    the tensor domain (adversarial, Gaussian with a 2^+-3 spread, and an exact selection
    precoder); blocks the emulation puts outside it must be the FFMA kernel's bits."""
    W, S, tags = adversarial_inputs()
    Wg = syn.precoders(47, 0, 2, 64, 36, "none")
    W = np.concatenate([W, Wg])
    Wsel = np.zeros((1, 64, 36), np.complex64)
    Wsel[0, np.arange(64), np.arange(64) % 36] = 1 - 2j
    W = np.concatenate([W, Wsel])
    G = len(W)
    Sg = syn.gaussian_symbols(47, 0, np.arange(6), 36, 60, 3)
    S = np.concatenate([S, Sg])
    tags = np.concatenate([tags, np.array([G - 3, G - 2, G - 1, G - 1, G - 3, G - 1], np.int32)])
    R, _ = run(W, S, tags, Variant.TENSOR)
    Rf, _ = run(W, S, tags, Variant.FFMA)
    n_model = 0
    for n in range(len(S)):
        g = tags[n]
        tau, exact, ok = tc_emulate.group_scale(W[g].real, W[g].imag)
        assert ok
        in_dom = tc_emulate.row_in_domain(S[n].real.T, S[n].imag.T, exact)   # per RE j
        if not in_dom.all():
            assert_bitwise(R[n], Rf[n], f"block {n}: outside the domain -> FFMA fix-up")
            continue
        n_model += 1
        # element (i, j): s = S[n][:, j], w = W[g][i, :]
        sr = np.broadcast_to(S[n].real.T[None], (64, 60, 36))
        si = np.broadcast_to(S[n].imag.T[None], (64, 60, 36))
        wr = np.broadcast_to(W[g].real[:, None, :], (64, 60, 36))
        wi = np.broadcast_to(W[g].imag[:, None, :], (64, 60, 36))
        re, im = tc_emulate.kernel_element(sr, si, wr, wi, tau, exact)
        assert_bitwise(R[n].real.copy(), re, f"block {n} re")
        assert_bitwise(R[n].imag.copy(), im, f"block {n} im")
    # (the exact group's rows need every component within 2^15 of the row maximum — Gaussian
    # components near zero send some of its blocks to the fix-up; every other block is modelled)
    assert n_model >= len(S) - int(np.sum(tags == G - 1)), n_model


# ---------------------------------------------------------------------------
# the tensor domain: out-of-range S blocks and W groups take the FFMA fix-up
# ---------------------------------------------------------------------------
def extreme_blocks(f, n, seed):
    """QAM blocks with some blocks carrying values outside the tensor domain."""
    S = syn.qam_symbols(seed, f, np.arange(n), f, 60, 64)
    bad = {}
    rng = np.random.default_rng(seed)
    picks = rng.choice(n, size=min(n, 12), replace=False)
    kinds = ["tiny", "huge", "tiny_all", "huge_all", "subnormal", "flt_max", "edge_lo", "edge_hi"]
    for i, b in enumerate(picks):
        kind = kinds[i % len(kinds)]
        k, j = int(rng.integers(f)), int(rng.integers(60))
        if kind == "tiny":
            S[b, k, j] = np.float32(2.0 ** -60) * (1 - 1j)
        elif kind == "huge":
            S[b, k, j] = np.float32(1.5 * 2.0 ** 60) * (1 + 0.5j)
        elif kind == "tiny_all":
            S[b] *= np.float32(2.0 ** -70)
        elif kind == "huge_all":
            S[b] *= np.float32(2.0 ** 70)
        elif kind == "subnormal":          # a whole element subnormal (relative range)
            S[b, k, j] = np.float32(3 * 2.0 ** -140) * (1 + 1j)
        elif kind == "flt_max":
            S[b] = 0
            S[b, k, j] = np.float32(1.5 * 2.0 ** 127)
        elif kind == "edge_lo":
            S[b, k, j] = np.float32(np.nextafter(np.float32(2.0 ** -40), np.float32(0)))
        elif kind == "edge_hi":
            S[b, k, j] = np.float32(2.0 ** 40)
        bad[int(b)] = kind
    return S, bad


@pytest.mark.parametrize("layout", [Layout.INTERLEAVED, Layout.PLANAR,
                                    Layout.INTERLEAVED_F16OUT, Layout.INTERLEAVED_I16OUT])
@pytest.mark.parametrize("f", [3, 17, 36])
def test_out_of_domain_blocks_fixed_up(f, layout):
    """Blocks with |s| outside [2^-40, 2^40) (tiny, huge, subnormal, near FLT_MAX) mixed with
    normal ones: the tensor launch returns the FFMA kernel's bits for those blocks, its own
    result elsewhere, and every fp32 element within the contract."""
    n, G = 301, 4
    S, bad = extreme_blocks(f, n, 7 + f)
    W = syn.precoders(9, f, G, 64, f, "unit_columns")
    tags = syn.subband_tags(9, np.arange(n), G)
    Rt, _ = run(W, S, tags, Variant.TENSOR, layout, share=3)
    Rf, _ = run(W, S, tags, Variant.FFMA, layout)
    Rg, _ = run(W, S, tags, Variant.TENSOR, layout)          # full grid: other CTA ranges
    badi = np.array(sorted(bad))
    assert_bitwise(Rt[badi], Rf[badi], "fixed-up blocks == FFMA kernel")
    assert_bitwise(Rg, Rt, "independent of the partition")
    if layout in (Layout.INTERLEAVED, Layout.PLANAR):
        R_ref, T, _ = oracle.beamform(W, S, tags, n_threads=NT)
        assert_parity(Rt, R_ref, T, what=f"f={f} with out-of-domain blocks")
        good = np.setdiff1d(np.arange(n), badi)
        Rc, _ = run(W, np.ascontiguousarray(S[good]), tags[good], Variant.TENSOR, layout)
        assert_bitwise(Rt[good], Rc, "in-domain blocks unchanged by their neighbours")


def test_fixup_list_overflow_rescans():
    """More out-of-domain blocks per CTA than the kernel's list holds (64): the CTA rescans
    its range; every block equals the FFMA kernel bitwise."""
    f, n = 4, 2 * 148 * 70
    S = syn.qam_symbols(13, 0, np.arange(n), f, 60, 16) * np.float32(2.0 ** -50)
    S[::7] *= np.float32(2.0 ** 50)                          # some blocks back in the domain
    W = syn.precoders(13, 0, 2, 64, f, "unit_columns")
    tags = syn.subband_tags(13, np.arange(n), 2)
    Rt, _ = run(W, S, tags, Variant.TENSOR)
    Rf, _ = run(W, S, tags, Variant.FFMA)
    bad = np.ones(n, bool)
    bad[::7] = False
    assert_bitwise(Rt[bad], Rf[bad], "rescanned blocks == FFMA kernel")
    sel = np.arange(0, n, 37)
    R_ref, T, _ = oracle.beamform(W, S[sel], tags[sel], n_threads=NT)
    assert_parity(Rt[sel], R_ref, T, what="overflow rescan")


@pytest.mark.parametrize("value", [2.0 ** 45, 2.0 ** -45, 2.0 ** -17, float("inf")],
                         ids=["huge", "tiny", "rel_small", "inf"])
def test_out_of_domain_precoders(value):
    """A group with a W entry outside the tensor domain (absolute range, or — rel_small — an
    element far more than 2^14 below the group's largest component): AUTO resolves to the
    FFMA kernel; an explicit tensor plan fixes that group's blocks up (bitwise FFMA), others
    unchanged."""
    f, n, G = 12, 400, 3
    W = syn.precoders(17, f, G, 64, f, "unit_columns")
    W[1, 5, 3] = np.float32(value)
    S = syn.qam_symbols(17, f, np.arange(n), f, 60, 64)
    tags = syn.subband_tags(17, np.arange(n), G)
    Ra, resolved = run(W, S, tags, Variant.AUTO)
    assert resolved == Variant.FFMA
    Rt, _ = run(W, S, tags, Variant.TENSOR)
    Rf, _ = run(W, S, tags, Variant.FFMA)
    assert_bitwise(Ra, Rf, "AUTO == FFMA")
    g1 = tags == 1
    assert_bitwise(Rt[g1], Rf[g1], "out-of-domain group fixed up")
    W2 = W.copy()
    W2[1] = syn.precoders(17, f, G, 64, f, "unit_columns")[1]
    Rc, resolved2 = run(W2, S, tags, Variant.TENSOR)
    assert_bitwise(Rt[~g1], Rc[~g1], "other groups unchanged")
    if np.isfinite(value):
        R_ref, T, _ = oracle.beamform(W, S, tags, n_threads=NT)
        assert_parity(Rt, R_ref, T, what="out-of-domain precoders")


def test_out_of_domain_blocks_in_a_batch():
    """bf_apply_batch over jobs of different f, some holding out-of-domain blocks: each job's
    result equals its own FFMA-variant apply bitwise on the fixed-up blocks and its own
    tensor apply elsewhere (the batch kernel's fix-up uses the job's own precoders)."""
    jobs, refs = [], []
    for i, f in enumerate((3, 17, 36)):
        n, G = 257 + 31 * i, 3
        S, bad = extreme_blocks(f, n, 40 + f)
        W = syn.precoders(50 + i, f, G, 64, f, "unit_columns")
        tags = syn.subband_tags(50 + i, np.arange(n), G)
        p = Plan(f=f, variant=Variant.TENSOR)
        p.set_precoders(torch.from_numpy(W).to(DEV))
        Sd = torch.from_numpy(np.ascontiguousarray(S)).to(DEV)
        perm, offs = p.route(torch.from_numpy(tags).to(DEV))
        R = torch.empty(p.r_shape(n), dtype=p.r_dtype, device=DEV)
        jobs.append((p, Sd, perm, offs, R))
        Rf, _ = run(W, S, tags, Variant.FFMA)
        Rt, _ = run(W, S, tags, Variant.TENSOR)
        refs.append((Rf, Rt, np.array(sorted(bad))))
    bf.apply_batch(jobs)
    torch.cuda.synchronize()
    for (p, Sd, perm, offs, R), (Rf, Rt, badi) in zip(jobs, refs):
        got = R.cpu().numpy()
        assert_bitwise(got[badi], Rf[badi], f"f={p.f}: fixed-up blocks == FFMA kernel")
        good = np.setdiff1d(np.arange(len(got)), badi)
        assert_bitwise(got[good], Rt[good], f"f={p.f}: other blocks == tensor apply")
        p.close()


def test_subnormal_components_stay_on_the_tensor_path():
    """A component far below its element's other component (here fp32 subnormal) is inside
    the tensor domain (the relative range is per element, max(|re|, |im|)): such blocks are
    not fixed up, equal the emulated kernel bit for bit and meet the bound."""
    f, n = 36, 4
    W = syn.precoders(61, 0, 1, 64, f, "none")
    S = syn.qam_symbols(61, 0, np.arange(n), f, 60, 64)
    S[0, 3, 7] = np.float32(3 * 2.0 ** -140) + 1j * S[0, 3, 7].imag
    S[1, :, 11] = S[1, :, 11].real + 1j * np.float32(2.0 ** -100)
    S[2, 5, :] = np.float32(2.0 ** -30) + 1j * S[2, 5, :].imag
    R, _ = run(W, S)
    tau, exact, ok = tc_emulate.group_scale(W[0].real, W[0].imag)
    assert ok and not exact
    for b in range(n):
        assert tc_emulate.row_in_domain(S[b].real.T, S[b].imag.T, exact).all()
        sr = np.broadcast_to(S[b].real.T[None], (64, 60, f))
        si = np.broadcast_to(S[b].imag.T[None], (64, 60, f))
        wr = np.broadcast_to(W[0].real[:, None, :], (64, 60, f))
        wi = np.broadcast_to(W[0].imag[:, None, :], (64, 60, f))
        re, im = tc_emulate.kernel_element(sr, si, wr, wi, tau, exact)
        assert_bitwise(R[b].real.copy(), re, f"block {b} re")
        assert_bitwise(R[b].imag.copy(), im, f"block {b} im")
    R_ref, T, _ = oracle.beamform(W, S, None, n_threads=NT)
    worst = assert_parity(R, R_ref, T, what="subnormal components")
    assert worst <= TC_BOUND, worst


@pytest.mark.parametrize("exact_w", [False, True], ids=["general_w", "exact_w"])
def test_relative_range_edges(exact_w):
    """The relative-range rule at its edges: a row whose smallest nonzero
    element sits 14 binades below the row's largest component is inside the tensor domain,
    15 binades is outside (the block is the FFMA kernel's bits); for exact W every nonzero
    component must also lie within 15 binades (block 8: an element inside, one of its
    components 16 binades below).  The emulation's row_in_domain decides every block the same
    way, and in-domain blocks equal the emulated kernel bit for bit."""
    f, n = 12, 9
    if exact_w:
        W = np.zeros((1, 64, f), np.complex64)
        W[0, np.arange(64), np.arange(64) % f] = 1
    else:
        W = syn.precoders(71, 0, 1, 64, f, "none")
    S = syn.qam_symbols(71, 0, np.arange(n), f, 60, 4)          # QPSK: components 2^-0.5
    big = np.float32(2.0 ** 3)
    for b, d in enumerate([13, 14, 15, 16]):                   # binades below the largest
        S[2 * b, 0, 5] = big * (1 + 1j)
        S[2 * b, 3, 5] = np.float32(2.0 ** (3 - d)) * (1 + 0j)
        S[2 * b + 1, 0, 9] = big * (1 + 1j)
        S[2 * b + 1, 4, 9] = np.float32(2.0 ** (3 - d)) * (1 + 0.5j)
    S[8, 0, 5] = big * (1 + 1j)
    S[8, 2, 5] = np.float32(2.0 ** -10) + 1j * np.float32(2.0 ** -13)
    R, _ = run(W, S)
    Rf, _ = run(W, S, variant=Variant.FFMA)
    tau, exact, ok = tc_emulate.group_scale(W[0].real, W[0].imag)
    assert ok and exact == exact_w
    decisions = []
    for b in range(n):
        inside = bool(tc_emulate.row_in_domain(S[b].real.T, S[b].imag.T, exact).all())
        decisions.append(inside)
        if not inside:
            assert_bitwise(R[b], Rf[b], f"block {b}: outside -> FFMA fix-up")
            continue
        sr = np.broadcast_to(S[b].real.T[None], (64, 60, f))
        si = np.broadcast_to(S[b].imag.T[None], (64, 60, f))
        wr = np.broadcast_to(W[0].real[:, None, :], (64, 60, f))
        wi = np.broadcast_to(W[0].imag[:, None, :], (64, 60, f))
        re, im = tc_emulate.kernel_element(sr, si, wr, wi, tau, exact)
        assert_bitwise(R[b].real.copy(), re, f"block {b} re")
        assert_bitwise(R[b].imag.copy(), im, f"block {b} im")
    assert decisions == [True] * 4 + [False] * 4 + [not exact_w], decisions
    R_ref, T, _ = oracle.beamform(W, S, None, n_threads=NT)
    assert_parity(R, R_ref, T, what="relative-range edges")


def test_batch_with_an_auto_plan_outside_the_domain():
    """bf_apply_batch packs AUTO plans into its tensor launch unless their precoders leave the
    tensor domain: such a job runs on its own (FFMA, bitwise its own apply_routed), the other
    jobs stay bitwise equal to their tensor-variant apply_routed."""
    jobs, refs = [], []
    for i, f in enumerate((9, 20, 33)):
        n, G = 300 + 17 * i, 3
        W = syn.precoders(80 + i, f, G, 64, f, "unit_columns")
        if i == 1:
            W[2, 7, 4] = np.float32(2.0 ** -17)           # relative range: group 2 outside
        S = syn.qam_symbols(80 + i, f, np.arange(n), f, 60, 64)
        tags = torch.from_numpy(syn.subband_tags(80 + i, np.arange(n), G)).to(DEV)
        p = Plan(f=f)                                      # AUTO
        p.set_precoders(torch.from_numpy(W).to(DEV))
        assert p.variant == (Variant.FFMA if i == 1 else Variant.TENSOR)
        Sd = torch.from_numpy(S).to(DEV)
        perm, offs = p.route(tags)
        R = torch.empty(p.r_shape(n), dtype=p.r_dtype, device=DEV)
        jobs.append((p, Sd, perm, offs, R))
        q = Plan(f=f, variant=Variant.TENSOR if i != 1 else Variant.FFMA)
        q.set_precoders(torch.from_numpy(W).to(DEV))
        ref = torch.empty_like(R)
        q.apply_routed(Sd, perm, offs, out=ref)
        refs.append((q, ref))
    bf.apply_batch(jobs)
    torch.cuda.synchronize()
    for i, ((p, _, _, _, R), (q, ref)) in enumerate(zip(jobs, refs)):
        assert_bitwise(R.cpu().numpy(), ref.cpu().numpy(), f"job {i}")
        p.close()
        q.close()
