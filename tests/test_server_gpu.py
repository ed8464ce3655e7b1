"""GPU tests of the slot server (include/bf.h bf_server_*): one persistent launch serving
untagged applies through a mapped-memory mailbox.  Results must equal bf_apply with the
tensor variant bit for bit (same kernel arithmetic), and the oracle within the contract.

While a server runs it holds every SM of its plan's share, so other kernels (a fill, the
reference apply) would wait for it: inputs are prepared before start, references computed
after stop."""
import numpy as np
import pytest

import bf_synth as syn
import oracle
from helpers import assert_bitwise, assert_parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():   # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1810_11451_b200 as bf  # noqa: E402
from paper_1810_11451_b200 import Layout, Plan, Server, Variant  # noqa: E402

DEV = torch.device("cuda", 0)
NT = oracle.max_threads()


def make_plan(f, layout=Layout.INTERLEAVED, seed=3):
    W = syn.precoders(seed, f, 1, 64, f, "unit_columns")
    p = Plan(f=f, layout=layout, variant=Variant.TENSOR)
    conv = syn.to_planar if layout == Layout.PLANAR else np.ascontiguousarray
    p.set_precoders(torch.from_numpy(conv(W)).to(DEV))
    return p, W


def slot_inputs(p, f, n, seed, layout=Layout.INTERLEAVED):
    S = syn.qam_symbols(seed, f, np.arange(n), f, 60, 64)
    conv = syn.to_planar if layout == Layout.PLANAR else np.ascontiguousarray
    Sd = torch.from_numpy(conv(S)).to(DEV)
    R = torch.full(p.r_shape(n), 0, dtype=p.r_dtype, device=DEV)
    return S, Sd, R


@pytest.mark.parametrize("layout", [Layout.INTERLEAVED, Layout.PLANAR, Layout.INTERLEAVED_F16OUT,
                                    Layout.INTERLEAVED_I16OUT])
@pytest.mark.parametrize("f", [5, 36])
def test_server_equals_apply(f, layout):
    """Slots of ragged sizes (1, 2, 301, 770, 5000 blocks) served one after another: every R
    equals plan.apply (tensor variant) bit for bit; fp32 layouts also against the oracle."""
    p, W = make_plan(f, layout)
    slots = [slot_inputs(p, f, n, 100 + i, layout) for i, n in enumerate([770, 1, 2, 301, 5000, 770])]
    torch.cuda.synchronize()
    srv = Server(p).start(torch.cuda.Stream(DEV))
    try:
        for S, Sd, R in slots:
            t = srv.submit(Sd, R)
            srv.wait(t, timeout_s=20)
            assert srv.slot_time_us(t) > 0
    finally:
        srv.stop()
        srv.close()
    for i, (S, Sd, R) in enumerate(slots):
        ref = p.apply(Sd)
        torch.cuda.synchronize()
        assert_bitwise(R.cpu().numpy(), ref.cpu().numpy(), f"slot {i} (n={len(S)})")
        if layout in (Layout.INTERLEAVED, Layout.PLANAR) and len(S) <= 770:
            got = R.cpu().numpy()
            got = syn.from_planar(got) if layout == Layout.PLANAR else got
            R_ref, T, _ = oracle.beamform(W, S, None, n_threads=NT)
            assert_parity(got, R_ref, T, what=f"server slot {i}")
    p.close()


def test_server_pipelined_slots_and_restart():
    """Eight slots posted back to back (more than the 4 in flight: submit waits for the
    oldest), then all waited; stop and start again on the same plan."""
    p, W = make_plan(36)
    for rnd in range(2):
        slots = [slot_inputs(p, 36, 770, 200 + 10 * rnd + i) for i in range(8)]
        torch.cuda.synchronize()
        srv = Server(p).start(torch.cuda.Stream(DEV))
        try:
            tickets = [srv.submit(Sd, R) for _, Sd, R in slots]
            for t in tickets:
                srv.wait(t, timeout_s=20)
        finally:
            srv.close()              # destroy stops a running server
        for t, (_, Sd, R) in zip(tickets, slots):
            assert_bitwise(R.cpu().numpy(), p.apply(Sd).cpu().numpy(), f"round {rnd} slot {t}")
    p.close()


def test_server_rejects_and_reports():
    """Unsupported plans are refused; S outside the tensor domain is reported by wait."""
    q = Plan(f=8, variant=Variant.TENSOR)
    q.set_precoders(torch.from_numpy(syn.precoders(4, 8, 2, 64, 8, "unit_columns")).to(DEV))
    with pytest.raises(bf.BfError) as e:
        Server(q)
    assert e.value.status == bf.Status.UNSUPPORTED
    q.close()
    p, W = make_plan(12)
    srv = Server(p)
    small = slot_inputs(p, 12, 4, 1)
    S, Sd, R = slot_inputs(p, 12, 50, 7)
    Sd[3, 2, 5] = 2.0 ** 50                                   # outside [2^-40, 2^40)
    bad_out = torch.empty((3, 64, 60), dtype=torch.complex64, device=DEV)
    torch.cuda.synchronize()
    with pytest.raises(bf.BfError):
        srv.submit(small[1], small[2])                        # not started
    srv.start(torch.cuda.Stream(DEV))
    try:
        t = srv.submit(Sd, R)
        with pytest.raises(bf.BfError) as e:
            srv.wait(t, timeout_s=20)
        assert e.value.status == bf.Status.INVALID_VALUE
        with pytest.raises((bf.BfError, ValueError)):
            srv.submit(Sd, bad_out)                           # wrong output shape
    finally:
        srv.stop()
        srv.close()
        p.close()
