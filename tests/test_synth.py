"""The seeded input generator (bf_synth): hash known answers and workload properties."""
import math

import numpy as np
import pytest

import bf_synth as syn


def test_splitmix64_known_answers():
    """Textbook SplitMix64 (Steele, Lea, Flood 2014) with seed 0: published first outputs."""
    assert syn.splitmix64_sequence(0, 3) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                             0x06C45D188009454F]


def test_counter_hash_is_the_splitmix_sequence():
    key = syn.stream_key(7, syn.KIND_S, 3)
    seq = syn.splitmix64_sequence(key, 20)
    got = syn.counter_hash(key, np.arange(20, dtype=np.uint64))
    assert [int(x) for x in got] == seq


@pytest.mark.parametrize("M,den", [(4, 2.0), (16, 10.0), (64, 42.0)])
def test_qam_levels_unit_power(M, den):
    lv = syn.qam_levels(M).astype(np.float64)
    L = int(math.sqrt(M))
    assert np.allclose(lv * math.sqrt(den), np.arange(-(L - 1), L, 2), atol=1e-6)
    # average power over the full constellation: 2 * mean(level^2) = 1
    assert 2 * np.mean(lv ** 2) == pytest.approx(1.0, abs=1e-6)


def test_qam_symbols_in_constellation_and_power():
    S = syn.qam_symbols(1, 0, np.arange(200), 36, 60, 64)
    lv = set(syn.qam_levels(64).tolist())
    assert set(np.unique(S.real).tolist()) == lv and set(np.unique(S.imag).tolist()) == lv
    assert np.mean(np.abs(S.astype(np.complex128)) ** 2) == pytest.approx(1.0, abs=0.01)


def test_symbols_independent_of_chunking():
    a = syn.qam_symbols(2, 5, np.arange(100), 12, 60, 16)
    b = np.concatenate([syn.qam_symbols(2, 5, np.arange(0, 37), 12, 60, 16),
                        syn.qam_symbols(2, 5, np.arange(37, 100), 12, 60, 16)])
    assert np.array_equal(a, b)
    # and block n's symbols do not depend on f (prefix rows agree)
    c = syn.qam_symbols(2, 5, np.arange(100), 7, 60, 16)
    assert np.array_equal(a[:, :7], c)


def test_precoder_normalisations():
    W = syn.precoders(1, 0, 3, 64, 36, "unit_columns")
    assert np.allclose(np.sum(np.abs(W.astype(np.complex128)) ** 2, axis=1), 1.0, atol=1e-6)
    W0 = syn.complex_gaussian(0, 0, 1, 64, 8)
    W1 = syn.precoders(0, 0, 1, 64, 8, "scale_inv_sqrt8")
    assert np.allclose(W1, (W0 / math.sqrt(8)).astype(np.complex64))
    big = syn.complex_gaussian(9, 0, 4, 64, 64)
    assert np.mean(np.abs(big) ** 2) == pytest.approx(1.0, abs=0.03)   # CN(0,1)
    assert abs(np.mean(big.real * big.imag)) < 0.02


def test_tags_modulations_cells():
    t = syn.subband_tags(3, np.arange(1 << 16), 55)
    assert t.min() == 0 and t.max() == 54 and t.dtype == np.int32
    counts = np.bincount(t, minlength=55)
    assert counts.min() > 0.8 * (1 << 16) / 55
    m = syn.block_modulations(4, np.arange(3000))
    assert set(np.unique(m).tolist()) == {4, 16, 64}
    fc = syn.cell_flows(4, 8)
    assert ((fc >= 1) & (fc <= 36)).all()


def test_planar_roundtrip():
    S = syn.qam_symbols(1, 0, np.arange(3), 5, 60, 16)
    P = syn.to_planar(S)
    assert P.shape == (3, 2, 5, 60)
    assert np.array_equal(syn.from_planar(P), S)


def test_workloads():
    assert syn.workload("c4").block_flops == 8 * 64 * 60 * 36
    assert syn.workload("c4").block_bytes == 480 * (36 + 64)
    for f in syn.C3_FLOWS:
        assert syn.workload("c3", f).f == f
    with pytest.raises(ValueError):
        syn.workload("c3", 5)
