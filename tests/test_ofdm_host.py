"""Host-side facts of the OFDM output stage (no GPU): workload shape and the algorithmic
bytes DESIGN.md §10 row 4 quotes, the bench's config routing, the header's contract."""
import os
import re

import bf_synth as syn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_of1_algorithmic_bytes():
    wl = syn.ofdm_workload("of1")
    assert (wl.n_sym, wl.nb, wl.f, wl.n, wl.cp) == (1 << 15, 26, 36, 2048, 144)
    assert wl.nb * wl.b <= wl.n
    # S read 26*60*36*8 + y written 64*(144+2048)*8; + R written and read 2*26*60*64*8
    assert wl.symbol_bytes(fused=True) == 449_280 + 1_122_304 == 1_571_584
    assert wl.symbol_bytes(fused=False) == 1_571_584 + 1_597_440 == 3_169_024
    # the IFFT kernel's bytes per (symbol, antenna): R run read + y written
    assert 8 * (wl.nb * wl.b + wl.cp + wl.n) == 30_016


def test_bench_routes_of_configs():
    import argparse
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    wl = bench.workload_of(argparse.Namespace(config="of1", f=36))
    assert isinstance(wl, syn.OfdmWorkload) and wl.name == "of1"


def test_header_states_the_readings_and_cites_the_paper():
    src = open(os.path.join(ROOT, "include", "bf_ofdm.h")).read()
    for tag in ("O1", "O2", "O3", "O4", "O5", "PAPER.md:41", "PAPER.md:84-86"):
        assert tag in src, tag
    names = set(re.findall(r"\b(bf_ofdm_[a-z_]+)\s*\(", re.sub(r"/\*.*?\*/", "", src, flags=re.S)))
    assert {"bf_ofdm_plan_create", "bf_ofdm_apply", "bf_ofdm_ifft", "bf_ofdm_destroy"} <= names
