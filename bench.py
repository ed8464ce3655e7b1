#!/usr/bin/env python3
"""Benchmark of the beamforming hot path (BASELINE.json metric: beamformed REs/s
at 64 antennas, f = 36, b = 60, and % of roofline at 1/2/4/8 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N      (one rank per GPU, NCCL)

A step is one bf_apply over the whole (per-rank shard of the) workload: block ->
group routing + the beamforming kernel AUTO picks (the tcgen05 split-precision
kernel at f = 36), inputs resident in HBM.  The
default workload is config c4 (BASELINE.json configs[3], the metric's
headline: 55 precoders 64x36, 2^20 tagged 64-QAM blocks), which fits one GPU;
S (18.1 GB) + R (32.2 GB) exceed the 126 MB L2, so no flush is needed.
Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle (the
only reference this paper-only build has) on bounded samples of the same
workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c4", help="c2 | c3 | c4 (default) | c5 | fl0 | fl1 | of0 | of1")
    ap.add_argument("--f", type=int, default=36, help="flow count for --config c3 (and of*: 36 is theirs)")
    ap.add_argument("--layout", default="interleaved",
                    choices=["interleaved", "planar", "interleaved_f16out", "interleaved_i16out"])
    ap.add_argument("--variant", default="auto", choices=["auto", "ffma", "tensor"],
                    help="kernel variant (auto = libbf's measured per-f table)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-blocks", type=int, default=0,
                    help="blocks per rank for the host-buffer e2e leg (0 = whole shard if RAM allows)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU work of the oracle baseline sample")
    ap.add_argument("--c5-chunks", type=int, default=0, help="c5: chunks per step (0 = all 2048)")
    ap.add_argument("--timeline", default="", help="c5: write a chrome-trace timeline (torch.profiler "
                    "over CUPTI: kernels per stream and the NVTX ranges libbf emits) of one replayed "
                    "step after the timed ones to this path")
    ap.add_argument("--no-graph", action="store_true", help="c5: launch eagerly, no CUDA graph")
    ap.add_argument("--steady-seconds", type=float, default=10.0,
                    help="after the timed burst, back-to-back steps for this long: steady-state "
                         "throughput, SM clock and power under the board's power cap (0 = off)")
    ap.add_argument("--no-server", action="store_true",
                    help="c2: skip the slot-server latency leg (bf_server_*)")
    ap.add_argument("--server-slots", type=int, default=200, help="c2: timed slots of the server leg")
    ap.add_argument("--parity-stride", type=int, default=16,
                    help="check every k-th block of each rank's output against the oracle after "
                         "the timed region (c4: 65 536 of 2^20 blocks; c2: every block)")
    ap.add_argument("--ofdm-out", default="f32", choices=["f32", "i16"],
                    help="of*: output samples as complex fp32 or int16 (re, im) x 2^12 fronthaul samples")
    ap.add_argument("--ofdm-chunk", type=int, default=0,
                    help="of*: symbols per bf_apply + IFFT pair inside bf_ofdm_apply (0 = libbf default)")
    ap.add_argument("--c5-batch", type=int, default=16,
                    help="c5: consecutive chunks per bf_apply_batch launch (1 = one bf_apply_routed per "
                         "chunk; 16 = two of every cell, the kernel's job limit)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_of(args):
    import bf_synth as syn
    if args.config.startswith("of"):
        import dataclasses
        wl = syn.ofdm_workload(args.config)
        f = getattr(args, "f", wl.f)
        if f != wl.f:         # --f: the same symbols with another flow count (sweeps)
            wl = dataclasses.replace(wl, f=int(f), name=f"{wl.name}-f{int(f)}",
                                     desc=wl.desc.replace("f = 36", f"f = {int(f)}"))
        return wl
    if args.config.startswith("fl"):
        return syn.filter_workload(args.config)
    if args.config == "c3":
        return syn.workload("c3", args.f)
    return syn.workload(args.config)


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle on bounded samples of the same workload
# ---------------------------------------------------------------------------
def oracle_rate(wl, seconds: float, threads: int, seed: int = 0):
    """Oracle REs/s on a seeded sample of the workload sized to ~`seconds` of CPU work."""
    import bf_synth as syn
    import oracle
    rng = np.random.default_rng(seed)
    f = wl.f if wl.f >= 0 else 36

    def sample(nb):
        ids = np.sort(rng.choice(wl.n_blocks, size=nb, replace=False))
        if wl.f >= 0:
            W, S, tags = syn.workload_inputs(wl, ids)
        else:   # c5: one cell's chunk worth of mixed-modulation blocks
            fc = syn.cell_flows(wl.seed, 8)
            cell = int(syn.c5_cell_of_block(ids[:1])[0])
            W = syn.precoders(wl.seed, cell, 55, 64, int(fc[cell]), "none")
            S = syn.qam_symbols(wl.seed, 0, ids, int(fc[cell]), 60, syn.block_modulations(wl.seed, ids))
            tags = syn.subband_tags(wl.seed, ids, 55)
        return W, S, tags

    W, S, tags = sample(max(threads, 8))
    t0 = time.perf_counter()
    oracle.beamform(W, S, tags, n_threads=threads, bound=False)
    per_block = max((time.perf_counter() - t0) / len(S), 1e-7)
    nb = int(min(wl.n_blocks, max(threads, seconds / per_block)))
    W, S, tags = sample(nb)
    t0 = time.perf_counter()
    oracle.beamform(W, S, tags, n_threads=threads, bound=False)
    dt = time.perf_counter() - t0
    return nb * wl.b / dt, nb, dt, f


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import benchkit
    import bf_synth as syn
    import oracle
    wl = workload_of(args)
    threads = oracle.max_threads()
    if isinstance(wl, syn.FilterWorkload):
        rates = []
        for st in range(args.warmup + args.steps):
            nb = max(threads, 32)
            ss = syn.filter_signals(wl.seed, 0, np.arange(st * nb, (st + 1) * nb), wl.n, wl.M)
            t0 = time.perf_counter()
            oracle.filter_apply(ss, syn.filter_taps(wl.n), n_threads=threads)
            if st >= args.warmup:
                rates.append((nb * wl.n, time.perf_counter() - t0))
        value = sum(r for r, _ in rates) / sum(t for _, t in rates)
        print(json.dumps({
            "impl": "reference", "metric": "filtered samples/s (IFFT(MULT(FFT(s))), n=2048)",
            "value": value, "unit": "samples/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(t for _, t in rates) / len(rates),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": wl.name, "n": wl.n},
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": "oracle",
                             "sample": f"{args.steps} steps of {max(threads, 32)} signals (fp64 O(n^2) DFTs)"},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return 0
    if isinstance(wl, syn.OfdmWorkload):
        # each step: a bounded sample of consecutive symbols (all 64 antennas) through the
        # fp64 OFDM oracle (W x S, bin map, O(n Nsc) IDFT, cyclic prefix)
        scale = float(np.float32(1.0 / np.sqrt(wl.n)))
        ns = max(1, min(wl.n_sym, threads // wl.n_ant or 1))
        rates = []
        for st in range(args.warmup + args.steps):
            W, S, tags = syn.ofdm_inputs(wl, (np.arange(ns) + st * ns) % wl.n_sym)
            t0 = time.perf_counter()
            oracle.ofdm(W, S, wl.nb, n=wl.n, cp=wl.cp, scale=scale, group_idx=tags, n_threads=threads)
            if st >= args.warmup:
                rates.append((ns * wl.nb * wl.b, time.perf_counter() - t0))
        value = sum(r for r, _ in rates) / sum(t for _, t in rates)
        print(json.dumps({
            "impl": "reference",
            "metric": "beamformed + OFDM-modulated REs/s (W x S, 2048-pt IFFT + CP per antenna)",
            "value": value, "unit": "REs/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(t for _, t in rates) / len(rates),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": wl.name, "nb": wl.nb, "f": wl.f, "n": wl.n,
                                            "cp": wl.cp},
            "cpu_baseline": {"value": value, "unit": "REs/s", "cores": threads, "kind": "oracle",
                             "sample": f"{args.steps} steps of {ns} symbols x 64 antennas (fp64 oracle)"},
            "e2e": {"value": value, "unit": "REs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return 0
    rates = []
    per_step_seconds = max(2.0, min(args.cpu_seconds, 150.0 / max(1, args.steps + args.warmup)))
    for s in range(args.warmup + args.steps):
        r, nb, dt, f = oracle_rate(wl, per_step_seconds, threads, seed=s)
        if s >= args.warmup:
            rates.append((r, nb, dt))
    total_res = sum(nb * wl.b for _, nb, _ in rates)
    total_t = sum(dt for _, _, dt in rates)
    value = total_res / total_t
    sample = (f"{args.steps} steps, each a seeded random sample of {rates[0][1]}-{max(r[1] for r in rates)} "
              f"blocks of {wl.name} (~{per_step_seconds:.0f} s of CPU work per step)")
    line = {
        "impl": "reference", "metric": "beamformed REs/s (64 ant, f=36, b=60)", "value": value,
        "unit": "REs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_t / len(rates), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl.name, "desc": wl.desc, "n_ant": wl.n_ant, "f": wl.f, "b": wl.b},
        "cpu_baseline": {"value": value, "unit": "REs/s", "cores": threads, "kind": "oracle",
                         "sample": sample, "cpu": benchkit.cpu_model()},
        "e2e": {"value": value, "unit": "REs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# parity of the timed output (outputs are checked against the oracle
# before a number is printed).  Runs after the timed region, on the R it
# left behind; every rank checks its own shard.
# ---------------------------------------------------------------------------
TOL = 1e-5   # BASELINE.json north_star item 4: |R_gpu - R_ref| <= 1e-5 sum_k |w_ik| |s_kj|


def _bound_T(W, S, tags):
    """T[n][i][j] = sum_k |W[g(n)][i][k]| |S[n][k][j]| in fp64 (the tolerance scale), as a
    plain matrix product of the moduli."""
    Wa = np.abs(W.astype(np.complex128))
    Sa = np.abs(S.astype(np.complex128))
    g = np.zeros(len(S), np.int64) if tags is None else tags.astype(np.int64)
    return np.matmul(Wa[g], Sa)


def compare_block_sample(R_ref, T, got, layout: str, out_exp: int = 12):
    """Worst error of sampled output blocks in units of their limit (<= 1 passes):
    fp32 layouts |dR| <= 1e-5 T (complex modulus); fp16 output |dR| <= sqrt(2) 2^-11 |R| +
    1e-5 T + 2^-24; int16 output |R16 2^-e - R| <= sqrt(2) 2^-(e+1) + 1e-5 T off saturation."""
    ref = R_ref.astype(np.complex128)
    if layout in ("interleaved", "planar"):
        err = np.abs(got.astype(np.complex128) - ref)
        lim = TOL * T
        rel = np.where(T > 0, err / np.where(T > 0, T, 1.0), np.where(err > 0, np.inf, 0.0))
        worst_T = float(rel.max()) if rel.size else 0.0
        ok = bool((err <= lim).all())
        return {"worst_err_over_T": worst_T, "ok": ok}
    g = got.astype(np.float64)
    if layout == "interleaved_f16out":
        val = g[..., 0] + 1j * g[..., 1]
        lim = np.sqrt(2) * 2.0 ** -11 * np.abs(ref) + TOL * T + 2.0 ** -24
        unsat = np.ones(val.shape, bool)
    else:
        val = (g[..., 0] + 1j * g[..., 1]) * 2.0 ** -out_exp
        lim = np.sqrt(2) * 2.0 ** -(out_exp + 1) + TOL * T
        big = 32767 * 2.0 ** -out_exp
        unsat = (np.abs(ref.real) < big) & (np.abs(ref.imag) < big)
    err = np.abs(val - ref)
    rel = np.where(unsat, err / lim, 0.0)
    return {"worst_err_over_limit": float(rel.max()) if rel.size else 0.0,
            "ok": bool((rel <= 1.0).all()), "saturated_elements": int((~unsat).sum())}


def parity_of_blocks(wl, R_dev, local_pos, global_ids, layout, out_exp=12, chunk=4096,
                     inputs=None):
    """Regenerate the sampled blocks on the host (bf_synth), run the oracle on them and
    compare with the device output R_dev[local_pos].  inputs(global_ids) -> (W, S, tags)
    overrides the workload's own generator (c5)."""
    import torch

    import bf_synth as syn
    import oracle
    thr = oracle.max_threads()
    res = {"blocks": int(len(local_pos)), "ok": True}
    worst_key = "worst_err_over_T" if layout in ("interleaved", "planar") else "worst_err_over_limit"
    worst = 0.0
    sat = 0
    t0 = time.perf_counter()
    for c0 in range(0, len(local_pos), chunk):
        lp = np.asarray(local_pos[c0:c0 + chunk])
        gid = np.asarray(global_ids[c0:c0 + chunk])
        W, S, tags = inputs(gid) if inputs else syn.workload_inputs(wl, gid)
        R_ref, _, _ = oracle.beamform(W, S, tags, n_threads=thr, bound=False)
        T = _bound_T(W, S, tags)
        got = R_dev[torch.from_numpy(lp).to(R_dev.device)].cpu().numpy()
        if layout == "planar":
            got = syn.from_planar(got)
        r = compare_block_sample(R_ref, T, got, layout, out_exp)
        worst = max(worst, r[worst_key])
        sat += r.get("saturated_elements", 0)
        res["ok"] = res["ok"] and r["ok"]
    res[worst_key] = worst
    if layout == "interleaved_i16out":
        res["saturated_elements"] = sat
    res["tol"] = TOL
    res["oracle_threads"] = thr
    res["check_s"] = time.perf_counter() - t0
    return res


def reduce_parity(res: dict, dev, world: int) -> dict:
    """Every rank's parity result on rank 0: ok = all ranks ok, worst = max over ranks."""
    if world == 1:
        return res
    import torch
    import torch.distributed as dist
    key = "worst_err_over_T" if "worst_err_over_T" in res else "worst_err_over_limit"
    t = torch.tensor([res[key], 0.0 if res["ok"] else 1.0, float(res["blocks"])], dtype=torch.float64,
                     device=dev)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    rows = [o.cpu().tolist() for o in out]
    return {**res, key: max(r[0] for r in rows), "ok": all(r[1] == 0.0 for r in rows),
            "blocks": int(sum(r[2] for r in rows)),
            "per_rank": [{key: r[0], "ok": r[1] == 0.0, "blocks": int(r[2])} for r in rows]}


def refuse(line: dict, parity: dict) -> int:
    """A parity failure prints no throughput (the number would be of a wrong result)."""
    print(json.dumps({"metric": line.get("metric"), "value": None, "error": "parity check failed",
                      "parity": parity, "config": line.get("config")}), flush=True)
    return 3


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def host_ram_available() -> int:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def peak_basis(peaks: dict) -> str:
    """Where the HBM peak came from: the driver-written measurement, else the fallback."""
    if peaks.get("source", "").startswith("measured"):
        return "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    return f"of fallback: {peaks['hbm_gbs']} GB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


# What the beamforming product is computed in (the line's "dtype" is its fp32 summary).
ARITH = {
    "tensor": "tcgen05 split precision on scaled operands (rows of S, groups of W by powers of two), "
              "11-bit terms as fp16, kind::f16 MMAs (exact products): S2*W1 + S1*W2 + S1*W1, fp32 "
              "accumulate in TMEM, exact unscale (exact W: S2*W1 + S3*W1 + S1*W1, bit-exact copies); "
              "blocks outside the tensor domain recomputed with FFMA arithmetic; DESIGN.md §7",
    "ffma": "fp32 FFMA, 4 per complex MAC, k ascending",
}


def pcie_probe(torch, dev, nbytes: int = 1 << 30, reps: int = 4) -> dict:
    """Pinned H2D and D2H copy bandwidth, each direction alone and both concurrently (two
    streams, CUDA events).  The alone figures bound an e2e step whose copies overlap each
    other and the kernels from above."""
    hs = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    hr = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def run(h2d: bool, d2h: bool, n: int):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize(dev)
        if h2d:
            with torch.cuda.stream(s1):
                ev[0].record(s1)
                for _ in range(n):
                    d1.copy_(hs, non_blocking=True)
                ev[1].record(s1)
        if d2h:
            with torch.cuda.stream(s2):
                ev[2].record(s2)
                for _ in range(n):
                    hr.copy_(d2, non_blocking=True)
                ev[3].record(s2)
        torch.cuda.synchronize(dev)
        gbs = lambda a, b: n * nbytes / (a.elapsed_time(b) * 1e-3) / 1e9  # noqa: E731
        return (gbs(ev[0], ev[1]) if h2d else None), (gbs(ev[2], ev[3]) if d2h else None)

    run(True, True, 1)                         # warm-up
    h2d_alone, _ = run(True, False, reps)
    _, d2h_alone = run(False, True, reps)
    h2d_conc, d2h_conc = run(True, True, reps)
    del hs, hr, d1, d2
    return {"h2d_gbs": h2d_alone, "d2h_gbs": d2h_alone,
            "h2d_gbs_concurrent": h2d_conc, "d2h_gbs_concurrent": d2h_conc,
            "how": f"pinned copies, {nbytes >> 20} MiB x {reps}, each direction alone and both "
                   "at once on two streams"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun (one rank per GPU)")
    # Test hooks only (tests/test_bench_gpu.py, a box with one GPU): BF_BENCH_SHARE_GPU=1
    # maps every rank to GPU local % count and BF_BENCH_DIST_BACKEND=gloo replaces NCCL
    # (which refuses two ranks on one GPU).  The ranks never wait on one another on the
    # device (no data-path collective), so sharing a GPU exercises the N > 1 host path.
    backend = os.environ.get("BF_BENCH_DIST_BACKEND", "nccl")
    if os.environ.get("BF_BENCH_SHARE_GPU") == "1":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            # NCCL's communicator-init log (ranks, NVLS / NVLink transport) for the run's
            # record; to stderr so that stdout keeps the single JSON line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    import benchkit
    import bf_synth as syn
    import bf_synth.cuda as sync
    import paper_1810_11451_b200 as bf
    from paper_1810_11451_b200 import shard

    wl = workload_of(args)
    if isinstance(wl, syn.FilterWorkload):
        return run_filter(args, wl, world, rank, local, dev)
    if isinstance(wl, syn.OfdmWorkload):
        return run_ofdm(args, wl, world, rank, local, dev)
    if wl.f < 0:
        return run_c5(args, wl, world, rank, local, dev)
    planar = args.layout == "planar"

    # ---- shard (host logic, identical on every rank) ------------------------------
    if wl.tagged:
        tags_all = syn.subband_tags(wl.seed, np.arange(wl.n_blocks), wl.n_groups)
        ids = shard.subband_shard(tags_all, rank, world)
        natural = world == 1
    else:
        first, cnt = shard.even_range(wl.n_blocks, rank, world)
        ids = np.arange(first, first + cnt, dtype=np.int64)
        natural = True
    n_local = len(ids)

    # ---- inputs resident in HBM ---------------------------------------------------
    ids_d = None if natural else torch.from_numpy(ids).to(dev)
    S, tags = sync.workload_device(wl, dev, first=int(ids[0]) if natural else 0, n=n_local,
                                   ids=ids_d, planar=planar)
    W = torch.empty((wl.n_groups, wl.n_ant, wl.f), dtype=torch.complex64, device=dev)
    if rank == 0:
        W.copy_(torch.from_numpy(syn.precoders(wl.seed, wl.sub, wl.n_groups, wl.n_ant, wl.f,
                                               wl.w_norm)))
    torch.cuda.synchronize()
    t_bc = time.perf_counter()
    shard.broadcast_precoders(W, src=0)          # NCCL over NVLink; once, untimed
    torch.cuda.synchronize()
    t_bc = time.perf_counter() - t_bc
    if planar:
        W = torch.from_numpy(syn.to_planar(W.cpu().numpy())).to(dev)

    plan = bf.Plan(f=wl.f, layout=args.layout, variant=args.variant)
    plan.set_precoders(W)
    R = torch.empty(plan.r_shape(n_local), dtype=plan.r_dtype, device=dev)
    stream = torch.cuda.current_stream()

    # ---- warm-up, then K timed steps ---------------------------------------------
    for _ in range(max(args.warmup, 0)):
        plan.apply(S, tags, out=R)
    torch.cuda.synchronize()
    clocks = benchkit.ClockSampler(local, period_ms=25).start() if rank == 0 else None
    plan.set_profiling(True)
    plan.kernel_time()
    launches0 = plan.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    small = (wl.block_bytes * n_local) < 4 * 126e6     # working set not >> the 126 MB L2
    if not small:
        e0.record(stream)
        for _ in range(args.steps):
            plan.apply(S, tags, out=R)
        e1.record(stream)
        torch.cuda.synchronize()
        elapsed_ms = e0.elapsed_time(e1)
    else:
        # Cold-L2 timing: overwrite a 512 MB buffer between steps (outside the events)
        # and sum the per-step device times.  The step is submitted as a replay of a CUDA
        # graph holding the same launches (a slot pipeline submits fixed-shape work that
        # way; --no-graph: eager), so host submission stays out of the per-slot time; the
        # kernel's own duration comes from K extra eager cold-L2 steps with libbf's events
        # (events recorded inside a graph cannot be read back per replay).
        flush = torch.empty(128 << 20, dtype=torch.float32, device=dev)
        graph = None
        if not args.no_graph:
            plan.set_profiling(False)
            try:
                lc0 = plan.launch_count()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    plan.apply(S, tags, out=R)
                launches_per_step = plan.launch_count() - lc0
                graph.replay()
                torch.cuda.synchronize()
                submission = "cuda_graph"
            except Exception as ex:  # pragma: no cover - reported, eager path measured instead
                graph, submission = None, f"eager (graph capture failed: {ex})"
            plan.set_profiling(True)
            plan.kernel_time()
        else:
            submission = "eager"
        elapsed_ms = 0.0
        for _ in range(args.steps):
            sync.fill_u32(flush, 0)
            e0.record(stream)
            if graph is not None:
                graph.replay()
            else:
                plan.apply(S, tags, out=R)
            e1.record(stream)
            torch.cuda.synchronize()
            elapsed_ms += e0.elapsed_time(e1)
        if graph is not None:
            for _ in range(args.steps):
                sync.fill_u32(flush, 0)
                plan.apply(S, tags, out=R)
            torch.cuda.synchronize()
        del flush
    if world > 1:
        dist.barrier()
    kern_ms, kern_n = plan.kernel_time()
    launches = plan.launch_count() - launches0
    if small and graph is not None:
        launches = launches_per_step * args.steps      # the timed replays' launches
    plan.set_profiling(False)
    clk = clocks.stop() if clocks else None

    elapsed_ms = shard.max_over_ranks(elapsed_ms, dev)
    # f = 0 launches no beamforming kernel (a8: R := +0 by cudaMemsetAsync): the memset
    # is the step's only work, timed by the step events
    memset_only = kern_n == 0
    kern_avg_ms = shard.max_over_ranks(elapsed_ms / args.steps if memset_only else kern_ms / kern_n, dev)
    launches = int(shard.sum_over_ranks(launches, dev))
    total_blocks = wl.n_blocks
    value = total_blocks * wl.b * args.steps / (elapsed_ms * 1e-3)

    # ---- roofline of the dominant kernel (AUTO: bf_tc_kernel at f = 36) -------------
    peaks = benchkit.measured_peaks()
    cfg = plan.kernel_config(n_local)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_max = benchkit.fp32_peak_tflops(sms, peaks.get("sm_max_mhz", 1965.0))
    flops_launch = wl.block_flops * n_local
    r_blk = 15360 if args.layout in ("interleaved_f16out", "interleaved_i16out") else 30720
    blk_bytes = 480 * wl.f + r_blk
    bytes_launch = blk_bytes * n_local
    achieved_tf = flops_launch / (kern_avg_ms * 1e-3) / 1e12
    achieved_gbs = bytes_launch / (kern_avg_ms * 1e-3) / 1e9
    hbm = peaks["hbm_gbs"]
    ai = wl.block_flops / blk_bytes
    variant = plan.variant.name.lower()
    # FFMA kernel: bound by the FP32 pipe when AI x HBM exceeds the FFMA peak.
    # Tensor kernel: 3 KP/16 fp16 MMAs (K = 16, KP = 16 ceil(2f / 16)) per 2-block tile at
    # ~2.2 PFLOP/s nominal leave it HBM-bound at every f (tensor pipe < 30 % busy).
    fp32_bound = variant == "ffma" and ai * hbm / 1e3 > peak_max
    # dram bytes of the same kernel from the committed `ncu --set full` capture
    # (profiles/traffic.json, per block), scaled to this launch's block count
    traffic, traffic_basis = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    kname = f"{'bf_tc_kernel' if plan.variant.name == 'TENSOR' else 'bf_ffma_kernel'}" \
            f"<{wl.f},{int(plan.layout)}>"
    if os.path.exists(tpath):
        try:
            tr = json.load(open(tpath)).get(kname)
        except ValueError:
            tr = None
        if tr:
            traffic = tr["dram_bytes_per_block"] * n_local
            traffic_basis = (f"{tr['capture']}: {tr['dram_bytes_per_block']:.0f} B/block "
                             f"x {n_local} blocks")
    if fp32_bound:
        roof = {"bound": "alu", "achieved": achieved_tf, "peak": peak_max, "unit": "TFLOP/s",
                "frac": achieved_tf / peak_max, "traffic": traffic,
                "peak_basis": f"derived: {sms} SMs x 128 FP32 lanes x 2 x {peaks.get('sm_max_mhz', 1965.0):.0f} MHz",
                "hbm": {"achieved": achieved_gbs, "peak": hbm, "unit": "GB/s", "frac": achieved_gbs / hbm}}
    else:
        roof = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s",
                "frac": achieved_gbs / hbm, "traffic": traffic,
                "peak_basis": peak_basis(peaks),
                "fp32_equivalent": {"achieved": achieved_tf, "unit": "TFLOP/s",
                                    "frac_of_derived_fp32_peak": achieved_tf / peak_max}}
    roof["kernel"] = "cudaMemsetAsync (f = 0: R := +0)" if memset_only else \
        f"{'bftc::bf_tc_kernel' if variant == 'tensor' else 'bfk::bf_ffma_kernel'}<{wl.f},{int(plan.layout)}>"
    roof["variant"] = variant
    if clk and clk.get("sm_mhz"):
        roof["frac_at_observed_clock"] = achieved_tf / benchkit.fp32_peak_tflops(sms, clk["sm_mhz"]) \
            if fp32_bound else None
    roof["traffic_basis"] = traffic_basis
    roof["kernel_ms"] = kern_avg_ms
    roof["kernel_share_of_step"] = kern_avg_ms * args.steps / elapsed_ms
    roof["algorithmic_bytes_per_launch"] = bytes_launch
    roof["algorithmic_flops_per_launch"] = flops_launch

    # ---- parity of the timed output: a seeded sample of every rank's blocks vs the oracle
    stride = 1 if n_local <= 4096 else max(1, args.parity_stride)
    local_pos = np.arange(0, n_local, stride, dtype=np.int64)
    parity = parity_of_blocks(wl, R, local_pos, ids[local_pos], args.layout, out_exp=12)
    parity["sample"] = (f"every {stride}th block of each rank's output after the timed steps, "
                        "regenerated on the host (bf_synth) and compared with the fp64 oracle")
    parity = reduce_parity(parity, dev, world)

    # ---- c2: the slot server — one persistent launch serving slot after slot (bf_server_*)
    server = None
    if wl.name == "c2" and world == 1 and not args.no_server:
        server = server_latency(args, plan, S, R, dev)

    # ---- steady state: the same step back to back for --steady-seconds (the timed burst
    #      above is ~0.2 s; the board's 1000 W cap takes ~0.3 s to bite)
    steady = None
    if args.steady_seconds > 0 and not small:
        steady = steady_state(args, plan, S, tags, R, local, rank, world, dev,
                              bytes_launch, n_local * wl.b, peaks["hbm_gbs"])

    # ---- e2e through the public API with host buffers ---------------------------------
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        del R
        torch.cuda.empty_cache()
        s_blk = 480 * wl.f
        need = n_local * (s_blk + r_blk + 4)
        budget = int(host_ram_available() * 0.6) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world)))
        n_e2e = n_local if args.e2e_blocks <= 0 else min(args.e2e_blocks, n_local)
        if n_e2e * (s_blk + r_blk + 4) > budget:
            n_e2e = max(1, budget // (s_blk + r_blk + 4))
        Sh = torch.empty(plan.s_shape(n_e2e), dtype=plan.dtype).pin_memory()
        Sh.copy_(S[:n_e2e])
        th = None
        if tags is not None:
            th = torch.empty(n_e2e, dtype=torch.int32).pin_memory()
            th.copy_(tags[:n_e2e])
        del S
        torch.cuda.empty_cache()
        Rh = torch.empty(plan.r_shape(n_e2e), dtype=plan.r_dtype).pin_memory()
        plan.apply_host(Sh, th, Rh)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(args.e2e_steps):
            plan.apply_host(Sh, th, Rh)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = shard.max_over_ranks(e0.elapsed_time(e1), dev)
        n_e2e_total = int(shard.sum_over_ranks(n_e2e, dev))
        e2e = {"value": n_e2e_total * wl.b * args.e2e_steps / (e2e_ms * 1e-3), "unit": "REs/s",
               "h2d_bytes_per_step": int(n_e2e_total * (s_blk + (4 if tags is not None else 0))),
               "d2h_bytes_per_step": int(n_e2e_total * r_blk),
               "steps": args.e2e_steps, "blocks_per_step": n_e2e_total,
               "ms_per_step": e2e_ms / args.e2e_steps,
               "path": "bf_apply_host: pinned host S/tags -> H2D -> route+kernel -> D2H pinned R, "
                       "chunked on 3 streams"}
        del Sh, Rh
        torch.cuda.empty_cache()
        pc = pcie_probe(torch, dev)
        t_floor = max(e2e["h2d_bytes_per_step"] / (pc["h2d_gbs"] * 1e9),
                      e2e["d2h_bytes_per_step"] / (pc["d2h_gbs"] * 1e9)) / max(1, world)
        pc["ceiling"] = n_e2e_total * wl.b / t_floor
        pc["frac"] = e2e["value"] / pc["ceiling"]
        e2e["pcie"] = pc

    # ---- CPU oracle baseline (rank 0, N = 1 only) -----------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        thr = oracle.max_threads()
        r, nb, dt, _ = oracle_rate(wl, args.cpu_seconds, thr)
        cpu = {"value": r, "unit": "REs/s", "cores": thr, "kind": "oracle",
               "sample": f"seeded random sample of {nb} blocks of {wl.name} ({dt:.1f} s, "
                         f"{thr} threads, fp64 triple loop)", "cpu": benchkit.cpu_model()}

    if rank == 0:
        gpu_name = torch.cuda.get_device_name(dev)
        line = {
            "metric": "beamformed REs/s (64 ant, f=36, b=60)", "value": value, "unit": "REs/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "parity": parity,
            "config": {"workload": wl.name, "desc": wl.desc, "n_ant": wl.n_ant, "f": wl.f,
                       "b": wl.b, "blocks": wl.n_blocks, "groups": wl.n_groups,
                       "layout": args.layout, "parallelism": f"dp{world} (blocks sharded by subband)"
                       if wl.tagged else f"dp{world}",
                       "world_size": world, "backend": dist.get_backend() if world > 1 else None,
                       "l2": "inputs larger than L2 (S+R >> 126 MB)" if not small
                       else "L2 flushed between steps (512 MB write outside the timed events)",
                       "submission": "eager" if not small else submission,
                       "kernel": cfg, "gpu": gpu_name, "w_broadcast_ms": t_bc * 1e3,
                       "arith": "none (f = 0: R := +0, memset)" if memset_only
                       else ARITH.get(roof.get("variant"), "?")},
            "flops_per_s": total_blocks * wl.block_flops * args.steps / (elapsed_ms * 1e-3),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk, "steady": steady, "server": server,
        }
        if "tflops" in os.environ.get("BF_BENCH_PROBE", "tflops"):
            try:
                line["ffma_probe"] = benchkit.ffma_probe()
            except Exception as ex:  # pragma: no cover
                line["ffma_probe"] = {"error": str(ex)}
        if not parity["ok"]:
            rc = refuse(line, parity)
        else:
            print(json.dumps(line), flush=True)
            rc = 0
    else:
        rc = 0 if parity["ok"] else 3
    if world > 1:
        dist.destroy_process_group()
    return rc


def server_latency(args, plan, S, R_ref, dev) -> dict:
    """One slot at a time through the slot server (include/bf.h bf_server_*): submit, wait,
    next.  16 distinct S / R buffers in rotation (16 x 37 MB > the 126 MB L2: every slot
    reads and writes cold memory).  Device time per slot from the server's %globaltimer
    stamps (CTA 0 sees the doorbell -> last CTA done); host round trip submit -> wait.
    The last results are checked bit for bit against the timed bf_apply output."""
    import statistics

    import torch

    import paper_1810_11451_b200 as bf
    nbuf = 16
    Ss = [S.clone() for _ in range(nbuf)]
    Rs = [torch.empty_like(R_ref) for _ in range(nbuf)]
    torch.cuda.synchronize()
    srv = bf.Server(plan)
    stream = torch.cuda.Stream(dev)
    srv.start(stream)
    dev_us, host_us = [], []
    try:
        for i in range(20 + args.server_slots):
            k = i % nbuf
            t0 = time.perf_counter()
            tk = srv.submit(Ss[k], Rs[k])
            srv.wait(tk, timeout_s=30)
            t1 = time.perf_counter()
            if i >= 20:
                dev_us.append(srv.slot_time_us(tk))
                host_us.append((t1 - t0) * 1e6)
    finally:
        srv.close()
    torch.cuda.synchronize()
    same = all(torch.equal(torch.view_as_real(Rs[k]), torch.view_as_real(R_ref)) for k in range(nbuf))
    n = R_ref.shape[0]
    med = statistics.median(dev_us)
    q = sorted(dev_us)
    return {"slots": len(dev_us), "blocks_per_slot": n,
            "device_us_median": med, "device_us_p10": q[len(q) // 10], "device_us_p90": q[9 * len(q) // 10],
            "host_roundtrip_us_median": statistics.median(host_us),
            "REs_per_s_at_device_latency": n * 60 / (med * 1e-6),
            "bitwise_equal_to_bf_apply": bool(same),
            "how": f"bf_server: one persistent launch; {len(dev_us)} slots submitted one at a time "
                   f"(submit -> wait), {nbuf} S/R buffers in rotation (cold L2); device time = "
                   "%globaltimer from CTA 0 seeing the doorbell to the last CTA done"}


def steady_state(args, plan, S, tags, R, local, rank, world, dev, bytes_launch, res_launch, hbm):
    """Back-to-back steps for args.steady_seconds of host time, the queue kept two batches
    deep; per-launch kernel times from libbf's CUDA events, clocks / power sampled by
    nvidia-smi.  Reports the mean over the window and one batch timed after it."""
    import statistics

    import torch
    import torch.distributed as dist

    import benchkit
    from paper_1810_11451_b200 import shard
    if world > 1:
        dist.barrier()
    clk = benchkit.ClockSampler(local, period_ms=50).start() if rank == 0 else None
    plan.set_profiling(True)
    plan.kernel_time()
    batch = max(1, int(0.15 / max(1e-4, bytes_launch / (hbm * 1e9))))   # ~150 ms per batch
    ev = [torch.cuda.Event(), torch.cuda.Event()]
    t0, nb, n_app = time.perf_counter(), 0, 0
    while time.perf_counter() - t0 < args.steady_seconds:
        for _ in range(batch):
            plan.apply(S, tags, out=R)
        n_app += batch
        ev[nb % 2].record()
        if nb >= 1:
            ev[(nb - 1) % 2].synchronize()          # keep one batch queued behind this one
        nb += 1
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    kms, kn = plan.kernel_time()
    plan.set_profiling(False)
    c = clk.stop() if clk else None
    per = kms / max(kn, 1)                      # mean over the whole window
    # one more batch, profiled on its own: the board is at its settled clock by now
    plan.set_profiling(True)
    plan.kernel_time()
    for _ in range(batch):
        plan.apply(S, tags, out=R)
    torch.cuda.synchronize()
    kms2, kn2 = plan.kernel_time()
    plan.set_profiling(False)
    late = kms2 / max(kn2, 1)
    late = shard.max_over_ranks(late, dev)
    per = shard.max_over_ranks(per, dev)
    out = {"seconds": wall, "applies": n_app,
           "kernel_ms_mean": per, "kernel_ms_settled": late,
           "REs_per_s_mean": res_launch * world / (per * 1e-3),
           "REs_per_s_settled": res_launch * world / (late * 1e-3),
           "GBps_mean": bytes_launch / (per * 1e-3) / 1e9,
           "GBps_settled": bytes_launch / (late * 1e-3) / 1e9,
           "frac_settled": bytes_launch / (late * 1e-3) / 1e9 / hbm,
           "how": f"{n_app} back-to-back steps over {wall:.1f} s (queue two {batch}-step batches "
                  f"deep), then {batch} more timed alone at the settled clock; per-launch kernel "
                  "time from libbf's CUDA events; nvidia-smi every 50 ms"}
    if c:
        out["clocks"] = c
    return out


def run_filter(args, wl, world, rank, local, dev):
    """Filter stage IFFT(MULT(FFT(s))), n = 2048:
    the fused bff kernel over the rank's share of the signals, resident in HBM."""
    import torch
    import torch.distributed as dist

    import benchkit
    import bf_synth as syn
    import bf_synth.cuda as sync
    from paper_1810_11451_b200 import FilterPlan, shard

    first, n_loc = shard.even_range(wl.n_signals, rank, world)
    s = torch.empty((n_loc, wl.n), dtype=torch.complex64, device=dev)
    sync.gen_filter_signals(s, wl.seed, 0, first=first, M=wl.M)
    y = torch.empty_like(s)
    plan = FilterPlan(wl.n)
    plan.set_taps(torch.from_numpy(syn.filter_taps(wl.n)).to(dev))
    for _ in range(max(args.warmup, 0)):
        plan.apply(s, out=y)
    torch.cuda.synchronize()
    clocks = benchkit.ClockSampler(local, period_ms=25).start() if rank == 0 else None
    plan.set_profiling(True)
    plan.kernel_time()
    l0 = plan.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    main = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(args.steps):
        plan.apply(s, out=y)
    e1.record(main)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed = shard.max_over_ranks(e0.elapsed_time(e1), dev)
    kms, kn = plan.kernel_time()
    kavg = shard.max_over_ranks(kms / max(kn, 1), dev)
    launches = int(shard.sum_over_ranks(plan.launch_count() - l0, dev))
    clk = clocks.stop() if clocks else None
    peaks = benchkit.measured_peaks()
    bytes_launch = wl.signal_bytes * n_loc
    achieved = bytes_launch / (kavg * 1e-3) / 1e9
    value = wl.n_signals * wl.n * args.steps / (elapsed * 1e-3)
    # parity of the timed output: every 256th signal of the rank vs the fp64 oracle
    # (per signal max_k |y - y_ref| <= 1e-5 ||s||_2 max|H|, reading F3)
    import oracle
    t0p = time.perf_counter()
    lp = np.arange(0, n_loc, 256, dtype=np.int64)
    ss = syn.filter_signals(wl.seed, 0, first + lp, wl.n, wl.M)
    y_ref, bnd = oracle.filter_apply(ss, syn.filter_taps(wl.n), n_threads=oracle.max_threads())
    got = y[torch.from_numpy(lp).to(dev)].cpu().numpy()
    rel = np.abs(got.astype(np.complex128) - y_ref.astype(np.complex128)).max(axis=1) / bnd
    parity = {"blocks": int(len(lp)), "unit": "signals", "worst_err_over_bound": float(rel.max()),
              "ok": bool((rel <= TOL).all()), "tol": TOL, "check_s": time.perf_counter() - t0p,
              "sample": "every 256th signal of each rank's output after the timed steps vs the "
                        "fp64 O(n^2) DFT oracle"}
    parity = reduce_parity({**parity, "worst_err_over_T": parity["worst_err_over_bound"]}, dev, world)
    # DRAM bytes per signal from the committed ncu capture, scaled to this launch
    traffic, tbasis = None, None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))["bff::filter_warp_kernel<2, true>"]
        traffic = tr["dram_bytes_per_signal"] * n_loc
        tbasis = f"{tr['capture']}: {tr['dram_bytes_per_signal']:.0f} B/signal x {n_loc} signals"
    except (OSError, KeyError, ValueError):
        pass

    # ---- e2e: pinned host signals -> H2D -> filter -> D2H, chunked on three streams --------
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        chunk = 16384
        n_e2e = n_loc if args.e2e_blocks <= 0 else min(args.e2e_blocks, n_loc)
        sh = torch.empty((n_e2e, wl.n), dtype=torch.complex64).pin_memory()
        sh.copy_(s[:n_e2e])
        yh = torch.empty_like(sh).pin_memory()
        del s, y
        torch.cuda.empty_cache()
        slots = 3
        dS = [torch.empty((chunk, wl.n), dtype=torch.complex64, device=dev) for _ in range(slots)]
        st_h2d, st_cmp, st_d2h = (torch.cuda.Stream(dev) for _ in range(3))
        ev_h = [torch.cuda.Event() for _ in range(slots)]
        ev_c = [torch.cuda.Event() for _ in range(slots)]
        ev_d = [torch.cuda.Event() for _ in range(slots)]

        def e2e_step():
            for i, c0 in enumerate(range(0, n_e2e, chunk)):
                k, nc = i % slots, min(chunk, n_e2e - c0)
                with torch.cuda.stream(st_h2d):
                    if i >= slots:
                        st_h2d.wait_event(ev_d[k])          # slot k's previous result left
                    dS[k][:nc].copy_(sh[c0:c0 + nc], non_blocking=True)
                    ev_h[k].record(st_h2d)
                st_cmp.wait_event(ev_h[k])
                plan.apply(dS[k][:nc], out=dS[k][:nc], stream=st_cmp)   # in place
                ev_c[k].record(st_cmp)
                with torch.cuda.stream(st_d2h):
                    st_d2h.wait_event(ev_c[k])
                    yh[c0:c0 + nc].copy_(dS[k][:nc], non_blocking=True)
                    ev_d[k].record(st_d2h)
            main.wait_stream(st_d2h)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(main)
        st_h2d.wait_stream(main)
        for _ in range(args.e2e_steps):
            e2e_step()
            st_h2d.wait_stream(main)
        f1.record(main)
        torch.cuda.synchronize()
        e2e_ms = shard.max_over_ranks(f0.elapsed_time(f1), dev)
        n_tot = int(shard.sum_over_ranks(n_e2e, dev))
        e2e = {"value": n_tot * wl.n * args.e2e_steps / (e2e_ms * 1e-3), "unit": "samples/s",
               "h2d_bytes_per_step": n_tot * wl.n * 8, "d2h_bytes_per_step": n_tot * wl.n * 8,
               "steps": args.e2e_steps, "signals_per_step": n_tot,
               "ms_per_step": e2e_ms / args.e2e_steps,
               "path": "pinned host signals -> H2D -> FilterPlan.apply (bff_apply, in place) -> "
                       "D2H pinned, 16384-signal chunks on three streams"}
        del sh, yh, dS
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import time as _t

        import oracle
        thr = oracle.max_threads()
        taps = syn.filter_taps(wl.n)
        nb = max(thr, 32)                  # probe, then a sample sized to ~--cpu-seconds
        t0 = _t.perf_counter()
        oracle.filter_apply(syn.filter_signals(wl.seed, 0, np.arange(nb), wl.n, wl.M), taps,
                            n_threads=thr)
        per = (_t.perf_counter() - t0) / nb
        nb = int(min(wl.n_signals, max(nb, args.cpu_seconds / max(per, 1e-9))))
        ss = syn.filter_signals(wl.seed, 0, np.arange(nb), wl.n, wl.M)
        t0 = _t.perf_counter()
        oracle.filter_apply(ss, taps, n_threads=thr)
        dt = _t.perf_counter() - t0
        cpu = {"value": nb * wl.n / dt, "unit": "samples/s", "cores": thr, "kind": "oracle",
               "sample": f"{nb} signals of {wl.name} ({dt:.1f} s, fp64 O(n^2) DFTs)"}
    if rank == 0:
        line = {
            "metric": "filtered samples/s (IFFT(MULT(FFT(s))), n=2048)", "value": value,
            "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": wl.name, "desc": wl.desc, "n": wl.n, "signals": wl.n_signals,
                       "parallelism": f"dp{world}", "l2": "inputs larger than L2",
                       "gpu": torch.cuda.get_device_name(dev)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                         "traffic_basis": tbasis,
                         "kernel": "bff::filter_warp_kernel<2, true> (one warp per signal, twiddles folded into the butterflies)", "kernel_ms": kavg,
                         "algorithmic_bytes_per_launch": bytes_launch,
                         "peak_basis": peak_basis(peaks)},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "parity": parity,
        }
        if parity["ok"]:
            print(json.dumps(line), flush=True)
        else:
            refuse(line, parity)
    if world > 1:
        dist.destroy_process_group()
    return 0 if parity["ok"] else 3


def run_ofdm(args, wl, world, rank, local, dev):
    """OFDM output stage (include/bf_ofdm.h): beamform every block of
    a symbol, then the per-antenna 2048-point IFFT with cyclic prefix
    (readings O1-O5), through bf_ofdm_apply over the rank's share of the symbols."""
    import torch
    import torch.distributed as dist

    import benchkit
    import bf_synth as syn
    import bf_synth.cuda as sync
    import oracle
    from paper_1810_11451_b200 import OfdmPlan, Plan, shard

    first, n_loc = shard.even_range(wl.n_sym, rank, world)
    nblk = n_loc * wl.nb
    S = torch.empty((nblk, wl.f, wl.b), dtype=torch.complex64, device=dev)
    sync.gen_symbols(S, wl.seed, 0, wl.f, wl.b, wl.M, first=first * wl.nb)
    tags = (torch.arange(first * wl.nb, first * wl.nb + nblk, device=dev) % wl.nb).to(torch.int32)
    W = syn.precoders(wl.seed, 0, wl.nb, wl.n_ant, wl.f, "unit_columns")
    scale = float(np.float32(1.0 / np.sqrt(wl.n)))
    plan = Plan(wl.f, variant=args.variant)
    plan.set_precoders(torch.from_numpy(W).to(dev))
    op = OfdmPlan(plan, wl.nb, n=wl.n, cp=wl.cp, scale=scale)
    if args.ofdm_chunk > 0:
        op.set_chunk(args.ofdm_chunk)
    out16 = args.ofdm_out == "i16"
    ob = 4 if out16 else 8                                  # bytes per output sample
    if out16:
        op.set_output("i16", 12)
    y = torch.empty(op.y_shape(n_loc), dtype=op.y_dtype, device=dev)
    for _ in range(max(args.warmup, 0)):
        op.apply(S, tags, out=y)
    torch.cuda.synchronize()
    clocks = benchkit.ClockSampler(local, period_ms=25).start() if rank == 0 else None
    plan.set_profiling(True)
    op.set_profiling(True)
    plan.kernel_time()
    op.kernel_time()
    l0 = plan.launch_count() + op.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    main = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(args.steps):
        op.apply(S, tags, out=y)
    e1.record(main)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed = shard.max_over_ranks(e0.elapsed_time(e1), dev)
    ifft_ms, ifft_n = op.kernel_time()
    bf_ms, bf_n = plan.kernel_time()
    ifft_ms = shard.max_over_ranks(ifft_ms, dev)
    bf_ms = shard.max_over_ranks(bf_ms, dev)
    launches = int(shard.sum_over_ranks(plan.launch_count() + op.launch_count() - l0, dev))
    clk = clocks.stop() if clocks else None
    plan.set_profiling(False)
    op.set_profiling(False)
    peaks = benchkit.measured_peaks()
    hbm = peaks["hbm_gbs"]
    ms_step = elapsed / args.steps
    value = wl.n_sym * wl.nb * wl.b * args.steps / (elapsed * 1e-3)
    # per-kernel algorithmic bytes (DESIGN.md §10 row 4): IFFT 8 Nsc read + 8 (cp + n) written
    # per (symbol, antenna); beamforming 8 f b read + 8 n_ant b written per block
    ifft_bytes = n_loc * wl.n_ant * (8 * wl.nb * wl.b + ob * (wl.cp + wl.n)) * args.steps
    bf_bytes = nblk * 8 * wl.b * (wl.f + wl.n_ant) * args.steps
    kern = {
        "bfofdm::ofdm_ifft_kernel": {"ms_per_step": ifft_ms / args.steps, "launches": ifft_n,
                                     "achieved_gbs": ifft_bytes / (ifft_ms * 1e-3) / 1e9},
        "bftc::bf_tc_kernel (via bf_apply, incl. routing)": {
            "ms_per_step": bf_ms / args.steps, "launches": bf_n,
            "achieved_gbs": bf_bytes / (bf_ms * 1e-3) / 1e9},
    }
    dom = max(kern, key=lambda k: kern[k]["ms_per_step"])
    ach = kern[dom]["achieved_gbs"]
    traffic, tbasis = None, None
    if dom.startswith("bfofdm") and not out16:      # the committed capture is of the fp32 output
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))["bfofdm::ofdm_ifft_kernel"]
            traffic = tr["dram_bytes_per_signal"] * n_loc * wl.n_ant
            tbasis = (f"{tr['capture']}: {tr['dram_bytes_per_signal']:.0f} B/signal (algorithmic "
                      f"{tr['algorithmic_bytes_per_signal']}) x {n_loc * wl.n_ant} signals per step")
        except (OSError, KeyError, ValueError):
            pass
    fused_b = wl.symbol_bytes(out_bytes=ob, fused=True) * n_loc
    unfused_b = wl.symbol_bytes(out_bytes=ob, fused=False) * n_loc
    step_gbs = fused_b / (ms_step * 1e-3) / 1e9

    # parity: every 1024th symbol of the rank (all 64 antennas) vs the fp64 oracle (O5)
    t0p = time.perf_counter()
    lp = np.arange(0, n_loc, max(1, min(1024, n_loc // 8 or 1)), dtype=np.int64)
    Wp, Sp, tp = syn.ofdm_inputs(wl, first + lp)
    y_ref, bnd = oracle.ofdm(Wp, Sp, wl.nb, n=wl.n, cp=wl.cp, scale=scale, group_idx=tp,
                             n_threads=oracle.max_threads())
    got = y[torch.from_numpy(lp).to(dev)].cpu().numpy()
    q_tol = 0.0
    if out16:       # int16 samples: the rounding to 2^-12 adds at most sqrt(2) 2^-13 per sample
        got = (got[..., 0].astype(np.float64) + 1j * got[..., 1]) / 2.0 ** 12
        q_tol = np.sqrt(2) * 2.0 ** -13
    rel = np.maximum(np.abs(got.astype(np.complex128) - y_ref.astype(np.complex128)).max(axis=2) - q_tol,
                     0.0) / bnd
    parity = {"blocks": int(len(lp) * wl.n_ant), "unit": "(symbol, antenna) signals",
              "worst_err_over_bound": float(rel.max()), "ok": bool((rel <= TOL).all()), "tol": TOL,
              "check_s": time.perf_counter() - t0p,
              "sample": f"every {int(lp[1] - lp[0]) if len(lp) > 1 else 1}th symbol of each rank's "
                        "output (all antennas) after the timed steps vs the fp64 oracle"}
    parity = reduce_parity({**parity, "worst_err_over_T": parity["worst_err_over_bound"]}, dev, world)
    del y_ref, got

    # ---- e2e: pinned host S + tags -> H2D -> bf_ofdm_apply -> D2H y, 3 streams ----------
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        chunk = 256
        n_e2e = min(n_loc, 2048 if args.e2e_blocks <= 0 else args.e2e_blocks)
        Sh = torch.empty((n_e2e * wl.nb, wl.f, wl.b), dtype=torch.complex64).pin_memory()
        Sh.copy_(S[:n_e2e * wl.nb])
        th = tags[:n_e2e * wl.nb].cpu().pin_memory()
        yh = torch.empty(op.y_shape(n_e2e), dtype=op.y_dtype).pin_memory()
        slots = 3
        dS = [torch.empty((chunk * wl.nb, wl.f, wl.b), dtype=torch.complex64, device=dev) for _ in range(slots)]
        dt_ = [torch.empty((chunk * wl.nb,), dtype=torch.int32, device=dev) for _ in range(slots)]
        dy = [torch.empty(op.y_shape(chunk), dtype=op.y_dtype, device=dev) for _ in range(slots)]
        st_h2d, st_cmp, st_d2h = (torch.cuda.Stream(dev) for _ in range(3))
        ev_h = [torch.cuda.Event() for _ in range(slots)]
        ev_c = [torch.cuda.Event() for _ in range(slots)]
        ev_d = [torch.cuda.Event() for _ in range(slots)]

        def e2e_step():
            for i, c0 in enumerate(range(0, n_e2e, chunk)):
                k, nc = i % slots, min(chunk, n_e2e - c0)
                with torch.cuda.stream(st_h2d):
                    if i >= slots:
                        st_h2d.wait_event(ev_d[k])
                    dS[k][:nc * wl.nb].copy_(Sh[c0 * wl.nb:(c0 + nc) * wl.nb], non_blocking=True)
                    dt_[k][:nc * wl.nb].copy_(th[c0 * wl.nb:(c0 + nc) * wl.nb], non_blocking=True)
                    ev_h[k].record(st_h2d)
                st_cmp.wait_event(ev_h[k])
                op.apply(dS[k][:nc * wl.nb], dt_[k][:nc * wl.nb], out=dy[k][:nc], stream=st_cmp)
                ev_c[k].record(st_cmp)
                with torch.cuda.stream(st_d2h):
                    st_d2h.wait_event(ev_c[k])
                    yh[c0:c0 + nc].copy_(dy[k][:nc], non_blocking=True)
                    ev_d[k].record(st_d2h)
            main.wait_stream(st_d2h)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(main)
        st_h2d.wait_stream(main)
        for _ in range(args.e2e_steps):
            e2e_step()
            st_h2d.wait_stream(main)
        f1.record(main)
        torch.cuda.synchronize()
        e2e_ms = shard.max_over_ranks(f0.elapsed_time(f1), dev)
        n_tot = int(shard.sum_over_ranks(n_e2e, dev))
        e2e = {"value": n_tot * wl.nb * wl.b * args.e2e_steps / (e2e_ms * 1e-3), "unit": "REs/s",
               "h2d_bytes_per_step": n_tot * wl.nb * (wl.f * wl.b * 8 + 4),
               "d2h_bytes_per_step": n_tot * wl.n_ant * (wl.cp + wl.n) * ob,
               "steps": args.e2e_steps, "symbols_per_step": n_tot,
               "ms_per_step": e2e_ms / args.e2e_steps,
               "path": "pinned host S + tags -> H2D -> OfdmPlan.apply (bf_ofdm_apply) -> D2H pinned "
                       "y, 256-symbol chunks on three streams"}
        del Sh, th, yh, dS, dt_, dy
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        thr = oracle.max_threads()
        ns = max(1, thr // wl.n_ant)
        Wc, Sc, tc = syn.ofdm_inputs(wl, np.arange(ns))
        t0 = time.perf_counter()
        oracle.ofdm(Wc, Sc, wl.nb, n=wl.n, cp=wl.cp, scale=scale, group_idx=tc, n_threads=thr)
        per = (time.perf_counter() - t0) / ns
        ns = int(min(wl.n_sym, max(1, args.cpu_seconds / max(per, 1e-9))))
        Wc, Sc, tc = syn.ofdm_inputs(wl, np.arange(ns))
        t0 = time.perf_counter()
        oracle.ofdm(Wc, Sc, wl.nb, n=wl.n, cp=wl.cp, scale=scale, group_idx=tc, n_threads=thr)
        dt = time.perf_counter() - t0
        cpu = {"value": ns * wl.nb * wl.b / dt, "unit": "REs/s", "cores": thr, "kind": "oracle",
               "sample": f"{ns} symbols of {wl.name} ({dt:.1f} s, fp64 W x S + O(n Nsc) IDFTs)"}
    if rank == 0:
        line = {
            "metric": "beamformed + OFDM-modulated REs/s (W x S, 2048-pt IFFT + CP per antenna)",
            "value": value, "unit": "REs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "output_dtype": "i16" if out16 else "f32",
            "config": {"workload": wl.name, "desc": wl.desc, "n_sym": wl.n_sym, "nb": wl.nb,
                       "f": wl.f, "n": wl.n, "cp": wl.cp, "scale": scale,
                       "chunk_symbols": args.ofdm_chunk or 4096, "variant": args.variant,
                       "output": "int16 (re, im) x 2^12" if out16 else "complex fp32",
                       "parallelism": f"dp{world}", "l2": "inputs larger than L2",
                       "gpu": torch.cuda.get_device_name(dev)},
            "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                         "frac": ach / hbm, "traffic": traffic, "traffic_basis": tbasis,
                         "algorithmic_bytes_per_step": ifft_bytes // args.steps if dom.startswith("bfofdm")
                         else bf_bytes // args.steps, "kernel": dom,
                         "kernel_ms_per_step": kern[dom]["ms_per_step"], "kernels": kern,
                         "step": {"fused_bytes_per_step": fused_b, "unfused_bytes_per_step": unfused_b,
                                  "achieved_gbs_fused_bytes": step_gbs, "frac_fused_bound": step_gbs / hbm,
                                  "frac_unfused_bound": unfused_b / (ms_step * 1e-3) / 1e9 / hbm,
                                  "note": "fused = S read + y written per symbol (no R round trip); "
                                          "unfused = + R written and read back"},
                         "peak_basis": peak_basis(peaks)},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "parity": parity,
        }
        if parity["ok"]:
            print(json.dumps(line), flush=True)
        else:
            refuse(line, parity)
    if world > 1:
        dist.destroy_process_group()
    return 0 if parity["ok"] else 3


def run_c5(args, wl, world, rank, local, dev):
    """Config c5 (BASELINE.json configs[4]): 8 cells x 55 precoders 64 x f_c, 2^23 blocks
    in 4096-block chunks (chunk c -> cell c mod 8), mixed QPSK/16/64-QAM per block.

    S of every chunk is generated before the timed region and stays in HBM; R (258 GB)
    streams through a ring.  A step processes every chunk as its own routed apply
    (routing on a side stream on 2 SMs kept free of apply CTAs, two apply streams, all
    captured in one CUDA graph); each rank takes an even share of every chunk.  `value` counts the whole
    stream's REs over the step's device time; the roofline is the mixed-f one (sum
    over chunks of algorithmic bytes / measured HBM bandwidth).
    """
    import torch
    import torch.distributed as dist

    import benchkit
    import bf_synth as syn
    import bf_synth.cuda as sync
    import paper_1810_11451_b200 as bf
    from paper_1810_11451_b200 import shard

    n_cells, chunk = wl.extra["n_cells"], wl.extra["chunk"]
    n_chunks = wl.n_blocks // chunk if args.c5_chunks <= 0 else min(args.c5_chunks, wl.n_blocks // chunk)
    fc = syn.cell_flows(wl.seed, n_cells)
    plans = []
    t_bc = time.perf_counter()
    for cell in range(n_cells):
        f = int(fc[cell])
        W = torch.empty((wl.n_groups, 64, f), dtype=torch.complex64, device=dev)
        if rank == 0:
            W.copy_(torch.from_numpy(syn.precoders(wl.seed, cell, wl.n_groups, 64, f, "none")))
        shard.broadcast_precoders(W, src=0)
        pl = bf.Plan(f=f, variant=args.variant)
        pl.set_precoders(W)
        plans.append(pl)
    torch.cuda.synchronize()
    t_bc = time.perf_counter() - t_bc
    # Whole windows of B consecutive chunks (two of every cell at the default B = 16) are dealt
    # round-robin to ranks (window w -> rank w mod world; shard.window_shard): every rank
    # sees the same per-cell f mix and each launch keeps whole 4096-block chunks.
    B = max(1, args.c5_batch)                # chunks per bf_apply_batch launch (window)
    my_wins = shard.window_shard(n_chunks, B, rank, world)
    my_chunks = [c for w in my_wins for c in w]
    nloc = chunk
    # The apply kernels leave 2 SMs free so the routing of the next chunks (one CTA
    # each, on the route stream) never waits for an SM (bf_plan_set_sm_share).
    # tools/c5_exp.py measured the alternatives: one stream per cell with SM shares
    # proportional to the cell's work (50-61 % of roofline: large-f cells run slower
    # per SM than their byte share, and static per-CTA ranges cannot rebalance), deep
    # routing rings (no gain) and routing inline on the apply stream (65 %); this
    # two-stream pipeline reaches 72 % over 1024 chunks, untagged applies 80 %.
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    route_sms = 2
    for pl in plans:
        pl.set_sm_share(sms - route_sms)
    # S (and tags) of every chunk of this rank are generated up front and stay resident
    # in HBM (74.5 GB at N = 1), so the timed region holds only the method: per chunk,
    # the routing (bf_route, on the "route" stream) and the beamforming.  Chunks are
    # beamformed in windows of B consecutive chunks (--c5-batch, default 8: one chunk of
    # each cell), one bf_apply_batch launch per window, so the tensor kernel's fill and
    # drain is paid once per window; B = 1 is one bf_apply_routed per chunk.  R (257.7 GB
    # in total) cannot stay resident: windows write a 4-slot ring.  Window w applies on
    # stream w % 2, so one window's tail overlaps the next one's head.
    NSLOT = 4
    pos = {c: i for i, c in enumerate(my_chunks)}          # chunk id -> local slot in S_all
    chunk_f = {c: int(fc[c % n_cells]) for c in my_chunks}
    s_off = np.concatenate([[0], np.cumsum([nloc * chunk_f[c] * 60 for c in my_chunks])]).astype(np.int64)
    S_all = torch.empty(max(1, int(s_off[-1])), dtype=torch.complex64, device=dev)
    T_all = torch.empty((max(1, len(my_chunks)), nloc), dtype=torch.int32, device=dev)

    def s_view(c):
        o = int(s_off[pos[c]])
        return S_all[o:o + nloc * chunk_f[c] * 60].view(nloc, chunk_f[c], 60)

    for c in my_chunks:
        sync.gen_symbols(s_view(c), wl.seed, 0, chunk_f[c], 60, 0, first=c * chunk)
        sync.gen_tags(T_all[pos[c]], wl.seed, wl.n_groups, first=c * chunk)
    torch.cuda.synchronize()
    n_win = len(my_wins)
    P_ring = [[torch.empty(nloc, dtype=torch.int32, device=dev) for _ in range(B)] for _ in range(NSLOT)]
    O_ring = [[torch.empty(wl.n_groups + 2, dtype=torch.int32, device=dev) for _ in range(B)]
              for _ in range(NSLOT)]
    route_plan = bf.Plan(f=1, variant=args.variant)   # routing needs only the precoder count
    route_plan.set_precoders(torch.zeros((wl.n_groups, 64, 1), dtype=torch.complex64, device=dev))
    route_plans = [route_plan]
    R_ring = [[torch.empty((nloc, 64, 60), dtype=torch.complex64, device=dev) for _ in range(B)]
              for _ in range(NSLOT)]
    rstream = torch.cuda.Stream(device=dev)
    side = torch.cuda.Stream(device=dev)
    main = torch.cuda.current_stream()
    ev_rt = [torch.cuda.Event() for _ in range(NSLOT)]
    ev_use = [torch.cuda.Event() for _ in range(NSLOT)]
    ev_fork, ev_join = torch.cuda.Event(), torch.cuda.Event()

    def step():
        ev_fork.record(main)                # fork the side streams from main (graph-safe)
        rstream.wait_event(ev_fork)
        side.wait_event(ev_fork)
        for s_ in range(NSLOT):
            ev_use[s_].record(main)
        for w, win in enumerate(my_wins):
            s = w % NSLOT
            ap = main if w % 2 == 0 else side
            jobs = []
            with torch.cuda.stream(rstream):
                rstream.wait_event(ev_use[s])
                for i, c in enumerate(win):
                    route_plan.route_into(T_all[pos[c]], P_ring[s][i], O_ring[s][i])
                    jobs.append((plans[c % n_cells], s_view(c), P_ring[s][i], O_ring[s][i],
                                 R_ring[s][i]))
                ev_rt[s].record(rstream)
            ap.wait_event(ev_rt[s])
            if B == 1:
                pl, Sv, pm, of, Rv = jobs[0]
                pl.apply_routed(Sv, pm, of, out=Rv, stream=ap)
            else:
                bf.apply_batch(jobs, stream=ap)
            ev_use[s].record(ap)
        ev_join.record(side)                # join the side streams back into main
        main.wait_event(ev_join)
        ev_join.record(rstream)
        main.wait_event(ev_join)

    step()                                  # grows every workspace before any capture
    torch.cuda.synchronize()
    # The step (n_chunks routings and beamforming kernels) is captured once into a
    # CUDA graph and replayed, so host launch overhead stays out of it.
    graph, mode = None, "eager"
    if not args.no_graph:
        try:
            launches_cap0 = sum(pl.launch_count() for pl in plans + route_plans)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                main = torch.cuda.current_stream()
                step()
            launches_per_step = sum(pl.launch_count() for pl in plans + route_plans) - launches_cap0
            mode = "cuda_graph"
        except Exception as ex:  # pragma: no cover - reported, eager path measured instead
            graph, mode = None, f"eager (graph capture failed: {ex})"
            main = torch.cuda.current_stream()
    run_step = graph.replay if graph is not None else step
    for _ in range(max(args.warmup, 0)):
        run_step()
    torch.cuda.synchronize()
    clocks = benchkit.ClockSampler(local, period_ms=25).start() if rank == 0 else None
    if graph is None:
        for pl in plans:
            pl.set_profiling(True)
            pl.kernel_time()
    launches0 = sum(pl.launch_count() for pl in plans + route_plans)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    main = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(args.steps):
        run_step()
    e1.record(main)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed_ms = shard.max_over_ranks(e0.elapsed_time(e1), dev)
    if graph is not None:
        # events recorded inside a graph cannot be queried: time the kernels of one
        # extra eager step (same launches, outside the timed region)
        for pl in plans:
            pl.set_profiling(True)
            pl.kernel_time()
        step()
        torch.cuda.synchronize()
        kern_ms = sum(pl.kernel_time()[0] for pl in plans) * args.steps
        launches = launches_per_step * args.steps
    else:
        kern_ms = sum(pl.kernel_time()[0] for pl in plans)
        launches = sum(pl.launch_count() for pl in plans + route_plans) - launches0
    kern_ms = shard.max_over_ranks(kern_ms, dev)
    launches = int(shard.sum_over_ranks(launches, dev))
    clk = clocks.stop() if clocks else None
    if args.timeline and rank == 0:
        # one more step under the profiler (outside the timed region): the kernels of the
        # route stream and the two apply streams, and libbf's NVTX ranges
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
            run_step()
            torch.cuda.synchronize()
        prof.export_chrome_trace(args.timeline)
    # ---- parity: the ring still holds the R of this rank's last NSLOT windows of the last
    #      step; every 8th block of each of those chunks against the oracle
    def c5_inputs(cell, f):
        def gen(gid):
            W = syn.precoders(wl.seed, cell, wl.n_groups, 64, f, "none")
            S = syn.qam_symbols(wl.seed, 0, gid, f, 60, syn.block_modulations(wl.seed, gid))
            return W, S, syn.subband_tags(wl.seed, gid, wl.n_groups)
        return gen
    parts = []
    for w in range(max(0, n_win - NSLOT), n_win):
        for i, c in enumerate(my_wins[w]):
            lp = np.arange(0, nloc, 8, dtype=np.int64)
            parts.append(parity_of_blocks(wl, R_ring[w % NSLOT][i], lp, c * chunk + lp, "interleaved",
                                          inputs=c5_inputs(c % n_cells, chunk_f[c])))
    parity = {"blocks": sum(p_["blocks"] for p_ in parts), "ok": all(p_["ok"] for p_ in parts),
              "worst_err_over_T": max([p_["worst_err_over_T"] for p_ in parts] or [0.0]),
              "tol": TOL, "check_s": sum(p_["check_s"] for p_ in parts),
              "sample": f"every 8th block of the chunks of each rank's last {NSLOT} windows "
                        "(the R ring after the timed steps) vs the fp64 oracle"}
    parity = reduce_parity(parity, dev, world)
    total_blocks = n_chunks * chunk
    blocks_by_f = [(int(fc[c % n_cells]), chunk) for c in range(n_chunks)]
    bytes_all = sum(480 * (f + 64) * nb for f, nb in blocks_by_f) * args.steps
    flops_all = sum(30720 * f * nb for f, nb in blocks_by_f) * args.steps
    value = total_blocks * 60 * args.steps / (elapsed_ms * 1e-3)
    peaks = benchkit.measured_peaks()
    hbm = peaks["hbm_gbs"]
    # Kernels of consecutive chunks overlap (two apply streams), so per-kernel event
    # times are not additive; the roofline uses the whole pipeline's device time.
    achieved = bytes_all / world / (elapsed_ms * 1e-3) / 1e9
    variant = plans[0].variant.name.lower()
    if rank == 0:
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": None,
                "peak_basis": peak_basis(peaks),
                "kernel": (f"bftc::bf_tc_kernel<0,0> (bf_apply_batch, {B} chunks per launch, "
                           f"f_c = {','.join(str(int(x)) for x in fc)})") if B > 1 else
                          (f"{'bftc::bf_tc_kernel' if variant == 'tensor' else 'bfk::bf_ffma_kernel'}"
                           f"<f_c,0> (f_c = {','.join(str(int(x)) for x in fc)})"),
                "variant": "tensor" if B > 1 and args.variant != "ffma" else variant,
                "basis": "pipeline: algorithmic bytes of every chunk / step device time",
                "kernel_ms_eager_sum": kern_ms / args.steps,
                "mixed_f_roofline_ms": bytes_all / world / hbm / 1e6 / args.steps,
                "algorithmic_bytes_per_step": bytes_all // args.steps,
                "algorithmic_flops_per_step": flops_all // args.steps}
        line = {
            "metric": "beamformed REs/s (64 ant, f=36, b=60)", "value": value, "unit": "REs/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "c5", "desc": wl.desc, "chunks_per_step": n_chunks,
                       "blocks_per_step": total_blocks, "cells_f": [int(x) for x in fc],
                       "parallelism": f"dp{world} (whole {B}-chunk windows dealt round-robin to ranks)",
                       "world_size": world, "backend": dist.get_backend() if world > 1 else None,
                       "l2": "S resident (74.5 GB at N=1, >> L2); R streamed through a 4-slot ring",
                       "gpu": torch.cuda.get_device_name(dev), "w_broadcast_ms": t_bc * 1e3,
                       "launch_mode": mode, "apply_streams": 2, "ring_slots": NSLOT,
                       "chunks_per_launch": B, "launches_per_step": n_win,
                       "apply_sms": sms - route_sms, "route_sms": route_sms,
                       },
            "flops_per_s": flops_all / (elapsed_ms * 1e-3), "roofline": roof, "cpu_baseline": None,
            "e2e": None, "gpu_launches": launches, "clocks": clk, "parity": parity,
        }
        if parity["ok"]:
            print(json.dumps(line), flush=True)
        else:
            refuse(line, parity)
    if world > 1:
        dist.destroy_process_group()
    return 0 if parity["ok"] else 3


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
