#!/usr/bin/env python3
"""Small cases of every libbf entry point for compute-sanitizer runs:

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick

c1, a ragged small-f c3 case, tagged c4 blocks (with routing), the host
pipeline and f = 0, for both kernel variants and both layouts.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bf_synth as syn  # noqa: E402
import paper_1810_11451_b200 as bf  # noqa: E402


def run(W, S, tags, variant, layout="interleaved"):
    dev = torch.device("cuda", 0)
    plan = bf.Plan(f=W.shape[-1], variant=variant, layout=layout)
    if layout == "planar":
        W, S = syn.to_planar(W), syn.to_planar(S)
    plan.set_precoders(torch.from_numpy(np.ascontiguousarray(W)).to(dev))
    R = plan.apply(torch.from_numpy(np.ascontiguousarray(S)).to(dev),
                   None if tags is None else torch.from_numpy(tags).to(dev))
    torch.cuda.synchronize()
    plan.close()
    return R


def main():
    quick = "--quick" in sys.argv
    for variant in ("ffma", "tensor"):
        W, S, _ = syn.workload_inputs(syn.workload("c1"))
        run(W, S, None, variant)
        W, S, _ = syn.workload_inputs(syn.workload("c3", 7), np.arange(37))
        run(W, S, None, variant, "planar")
        if quick:
            continue
        W, S, tags = syn.workload_inputs(syn.workload("c4"), np.arange(301))
        run(W, S, tags, variant)
        plan = bf.Plan(f=36, variant=variant)
        plan.set_host_chunk(128)
        plan.set_precoders(torch.from_numpy(W).cuda())
        Rh = torch.empty((301, 64, 60), dtype=torch.complex64).pin_memory()
        plan.apply_host(torch.from_numpy(S).pin_memory(), torch.from_numpy(tags).pin_memory(), Rh)
        torch.cuda.synchronize()
        plan.close()
    # many groups, a share of the SMs (cost-balanced ranges, W double buffer, group walk)
    ids = np.arange(700)
    W = syn.precoders(3, 0, 300, 64, 12, "unit_columns")
    S = syn.qam_symbols(3, 0, ids, 12, 60, 16)
    tags = syn.subband_tags(3, ids, 300)
    for variant in ("ffma", "tensor"):
        plan = bf.Plan(f=12, variant=variant)
        plan.set_sm_share(7)
        plan.set_precoders(torch.from_numpy(W).cuda())
        plan.apply(torch.from_numpy(S).cuda(), torch.from_numpy(tags).cuda())
        torch.cuda.synchronize()
        plan.close()
    # the filter stage
    fp = bf.FilterPlan()
    fp.set_taps(torch.from_numpy(syn.filter_taps()).cuda())
    fp.apply(torch.from_numpy(syn.filter_signals(5, 0, np.arange(3))).cuda())
    torch.cuda.synchronize()
    fp.close()
    p0 = bf.Plan(f=0)
    p0.set_precoders(torch.zeros((1, 64, 0), dtype=torch.complex64, device="cuda"))
    p0.apply(torch.zeros((5, 0, 60), dtype=torch.complex64, device="cuda"))
    torch.cuda.synchronize()
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
