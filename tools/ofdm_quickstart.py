"""The README's OFDM quick start, run as written (a check that the documented calls work)."""
import sys; sys.path.insert(0, ".")
import __graft_entry__; __graft_entry__.build()
import torch, bf_synth as syn
from paper_1810_11451_b200 import Plan, OfdmPlan
wl = syn.ofdm_workload("of0")
W, S, tags = syn.ofdm_inputs(wl)
plan = Plan(f=wl.f); plan.set_precoders(torch.from_numpy(W).cuda())
op = OfdmPlan(plan, nb=wl.nb, cp=wl.cp, scale=2048 ** -0.5)
y = op.apply(torch.from_numpy(S).cuda(), torch.from_numpy(tags).cuda())
print(tuple(y.shape), y.dtype)
op.set_output("i16", 12)
y16 = op.apply(torch.from_numpy(S).cuda(), torch.from_numpy(tags).cuda())
print(tuple(y16.shape), y16.dtype, int(y16.abs().max()))
