"""Routing time (bf_route) for a few (n, groups): CUDA events over 50 back-to-back calls."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np, bf_synth as syn, paper_1810_11451_b200 as bf
dev=torch.device("cuda",0)
for n,G in ((1<<20,55),(1<<20,1024),(100000,300)):
    pl=bf.Plan(f=36); pl.set_precoders(torch.zeros((G,64,36),dtype=torch.complex64,device=dev))
    td=torch.from_numpy(syn.subband_tags(3,np.arange(n),G)).to(dev)
    perm=torch.empty(n,dtype=torch.int32,device=dev); offs=torch.empty(G+2,dtype=torch.int32,device=dev)
    for _ in range(3): pl.route_into(td,perm,offs)
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(50): pl.route_into(td,perm,offs)
    e1.record(); torch.cuda.synchronize()
    print(n,G,"route us", e0.elapsed_time(e1)*1e3/50)
