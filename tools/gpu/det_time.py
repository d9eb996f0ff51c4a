"""cfg2 real-space stage time (binning + kernel, CUDA events) in the default
(Newton) and the deterministic (full shell) mode.   python tools/gpu/det_time.py"""
import sys, os, numpy as np, torch
ROOT=os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0]=[ROOT,os.path.join(ROOT,'tools')]
import workloads, paper_1712_04732_b200 as se
from paper_1712_04732_b200 import _native, device as sedev
w=workloads.ALL['cfg2'](); dev=torch.device('cuda',0)
pos=torch.from_numpy(w['pos']).to(dev); q=torch.from_numpy(w['q']).to(dev)
prm=se.SEParams(**w['prm']); peri=se.Periodicity(3); N=q.shape[0]
phi=torch.empty(N,dtype=torch.float64,device=dev)
for det in (False, True):
    se.set_deterministic(det)
    pl=sedev.plan(w['L'],prm,peri,dev)
    for _ in range(2): _native.call("se_realspace_dev",pl.handle,_native.ptr(pos),_native.ptr(q),N,_native.ptr(phi),1)
    torch.cuda.synchronize()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): _native.call("se_realspace_dev",pl.handle,_native.ptr(pos),_native.ptr(q),N,_native.ptr(phi),1)
    b.record(); torch.cuda.synchronize()
    print('deterministic' if det else 'default', a.elapsed_time(b)/5, 'ms real space (incl. binning)')
se.set_deterministic(False)
