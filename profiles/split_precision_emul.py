#!/usr/bin/env python
"""fp64 emulation of the K1 policy forward under the tensor-core operand splits
(3xTF32, 3xFP16, 3xFP16 with the weight pre-scale, and the rejected ELU+1 shift):
relative output error against float64 on 20k dubins inputs."""
import numpy as np, sys
sys.path.insert(0,'/root/repo')
from paper_2602_19699_b200 import specs, nets as B
spec,fld=specs.config("dubins")
rng=np.random.default_rng(0)
c,h=specs.normalisation(spec)
d=spec.n+1
actor=B.init_mlp([d,64,64,64,spec.m],rng,head="tanh",out_scale=spec.u_bound,in_center=c,in_half=h)
actor=actor.with_params([q*(10.0 if i==6 else 1.0) for i,q in enumerate(actor.flat_params())])
lo,hi=specs.region_box(spec)
X=np.concatenate([rng.uniform(size=(20000,spec.n))*(hi-lo)+lo, rng.integers(0,100,(20000,1))],1)
xn=(X-c)/h
def f16(x): return x.astype(np.float16).astype(np.float64)
def tf32(x):
    u=x.astype(np.float32).view(np.uint32); return ((u+np.uint32(0x1000))&np.uint32(0xFFFFE000)).view(np.float32).astype(np.float64)
def split_dot(a,W,sp):
    a=a.astype(np.float32).astype(np.float64); W=W.astype(np.float32).astype(np.float64)
    ah=sp(a); al=sp((a-ah)); wh=sp(W); wl=sp(W-wh)
    return ah@wh.T+ah@wl.T+al@wh.T
def fwd(mode):
    a=xn.copy()
    L=len(actor.weights)
    for i,(W,b) in enumerate(zip(actor.weights,actor.biases)):
        if mode=="f64": z=a@W.T+b
        elif mode=="tf32": z=split_dot(a,W,tf32)+b
        elif mode=="f16": z=split_dot(a,W,f16)+b
        elif mode=="f16s":   # scaled + shifted like the kernel
            S=8*1.4426950408889634 if i<L-1 else 8.0
            Ws=(W*S).astype(np.float32)
            if i==0: bb=S*b; aa=a
            else: bb=S*(b-W.sum(1)); aa=a  # a is already ELU+1
            z=(split_dot(aa,Ws,f16)+bb)/S
        if i<L-1:
            if mode=="f16s": a=np.maximum(z,0)+np.exp(np.minimum(z,0))
            else: a=np.where(z>0,z,np.expm1(np.minimum(z,0)))
        else: o=z
    return o
ref=fwd("f64")
for mm in ("tf32","f16","f16s"):
    o=fwd(mm); e=np.abs(o-ref)/np.maximum(1,np.abs(ref))
    print(mm, "median %.2e p99 %.2e max %.2e"%(np.median(e),np.quantile(e,.99),e.max()))
def fwd2(scale, shift, sp=f16):
    a=xn.copy(); L=len(actor.weights)
    for i,(W,b) in enumerate(zip(actor.weights,actor.biases)):
        S=(8*1.4426950408889634 if i<L-1 else 8.0) if scale else 1.0
        Ws=(W*S).astype(np.float32)
        bb=S*(b-W.sum(1)) if (shift and i>0) else S*b
        z=(split_dot(a,Ws,sp)+bb)/S
        if i<L-1:
            e=np.exp(np.minimum(z,0)); a=np.maximum(z,0)+e if shift else np.maximum(z,0)+e-1
        else: o=z
    return o
for sc in (0,1):
  for shf in (0,1):
    o=fwd2(sc,shf); e=np.abs(o-ref)/np.maximum(1,np.abs(ref))
    print("scale",sc,"shift",shf,"median %.2e p99 %.2e max %.2e"%(np.median(e),np.quantile(e,.99),e.max()))
o=fwd2(1,0,tf32); e=np.abs(o-ref)/np.maximum(1,np.abs(ref)); print("tf32 scaled", np.median(e))
