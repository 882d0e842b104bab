"""CPU simulation of the per-row logp bias that the FFMA rounding of the
logsumexp argument d = fl(x * c - Mc) leaves (DESIGN.md §3 "Row arithmetic"):
bf16 N(0, 2^2) rows of V = 151 936 with a planted target above the bulk, the
top element excluded as K2 does, exact fp64 2^d of the rounded vs the exact
argument. 'plain': c = fl(log2 e); 'cdither': c moved by -8..8 ulp per row.
    python scripts/round_bias_sim.py
"""
import numpy as np
rng=np.random.default_rng(1)
V=151936
c32=np.float32(1.4426950408889634)
c=float(c32)
def bf16(a):
    b=a.astype(np.float32).view(np.uint32)
    b=((b+0x7fff+((b>>16)&1))&0xffff0000).astype(np.uint32)
    return b.view(np.float32).astype(np.float64)
def row_bias(x, M, cc):
    e=x*cc-M                      # exact in fp64 (bf16 * fp32 fits)
    d=e.astype(np.float32).astype(np.float64)   # one rounding = FFMA
    w=np.exp2(e); wf=np.exp2(d)
    return np.log(wf.sum()/w.sum())   # logp error (negative of) from d rounding
for mode in ("plain","cdither"):
    bs=[]
    for r in range(300):
        x=bf16(rng.normal(0,2,V))
        xt=x.max()+rng.uniform(0,5)          # planted target above bulk
        x[0]=float(bf16(np.array([xt]))[0])
        cc=c
        if mode=="cdither":
            k=int(rng.integers(-8,9)); cc=float((np.array([c32]).view(np.int32)+k).view(np.float32)[0])
        M=np.ceil(x.max()*cc)
        # exclude the top element (exact in the kernel)
        xs=np.delete(x, np.argmax(x))
        bs.append(row_bias(xs,M,cc))
    bs=np.array(bs)
    print(mode, "mean", bs.mean(), "sd", bs.std(), "sd/sqrt(n)", bs.std()/np.sqrt(len(bs)))
