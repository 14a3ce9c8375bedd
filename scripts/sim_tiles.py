"""Tile-schedule model of the bench point (configs[1]: N = 8192, exp. decay 0.99, tau = 1e-6, BF16):
kept set from Toeplitz tile norms, per macro-tile k-steps, MMA-run tensor cycles (N <= 128 runs cost
>= 66 cycles, scripts/probe_mma_rate.cu), operand bytes through L2, and the LPT load of 8x8 tiles over
148 CTAs.  Analysis only: python scripts/sim_tiles.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
N=8192; T=32; lam=0.99; tau=1e-6
tab = synth.decay_table('exp', N, lam)  # float32 table
# bf16-rounded Toeplitz tile norms by offset D
tb = synth.round_to_bf16(tab.astype(np.float32)).astype(np.float64)
B = N//T
nD = {}
r = np.arange(T)
for D in range(-(B-1), B):
    d = np.abs((D*T + r[:,None]) - r[None,:])
    nD[D] = np.sqrt((tb[d]**2).sum())
nvec = np.array([nD[D] for D in range(-(B-1), B)])
def nA(i,k): return nvec[(i-k)+(B-1)]
I = np.arange(B)
# keep[i,k,j]
keep = np.zeros((B,B,B), bool)
for k in range(B):
    a = nA(I, k)           # over i
    b = nA(k, I)           # over j (nB[k,j] = n(k-j))
    keep[:,k,:] = (a[:,None]*b[None,:]) >= tau
print('kept', keep.sum(), 'vr', keep.sum()/B**3)
def mma_cyc(length): return max(66, 16*length)
def runs_of(mask4x8):   # mask [4,8] bool -> list of run lengths
    pats = [tuple(mask4x8[:,j]) for j in range(8)]
    out=[]; j=0
    while j<8:
        j1=j+1
        while j1<8 and pats[j1]==pats[j]: j1+=1
        if any(pats[j]): out.append(j1-j)
        j=j1
    return out
def design(MI, MJ):
    tiles=[]
    for ti in range(B//MI):
        for tj in range(B//MJ):
            sub = keep[ti*MI:(ti+1)*MI, :, tj*MJ:(tj+1)*MJ]  # MI,B,MJ
            ks = np.nonzero(sub.any(axis=(0,2)))[0]
            cyc_halves=[0]*(MI//4); byts=0; steps=len(ks)
            for k in ks:
                m = sub[:,k,:]
                for h in range(MI//4):
                    mh = m[4*h:4*h+4]
                    if mh.any():
                        cyc_halves[h] += sum(2*mma_cyc(l) for l in runs_of(mh))
                    byts += 128*64  # A rows loaded (always)
                cols = m.any(axis=0); nz=np.nonzero(cols)[0]
                byts += (nz[-1]-nz[0]+1)*2048
            tiles.append((steps, cyc_halves, byts))
    return tiles
for MI,MJ in ((4,8),(8,8)):
    t = design(MI,MJ)
    steps = sum(x[0] for x in t); cyc = sum(sum(x[1]) for x in t); byts = sum(x[2] for x in t)
    nonempty = sum(1 for x in t if x[0])
    print(f'{MI}x{MJ}: tiles {len(t)} nonempty {nonempty} ksteps {steps} pipe cycles total {cyc:.3e} -> per SM {cyc/148/1.965e3:.1f} us; L2 bytes {byts/1e9:.2f} GB -> at 12 TB/s {byts/12e12*1e6:.1f} us')
    # LPT sim: 1 issuer-pair per SM for 8x8 (cost = max over halves + overhead), per-tile cost
    per = sorted([max(x[1]) if x[1] else 0 for x in t], reverse=True) if MI==8 else sorted([sum(x[1]) for x in t], reverse=True)
    slots = 148 if MI==8 else 296
    import heapq
    h=[(0,i) for i in range(slots)]
    for c in per:
        l,i=heapq.heappop(h); heapq.heappush(h,(l+c,i))
    mx=max(l for l,i in h); avg=sum(per)/slots
    print(f'   LPT {slots} slots: max {mx/1.965e3:.1f} us avg {avg/1.965e3:.1f} us')

# U distribution for 8x8 tiles and dynamic LPT claiming with cost ~ U
t = design(8,8)
U = sorted([x[0] for x in t if x[0]], reverse=True)
print('U top', U[:10], 'U tail', U[-10:], 'n', len(U), 'sum', sum(U))
import heapq
for slots in (148,):
    h=[(0,i) for i in range(slots)]
    for c in U:
        l,i=heapq.heappop(h); heapq.heappush(h,(l+c+3,i))
    loads=[l for l,i in h]
    print('LPT loads max', max(loads), 'mean', sum(loads)/slots, 'min', min(loads))
