"""Host model of the tensor path's 128-row MMA granularity on configs[4] (N = 65536, lambda = 0.999,
BF16, tau = 1e-6): kept (i,k,j) pairs / pair slots the issued MMA runs cover.  Prints 0.994."""
import numpy as np, synth, oracle
N=65536; T=32; BD=N//T; tau=1e-6
table=synth.round_to_bf16(synth.decay_table("exp", N, 0.999).astype(np.float32))
r = oracle.tile_norms(synth.toeplitz_block(table, 0, T, 0, 2048*T//8), T)[0]   # offsets 0..255 tiles
r = np.concatenate([r, np.zeros(4096)])
W=800
issued=0.0; kept=0.0; ksteps=0
li=np.arange(8)
for d1 in range(-W, W):          # d1 = 8I - k  (row offset of the tile's first row)
    a = r[np.abs(d1+li)]         # norms of rows 0..7
    for d2 in range(-W, W):
        if (d1+d2) % 8: continue
        b = r[np.abs(d2-li)]     # cols: j = 8J+lj, offset k-j = d2 - lj
        m = (a[:,None]*b[None,:]) >= tau
        if not m.any(): continue
        ksteps += 1
        for h in range(2):
            mh = m[4*h:4*h+4]
            nc = mh.any(axis=0).sum()
            issued += 4*nc
            kept += mh.sum()
print("kept/issued pair slots", kept/issued, "steps", ksteps)
