import torch, numpy as np, ctypes
import synth, oracle
from paper_2103_13042_b200 import spamm as sp
M=N=K=256
A = synth.perturbed_decay_matrix(K, 0.95, seed=11, m=M)
plan = sp.Plan(M,N,K,0.0,"fp32")
Ad = torch.from_numpy(A).cuda()
plan.norms(Ad, Ad); plan.build_skipmap(); torch.cuda.synchronize()
print(plan.stats())
V, rw = sp.spamm_get_counts(plan.handle)
print("V sum", V.sum().item(), "rw", rw.tolist())
ptr, ent, order, GM, GN = sp.spamm_get_macro(plan.handle)
print("macro_ptr", ptr.tolist(), "order", order.tolist())
