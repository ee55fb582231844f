import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2208_02995_b200.multilevel import emin_multilevel
from workloads.problems import coarse_split, make_config
prob = make_config("3")
dims, zlo = prob.meta["dims"], 0
iscs = []
for _ in range(4):
    isc, dims, zlo = coarse_split(dims, zlo)
    iscs.append(torch.from_numpy(isc.astype(np.uint8)).cuda())
t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
for stag in (1e-30, 0.0):
    try:
        lv = emin_multilevel(t(prob.A_rowptr), t(prob.A_col), t(prob.A_val), iscs, t(prob.B), P_rowptr=t(prob.P_rowptr),
                             P_col=t(prob.P_col), P_val=None, iters=40, stagnation_rel=stag)
        for l in lv: print(stag, l["level"], l["k_done"], l["E0"], l["E"], float(l["dE"][-1] / l["dE"][0]))
    except Exception as e:
        print(stag, "ERR", e)
