import sys, json, numpy as np, torch
sys.path.insert(0, ".")
from paper_2208_02995_b200 import emin as E
from workloads.problems import make_config
p = make_config("5")
keys = ["A_rowptr", "A_col", "A_val", "is_coarse", "P_rowptr", "P_col", "P_val", "B", "Bc"]
dev = {k: (None if getattr(p, k) is None else torch.from_numpy(np.ascontiguousarray(getattr(p, k))).cuda()) for k in keys}
h = E.emin_setup(p.n, p.nc, dev["A_rowptr"], dev["A_col"], dev["A_val"], dev["is_coarse"], dev["P_rowptr"], dev["P_col"],
                 dev["P_val"], p.nv, dev["B"], dev["Bc"], block_size=3, stagnation_rel=0.0)
E0 = E.emin_report(h)["E0"]
kd, dE = E.emin_iterate(h, 40, want=True)
Ek = E0 - np.cumsum(dE)
print(json.dumps({"E0": E0, "E_k": Ek.tolist(), "target_sgs10": 143823.72133763676,
                  "first_k_at_or_below": int(np.argmax(Ek <= 143823.72133763676)) + 1 if (Ek <= 143823.72133763676).any() else None}))
