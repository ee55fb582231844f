"""Wall time of emin_pattern (host inputs, includes the H2D copies) per config."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2208_02995_b200 import emin as E  # noqa: E402
from workloads.problems import make_config  # noqa: E402

for cfg in sys.argv[1:] or ["3", "5"]:
    p = make_config(cfg)
    E.emin_pattern(p.n, p.A_rowptr, p.A_col, p.is_coarse, p.block_size, p.nv, p.Bc, p.nc)
    torch.cuda.synchronize()
    t = time.perf_counter()
    rp, col = E.emin_pattern(p.n, p.A_rowptr, p.A_col, p.is_coarse, p.block_size, p.nv, p.Bc, p.nc)
    dt = time.perf_counter() - t
    ok = np.array_equal(rp, p.P_rowptr) and np.array_equal(col, p.P_col)
    print(cfg, "emin_pattern s", round(dt, 3), "equal to generator", ok, flush=True)
