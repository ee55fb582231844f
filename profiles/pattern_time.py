"""Time of emin_pattern per config: device inputs (CUDA events around the
call, count + fill passes, after a warm-up call) and, for reference, the
wall time with host (pageable numpy) inputs, which adds the copies."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2208_02995_b200 import emin as E  # noqa: E402
from workloads.problems import make_config  # noqa: E402

for cfg in sys.argv[1:] or ["3", "5"]:
    p = make_config(cfg)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    dA = (t(p.A_rowptr), t(p.A_col), t(p.is_coarse), t(p.Bc))
    E.emin_pattern(p.n, dA[0], dA[1], dA[2], p.block_size, p.nv, dA[3], p.nc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rp, col = E.emin_pattern(p.n, dA[0], dA[1], dA[2], p.block_size, p.nv, dA[3], p.nc)
    e1.record()
    e1.synchronize()
    ok = np.array_equal(rp.cpu().numpy(), p.P_rowptr) and np.array_equal(col.cpu().numpy(), p.P_col)
    th = time.perf_counter()
    E.emin_pattern(p.n, p.A_rowptr, p.A_col, p.is_coarse, p.block_size, p.nv, p.Bc, p.nc)
    wall = time.perf_counter() - th
    print(cfg, "emin_pattern device ms", round(e0.elapsed_time(e1), 2), "host-input wall s", round(wall, 3),
          "equal to generator", ok, flush=True)
