"""Masked SpGEMM A/B driver: set up one config (device inputs) with the given
emin_opts.debug_flags, run emin_iterate(k) twice (warm-up, then timed with the
library's per-kernel CUDA events) and print the SpGEMM's average launch time.

  python profiles/spgemm_once.py [config] [debug_flags] [k]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2208_02995_b200 import Emin, emin_kernel_times, emin_set_profiling  # noqa: E402
from workloads.problems import make_config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "3"
dbg = int(sys.argv[2]) if len(sys.argv) > 2 else 0
k = int(sys.argv[3]) if len(sys.argv) > 3 else 10
prob = make_config(cfg)
g = Emin.from_problem(prob, stagnation_rel=0.0, debug_flags=dbg)
g.iterate(k, want=False)
torch.cuda.synchronize()
g.reset()
emin_set_profiling(g.h, 1)
g.iterate(k, want=False)
kt = emin_kernel_times(g.h)
ms, n = kt["spgemm"]
print(f"config {cfg} dbg {dbg}: spgemm {1e3 * ms / max(n, 1):.1f} us/launch over {n}; "
      f"stage1 {1e3 * kt['stage1'][0] / max(1, kt['stage1'][1]):.1f} us, "
      f"stage2 {1e3 * kt['stage2'][0] / max(1, kt['stage2'][1]):.1f} us, kernel_path {g.report()['kernel_path']}",
      flush=True)
