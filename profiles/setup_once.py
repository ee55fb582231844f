"""One emin_setup + 1 iteration + energy + get_P of a config from device
inputs (for launch lists of the setup: ncu --metrics gpu__time_duration.sum)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2208_02995_b200 import Emin  # noqa: E402
from workloads.problems import make_config  # noqa: E402

prob = make_config(sys.argv[1] if len(sys.argv) > 1 else "5")
g = Emin.from_problem(prob, device="cuda", stagnation_rel=0.0)
g.iterate(1)
g.energy()
g.get_P()
g.close()
torch.cuda.synchronize()
print("ok")
