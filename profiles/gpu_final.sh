#!/bin/bash
# Round checkpoint on one B200: full GPU suite, smoke, default bench, launch
# list and one ncu --set full capture of the dominant kernel.
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q > $O/gputests_final.log 2>&1; echo "pytest rc=$?" >> $O/gputests_final.log
tail -2 $O/gputests_final.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_final.json 2> $O/bench_final.err; echo "bench rc=$?"
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$P > $O/plain_l.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_final.csv $P > $O/ncu_l.log 2>&1
$P > $O/plain_f.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spgemm_win2 -s 20 -c 1 -o $O/prof_final $P > $O/ncu_f.log 2>&1
echo "ncu rc=$?"
timeout 600 python - > $O/pattern_c5.log 2>&1 <<'PY'
import time, numpy as np, torch, sys
sys.path.insert(0, ".")
from workloads.problems import make_config
from paper_2208_02995_b200 import emin as E
for cfg in ("3", "5"):
    p = make_config(cfg)
    E.emin_pattern(p.n, p.A_rowptr, p.A_col, p.is_coarse, p.block_size, p.nv, p.Bc, p.nc)
    torch.cuda.synchronize(); t = time.perf_counter()
    rp, col = E.emin_pattern(p.n, p.A_rowptr, p.A_col, p.is_coarse, p.block_size, p.nv, p.Bc, p.nc)
    dt = time.perf_counter() - t
    print(cfg, "emin_pattern s", round(dt, 3), "equal to generator", np.array_equal(rp, p.P_rowptr) and np.array_equal(col, p.P_col))
PY
tail -2 $O/pattern_c5.log
