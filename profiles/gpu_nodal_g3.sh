#!/bin/bash
# Nodal y^ with three blocks per round (9 gathers in flight per lane; the single
# position chunk frees the registers), nodal parity tests,
# SpGEMM / iteration times on configs 4 / 5, ncu --set full of one config-4
# launch.
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 300 python profiles/spgemm_once.py 4 0 30 2>&1 | tee $O/sp4.log
timeout 300 python profiles/iter_time.py 4 0 30 3 2>&1 | tee $O/it4.log
timeout 600 python profiles/spgemm_once.py 5 0 5 2>&1 | tee $O/sp5.log
timeout 1500 python -m pytest tests -m gpu -q -x -k "elasticity or nodal or multirank or multilevel or config4 or 4" > $O/t_g3.log 2>&1; echo "pytest rc=$?"; tail -2 $O/t_g3.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spgemm_nodal -s 12 -c 1 -o $O/prof_c4_g3 python profiles/spgemm_once.py 4 0 10 > $O/ncu4.log 2>&1
echo "ncu4 rc=$?"
