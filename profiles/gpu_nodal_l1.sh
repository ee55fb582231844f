#!/bin/bash
# Nodal y^ with the second position chunk spread over lane groups
# (n3 = 36: 4 positions x 8 lanes): GPU parity / multirank / multilevel
# suites, SpGEMM and iteration times on configs 4 / 5, ncu --set full of one
# config-4 nodal launch.
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > $O/t_l1.log 2>&1; echo "pytest rc=$?"; tail -2 $O/t_l1.log
timeout 300 python profiles/spgemm_once.py 4 0 30 2>&1 | tee $O/sp4.log
timeout 300 python profiles/iter_time.py 4 0 30 3 2>&1 | tee $O/it4.log
timeout 600 python profiles/spgemm_once.py 5 0 5 2>&1 | tee $O/sp5.log
timeout 600 python profiles/iter_time.py 5 0 10 2 2>&1 | tee $O/it5.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spgemm_nodal -s 12 -c 1 -o $O/prof_c4_l1 python profiles/spgemm_once.py 4 0 10 > $O/ncu4.log 2>&1
echo "ncu4 rc=$?"
