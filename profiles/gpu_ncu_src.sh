#!/bin/bash
# ncu --set full with source counters of the masked SpGEMM (scalar win2 on
# config 3, nodal v2x on config 4), one launch each, via profiles/spgemm_once.py
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
python profiles/spgemm_once.py 3 0 10 > $O/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spgemm_win2" -s 5 -c 1 -o $O/src_win2 python profiles/spgemm_once.py 3 0 10 > $O/ncu3.log 2>&1
echo "ncu3 rc=$?"
python profiles/spgemm_once.py 4 0 10 > $O/plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spgemm_nodal" -s 5 -c 1 -o $O/src_nodal4 python profiles/spgemm_once.py 4 0 10 > $O/ncu4.log 2>&1
echo "ncu4 rc=$?"
