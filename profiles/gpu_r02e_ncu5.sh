#!/bin/bash
# ncu --set full of one config-5 ITERATION launch of the nodal masked SpGEMM
# (launch order in spgemm_once.py: setup r0/E0 pass, 3 warm-up iterations, the
# reset's r0/E0 pass, 3 timed iterations -> skip 5).
O=gpurun_out
python profiles/spgemm_once.py 5 0 3 > $O/plain5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none -k regex:"k_spgemm_nodal" -s 5 -c 2 -o $O/prof_c5it python profiles/spgemm_once.py 5 0 3 > $O/ncu5it.log 2>&1
echo "ncu5 rc=$?"
ncu -i $O/prof_c5it.ncu-rep --page details > $O/ncu_c5_iter_full.txt 2>&1
ncu -i $O/prof_c5it.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > $O/ncu_c5_iter_traffic.csv 2>&1
