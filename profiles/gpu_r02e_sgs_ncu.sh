#!/bin/bash
# launch list of SGS (colouring) iterations on configs 3 and 4
O=gpurun_out
SGS_ONLY=sgs:color timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_sgs_c3.csv python profiles/sgs_vs_jacobi.py 3 5 > $O/ncu_sgs3.log 2>&1; echo "rc=$?"
SGS_ONLY=sgs:color timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_sgs_c4.csv python profiles/sgs_vs_jacobi.py 4 5 > $O/ncu_sgs4.log 2>&1; echo "rc=$?"
