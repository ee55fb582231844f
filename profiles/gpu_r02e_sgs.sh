#!/bin/bash
# Jacobi vs projected SGS per iteration at HEAD (configs 3, 4: 20 steps; config 5: 5 steps)
O=gpurun_out
timeout 600 python profiles/sgs_vs_jacobi.py 3 20 > $O/sgs_vs_jacobi_c3.log 2>&1; echo "c3 rc=$?"
timeout 900 python profiles/sgs_vs_jacobi.py 4 20 > $O/sgs_vs_jacobi_c4.log 2>&1; echo "c4 rc=$?"
SGS_ONLY=jacobi:None timeout 900 python profiles/sgs_vs_jacobi.py 5 5 > $O/sgs_vs_jacobi_c5_jacobi.log 2>&1; echo "c5j rc=$?"
SGS_ONLY=sgs:color timeout 1200 python profiles/sgs_vs_jacobi.py 5 5 > $O/sgs_vs_jacobi_c5_sgs.log 2>&1; echo "c5s rc=$?"
