#!/bin/bash
# ncu --set full of the setup-side kernels of one emin_setup on config 3
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
python profiles/setup_once.py 3 > $O/setup_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fill|k_plan_entries|k_alg2_nv1_wd|k_spgemm_wdm|k_rows|k_plan_pdesc|k_plan_wdesc|k_get_P_win" -c 12 -o $O/prof_setup python profiles/setup_once.py 3 > $O/ncu_setup.log 2>&1
echo "ncu rc=$?"
