#!/bin/bash
# A/B of the scalar masked SpGEMM: pair-lane kernel (k_spgemm_wp) variants
# (debug_flags bits 10-12) vs one entry per lane (k_spgemm_wd, flag 128)
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pair_kernel or kernel_paths or setup_energy" > $O/t_wp.log 2>&1; echo "pytest rc=$?"; tail -2 $O/t_wp.log
for f in 128 0 1024 2048 3072 0 1024 2048 3072; do timeout 300 python profiles/spgemm_once.py 3 $f 20; done
for f in 0 1024 2048 3072; do timeout 300 python profiles/iter_time.py 3 $f 20 5; done
if [ -n "$1" ]; then eval "$1"; fi
