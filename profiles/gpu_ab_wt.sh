#!/bin/bash
# A/B of the scalar masked SpGEMM: window-transposed records (k_spgemm_wt,
# default) vs row-contiguous records (k_spgemm_wd, EMIN_DBG_AB2 = 128)
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "transposed or kernel_paths or setup_energy" > $O/t_wt.log 2>&1; echo "pytest rc=$?"; tail -2 $O/t_wt.log
for r in 1 2; do
  for f in 0 128; do timeout 300 python profiles/spgemm_once.py 3 $f 20; done
done
for f in 0 128; do timeout 300 python profiles/iter_time.py 3 $f 20 5; done
if [ -n "$1" ]; then eval "$1"; fi
