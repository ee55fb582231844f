#!/bin/bash
# A/B of the masked SpGEMM variant selected by EMIN_DBG_AB1 (64): bitwise check
# against the default, then us per launch (profiles/spgemm_once.py) for each
# config given.  args: configs (default "3")
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for c in ${@:-3}; do
  timeout 600 python profiles/ab_bitwise.py $c 64 10 2>&1 | tail -1
  for rep in 1 2; do
    timeout 600 python profiles/spgemm_once.py $c 0 10 2>&1 | tail -1
    timeout 600 python profiles/spgemm_once.py $c 64 10 2>&1 | tail -1
  done
done
