#!/bin/bash
# A/B of EMIN_DBG_AB1 sub-variants (debug_flags = 64 | v << 8): bitwise check, us per launch.
# args: config variant...
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
c=$1; shift
timeout 600 python profiles/spgemm_once.py $c 0 10 2>&1 | tail -1
for v in "$@"; do
  f=$((64 | (v << 8)))
  timeout 600 python profiles/ab_bitwise.py $c $f 10 2>&1 | tail -1
  timeout 600 python profiles/spgemm_once.py $c $f 10 2>&1 | tail -1
done
timeout 600 python profiles/spgemm_once.py $c 0 10 2>&1 | tail -1
