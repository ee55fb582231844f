#!/bin/bash
# ncu --set full (source-level) of the scalar masked SpGEMM variants on config 3
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for f in ${FLAGS:-0 5120}; do
  python profiles/spgemm_once.py 3 $f 10 > $O/plain_$f.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spgemm_w" -s 5 -c 1 -o $O/prof_wp_$f python profiles/spgemm_once.py 3 $f 10 > $O/ncu_$f.log 2>&1
  echo "ncu $f rc=$?"
done
