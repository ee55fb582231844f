#!/bin/bash
# ncu --set full of one launch of each SpGEMM variant (plain run first).
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for spec in "3 win2 k_spgemm_win2" "3 win4 k_spgemm_win4" "3 hdr k_spgemm_hdr" "4 EMIN_NODAL=s k_spgemm_nodal_s" "4 EMIN_NODAL=v2 k_spgemm_nodal_v2"; do
  set -- $spec
  tag=$(echo $2 | tr '=' '_')
  python profiles/spgemm_variants.py $1 $2 > $O/plain_$tag.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s 5 -c 1 -o $O/ab_$tag python profiles/spgemm_variants.py $1 $2 > $O/ncu_$tag.log 2>&1
  echo "$spec rc=$?"
done
