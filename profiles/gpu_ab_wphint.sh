#!/bin/bash
# A/B: cache hints on the once-per-launch streams of the scalar y^ kernel
# (-DWP_V: 1 = Q by ld.cs, 2 = Q by ld.cs + y^ by st.cs, 3 = Q by ld.cg,
# 4 = Q and the lane descriptors by ld.cs) vs the default.
O=gpurun_out
run() {
  for r in 1 2; do
    timeout 300 python profiles/spgemm_once.py 3 0 20 2>&1 | tail -n 1 | tee -a $O/wphint_$1.log
    timeout 300 python profiles/iter_time.py 3 0 20 5 2>&1 | tail -n 1 | tee -a $O/wphint_$1.log
  done
}
rm -f $O/wphint_*.log
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
run v0
for V in 1 2 3 4; do
  touch paper_2208_02995_b200/csrc/kernels_fast.cuh
  EMIN_NVCC_EXTRA=-DWP_V=$V python -c "import __graft_entry__ as g; g.build()" > $O/build_v$V.log 2>&1 || { tail $O/build_v$V.log; exit 1; }
  run v$V
done
