#!/bin/bash
# A/B: the scalar y^ record stream read with an L2 evict-first policy
# (-DWP_EVF, createpolicy + ld.global.nc.L2::cache_hint) vs the default __ldg.
O=gpurun_out
run() {
  timeout 300 python profiles/spgemm_once.py 3 0 20 2>&1 | tail -n 1 | tee -a $O/evf_$1.log
  timeout 300 python profiles/iter_time.py 3 0 20 5 2>&1 | tail -n 1 | tee -a $O/evf_$1.log
  timeout 300 python profiles/spgemm_once.py 3 0 20 2>&1 | tail -n 1 | tee -a $O/evf_$1.log
  timeout 300 python profiles/iter_time.py 3 0 20 5 2>&1 | tail -n 1 | tee -a $O/evf_$1.log
}
rm -f $O/evf_*.log
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
run base
touch paper_2208_02995_b200/csrc/kernels_fast.cuh
EMIN_NVCC_EXTRA=-DWP_EVF python -c "import __graft_entry__ as g; g.build()" > $O/build_evf.log 2>&1 || { tail $O/build_evf.log; exit 1; }
run evf
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "full_size_scalar or parity_small or config3" > $O/evf_tests.log 2>&1; echo "pytest rc=$?"; tail -n 2 $O/evf_tests.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c3_evf.json 2> $O/bench_c3_evf.err; echo "bench rc=$?"
