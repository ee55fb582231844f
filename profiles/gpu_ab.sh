#!/bin/bash
# GPU A/B session: variant parity tests, then per-variant kernel timings.
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "kernel_paths_agree or parity_small or composable" > $O/gputests_ab.log 2>&1; echo "pytest rc=$?" >> $O/gputests_ab.log
tail -3 $O/gputests_ab.log
#timeout 600 python profiles/spgemm_variants.py 3 win2 EMIN_PINGPONG=0 > $O/ab_c3.log 2>&1; tail -4 $O/ab_c3.log
timeout 600 python profiles/spgemm_variants.py 4 EMIN_NODAL=v2 EMIN_NODAL=v3 > $O/ab_c4.log 2>&1; tail -3 $O/ab_c4.log
