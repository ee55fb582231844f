#!/bin/bash
# End-of-round-2 evidence on one B200 (HEAD after the nodal lane-group kernel
# and the pending-dW flush): default bench first (fresh box), launch list,
# ncu --set full of the masked SpGEMM of configs 3 / 4 / 5, the GPU suite,
# smoke, then the config 4 / 5 benches.
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench3 rc=$?"
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$P > $O/plain_l.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv $P > $O/ncu_l.log 2>&1
echo "ncu-list rc=$?"
python profiles/spgemm_once.py 3 0 10 > $O/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spgemm|k_stage" -s 15 -c 3 -o $O/prof_c3 python profiles/spgemm_once.py 3 0 10 > $O/ncu3.log 2>&1
echo "ncu3 rc=$?"
python profiles/spgemm_once.py 4 0 10 > $O/plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spgemm_nodal" -s 12 -c 1 -o $O/prof_c4 python profiles/spgemm_once.py 4 0 10 > $O/ncu4.log 2>&1
echo "ncu4 rc=$?"
python profiles/spgemm_once.py 5 0 3 > $O/plain5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none -k regex:"k_spgemm_nodal" -s 4 -c 1 -o $O/prof_c5 python profiles/spgemm_once.py 5 0 3 > $O/ncu5.log 2>&1
echo "ncu5 rc=$?"
for c in 3 4 5; do
  [ -f $O/prof_c$c.ncu-rep ] && ncu -i $O/prof_c$c.ncu-rep --page details > $O/ncu_c${c}_full.txt 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q -x > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
tail -n 2 $O/gputests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --config 4 --steps 10 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench4 rc=$?"
timeout 1500 python bench.py --config 5 --steps 3 > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench5 rc=$?"
timeout 600 python bench.py > $O/bench_c3_after.json 2> $O/bench_c3_after.err; echo "bench3b rc=$?"
