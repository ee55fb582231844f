#!/bin/bash
# End-of-session evidence on one B200 (round 1, after the multilevel /
# paired-gather changes): full GPU suite, smoke, benches of configs 3/4/5,
# launch list and one ncu --set full capture of the dominant kernels.
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q > $O/gputests_final.log 2>&1; echo "pytest rc=$?" >> $O/gputests_final.log
tail -2 $O/gputests_final.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c3_final.json 2> $O/bench_c3_final.err; echo "bench3 rc=$?"
timeout 900 python bench.py --config 4 --steps 10 > $O/bench_c4_final.json 2> $O/bench_c4_final.err; echo "bench4 rc=$?"
timeout 1500 python bench.py --config 5 --steps 3 > $O/bench_c5_final.json 2> $O/bench_c5_final.err; echo "bench5 rc=$?"
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$P > $O/plain_l.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_final.csv $P > $O/ncu_l.log 2>&1
$P > $O/plain_f.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spgemm_win2|k_stage" -s 20 -c 3 -o $O/prof_final $P > $O/ncu_f.log 2>&1
echo "ncu rc=$?"
P5="python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$P5 > $O/plain_f4.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spgemm_nodal_v2" -s 5 -c 1 -o $O/prof_c4 $P5 > $O/ncu_f4.log 2>&1
echo "ncu4 rc=$?"
