#!/bin/bash
# Round 2 evidence: GPU suite, smoke, default bench (config 3), config 4 / 5
# benches, launch list of the default step, ncu --set full of the masked
# SpGEMM (config 3 wd, config 4 nodal).
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -x > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
tail -2 $O/gputests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench3 rc=$?"
if [ "$1" == "all" ]; then
timeout 900 python bench.py --config 4 --steps 10 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench4 rc=$?"
timeout 1500 python bench.py --config 5 --steps 3 > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench5 rc=$?"
fi
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$P > $O/plain_l.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv $P > $O/ncu_l.log 2>&1
echo "ncu-list rc=$?"
python profiles/spgemm_once.py 3 0 10 > $O/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spgemm_wp|k_stage" -s 15 -c 3 -o $O/prof_c3 python profiles/spgemm_once.py 3 0 10 > $O/ncu3.log 2>&1
echo "ncu3 rc=$?"
