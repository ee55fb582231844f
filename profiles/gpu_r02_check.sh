#!/bin/bash
# Round 2 re-entry check on one B200: build, GPU suite, smoke, default bench,
# launch list of the default step.
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -x > $O/gputests_r02.log 2>&1; echo "pytest rc=$?" >> $O/gputests_r02.log
tail -3 $O/gputests_r02.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench3 rc=$?"
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$P > $O/plain_l.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv $P > $O/ncu_l.log 2>&1
echo "ncu rc=$?"
