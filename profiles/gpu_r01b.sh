#!/bin/bash
# GPU session: parity tests, config-3 bench, launch list, ncu --set full of
# the masked SpGEMM on configs 3 (scalar win2) and 4 (nodal).
set -x
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
timeout 900 python bench.py --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench rc=$?" >> $O/bench_c3.err
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$P > $O/plain3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv $P > $O/ncu_l3.log 2>&1
$P > $O/plain3b.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spgemm_win2 -s 20 -c 2 -o $O/prof_c3 $P > $O/ncu_c3.log 2>&1
P4="python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$P4 > $O/plain4.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spgemm_nodal -s 20 -c 2 -o $O/prof_c4 $P4 > $O/ncu_c4.log 2>&1
echo done
