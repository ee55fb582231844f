# A/B: record plan kernels (temporary debug bit 4096 = the previous kernel)
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for c in "3 4096 10 17" "1b 4096 20" "3 4096 10" "2b 4096 20 10"; do timeout 300 python profiles/ab_bitwise.py $c; done
timeout 300 python profiles/step_ab.py 3 4096 0 9
python profiles/setup_once.py 3 > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_setup.csv python profiles/setup_once.py 3 > /dev/null 2>&1; echo ncu rc=$?
