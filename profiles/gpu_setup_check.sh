O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/t_par.log 2>&1; echo "pytest rc=$?"; tail -2 $O/t_par.log
python profiles/step_breakdown.py 3 2>&1 | tail -3
python profiles/setup_once.py 3 > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_setup.csv python profiles/setup_once.py 3 > /dev/null 2>&1; echo ncu rc=$?
