# symmetric scaling on the nodal path: parity + multirank tests, then A/B vs EMIN_DBG_UNSCALED on configs 4 / 5
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 1700 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x > $O/t_sn.log 2>&1; echo "pytest rc=$?"; tail -3 $O/t_sn.log
for f in 512 0; do timeout 300 python profiles/iter_time.py 4 $f 30 3; done
for f in 512 0; do timeout 600 python profiles/iter_time.py 5 $f 10 2; done
