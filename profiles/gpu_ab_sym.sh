# symmetric Jacobi scaling (default) vs the unscaled CG (EMIN_DBG_UNSCALED = 512)
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > $O/t_par.log 2>&1; echo "pytest rc=$?"; tail -3 $O/t_par.log
for f in 512 0 512 0; do timeout 300 python profiles/spgemm_once.py 3 $f 20; done
for f in 512 0; do timeout 300 python profiles/iter_time.py 3 $f 40 5; done
timeout 300 python profiles/step_ab.py 3 512 0 9
