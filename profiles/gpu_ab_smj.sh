# A/B: slot-major scaled records with an L1 prefetch of the window's block (temporary debug bit 4096)
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for c in "3 4096 10 17" "1b 4096 20" "3 4096 20" "2b 4096 20 10"; do timeout 300 python profiles/ab_bitwise.py $c; done
for r in 1 2; do for f in 0 4096; do timeout 300 python profiles/spgemm_once.py 3 $f 20; done; done
for f in 0 4096; do timeout 300 python profiles/iter_time.py 3 $f 40 5; done
timeout 300 python profiles/step_ab.py 3 0 4096 9
