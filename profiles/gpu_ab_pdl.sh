# A/B: programmatic dependent launch between the iteration's kernels (temporary debug bit 4096)
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for c in "3 4096 20 17" "1b 4096 20" "3 4096 40" "2b 4096 30 10"; do timeout 300 python profiles/ab_bitwise.py $c; done
for f in 0 4096 0 4096; do timeout 300 python profiles/iter_time.py 3 $f 40 5; done
timeout 300 python profiles/step_ab.py 3 0 4096 9
