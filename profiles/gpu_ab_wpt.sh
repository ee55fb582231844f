O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for c in "3 6144 10 17" "1b 6144 20"; do timeout 300 python profiles/ab_bitwise.py $c; done
for f in 0 5120 6144 0 5120 6144; do timeout 300 python profiles/spgemm_once.py 3 $f 20; done
for f in 0 5120 6144; do timeout 300 python profiles/iter_time.py 3 $f 20 5; done
