# A/B of launch shapes of the scaled pair kernel (temporary debug bits 12-14)
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for f in 4096 12288 20480; do timeout 300 python profiles/ab_bitwise.py 3 $f 10 17; done
for r in 1 2; do for f in 0 4096 8192 12288 16384 20480 24576 28672; do timeout 300 python profiles/spgemm_once.py 3 $f 20; done; done
