# A/B of k_spgemm_wp variants selected by temporary debug bits (see profiles/r02/spgemm_ab_c3.txt)
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for f in $FL; do for c in "3 $f 10 17" "1b $f 20"; do timeout 300 python profiles/ab_bitwise.py $c; done; done
for r in 1 2; do for f in 0 $FL; do timeout 300 python profiles/spgemm_once.py 3 $f 20; done; done
for f in 0 $FL; do timeout 300 python profiles/iter_time.py 3 $f 20 5; done
