#!/bin/bash
# full GPU test suite + A/B of given variant specs on given configs
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
tail -3 $O/gputests.log
for spec in "$@"; do
  timeout 600 python profiles/spgemm_variants.py $spec > $O/ab.log 2>&1; grep -v '^{' $O/ab.log | tail -4
done
