#!/bin/bash
# build + the GPU test suite (+ optional extra command)
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -x > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
tail -3 $O/gputests.log
if [ -n "$1" ]; then eval "$1"; fi
