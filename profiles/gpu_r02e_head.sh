#!/bin/bash
# HEAD confirmation after the A/B sessions: build, GPU suite, smoke, default bench
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 600 python bench.py > $O/bench_c3_head.json 2> $O/bench_c3_head.err; echo "bench rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -x > $O/gputests_head.log 2>&1; echo "pytest rc=$?" >> $O/gputests_head.log
tail -n 2 $O/gputests_head.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_head.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_head.json 2> $O/bench_ref_head.err; echo "ref rc=$?"
