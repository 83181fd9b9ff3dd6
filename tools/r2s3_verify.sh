#!/bin/bash
# Session-3 check of the restored build on one B200: GPU tests, smoke, default bench line.
O=gpurun_out/r2s3; mkdir -p $O
start=$(date +%s)
timeout 1500 python -m pytest tests -x -q -m gpu --durations=10 > $O/tests.log 2>&1; echo "tests rc=$? in $(( $(date +%s) - start )) s" >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --config C4 > $O/bench_C4.json 2> $O/bench_C4.err
