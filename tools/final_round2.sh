#!/bin/bash
# Round-2 end validation on one B200: all GPU tests, smoke, bench lines for every config, the reference arm,
# the default bench's launch list, and ncu captures of the dominant kernels (via tools/kernel_run.py).
O=gpurun_out/final2; mkdir -p $O
start=$(date +%s)
timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > $O/tests.log 2>&1; echo "tests rc=$? in $(( $(date +%s) - start )) s" >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > $O/smoke.log 2>&1
for C in C2 C1 C3 C4; do
  timeout 900 python bench.py --config $C > $O/bench_$C.json 2> $O/bench_$C.err
done
timeout 1500 python bench.py --config C5 > $O/bench_C5.json 2> $O/bench_C5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python tools/launches_summary.py $O/launches.csv > $O/launches.txt 2>&1
tools/ncu_cap.sh $O ncu_C4_s3d "k_schwarz3d" 1 1 python tools/kernel_run.py C4 sweep 2
tools/ncu_cap.sh $O ncu_C5_s3d "k_schwarz3d" 1 1 python tools/kernel_run.py C5 sweep 2
tools/ncu_cap.sh $O ncu_C5_band "k_band" 3 3 python tools/kernel_run.py C5 prolong 2
ls -la $O
