#!/bin/bash
# Round-end validation on one B200: GPU parity tests, smoke, bench lines for every config, the
# reference arm, the C2 launch list and one `ncu --set full` capture of each config's Schwarz kernel.
set -x
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 1500 python -m pytest tests -x -q -m gpu > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > $O/smoke.log 2>&1
for C in C2 C1 C3 C4 C5; do
  timeout 600 python bench.py --config $C > $O/bench_$C.json 2> $O/bench_$C.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
for C in C2 C1 C3 C4 C5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_schwarz --launch-skip 10 --launch-count 3 \
    -o $O/ncu_traffic_$C python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_traffic_$C.log 2>&1
  # reports are ~50 MB each (gpurun returns <= 64 MiB): keep the text summary and the raw metrics only
  ncu -i $O/ncu_traffic_$C.ncu-rep --page details > $O/ncu_traffic_$C.txt 2>&1
  ncu -i $O/ncu_traffic_$C.ncu-rep --page raw --csv > $O/ncu_traffic_${C}_raw.csv 2>&1
  python tools/ncu_hot.py $O/ncu_traffic_$C.ncu-rep 30 > $O/ncu_traffic_${C}_hot.txt 2>&1
  rm -f $O/ncu_traffic_$C.ncu-rep
done
ls -la $O
