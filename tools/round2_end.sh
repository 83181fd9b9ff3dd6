#!/bin/bash
# Round-2 end evidence on one B200: GPU tests + smoke, bench lines for every config (+ the slab mode at N=1 and
# the reference arm), the default bench's launch list, and ncu --set full captures of each config's dominant
# colour kernel (text, raw csv for tools/traffic.py, hot lines).
O=gpurun_out/r2end; mkdir -p $O
start=$(date +%s)
timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > $O/tests.log 2>&1; echo "tests rc=$? in $(( $(date +%s) - start )) s" >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > $O/smoke.log 2>&1
for C in C2 C1 C3 C4; do
  timeout 900 python bench.py --config $C > $O/bench_$C.json 2> $O/bench_$C.err
done
timeout 1500 python bench.py --config C5 > $O/bench_C5.json 2> $O/bench_C5.err
timeout 900 python bench.py --config C4 --shard slab --steps 50 > $O/bench_C4_slab1.json 2> $O/bench_C4_slab1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python tools/launches_summary.py $O/launches.csv > $O/launches.txt 2>&1
cap() {  # name, kernel regex, launch skip, count, command...
  local n=$1 k=$2 s=$3 c=$4; shift 4
  timeout 900 ncu --set full --clock-control none --import-source on --graph-profiling node -k "regex:$k" \
    --launch-skip $s --launch-count $c -o $O/$n "$@" > $O/$n.log 2>&1
  ncu -i $O/$n.ncu-rep --page details > $O/$n.txt 2>&1
  ncu -i $O/$n.ncu-rep --page raw --csv > $O/${n}_raw.csv 2>&1
  python tools/ncu_hot.py $O/$n.ncu-rep 25 > $O/${n}_hot.txt 2>&1
  rm -f $O/$n.ncu-rep
}
cap ncu_C2_s2d_p5 "k_schwarz2d_mma" 10 2 python tools/kernel_run.py C2p5 sweep 14
cap ncu_C1_s2d "k_schwarz2d_mma" 10 3 python bench.py --config C1 --steps 1 --warmup 3 --no-cpu-baseline
cap ncu_C3_s2d "k_schwarz2d_mm" 10 2 python tools/kernel_run.py C3 sweep 14
cap ncu_C4_s3dw "k_schwarz3d_w" 1 1 python tools/kernel_run.py C4 sweep 2
cap ncu_C5_s3dw "k_schwarz3d_w" 1 1 python tools/kernel_run.py C5 sweep 2
python tools/traffic.py C1=$O/ncu_C1_s2d_raw.csv@ncu_C1_s2d_r02.txt C2=$O/ncu_C2_s2d_p5_raw.csv@ncu_C2_s2d_p5_r02.txt \
  C3=$O/ncu_C3_s2d_raw.csv@ncu_C3_s2d_r02.txt C4=$O/ncu_C4_s3dw_raw.csv@ncu_C4_s3dw_r02.txt \
  C5=$O/ncu_C5_s3dw_raw.csv@ncu_C5_s3dw_r02.txt > $O/schwarz_traffic.json 2> $O/traffic.err
ls -la $O
