#!/bin/bash
# Round-2 (session 3) end evidence on one B200: ncu of the C5 z-chain colour kernel first (its DRAM bytes per launch
# feed bench.py's roofline.traffic), GPU tests + smoke, bench lines for every config and the reference arm, the
# default bench's launch list.
O=gpurun_out/r2s3end; mkdir -p $O
cap() {  # name, kernel regex, launch skip, count, command...
  local n=$1 k=$2 s=$3 c=$4; shift 4
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" \
    --launch-skip $s --launch-count $c -o $O/$n "$@" > $O/$n.log 2>&1
  ncu -i $O/$n.ncu-rep --page details > $O/$n.txt 2>&1
  ncu -i $O/$n.ncu-rep --page raw --csv > $O/${n}_raw.csv 2>&1
  python tools/ncu_hot.py $O/$n.ncu-rep 25 > $O/${n}_hot.txt 2>&1
  rm -f $O/$n.ncu-rep
}
cap ncu_C5_s3dzc "k_schwarz3d_zc" 1 1 python tools/kernel_run.py C5 sweep 2
python tools/traffic.py C5=$O/ncu_C5_s3dzc_raw.csv@ncu_C5_s3dzc_r02.txt > $O/traffic_C5.json 2> $O/traffic.err
python - <<'PY'
import json
p = "profiles/schwarz_traffic.json"
d = json.load(open(p)); d.update(json.load(open("gpurun_out/r2s3end/traffic_C5.json")))
json.dump(d, open(p, "w"), indent=1)
PY
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
ls -la $O
