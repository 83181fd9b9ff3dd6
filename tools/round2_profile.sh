#!/bin/bash
# Round-2 evidence on one B200: bench lines for every config, the default bench's launch list, and
# `ncu --set full` captures (text summaries) of the dominant and the HBM-phase kernels.
O=gpurun_out/r2prof
mkdir -p $O
for C in C2 C1 C3 C4 C5; do
  timeout 900 python bench.py --config $C > $O/bench_$C.json 2> $O/bench_$C.err
done
timeout 900 python bench.py --config C4 --shard slab --steps 50 > $O/bench_C4_slab1.json 2> $O/bench_C4_slab1.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python tools/launches_summary.py $O/launches.csv > $O/launches.txt 2>&1
cap() {  # name, kernel regex, launch skip, count, command...
  local n=$1 k=$2 s=$3 c=$4; shift 4
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" --launch-skip $s --launch-count $c \
    -o $O/$n "$@" > $O/$n.log 2>&1
  ncu -i $O/$n.ncu-rep --page details > $O/$n.txt 2>&1
  ncu -i $O/$n.ncu-rep --page raw --csv > $O/${n}_raw.csv 2>&1
  python tools/ncu_hot.py $O/$n.ncu-rep 25 > $O/${n}_hot.txt 2>&1
  rm -f $O/$n.ncu-rep
}
cap ncu_C2_s2d_p5 "k_schwarz2d_mma<5" 10 3 python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline
cap ncu_C2_s2d_p3 "k_schwarz2d_mma<3" 10 3 python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline
cap ncu_C3_s2d "k_schwarz2d_mma" 10 2 python tools/kernel_run.py C3 sweep 2
cap ncu_C4_s3d "k_schwarz3d" 1 1 python tools/kernel_run.py C4 sweep 2
cap ncu_C5_s3d "k_schwarz3d" 1 1 python tools/kernel_run.py C5 sweep 2
cap ncu_C4_apply3d "k_apply3d_tma" 1 1 python tools/kernel_run.py C4 apply 2
cap ncu_C5_apply3d "k_apply3d_tma" 1 1 python tools/kernel_run.py C5 apply 2
cap ncu_C3_apply2d "k_apply2d_t" 1 1 python tools/kernel_run.py C3 apply 2
cap ncu_C5_prolong "k_band_axis" 3 3 python tools/kernel_run.py C5 prolong 2
cap ncu_C3_transfer "k_transfer2d_sep" 1 1 python tools/kernel_run.py C3 defect 2
cap ncu_C5_vcycle_gs "k_q_gs" 54 2 python tools/kernel_run.py C5 coarse 2
cap ncu_C5_vcycle_smem "k_vcycle_smem" 1 1 python tools/kernel_run.py C5 coarse 2
cap ncu_C2_vcycle_smem "k_vcycle_smem" 1 1 python tools/kernel_run.py C2p5 coarse 2
ls -la $O
