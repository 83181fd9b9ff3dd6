#!/bin/bash
# A/B of the interior block-inverse paths (2D s^2 <= 32 DMMA kernel, 3D s = 3 pencil kernel) + their tests.
mkdir -p gpurun_out/ab
O=gpurun_out/ab
timeout 900 python -m pytest tests -x -q -m gpu -k "inverse or one_sweep or temporal or multiblock or batch or solve_matches or five_iter" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 900 python tools/variants.py IGA2L_MMA_INV 0,1 C2p3,C2p4,C2p5,C1 10 > $O/inv2d.txt 2>&1
timeout 900 python tools/variants.py IGA2L_S3D_INV 0,1 C4 5 > $O/inv3d.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > $O/bench_C2.json 2> $O/bench_C2.err
timeout 300 python bench.py --config C4 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
for C in C2 C4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_schwarz --launch-skip 10 --launch-count 3 \
    -o $O/ncu_$C python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_$C.log 2>&1
  ncu -i $O/ncu_$C.ncu-rep --page details > $O/ncu_$C.txt 2>&1
  ncu -i $O/ncu_$C.ncu-rep --page raw --csv > $O/ncu_${C}_raw.csv 2>&1
  python tools/ncu_hot.py $O/ncu_$C.ncu-rep 30 > $O/ncu_${C}_hot.txt 2>&1
  rm -f $O/ncu_$C.ncu-rep
done
