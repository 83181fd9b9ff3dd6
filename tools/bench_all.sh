#!/bin/bash
# bench.py for every config (one B200), lines into gpurun_out/benchall/
mkdir -p gpurun_out/benchall
for C in C2 C1 C3 C4 C5; do
  timeout 600 python bench.py --config $C > gpurun_out/benchall/bench_$C.json 2> gpurun_out/benchall/bench_$C.err
done
