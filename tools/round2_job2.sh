O=gpurun_out/r2b; mkdir -p $O
timeout 1500 python tools/annulus_table.py > $O/annulus_table.txt 2>&1
timeout 1500 python bench.py --config C5 > $O/bench_C5.json 2> $O/bench_C5.err
tools/ncu_cap.sh $O ncu_C2p5_s2d "k_schwarz2d_mma" 10 2 python tools/kernel_run.py C2p5 sweep 14
tools/ncu_cap.sh $O ncu_C2p3_s2d "k_schwarz2d_mma" 10 2 python tools/kernel_run.py C2p3 sweep 14
tools/ncu_cap.sh $O ncu_C3_s2d "k_schwarz2d_mma" 10 1 python tools/kernel_run.py C3 sweep 12
ls $O
