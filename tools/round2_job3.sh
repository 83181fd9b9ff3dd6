O=gpurun_out/r2c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "3d or variants or persistent" > $O/t3d.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "C4_m48 or C5_m32" >> $O/t3d.log 2>&1
timeout 600 python -m pytest tests/test_gpu_annulus.py -q -x >> $O/t3d.log 2>&1
IGA2L_S3D_PERSIST=1 timeout 600 python tools/phase_times.py C4,C5 5 > $O/ph_v5.txt 2>&1
IGA2L_S3D_PERSIST=0 timeout 600 python tools/phase_times.py C4,C5 5 > $O/ph_v4.txt 2>&1
timeout 600 python tools/vcycle_probe.py C2p5,C3,C4,C5 > $O/vcycle_probe.txt 2>&1
timeout 1200 python tools/annulus_table.py 128,256 > $O/annulus_table_b.txt 2>&1
ls $O
