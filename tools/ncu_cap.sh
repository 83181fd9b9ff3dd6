#!/bin/bash
# ncu --set full capture of one kernel -> text details, raw csv and the hot-source summary (no .ncu-rep kept).
# usage: tools/ncu_cap.sh <outdir> <name> <kernel regex> <launch skip> <launch count> <command...>
O=$1 n=$2 k=$3 s=$4 c=$5; shift 5
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --graph-profiling node -k "regex:$k" \
  --launch-skip $s --launch-count $c -o $O/$n "$@" > $O/$n.log 2>&1
ncu -i $O/$n.ncu-rep --page details > $O/$n.txt 2>&1
ncu -i $O/$n.ncu-rep --page raw --csv > $O/${n}_raw.csv 2>&1
python tools/ncu_hot.py $O/$n.ncu-rep 25 > $O/${n}_hot.txt 2>&1
rm -f $O/$n.ncu-rep
