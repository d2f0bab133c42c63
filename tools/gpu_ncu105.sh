#!/bin/bash
# ncu evidence for U1 param 105 (config 4 default bench): launch list + full capture of k_u1t
O=gpurun_out/s2
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
CMD="python bench.py --steps 2 --warmup 3 --warm-seconds 0 --no-cpu-baseline --no-secondary"
$CMD > $O/plain.log 2>&1 && \
$NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv $CMD > $O/ncu_launch.log 2>&1
echo launch rc $? >> $O/rc.txt
CMD1="python bench.py --steps 1 --warmup 3 --warm-seconds 0 --no-cpu-baseline --no-secondary"
$CMD1 > $O/plain1.log 2>&1 && \
$NCU --set full --clock-control none --import-source on -k regex:k_u1t -s 2 -c 1 -o $O/ncu_u1t_cfg4 $CMD1 > $O/ncu_full.log 2>&1
echo full rc $? >> $O/rc.txt
