#!/bin/bash
# bench lines of configs 1, 3, 5 (and 2) with the current build
O=gpurun_out/${1:-s3}
mkdir -p $O
for c in ${CFGS:-1 3 5 2}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo cfg$c rc $? >> $O/rc.txt
done
