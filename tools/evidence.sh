#!/bin/bash
# Round evidence: bench lines for every config (+ sharded paths and the
# reference arm), the launch list of the default bench command, and ncu full
# captures of the top kernels. Run on the GPU box from the repo root:
#   gpurun -- 'bash tools/evidence.sh r01'
R=${1:-r01}
O=gpurun_out/$R
mkdir -p $O
for c in 2 1 3 4 5; do
  timeout 900 python bench.py --config $c --steps 30 --warmup 5 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 900 python bench.py --config 3 --shard --steps 30 --warmup 5 > $O/bench_cfg3_shard.json 2> $O/bench_cfg3_shard.err
timeout 900 python bench.py --config 5 --shard --steps 30 --warmup 5 > $O/bench_cfg5_shard.json 2> $O/bench_cfg5_shard.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_cfg2.json 2> $O/bench_reference_cfg2.err
# launch list of the default bench command (cold-cache, serialised per-launch times)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_cfg2.csv \
  python bench.py --steps 2 --warmup 3 --warm-seconds 0 --no-cpu-baseline > $O/ncu_launches.log 2>&1
# full captures
ncu --set full --clock-control none --import-source on -k regex:"k_s3" -c 2 -o $O/s3_cfg2 \
  python tools/prof_kernels.py --config 2 --kernels s3 --reps 1 --time-reps 1 > $O/ncu_s3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_u1s" -c 1 -o $O/u1s_cfg5 \
  python tools/prof_kernels.py --config 5 --kernels u1 --params 100 --reps 1 --time-reps 1 > $O/ncu_u1s5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_u1s" -c 1 -o $O/u1s_cfg1 \
  python tools/prof_kernels.py --config 1 --kernels u1 --params 100 --reps 1 --time-reps 1 > $O/ncu_u1s1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_u1s" -c 1 -o $O/u1s_cfg3 \
  python tools/prof_kernels.py --config 3 --kernels u1 --params 101 --reps 1 --time-reps 1 > $O/ncu_u1s3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_mgs_res" --launch-skip 25 -c 1 -o $O/mgs_cfg5 \
  python bench.py --config 5 --steps 1 --warmup 0 --warm-seconds 0 --no-cpu-baseline > $O/ncu_mgs.log 2>&1
echo done > $O/DONE
