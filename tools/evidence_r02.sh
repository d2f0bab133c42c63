#!/bin/bash
# Round-2 evidence batch (GPU box): smoke, the GPU suite, bench lines, reference
# arms, launch list, ncu captures. Outputs under gpurun_out/r02/; the summaries
# kept in profiles/ are made from them by tools/ncu_summary.py.
cd "$(dirname "$0")/.."
O=gpurun_out/r02
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
python -m pytest tests -q -m gpu --durations=20 > $O/pytest_gpu.log 2>&1
python bench.py > $O/bench_default.json 2> $O/bench_default.err
python bench.py --impl reference > $O/reference_release.json 2> $O/reference_release.err
python bench.py --impl reference --ref-build native --steps 20 > $O/reference_native.json 2> $O/reference_native.err
for c in 1 2 3; do python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
python bench.py --config 5 --gmres-full-reference > $O/bench_cfg5.json 2> $O/bench_cfg5.err
# launch list of the default bench command (per-launch times are cold-cache and serialised)
$NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 --warm-seconds 0 \
  --no-cpu-baseline --no-secondary > $O/ncu_launch.log 2>&1
# full captures: the headline kernel inside the bench command, then single plans
$NCU --set full --clock-control none --import-source on -k regex:k_u1v -c 1 \
  -o $O/ncu_u1v_cfg4 python bench.py --steps 1 --warmup 3 --warm-seconds 0 --no-cpu-baseline \
  --no-secondary > $O/ncu_full.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:k_u1v -c 1 \
  -o $O/ncu_u1v_cfg1 python tools/ncu_one.py 1 0 106 >> $O/ncu_full.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:k_u1v -c 1 \
  -o $O/ncu_s1v_cfg2 python tools/ncu_one.py 2 16 106 >> $O/ncu_full.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:k_s3 -c 2 \
  -o $O/ncu_s3_cfg2 python tools/ncu_one.py 2 18 0 >> $O/ncu_full.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:"k_u1s" -c 1 \
  -o $O/ncu_u1s101_cfg3 python tools/ncu_one.py 3 0 101 >> $O/ncu_full.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:"k_u3w|k_fixup_carries" -c 2 \
  -o $O/ncu_u3w_cfg3 python tools/ncu_one.py 3 2 1008 >> $O/ncu_full.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:"k_u1v" -c 1 \
  -o $O/ncu_u1v_cfg5 python tools/ncu_one.py 5 0 106 >> $O/ncu_full.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:"k_mgs_dma" --launch-skip 25 -c 1 \
  -o $O/ncu_mgs_cfg5 python bench.py --config 5 --steps 1 --warmup 0 --warm-seconds 0 \
  --no-cpu-baseline >> $O/ncu_full.log 2>&1
tools/exchange_bench > $O/exchange_bench.txt 2>&1
ls -la $O
