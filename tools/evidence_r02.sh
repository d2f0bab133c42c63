#!/bin/bash
# Round-2 evidence batch (GPU box): bench lines, reference arms, ncu.
cd "$(dirname "$0")/.."
O=gpurun_out/r02
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
python -m pytest tests -q -m gpu --durations=20 > $O/pytest_gpu.log 2>&1
python bench.py > $O/bench_default.json 2> $O/bench_default.err
python bench.py --impl reference > $O/reference_release.json 2> $O/reference_release.err
python bench.py --impl reference --ref-build native --steps 20 > $O/reference_native.json 2> $O/reference_native.err
tools/gather_bench > $O/gather.txt 2>&1
for c in 1 2 3; do python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
python bench.py --config 5 --gmres-full-reference > $O/bench_cfg5.json 2> $O/bench_cfg5.err
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 --warm-seconds 0 \
  --no-cpu-baseline --no-secondary > $O/ncu_launch.log 2>&1
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_u1s -c 1 \
  -o $O/ncu_u1s_cfg1 python bench.py --config 1 --steps 1 --warmup 3 --warm-seconds 0 \
  --no-cpu-baseline > $O/ncu_full.log 2>&1
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_u1p -c 1 \
  -o $O/ncu_u1p_cfg4 python bench.py --steps 1 --warmup 3 --warm-seconds 0 --no-cpu-baseline \
  --no-secondary >> $O/ncu_full.log 2>&1
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_s3 -c 2 \
  -o $O/ncu_s3_cfg2 python tools/ncu_one.py 2 18 0 >> $O/ncu_full.log 2>&1
ls -la $O
