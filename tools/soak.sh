#!/bin/bash
# Long soak of every fuzzer over many seeds (GPU box); one line per run.
cd "$(dirname "$0")/.."
O=gpurun_out/soak
mkdir -p $O
export FUZZ_WATCHDOG=900
for s in $(seq ${SOAK_FIRST:-101} ${SOAK_LAST:-112}); do
  timeout 1000 python tools/fuzz_u1v.py 400 $s 2>&1 | tail -1 >> $O/soak.txt
  timeout 1000 python tools/fuzz_all.py 48 $s 2>&1 | tail -1 >> $O/soak.txt
  timeout 1000 python tools/fuzz_dist.py 60 $s 2>&1 | tail -1 >> $O/soak.txt
  timeout 1000 python tools/fuzz_krylov.py 60 $s 2>&1 | tail -1 >> $O/soak.txt
  timeout 1000 python tools/fuzz_artefacts.py 30 $s 2>&1 | tail -1 >> $O/soak.txt
  timeout 1000 python tools/fuzz_threads.py 8 4 $s 2>&1 | tail -1 >> $O/soak.txt
  timeout 1000 python tools/fuzz_lanczos.py 12 $s 2>&1 | tail -1 >> $O/soak.txt
done
for s in ${SOAK_CHAOS:-201 202 203}; do
  KTB_LIB_NAME=libktb_chaos.so timeout 1000 python tools/fuzz_all.py 36 $s 2>&1 | tail -1 >> $O/soak.txt
  KTB_LIB_NAME=libktb_chaos.so timeout 1000 python tools/fuzz_dist.py 45 $s 2>&1 | tail -1 >> $O/soak.txt
  KTB_LIB_NAME=libktb_chaos.so timeout 1000 python tools/fuzz_threads.py 6 3 $s 2>&1 | tail -1 >> $O/soak.txt
done
grep -c . $O/soak.txt; grep -v "^fuzz_" $O/soak.txt | head -20
