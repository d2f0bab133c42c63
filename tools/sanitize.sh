#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py; one log per (tool, case) in
# gpurun_out/sanitize/, a summary line per run in gpurun_out/sanitize/summary.txt
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize
mkdir -p $OUT
: > $OUT/summary.txt
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for c in ${CASES:-s3 mgs ilu unsym halo}; do
    extra=""
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout ${T:-900} $CS --tool $tool $extra --print-limit 50 python tools/sanitize_cases.py $c \
        > $OUT/${tool}_${c}.log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $OUT/${tool}_${c}.log | tr '\n' ' ')" >> $OUT/summary.txt
  done
done
cat $OUT/summary.txt
