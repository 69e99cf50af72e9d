#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over both pipelines at
# C2/C3 sizes and small n (sparse path: 20M and 300K square and disk; full sort:
# 4K disk, 2K circle),
# logs in gpurun_out/san/ (summaries copied to profiles/ by hand).
out=gpurun_out/san
mkdir -p $out
for tool in memcheck racecheck synccheck; do
  for c in "square 20000000" "disk 20000000" "square 300000" "disk 300000" "disk 4000" "circle 2000"; do
    set -- $c
    timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 \
      python tools/one_call.py $1 $2 1 > $out/${tool}_$1_$2.log 2>&1
    echo "$tool $1 $2 rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $out/${tool}_$1_$2.log | tail -1)"
  done
done
