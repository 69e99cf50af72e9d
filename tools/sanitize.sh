#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over both pipelines at
# C2/C3 sizes and small n (sparse path on device-resident input -- the CUDA
# graph with programmatic dependent launch -- at 20M and 300K square and disk;
# the host entry with the overlapped ingest at 20M; full sort: 4K disk, 2K
# circle) and the sharded path (3 simulated ranks, 600K disk, the device-side
# data plane and the distributed F6). Logs in gpurun_out/san/ (summaries
# copied to profiles/ by hand).
out=gpurun_out/san
mkdir -p $out
run() {  # tool label command...
  local tool=$1 label=$2; shift 2
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 "$@" > $out/${tool}_${label}.log 2>&1
  echo "$tool $label rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $out/${tool}_${label}.log | tail -1)"
}
for tool in memcheck racecheck synccheck; do
  for c in "square 20000000" "disk 20000000" "square 300000" "disk 300000" "disk 4000" "circle 2000"; do
    set -- $c
    run $tool $1_$2 python tools/one_call.py $1 $2 1
  done
  ONE_CALL_HOST=1 run $tool host_square_20000000 python tools/one_call.py square 20000000 1
  run $tool sharded_disk_600000 python tools/sharded_check.py
done
