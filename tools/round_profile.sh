#!/bin/bash
# One GPU call that refreshes the round's measured artifacts into gpurun_out/:
# the GPU test suite, the bench line, the reference-arm line, the ncu launch
# list of a short bench run, and one ncu --set full capture of the hot kernels.
set -u
out=gpurun_out/prof
mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; tail -2 $out/pytest_gpu.txt
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err; tail -1 $out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err; tail -1 $out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $out/launch_run.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k "regex:k_extremes|k_sp_hist|k_sp_phi|k_sp_cand|k_gr_mid|k_gr_cert|k_gr_up|k_gr_down|k_sp_dup|k_sp_place_g|k_sp_sort_gathered|k_sp_walk" -c 18 -o $out/full \
  python tools/one_call.py square 20000000 1 > $out/full_run.log 2>&1
ncu -i $out/full.ncu-rep --page raw --csv > $out/full_raw.csv 2>/dev/null
ls -la $out
