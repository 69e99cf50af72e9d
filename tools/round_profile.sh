#!/bin/bash
# One GPU call that refreshes the round's measured artifacts into gpurun_out/prof2:
# the GPU test suite, smoke, the bench lines (C2 default + C1, C3, C4, C5), the
# reference arm, the ncu launch list of a short bench run, and one ncu --set full
# capture of the hot kernels on C2 and of F2 on C5.
set -u
out=gpurun_out/prof2
mkdir -p $out
timeout 1800 python -m pytest tests -m gpu -q > $out/pytest_gpu.txt 2>&1; tail -2 $out/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1; tail -1 $out/smoke.txt
timeout 600 python bench.py > $out/bench_C2.json 2> $out/bench_C2.err; tail -c 400 $out/bench_C2.json
for c in C1 C3 C4; do timeout 600 python bench.py --config $c --steps 20 > $out/bench_$c.json 2> $out/bench_$c.err; done
timeout 900 python bench.py --config C5 --steps 10 > $out/bench_C5.json 2> $out/bench_C5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 2 > $out/bench_ref_C2.json 2> $out/bench_ref_C2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $out/launch_run.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k "regex:k_extremes|k_sp_hist|k_sp_phi|k_sp_cand|k_gr_mid|k_gr_cert|k_gr_up|k_gr_down|k_sp_dup|k_sp_place_g|k_sp_sort_gathered|k_sp_walk|k_sp_lrank|k_sp_f2_patch" -c 20 -o $out/full \
  python tools/one_call.py square 20000000 1 > $out/full_run.log 2>&1
ncu -i $out/full.ncu-rep --page raw --csv > $out/full_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k "regex:k_sp_hist_ring|k_extremes_tma" -c 2 -o $out/c5 \
  python tools/big_check.py 1e9 > $out/c5_run.log 2>&1
ncu -i $out/c5.ncu-rep --page raw --csv > $out/c5_raw.csv 2>/dev/null
ls -la $out
