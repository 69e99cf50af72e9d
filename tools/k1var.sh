# time K1 (k_extremes_tma) for alternative builds
for v in ${@:-default}; do
  if [ "$v" = default ]; then lib=""; else lib=paper_1508_05931_b200/_lib/var/$v/libgscan.so; fi
  GSCAN_LIB=$lib timeout 120 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', 'K1', d['kernels_ms'].get('k_extremes_tma'), 'F2', d['kernels_ms'].get('k_sp_hist'), 'ms', d['ms_per_step'], 'parity', d['parity_vs_golden'])"
done
