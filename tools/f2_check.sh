#!/bin/bash
# F2 A/B on the GPU: the sparse GPU tests, a short bench, one ncu capture of F2.
out=gpurun_out/${1:-f2}
mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_golden.py -x -q > $out/pytest.txt 2>&1; tail -2 $out/pytest.txt
timeout 300 python bench.py --steps 30 --no-cpu-baseline > $out/bench.json 2> $out/bench.err
python - $out/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("ms", d["ms_per_step"], "parity", d["parity_vs_golden"], "roof", d["roofline"]["frac"], d["roofline"]["kernel_ms"])
k=d["kernels_ms"]; print({a:k[a] for a in sorted(k, key=lambda a:-k[a])[:12]})
PY
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_sp_hist -c 2 -o $out/f2 python tools/one_call.py square 20000000 1 > $out/ncu.log 2>&1
