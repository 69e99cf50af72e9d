"""One C2-sized hull call on device-resident input, the bench's `value` path
(for ncu captures): python tools/one_call.py [kind] [n] [calls]
ONE_CALL_HOST=1: through the host entry instead (hull_indices: overlapped ingest)."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1508_05931_b200 import Engine, PipelineConfig, generate  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "square"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000_000
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 1
eng = Engine(0)
if kind == "square":  # generated on the device, bit-identical to gen_square
    xs = torch.empty(n, dtype=torch.float64, device="cuda")
    ys = torch.empty_like(xs)
    eng.generate_square_device(1, 0, n, xs.data_ptr(), ys.data_ptr())
else:
    hx, hy = generate(kind, n, 1)
    xs, ys = torch.from_numpy(hx).cuda(), torch.from_numpy(hy).cuda()
torch.cuda.synchronize()
out = torch.empty(n, dtype=torch.int32, device="cuda")
for _ in range(calls):
    if os.environ.get("ONE_CALL_HOST"):
        idx, st = eng.hull_indices(xs.cpu().numpy(), ys.cpu().numpy(), PipelineConfig())
    else:
        k, st = eng.hull_device(xs.data_ptr(), ys.data_ptr(), n, out.data_ptr(), n, PipelineConfig())
print(kind, n, st.n_after_round1, st.n_after_round2, st.hull_size, eng.sparse_info(), flush=True)
