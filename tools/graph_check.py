import sys; sys.path.insert(0,'/root/repo')
import torch
from paper_1508_05931_b200 import Engine, PipelineConfig, generate
xs, ys = generate("square", 20_000_000, 1)
eng = Engine(0)
s = torch.cuda.current_stream()
print("torch stream", s.cuda_stream)
eng._lib.gscan_set_stream(eng.handle, s.cuda_stream)
d_xs = torch.from_numpy(xs).cuda(); d_ys = torch.from_numpy(ys).cuda()
out = torch.empty(20_000_000, dtype=torch.int32, device="cuda")
for i in range(3):
    k, st = eng.hull_device(d_xs.data_ptr(), d_ys.data_ptr(), 20_000_000, out.data_ptr(), 20_000_000, PipelineConfig())
    print(k, st.t_total_ms, eng.sparse_info())
