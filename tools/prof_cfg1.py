import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1402_0264_b200 as mmm
P = 469762049
rng = np.random.default_rng(1)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 14
a = torch.from_numpy(rng.integers(0, P, n).astype(np.uint32).view(np.int32)).cuda()
b = torch.from_numpy(rng.integers(1, P, n).astype(np.uint32).view(np.int32)).cuda()
f = torch.zeros(2 * n, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    mmm.mul_dev(P, a.data_ptr(), n, b.data_ptr(), n, f.data_ptr(), stream=st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    mmm.mul_dev(P, a.data_ptr(), n, b.data_ptr(), n, f.data_ptr(), stream=st)
e1.record(); torch.cuda.synchronize()
print("cfg1-shape product", e0.elapsed_time(e1) / 20 * 1e3, "us")
