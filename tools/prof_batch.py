"""Small driver for ncu captures of the batched kernels (cfg5 shapes, fewer
instances): python tools/prof_batch.py [mul|div] [count]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1402_0264_b200 as mmm  # noqa: E402

P = 469762049
what = sys.argv[1] if len(sys.argv) > 1 else "mul"
cnt = int(sys.argv[2]) if len(sys.argv) > 2 else 592
n = 4096
rng = np.random.default_rng(1)
A = torch.from_numpy(rng.integers(0, P, (cnt, 2 * n)).astype(np.uint32).view(np.int32)).cuda()
B = torch.from_numpy(rng.integers(1, P, (cnt, n)).astype(np.uint32).view(np.int32)).cuda()
F = torch.zeros((cnt, 2 * n), dtype=torch.int32, device="cuda")
R = torch.zeros((cnt, n), dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    if what == "mul":
        mmm.mul_batched_dev(P, A.data_ptr(), 2 * n, n, B.data_ptr(), n, n, cnt, F.data_ptr(),
                            2 * n, stream=st)
    else:
        mmm.divmod_batched_dev(P, A.data_ptr(), 2 * n, 2 * n, B.data_ptr(), n, n, cnt,
                               F.data_ptr(), n + 1, R.data_ptr(), n - 1, stream=st)
torch.cuda.synchronize()
print("ok", what, cnt)
