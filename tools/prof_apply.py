"""Run a few applies of one operator (ncu target): python tools/prof_apply.py <loop_bench spec> [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from tools.loop_bench import build  # noqa: E402

A, nd = build(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
u = torch.rand(nd, dtype=torch.float64, device="cuda") * 2 - 1
y = torch.empty_like(u)
st = torch.cuda.current_stream().cuda_stream
for _ in range(n):
    A.apply_into(u.data_ptr(), y.data_ptr(), st)
torch.cuda.synchronize()
print("ok", A.info["cell_engine"], A.info["face_engine"])
