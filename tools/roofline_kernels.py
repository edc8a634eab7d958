"""The 8 C2 bench applies once each (after a warm-up round), in bench order, for the
committed ncu capture of their cell kernels (tools/capture_roofline.sh):

    ncu --set full -k regex:cell_ -s 8 -c 8 python tools/roofline_kernels.py

Prints the order of the problems (one key per line) so the capture can be keyed.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_10226_b200 import operator as op  # noqa: E402

probs = []
for reorder in (False, True):
    for p in bench.DEGREES:
        m, dm, geo, bas = bench.build_problem(bench.N_MESH, p, reorder)
        A = op.CgPoissonOperator(m, dm, geo, bas)
        u = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)).cuda()
        probs.append((f"p{p}{'_reordered' if reorder else ''}", A, u, torch.empty_like(u)))
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for rnd in range(2):
    for key, A, u, y in probs:
        flush.fill_(1.0)
        A.apply_into(u.data_ptr(), y.data_ptr(), st)
        if rnd == 1:
            print(key, flush=True)
torch.cuda.synchronize()
