"""One fp32 apply + one V-cycle at 96^3 P3 (ncu target; developer tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_10226_b200 import mesh as M
from paper_2509_10226_b200.multigrid import PMultigrid
from paper_2509_10226_b200.reorder import reorder_mesh

m = reorder_mesh(M.kuhn_cube_mesh(int(sys.argv[1]) if len(sys.argv) > 1 else 96, seed=0))
mg = PMultigrid(m, (3, 2, 1), precision="mixed", coarse_matrix=True)
dm = mg.levels[0].dm
r = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)).cuda()
for _ in range(2):
    mg.vcycle(r)
torch.cuda.synchronize()
print("ok")
