"""What the y memset costs inside a CG apply (developer experiment): the full apply
(zero + cells) against the cell stage alone, CUDA events after an L2 flush."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from tools.loop_bench import build  # noqa: E402


def med(f, flush, n=30):
    ts = []
    for _ in range(n):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return round(float(np.median(ts)), 4)


for spec in sys.argv[1:]:
    A, nd = build(spec)
    u = torch.rand(nd, dtype=torch.float64, device="cuda") * 2 - 1
    y = torch.empty_like(u)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(5):
        A.apply_into(u.data_ptr(), y.data_ptr(), st)
    full = med(lambda: A.apply_stages(u.data_ptr(), y.data_ptr(), 1 | 2 | 8, stream=st), flush)
    cells = med(lambda: A.apply_stages(u.data_ptr(), y.data_ptr(), 2 | 8, stream=st), flush)
    zero = med(lambda: A.apply_stages(u.data_ptr(), y.data_ptr(), 1, stream=st), flush)
    empty = med(lambda: None, flush)
    print(json.dumps({"spec": spec, "zero_cells_ms": full, "cells_only_ms": cells, "zero_only_ms": zero,
                      "empty_event_pair_ms": empty}), flush=True)
