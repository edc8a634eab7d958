"""GPU-bound timing of back-to-back applies (no host gaps), with and without an L2
flush between applies; also the host enqueue cost per apply.  Developer tool."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from quick_bench_setup import build  # noqa: E402


def main():
    for spec in sys.argv[1:]:
        A, nd, meta = build(spec)
        u = torch.rand(nd, dtype=torch.float64, device="cuda") * 2 - 1
        y = torch.empty_like(u)
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
        st = torch.cuda.current_stream()
        for _ in range(5):
            A.apply_into(u.data_ptr(), y.data_ptr(), st.cuda_stream)
        torch.cuda.synchronize()
        n = 50
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(n):
            A.apply_into(u.data_ptr(), y.data_ptr(), st.cuda_stream)
        e1.record()
        host_us = (time.perf_counter() - t0) / n * 1e6
        e1.synchronize()
        hot = e0.elapsed_time(e1) / n
        e0.record()
        for _ in range(n):
            flush.fill_(1.0)
        e1.record()
        e1.synchronize()
        fl = e0.elapsed_time(e1) / n
        e0.record()
        for _ in range(n):
            flush.fill_(1.0)
            A.apply_into(u.data_ptr(), y.data_ptr(), st.cuda_stream)
        e1.record()
        e1.synchronize()
        cold = e0.elapsed_time(e1) / n - fl
        meta.update(ndof=nd, hot_ms=round(hot, 4), cold_ms=round(cold, 4), host_enqueue_us=round(host_us, 1),
                    gdofs_hot=round(nd / hot / 1e6, 3), gdofs_cold=round(nd / cold / 1e6, 3),
                    frac_fp64_cold=round(A.info["flops_alg"] / (cold * 1e-3) / 37.1e12, 3))
        print(json.dumps(meta), flush=True)


if __name__ == "__main__":
    main()
