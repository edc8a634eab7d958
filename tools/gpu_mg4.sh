set -x
timeout 900 python -m pytest tests/test_gpu_multigrid.py -x -q > gpurun_out/mg4_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python tools/bench_configs.py mg --n5 128 --precision mixed > gpurun_out/mg_128_mixed.jsonl 2> gpurun_out/mg_128_mixed.err; echo "rc=$?"
timeout 900 python tools/quick_bench.py cgv:3:128 > gpurun_out/q_cg3_128.jsonl 2>&1
python - > gpurun_out/f32_apply_times.jsonl 2>&1 <<'PY'
import json, sys, torch, numpy as np
sys.path.insert(0, '.')
from tools.bench_configs import setup
from paper_2509_10226_b200 import operator as op
for n, p in ((128, 3), (128, 2), (128, 1), (48, 4)):
    m, dm, geo, bas, ts = setup(n, p, "cg", True, tuple(range(6)))
    A = op.CgPoissonOperator(m, dm, geo, bas, op.OperatorConfig(f32_mirror=True))
    u = torch.rand(dm.n_global_dofs, dtype=torch.float64, device="cuda")
    y = torch.empty_like(u); u32 = u.float(); y32 = torch.empty_like(u32)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3): A.apply_into(u.data_ptr(), y.data_ptr(), st); A.apply_f32(u32, out=y32)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record()
    for _ in range(10): A.apply_into(u.data_ptr(), y.data_ptr(), st)
    e[1].record()
    for _ in range(10): A.apply_f32(u32, out=y32)
    e[2].record(); e[2].synchronize()
    t64, t32 = e[0].elapsed_time(e[1]) / 10, e[1].elapsed_time(e[2]) / 10
    print(json.dumps({"n": n, "p": p, "ndof": dm.n_global_dofs, "fp64_ms": round(t64, 4), "fp32_ms": round(t32, 4),
                      "rel_diff": float(torch.linalg.vector_norm(y32.double() - y) / torch.linalg.vector_norm(y))}), flush=True)
    del A
PY
echo done
