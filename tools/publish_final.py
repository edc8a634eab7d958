"""Copy the outputs of tools/gpu_final.sh from gpurun_out/ into profiles/r02/ (run here, after
the gpurun call): bench lines, config lines, test log, launch-list shares, the ncu --set full
summaries of the C2 cell kernels (tools/summarize_roofline.py) and of the face kernels."""
import csv
import gzip
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles", "r02")


def ncu_raw(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    return r.stdout


def main():
    shutil.copy(os.path.join(G, "final_bench.json"), os.path.join(P, "bench_c2.json"))
    shutil.copy(os.path.join(G, "final_bench_ref.json"), os.path.join(P, "bench_reference_arm.json"))
    shutil.copy(os.path.join(G, "final_configs.jsonl"), os.path.join(P, "configs_single_gpu.jsonl"))
    shutil.copy(os.path.join(G, "final_launches.csv"), os.path.join(P, "bench_launches_ncu.csv"))
    with open(os.path.join(P, "gpu_suite_head.log"), "w") as f:
        f.write(open(os.path.join(G, "final_smoke.log")).read())
        f.write("".join(open(os.path.join(G, "final_tests.log")).readlines()[-3:]))
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "summarize_roofline.py")], check=True,
                   stdout=subprocess.DEVNULL)
    with gzip.open(os.path.join(P, "ncu_c2_cell_kernels_raw.csv.gz"), "wt") as f:
        f.write(ncu_raw(os.path.join(G, "prof_c2.ncu-rep")))
    # face kernels
    path = os.path.join(P, "ncu_faces_splitmode.json")
    out = json.load(open(path))
    aft = {}
    names = {"dg_3": "C3 DG-SIPG P3 64^3 reordered, interior faces at HEAD",
             "helmk_2": "kappa-Helmholtz P2 64^3 reordered, interior faces at HEAD"}
    keys = [("duration_us", "gpu__time_duration.sum"), ("registers", "launch__registers_per_thread"),
            ("grid", "launch__grid_size"), ("block", "launch__block_size"),
            ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
            ("dram_read", "dram__bytes_read.sum"), ("dram_write", "dram__bytes_write.sum"),
            ("lts_throughput_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            ("l1_data_pipe_pct", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
            ("dmma_pipe_pct", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
            ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            ("l2_hit_pct", "lts__t_sector_hit_rate.pct"), ("l1_hit_pct", "l1tex__t_sector_hit_rate.pct"),
            ("l2_red_sectors", "lts__t_sectors_srcunit_tex_op_red.sum")]
    for t, name in names.items():
        rows = list(csv.reader(ncu_raw(os.path.join(G, f"ncu_face_{t}.ncu-rep")).splitlines()))
        hdr, units, r = rows[0], rows[1], rows[2]
        d = {"what": name, "kernel": r[hdr.index("Kernel Name")]}
        for k, h in keys:
            if h in hdr:
                d[k] = (r[hdr.index(h)] + " " + units[hdr.index(h)]).strip()
        st = {}
        for h in hdr:
            m = re.search(r"smsp__average_warps_issue_stalled_(.*)_per_issue_active", h)
            if m and float(r[hdr.index(h)]) > 0.3:
                st[m.group(1)] = round(float(r[hdr.index(h)]), 2)
        d["stalls_per_issue"] = dict(sorted(st.items(), key=lambda x: -x[1]))
        aft[t] = d
    out["at_head"] = aft
    json.dump(out, open(path, "w"), indent=1)
    # launch-list shares
    rows = list(csv.reader(open(os.path.join(G, "final_launches.csv"))))
    i0 = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i0]
    K, V, U = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = {}
    for r in rows[i0 + 1:]:
        if len(r) <= V:
            continue
        k = re.sub(r"\(.*", "", r[K])
        v = float(r[V].replace(",", ""))
        v = v / 1000.0 if r[U] in ("ns", "nsecond") else v * 1000.0 if r[U] in ("ms", "msecond") else v
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    json.dump({"what": "ncu --metrics gpu__time_duration.sum --clock-control none launch list of `bench.py --steps 2 "
                       "--warmup 3 --no-cpu --no-quadrature --c4-n 0` (every launch of the process: setup kernels, "
                       "L2-flush fills, warm-up and timed applies; per-launch times are cold-cache and serialised "
                       "-- the kernels' SHARES are what to compare with the bench line)",
               "total_us": tot,
               "kernels": [{"kernel": k, "launches": v[0], "us": round(v[1], 1), "share_pct": round(100 * v[1] / tot, 1)}
                           for k, v in sorted(agg.items(), key=lambda t: -t[1][1])]},
              open(os.path.join(P, "bench_launches_ncu.json"), "w"), indent=1)
    b = json.loads(open(os.path.join(P, "bench_c2.json")).read().strip().splitlines()[-1])
    print("bench", b["value"], b["ms_per_step"], "e2e", b["e2e"]["value"], b["e2e"]["link"]["frac"], "c4", b["c4_strong"]["value"])
    for k, v in b["per_degree"].items():
        print("  ", k, v["ms"], v["gdofs"], v["frac_engine"], v["frac_alg"])
    print("roofline", {k: b["roofline"][k] for k in ("achieved", "frac", "frac_alg", "traffic", "kernel_ms")})
    for t in aft:
        print(t, {k: aft[t].get(k) for k in ("duration_us", "dram_read", "dram_write", "l2_hit_pct", "dmma_pipe_pct", "l1_data_pipe_pct", "l2_red_sectors")})
    for k, v in sorted(agg.items(), key=lambda t: -t[1][1])[:6]:
        print(f"  {100 * v[1] / tot:5.1f}%  {k[:80]}")


if __name__ == "__main__":
    main()
