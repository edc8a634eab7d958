"""Summarise an ncu --set full report into a small JSON (kept under profiles/)."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_op_red.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "us": 1e-6, "ms": 1e-3, "ns": 1e-9,
        "Ghz": 1e9, "Mhz": 1e6}


def summarise(rep):
    """rep: an .ncu-rep, or the `ncu -i rep --page raw --csv` export of one."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else None}
        stalls = {}
        for i, name in enumerate(h):
            try:
                x = float(v[i].replace(",", ""))
            except ValueError:
                continue
            if name in KEYS:
                d[name] = x * UNIT.get(units[i], 1.0) if units[i] in UNIT else x
            if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
                stalls[name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = x
        d["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda t: -t[1])[:6])
        if "dram__bytes_read.sum" in d:
            d["dram_bytes_per_launch"] = d["dram__bytes_read.sum"] + d.get("dram__bytes_write.sum", 0.0)
        res.append(d)
    return res


if __name__ == "__main__":
    print(json.dumps(summarise(sys.argv[1]), indent=1))
