"""Print the key ncu 'details' metrics and the top stalled SASS lines of CSV exports
(tools/gpu_ncu_*.sh): python tools/ncu_brief.py gpurun_out/ncu_<name> [n_lines]"""
import csv
import sys

WANT = ["Duration", "L1/TEX Cache Throughput", "L2 Cache Throughput", "DRAM Throughput", "Achieved Occupancy",
        "Registers Per Thread", "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate", "Mem Busy", "Max Bandwidth",
        "Mem Pipes Busy", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block", "SM Active Cycles",
        "Elapsed Cycles", "Executed Ipc Active", "Theoretical Occupancy"]


def main(base, n=25):
    rows = list(csv.reader(open(base + "_details.csv")))
    h = rows[0]
    for r in rows[1:]:
        if r[h.index("Metric Name")] in WANT:
            print("   ", r[h.index("Metric Name")], r[h.index("Metric Value")], r[h.index("Metric Unit")])
    try:
        rows = list(csv.reader(open(base + "_sass.csv")))
    except FileNotFoundError:
        return
    h = rows[1]
    data = rows[2:]
    tot = sum(int(r[2]) for r in data if r[2].isdigit())
    print("  samples", tot)
    for r in sorted(data, key=lambda r: -int(r[2]) if r[2].isdigit() else 0)[:n]:
        st = {h[i][6:]: int(r[i]) for i in range(29, 46) if r[i].isdigit() and int(r[i]) > 0}
        st = dict(sorted(st.items(), key=lambda t: -t[1])[:2])
        print("  ", r[0][-5:], r[2].rjust(6), r[1][:58].ljust(58), st)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
