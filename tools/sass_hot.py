"""Top stall-sampled SASS instructions from `ncu -i rep --page source --csv --print-source sass`."""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    S = h.index("Source")
    W = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    data = []
    for r in rows[2:]:
        try:
            data.append((float(r[W] or 0), r))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1.0
    print(f"{len(data)} instructions, {tot:.0f} samples")
    for v, r in sorted(data, key=lambda x: -x[0])[:top]:
        st = sorted(((float(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:3]
        print(f"{100 * v / tot:5.1f}%  {r[S].strip()[:60]:60s} " + " ".join(f"{n}:{int(c)}" for c, n in st if c))
    # totals per stall reason
    agg = {h[i][6:]: sum(float(r[i] or 0) for _, r in data) for i in stall_cols}
    print({k: round(100 * v / tot, 1) for k, v in sorted(agg.items(), key=lambda t: -t[1])[:8]})


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
