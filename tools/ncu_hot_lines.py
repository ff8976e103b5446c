"""Hottest source lines of an ncu source page (stdin: `ncu -i X.ncu-rep --page
source --csv`): top 25 lines by warp stall samples, with their instruction
counts."""
import csv
import sys


def main():
    rows = list(csv.reader(l for l in sys.stdin if l.startswith('"')))
    if not rows:
        print("no source page")
        return
    # the page starts with file-name rows; the header is the first row that
    # names a "Source" column (repeated per kernel: the first is used)
    hdr = next((r for r in rows if any(c.strip() == "Source" for c in r)), rows[0])

    def col(*names):
        for n in names:
            for i, h in enumerate(hdr):
                if h.strip().lower() == n.lower():
                    return i
        return None
    si = col("Source")
    ws = col("Warp Stall Sampling (All Samples)", "Warp Stall Sampling (All Cycles)", "# Samples")
    ie = col("Instructions Executed")
    if si is None or ws is None:
        print("columns:", hdr)
        return
    data = []
    for r in rows:
        if r == hdr or len(r) <= max(si, ws):
            continue
        try:
            w = float(r[ws].replace(",", "") or 0)
        except ValueError:
            continue
        n = r[ie] if ie is not None and len(r) > ie else ""
        data.append((w, n, r[si].strip()))
    tot = sum(d[0] for d in data) or 1.0
    print(f"total samples {tot:.0f}")
    for w, n, src in sorted(data, key=lambda d: -d[0])[:25]:
        print(f"{100 * w / tot:5.1f}%  inst {n:>10}  {src[:120]}")


if __name__ == "__main__":
    main()
