"""Per-kernel launch counts and time shares from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv ...`).

    python tools/ncu_shares.py launches.csv [header line]
"""

import collections
import csv
import gzip
import sys


def main(path, header=None):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                      hdr.index("Metric Value"), hdr.index("Metric Unit"))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        v_us = v / 1e3 if unit in ("nsecond", "ns") else (v * 1e3 if unit in ("msecond", "ms") else v)
        name = r[ki].replace("(sg::StepArgs<T1>)", "").replace("sg::", "")[:60]
        tot[name] += v_us
        cnt[name] += 1
    all_us = sum(tot.values())
    if header:
        print(header)
    print("cold-cache, serialised launches: compare SHARES, not absolute times")
    for name, us in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{name:<60} launches={cnt[name]:6d} total={us / 1e3:9.3f} ms "
              f"share={100 * us / all_us:5.1f}% mean={us / cnt[name]:9.2f} us")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
