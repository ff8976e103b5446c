"""Dynamic SASS profile of one kernel from an ncu report (needs --set full):
stall reasons, hottest instructions, executed-instruction mix.

    python tools/ncu_sass_profile.py REPORT.ncu-rep [kernel index]
"""
import collections
import csv
import io
import subprocess
import sys


def main(path, which=0):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO("".join(l + "\n" for l in out.splitlines()
                                               if l.startswith('"')))))
    heads = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    if not heads:
        print("no SASS page in", path)
        return
    h0 = heads[min(which, len(heads) - 1)]
    end = next((i for i in heads if i > h0), len(rows) + 1) - 1
    hdr, data = rows[h0], [r for r in rows[h0 + 1:end] if len(r) > 10]
    ci = {n: i for i, n in enumerate(hdr)}
    name = rows[h0 - 1][1] if h0 > 0 else "?"
    f = lambda r, n: float(r[ci[n]].replace(",", "") or 0)
    tot = sum(f(r, "# Samples") for r in data) or 1.0
    execd = sum(f(r, "Instructions Executed") for r in data)
    print(f"kernel: {name}")
    print(f"static instructions {len(data)}, executed warp instructions {execd:.0f}, samples {tot:.0f}")
    stalls = [n for n in hdr if n.startswith("stall_") and "Not Issued" not in n]
    agg = {n: sum(f(r, n) for r in data) for n in stalls}
    print("stall reasons (share of samples):")
    for n, v in sorted(agg.items(), key=lambda kv: -kv[1])[:9]:
        print(f"  {n:26s} {100 * v / tot:5.1f}%")
    print("hottest instructions:")
    for r in sorted(data, key=lambda r: -f(r, "# Samples"))[:14]:
        print(f"  {100 * f(r, '# Samples') / tot:5.1f}%  executed {int(f(r, 'Instructions Executed')):>8}  "
              f"{r[1].strip()[:80]}")
    mix = collections.Counter()
    for r in data:
        parts = r[1].strip().split()
        if not parts:
            continue
        op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
        mix[op.split(".")[0]] += f(r, "Instructions Executed")
    print("executed-instruction mix:")
    print("  " + ", ".join(f"{k} {100 * v / execd:.1f}%" for k, v in mix.most_common(16)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
