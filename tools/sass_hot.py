"""Summarise an ncu '--page source --csv --print-source sass' export: stall reasons, hot instructions, and
samples per 100-instruction region (diagnostics for the INT8 product kernels)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) >= len(hdr) - 1]
si = hdr.index("Warp Stall Sampling (All Samples)")
ei = hdr.index("Instructions Executed")
reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]


def v(r, i):
    try:
        return int(r[i])
    except ValueError:
        return 0


tot = sum(v(r, si) for r in data)
print("total samples", tot, "instructions", len(data))
sums = {h: sum(v(r, i) for r in data) for i, h in reasons}
print(sorted(sums.items(), key=lambda x: -x[1])[:10])
step = int(sys.argv[2]) if len(sys.argv) > 2 else 100
for k in range(0, len(data), step):
    s = sum(v(r, si) for r in data[k:k + step])
    if s > tot * 0.01:
        ops = Counter((r[1].split()[1] if r[1].strip().startswith("@") else r[1].split()[0]) for r in data[k:k + step])
        st = Counter()
        for r in data[k:k + step]:
            for i, h in reasons:
                st[h[6:]] += v(r, i)
        print(f"{k:5d} {s:6d} ({100.0 * s / tot:4.1f}%)", ops.most_common(5), st.most_common(3))
