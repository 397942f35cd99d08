"""Summaries of ncu captures for profiles/ (run here on the .ncu-rep / CSV files gpurun brings back).

  python tools/ncu_summary.py launches <launch-list.csv>      per-kernel time share of one NS step
  python tools/ncu_summary.py kernel <capture.ncu-rep>        key metrics, stall reasons, top source lines
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in data:
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "second": 1e6, "byte": 1.0, "Kbyte": 1e3,
                 "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        per[r[ii]][r[mi]] = v * scale
        names[r[ii]] = r[ki].split("(")[0]
    agg = collections.OrderedDict()
    tot = 0.0
    for i, m in per.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        a = agg.setdefault(names[i], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += t
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        tot += t
    print(f"one NS step (graph-replayed) at 256^3: {len(per)} launches, {tot / 1e3:.3f} ms serialised (ncu, cold L2)")
    print(f"{'kernel':34s} {'launches':>8s} {'time_ms':>9s} {'share':>7s} {'dram_GB':>8s}")
    for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:34s} {c:8d} {t / 1e3:9.3f} {100 * t / tot:6.1f}% {b / 1e9:8.3f}")


def kernel(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u = r[0], r[1]
    want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "smsp__inst_executed.sum"]
    for v in r[2:]:  # every launch of the capture
        for w in want:
            if w in h:
                i = h.index(w)
                print(f"  {w:62s} {v[i]} {u[i]}")
        st = []
        for i, n in enumerate(h):
            if n.startswith("smsp__average_warps_issue_stalled") and n.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(v[i]), n.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        print("  stall cycles per issued instruction: " + ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:7]))
        print()
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, fn = [], None
    for row in csv.reader(io.StringIO(src)):
        if row and row[0] == "File Path":
            fn = row[1].split("/")[-1]
            continue
        if len(row) >= 5 and row[0] and row[0].isdigit():
            try:
                rows.append((int(row[4]), fn, int(row[0]), row[1].strip()[:96]))
            except ValueError:
                pass
    tot = sum(x[0] for x in rows) or 1
    print("  top source lines by warp-stall samples:")
    for s, f, l, text in sorted(rows, reverse=True)[:20]:
        print(f"    {100 * s / tot:5.1f}%  {f}:{l}  {text}")


if __name__ == "__main__":
    {"launches": launches, "kernel": kernel}[sys.argv[1]](sys.argv[2])
