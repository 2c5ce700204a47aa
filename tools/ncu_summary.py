"""Summarise an ncu capture exported by tools/ncu_visits.sh: duration, DRAM
throughput and bytes, SM/issue activity, occupancy, the warp-stall breakdown
and the SASS instruction mix of the hottest kernel.

    python tools/ncu_summary.py gpurun_out/mid/D16   # reads D16_{details,raw}.csv, D16_source.csv.gz
"""
import collections
import csv
import gzip
import io
import os
import sys


def details(prefix):
    out = {}
    with open(prefix + "_details.csv") as fh:
        rows = list(csv.reader(fh))
    hdr = rows[0]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        out[d.get("Metric Name")] = (d.get("Metric Value"), d.get("Metric Unit"))
    return out


def raw(prefix):
    with open(prefix + "_raw.csv") as fh:
        rows = list(csv.reader(fh))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def sass_mix(prefix):
    p = prefix + "_source.csv.gz"
    if not os.path.exists(p):
        return None
    rows = list(csv.reader(io.StringIO(gzip.open(p, "rt").read())))
    hi = [i for i, r in enumerate(rows) if len(r) > 4 and r[0] == "Line No"]
    sass = [r for r in rows[hi[0] + 1:] if len(r) > 8 and r[2].startswith("0x")]
    op = collections.Counter()
    for r in sass:
        t = r[3].split()
        if not t:
            continue
        m = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        op[m.split(".")[0]] += int(r[7] or 0)
    return op


def main(prefix):
    d = details(prefix)
    v, u = raw(prefix)
    keys = ["Duration", "DRAM Throughput", "Memory Throughput", "SM Active Cycles", "Elapsed Cycles",
            "Issue Slots Busy", "Achieved Active Warps Per SM", "Registers Per Thread", "Grid Size",
            "Block Size", "Waves Per SM", "Warp Cycles Per Issued Instruction", "L2 Hit Rate"]
    for k in keys:
        if k in d:
            print(f"  {k:36s} {d[k][0]} {d[k][1]}")
    rd = float(v.get("dram__bytes_read.sum", "0").replace(",", "") or 0)
    wr = float(v.get("dram__bytes_write.sum", "0").replace(",", "") or 0)
    print(f"  DRAM read+write                      {rd:.4g} + {wr:.4g} {u.get('dram__bytes_read.sum')}")
    st = {k.split("stalled_")[1].replace("_per_issue_active.ratio", ""): float(val)
          for k, val in v.items() if k.startswith("smsp__average_warps_issue_stalled_")
          and k.endswith("_per_issue_active.ratio") and float(val or 0) > 0.02}
    print("  stalls per issue: " + ", ".join(f"{k} {x:.2f}" for k, x in sorted(st.items(), key=lambda t: -t[1])))
    op = sass_mix(prefix)
    if op:
        tot = sum(op.values())
        print(f"  instructions {tot:.4g}: " + ", ".join(f"{k} {100*n/tot:.0f}%" for k, n in op.most_common(12)))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        main(p)


def hot_lines(prefix, top=25):
    """Top CUDA source lines by warp-stall samples (all files of the capture)."""
    rows = list(csv.reader(io.StringIO(gzip.open(prefix + "_source.csv.gz", "rt").read())))
    out = []
    fname = None
    for i, r in enumerate(rows):
        if len(r) == 2 and r[0] == "File Path":
            fname = os.path.basename(r[1])
        elif len(r) > 6 and r[0].isdigit() and not (len(r) > 2 and r[2].startswith("0x")):
            try:
                out.append((int(r[4] or 0), fname, int(r[0]), r[1].strip()[:90]))
            except ValueError:
                pass
    tot = sum(o[0] for o in out) or 1
    for s, f, ln, src in sorted(out, reverse=True)[:top]:
        print(f"  {100*s/tot:5.1f}%  {f}:{ln}  {src}")
