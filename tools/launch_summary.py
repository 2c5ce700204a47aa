"""Sum an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_*] --csv
--log-file) by kernel, for the profiles/ summaries.

    python tools/launch_summary.py launches.csv "command description" > summary.txt
"""
import collections
import csv
import re
import sys


def main(path, what):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    t = collections.defaultdict(float)
    n = collections.defaultdict(set)
    dram = collections.defaultdict(float)
    launches = set()
    for r in rows[1:]:
        name = re.sub(r"\(.*$", "", r[ix["Kernel Name"]]).replace("void ", "")
        launches.add(r[ix["ID"]])
        v = float(r[ix["Metric Value"]].replace(",", ""))
        if r[ix["Metric Name"]] == "gpu__time_duration.sum":
            scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0}.get(
                r[ix["Metric Unit"]], 1e-6)
            t[name] += v * scale
            n[name].add(r[ix["ID"]])
        elif r[ix["Metric Name"]].startswith("dram__bytes"):
            dram[name] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(
                r[ix["Metric Unit"]], 1)
    tot = sum(t.values())
    print(f"# {what}")
    print(f"# cold-cache, serialised per-launch times summed by kernel")
    print(f"# launches: {len(launches)}, total kernel time {tot:.3f} ms\n")
    for k in sorted(t, key=lambda k: -t[k]):
        extra = f"  dram {dram[k] / 1e9:8.3f} GB" if dram else ""
        print(f"{t[k]:9.3f} ms {100 * t[k] / tot:5.1f}%  n={len(n[k]):4d}  {k}{extra}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
