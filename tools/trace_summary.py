"""Summarise FMGSR_COARSE_TRACE=1 output (coarse kernels' per-phase clock
deltas of CTA 0) by phase and level.

    FMGSR_COARSE_TRACE=1 python tools/profile_solve.py --workload config2 > t.txt
    python tools/trace_summary.py t.txt
"""
import collections
import sys


def main(path):
    tot = collections.defaultdict(int)
    cnt = collections.defaultdict(int)
    launches, cycles = 0, 0
    for line in open(path):
        f = line.split()
        if not f or not f[0].startswith("coarse"):
            continue
        if f[1] == "1":
            launches += 1
        c = int(f[2])
        key = (f[3], int(f[4])) if len(f) >= 5 else ("phase", int(f[1]))
        tot[key] += c
        cnt[key] += 1
        cycles += c
    print(f"# {path}: {launches} coarse launches traced (CTA 0), {cycles} cycles in phases")
    print(f"# {'phase':12s} {'level':>5s} {'count':>6s} {'cycles':>9s} {'per call':>9s} {'share':>6s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"  {k[0]:12s} {k[1]:5d} {cnt[k]:6d} {v:9d} {v // cnt[k]:9d} {100 * v / cycles:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
