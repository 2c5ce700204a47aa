"""Build profiles/traffic.json (the `roofline.traffic` block bench.py reports)
from the `ncu --set full` raw pages that tools/round_evidence.sh writes.

    python tools/traffic_from_ncu.py            # every workload from its capture directory
"""
import csv
import json
import os
import sys

SETS = {  # workload -> (label, capture name) of its finest-level visits
    "config2": [("T_16", "T16"), ("U_16", "U16")],
    "config3": [("T_20", "T20"), ("U_20", "U20")],
    "config4": [("T_24", "T24"), ("U_24", "U24")],
}
DIRS = {"config2": "profiles/r01", "config3": "profiles/r01", "config4": "profiles/r02"}
SCRIPT = {"profiles/r01": "tools/round_evidence.sh", "profiles/r02": "tools/evidence_r02.sh"}
ALG = {"config2": 2.5 * 2 ** 16 * 1024 * 8, "config3": 2.5 * 2 ** 20 * 256 * 8,
       "config4": 2.5 * 2 ** 24 * 64 * 8}
NOTES = {"config3": "V(2,2): the forward sweep spills the window (1 word) and the backward sweep "
                    "re-reads it and f (2 words); T_20 also carries the fused restriction (writes 1 "
                    "word), so DRAM traffic is 5.5 (T) / 6 (U) words against the 2.5-word "
                    "algorithmic count"}
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
         "ns": 1e-3, "us": 1.0, "ms": 1e3,
         "msecond": 1e3}


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for h, u, v in zip(hdr, units, vals):
        try:
            out[h] = float(v.replace(",", "")) * UNITS.get(u, 1.0)
        except ValueError:
            out[h] = v
    return out


def main():
    res = {}
    for wl, caps in SETS.items():
        d = DIRS[wl]
        ks = {}
        for label, name in caps:
            p = os.path.join(d, f"{name}_raw.csv")
            if not os.path.exists(p):
                continue
            r = raw(p)
            ks[label] = {"kernel": r.get("Kernel Name"),
                         "dram_read_bytes": r["dram__bytes_read.sum"],
                         "dram_write_bytes": r["dram__bytes_write.sum"],
                         "ncu_duration_us": r["gpu__time_duration.sum"]}
        if not ks:
            continue
        tot = [k["dram_read_bytes"] + k["dram_write_bytes"] for k in ks.values()]
        res[wl] = {"kernels": ks, "alg_bytes_per_launch": ALG[wl],
                   "source": f"ncu --set full --clock-control none, {d}/"
                             f"{{{','.join(n for _, n in caps)}}}_raw.csv ({SCRIPT[d]})",
                   "bytes_per_launch": sum(tot) / len(tot)}
        if wl in NOTES:
            res[wl]["note"] = NOTES[wl]
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles",
                           "traffic.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
