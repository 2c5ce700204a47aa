#!/usr/bin/env bash
# ncu --set full of selected mid-level visits of config 2 (op-by-op solve).
#   tools/ncu_small.sh NAME REGEX SKIP
set -u
OUT=gpurun_out/ev
mkdir -p "$OUT"
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:$2" --launch-skip "$3" -c 1 \
    -o "$OUT/$1" python tools/profile_solve.py --workload "${WL:-config2}" > "$OUT/ncu_$1.log" 2>&1
ncu -i "$OUT/$1.ncu-rep" --page raw --csv > "$OUT/$1_raw.csv" 2>/dev/null
ncu -i "$OUT/$1.ncu-rep" --page details --csv > "$OUT/$1_details.csv" 2>/dev/null
ncu -i "$OUT/$1.ncu-rep" --page source --csv --print-source=cuda,sass > "$OUT/$1_source.csv" 2>/dev/null
gzip -f "$OUT/$1_source.csv"
rm -f "$OUT/$1.ncu-rep"
