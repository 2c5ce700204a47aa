#!/usr/bin/env bash
# ncu --set full of single level visits picked by their NVTX range (op-by-op solve).
#   tools/ncu_visits.sh OUTDIR "ARGS for profile_solve" NAME:RANGE [NAME:RANGE ...]
# e.g. tools/ncu_visits.sh gpurun_out/mid "--workload config4" D16:D_16 U16:U_16
set -u
OUT=$1; shift
ARGS=$1; shift
mkdir -p "$OUT"
cmd="python tools/profile_solve.py $ARGS"
$cmd > "$OUT/plain.log" 2>&1 || { echo "plain run failed"; exit 1; }
for spec in "$@"; do
  name=${spec%%:*}; rng=${spec#*:}
  ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "$rng/" -c 1 \
      -o "$OUT/$name" $cmd > "$OUT/ncu_$name.log" 2>&1
  echo "ncu $name rc=$?"
  ncu -i "$OUT/$name.ncu-rep" --page raw --csv > "$OUT/${name}_raw.csv" 2>/dev/null
  ncu -i "$OUT/$name.ncu-rep" --page details --csv > "$OUT/${name}_details.csv" 2>/dev/null
  ncu -i "$OUT/$name.ncu-rep" --page source --csv --print-source=cuda,sass > "$OUT/${name}_source.csv" 2>/dev/null
  gzip -f "$OUT/${name}_source.csv"
  rm -f "$OUT/$name.ncu-rep"
done
