#!/usr/bin/env bash
# Round-2 measurement evidence on a GPU box (run from the repo root under gpurun).
# Outputs go to gpurun_out/ev2/; the summaries that are judged get copied into
# profiles/r02/ afterwards.
#   ncu --set full of the config-4 finest visits (T_24, U_24) -> roofline.traffic
#   ncu launch list of a short default bench run (config 4)
#   usage: tools/evidence_r02.sh [profiles|launches|all]
set -u
OUT=gpurun_out/ev2
mkdir -p "$OUT"
prof() {  # name workload kernel-regex skip
  ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k "regex:$3" --launch-skip "$4" -c 1 \
      -o "$OUT/$1" python tools/profile_solve.py --workload "$2" > "$OUT/ncu_$1.log" 2>&1
  echo "ncu $1 rc=$?"
  ncu -i "$OUT/$1.ncu-rep" --page raw --csv > "$OUT/$1_raw.csv" 2>/dev/null
  ncu -i "$OUT/$1.ncu-rep" --page details --csv > "$OUT/$1_details.csv" 2>/dev/null
  ncu -i "$OUT/$1.ncu-rep" --page source --csv --print-source=cuda,sass > "$OUT/$1_source.csv" 2>/dev/null
  gzip -f "$OUT/$1_source.csv"
  [ "${KEEP_REPS:-0}" = "1" ] || rm -f "$OUT/$1.ncu-rep"  # gpurun copies back <= 64 MiB
}
what=${1:-all}
if [ "$what" = "profiles" ] || [ "$what" = "all" ]; then
  # plain run first (ncu only after the same command exited 0 without it)
  python tools/profile_solve.py --workload config4 > "$OUT/plain_config4.log" 2>&1 || exit 1
  # config 4 (B = 64: two RHS columns per lane on T; the SR up visit Pi + CR scalar)
  # T_m is the 11th V2 FMG-epilogue visit of a solve (levels 14..24)
  prof T24 config4 "visit_kernel<fmgsr::V2<double>, .int.2, .bool.0, .bool.1" 10
  prof U24 config4 "visit_kernel<double, .int.2, .bool.1, .bool.0" 0
fi
if [ "$what" = "launches" ] || [ "$what" = "all" ]; then
  cmd="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra --e2e-steps 1"
  $cmd > "$OUT/plain_bench.log" 2>&1 || exit 1
  ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv \
      --log-file "$OUT/launches_config4.csv" $cmd > "$OUT/ncu_launches.log" 2>&1
  echo "ncu launches rc=$?"
fi
ls -la "$OUT"
