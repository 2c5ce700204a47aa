#!/usr/bin/env bash
# Regenerate the round's measurement evidence on a GPU box (run from the repo
# root, e.g. under gpurun).  Outputs go to gpurun_out/ev/; the summaries that
# are judged get copied into profiles/rNN/ by hand afterwards.
#   bench lines (every workload; config2 with the CPU baseline, the reference arm)
#   ncu launch list of the default bench command
#   ncu --set full of the finest-level visits (config 2: T_16, U_16; config 3: T_20, U_20)
#   --profiles-only : just the ncu --set full captures
set -u
OUT=gpurun_out/ev
mkdir -p "$OUT"
prof() {  # name workload kernel-regex skip
  ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k "regex:$3" --launch-skip "$4" -c 1 \
      -o "$OUT/$1" python tools/profile_solve.py --workload "$2" > "$OUT/ncu_$1.log" 2>&1
  ncu -i "$OUT/$1.ncu-rep" --page raw --csv > "$OUT/$1_raw.csv" 2>/dev/null
  ncu -i "$OUT/$1.ncu-rep" --page details --csv > "$OUT/$1_details.csv" 2>/dev/null
  ncu -i "$OUT/$1.ncu-rep" --page source --csv --print-source=cuda,sass > "$OUT/$1_source.csv" 2>/dev/null
  gzip -f "$OUT/$1_source.csv"
  [ "${KEEP_REPS:-0}" = "1" ] || rm -f "$OUT/$1.ncu-rep"  # gpurun copies back <= 64 MiB
}
profiles() {
  # config 2 finest visits: T_16 runs two RHS columns per lane (V2<double>),
  # U_16 (Pi + Kaczmarz) one; U_11 is a mid-level FAS-correction visit (V2)
  prof T16 config2 "visit_kernel<fmgsr::V2<double>, .int.2, .bool.0, .bool.1, .bool.1, .bool.0, .bool.0>" 6
  prof U16 config2 "visit_kernel<double, .int.2, .bool.1, .bool.0, .bool.1, .bool.0, .bool.0>" 0
  prof U11 config2 "visit_kernel<fmgsr::V2<double>, .int.1, .bool.0, .bool.0, .bool.1, .bool.0, .bool.0>" 2
  # the on-chip coarse kernel, a V-segment launch (mode 1) of config 2
  prof C9 config2 "coarse_kernel<double, .int.8>" 3
  prof T20 config3 "ns2_kernel<double, .int.2, .bool.0, .bool.1, .bool.1, .bool.1>" 9
  prof U20 config3 "ns2_kernel<double, .int.2, .bool.1, .bool.1, .bool.1, .bool.0>" 0
}
if [ "${1:-}" = "--profiles-only" ]; then
  profiles
  ls -la "$OUT"
  exit 0
fi
python bench.py > "$OUT/bench_config2.jsonl" 2> "$OUT/bench_config2.err"
python bench.py --impl reference > "$OUT/bench_reference.jsonl" 2> "$OUT/bench_reference.err"
for w in config1 config3 config4 config5 config5_f32; do
  python bench.py --workload "$w" --no-cpu-baseline > "$OUT/bench_$w.jsonl" 2> "$OUT/bench_$w.err"
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches_config2.csv" \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$OUT/ncu_launches.log" 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file "$OUT/launches_config3_solve.csv" \
    python tools/profile_solve.py --workload config3 > "$OUT/ncu_launches3.log" 2>&1
profiles
ls -la "$OUT"
