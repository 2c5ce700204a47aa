#!/usr/bin/env bash
# Where the latency-bound visits spend their time (run from the repo root under gpurun):
#   fp64 dependent-op latency, config-5 table (all 32 cells), per-visit breakdowns of the
#   small-P geometry and of one 8-way shard of config 4, then ncu --set full of the
#   config-5 P = 16 finest T visit (picked by its NVTX range).
set -u
OUT=gpurun_out/lat
mkdir -p "$OUT"
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o "$OUT/fp64_latency" tools/micro/fp64_latency.cu \
  && "$OUT/fp64_latency" > "$OUT/fp64_latency.txt" 2>&1
python tools/config5_table.py --json "$OUT/config5_table.json" --md "$OUT/config5_table.md" \
  > "$OUT/config5_table.log" 2>&1
python tools/visit_breakdown.py --workload config5 --P 16 --b 8 --total > "$OUT/bd_c5_P16_b8.txt" 2>&1
python tools/visit_breakdown.py --workload config4 --shards 8 --rank 4 --total > "$OUT/bd_c4_s8.txt" 2>&1
if [ "${NCU:-1}" = "1" ]; then
  cmd="python tools/profile_solve.py --workload config5 --P 16 --b 8"
  $cmd > "$OUT/plain_P16.log" 2>&1 || exit 1
  ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "T_20/" -c 1 \
      -o "$OUT/T20_P16" $cmd > "$OUT/ncu_T20_P16.log" 2>&1
  echo "ncu rc=$?"
  ncu -i "$OUT/T20_P16.ncu-rep" --page raw --csv > "$OUT/T20_P16_raw.csv" 2>/dev/null
  ncu -i "$OUT/T20_P16.ncu-rep" --page details --csv > "$OUT/T20_P16_details.csv" 2>/dev/null
  ncu -i "$OUT/T20_P16.ncu-rep" --page source --csv --print-source=cuda,sass > "$OUT/T20_P16_source.csv" 2>/dev/null
  gzip -f "$OUT/T20_P16_source.csv"
  rm -f "$OUT/T20_P16.ncu-rep"
fi
ls -la "$OUT"
