#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python bench.py --workload c4 --steps 10 --warmup 3 > $OUT/bench_c4.json 2> $OUT/bench_c4.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_c4.csv python bench.py --workload c4 --steps 1 --warmup 3 --profile --no-cpu-baseline > $OUT/ncu_list_c4.log 2>&1
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"k_coarse_tc|k_exact_needed|k_refine_list|k_relayout|k_second_level" -c 6 \
  -f -o $OUT/coarse_c4 python bench.py --workload c4 --steps 1 --warmup 3 --profile --no-cpu-baseline > $OUT/ncu_coarse_c4.log 2>&1
