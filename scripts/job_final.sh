#!/bin/bash
# Final round-1 measurement: smoke, C4 bench line, ncu launch list of one step,
# ncu --set full of the scan kernel (source-correlated).  Outputs in gpurun_out/.
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_info.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > $OUT/bench_c4_final.json 2> $OUT/bench_c4_final.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_c4_final.csv python bench.py --workload c4 --steps 1 --warmup 3 --profile --no-cpu-baseline > $OUT/ncu_list_c4.log 2>&1
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_scan_fast2 -c 1 \
  -f -o $OUT/scan_c4_final python bench.py --workload c4 --steps 1 --warmup 3 --profile --no-cpu-baseline > $OUT/ncu_full_c4.log 2>&1
ls -la $OUT
