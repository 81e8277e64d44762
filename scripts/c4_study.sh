OUT=gpurun_out
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $OUT/launches_c4.csv python bench.py --workload c4 --steps 1 --warmup 3 --profile > $OUT/ncu_list_c4.log 2>&1
for u in 4 6 8; do
  VLQ_SCAN_U=$u timeout 600 python bench.py --workload deep100m --steps 5 --warmup 3 --no-cpu-baseline > $OUT/u${u}_deep100m.json 2> $OUT/u${u}_deep100m.log
done
