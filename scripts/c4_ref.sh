OUT=gpurun_out
timeout 1500 python bench.py --workload c4 --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_c4.json 2> $OUT/bench_ref_c4.log
free -g >> $OUT/bench_ref_c4.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_scan_fast -c 1 \
   -f -o $OUT/scan_c4 python bench.py --workload c4 --steps 1 --warmup 3 --profile > $OUT/ncu_full_c4.log 2>&1
