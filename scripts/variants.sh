# scan-kernel variant study; VLQ_SCAN_VARIANT: 0 default, 1 generic, 2 replicated LUT
timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-0 2}; do
  VLQ_SCAN_VARIANT=$v timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v${v}_c2.json 2> gpurun_out/v${v}_c2.log
  VLQ_SCAN_VARIANT=$v timeout 600 python bench.py --workload deep100m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v${v}_deep100m.json 2> gpurun_out/v${v}_deep100m.log
done
for w in ${NCU_WORKLOADS:-deep100m}; do
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_scan -c 1 \
    -f -o gpurun_out/scan_$w python bench.py --workload $w --steps 1 --warmup 3 --profile > gpurun_out/ncu_full_$w.log 2>&1
done
