set -x
timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for v in 0 1 3 4; do
  VLQ_SCAN_VARIANT=$v VLQ_SCAN_VARIANT=$v timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v${v}_c2.json 2> gpurun_out/v${v}_c2.log
  VLQ_SCAN_VARIANT=$v timeout 600 python bench.py --workload deep100m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v${v}_deep100m.json 2> gpurun_out/v${v}_deep100m.log
done
