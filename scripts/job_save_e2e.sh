#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log
timeout 600 python scripts/e2e_probe.py --workload c2 > $OUT/e2e_probe_c2.json 2> $OUT/e2e_probe_c2.log
( time timeout 1800 python bench.py --workload c4 --impl reference --steps 2 --warmup 3 ) > $OUT/bench_ref_c4.json 2> $OUT/bench_ref_c4.log
