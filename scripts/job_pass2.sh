#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log
timeout 900 python scripts/scan_study.py --workload c4 --steps 5 --configs "tc_pass2_single=0" "tc_pass2_single=1" "tc_pass2_single=0" "tc_pass2_single=1" > $OUT/study_pass2_c4.jsonl 2> $OUT/study_pass2_c4.log
