#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
VLQ_SCAN_VARIANT=11 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > $OUT/pytest_v11.log 2>&1; echo rc=$? >> $OUT/pytest_v11.log
timeout 1500 python scripts/scan_study.py --workload c4 --steps 5 --configs \
  "scan_variant=0,scan_cap=0,scan_keep_min=0" \
  "scan_variant=11,scan_cap=0,scan_keep_min=512" \
  "scan_variant=12,scan_cap=0,scan_keep_min=512" \
  "scan_variant=11,scan_cap=0,scan_keep_min=0" \
  "scan_variant=9,scan_cap=4096,scan_keep_min=512" \
  "scan_variant=0,scan_cap=0,scan_keep_min=0" > $OUT/study_bulkq8_c4.jsonl 2> $OUT/study_bulkq8_c4.log
