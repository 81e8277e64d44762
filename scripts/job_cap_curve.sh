#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python scripts/scan_study.py --workload c4 --steps 5 --configs \
  "scan_variant=0,scan_cap=0,scan_keep_min=0" "scan_variant=0,scan_cap=4096,scan_keep_min=0" \
  "scan_variant=9,scan_cap=4096,scan_keep_min=512" "scan_variant=9,scan_cap=8192,scan_keep_min=512" \
  "scan_variant=0,scan_cap=0,scan_keep_min=0" > $OUT/study_cap_c4.jsonl 2> $OUT/study_cap_c4.log
timeout 1500 python scripts/curve.py --workload c4 --nqs 10000 --w1s 16,32,64,128 > $OUT/curve_c4.jsonl 2> $OUT/curve_c4.log
timeout 1500 python scripts/curve.py --workload c5 --queries heldout > $OUT/curve_c5_heldout.jsonl 2> $OUT/curve_c5_heldout.log
