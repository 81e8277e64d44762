#!/bin/bash
# v7 (bulk-async staged scan) parity + A/B study on C4.  Outputs in gpurun_out/.
OUT=gpurun_out; mkdir -p $OUT
for v in ${PARITY_VARIANTS:-5 6}; do
  VLQ_SCAN_VARIANT=$v timeout 600 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $OUT/pytest_v$v.log 2>&1; echo "rc=$?" >> $OUT/pytest_v$v.log
done
timeout 1500 python scripts/scan_study.py --workload ${W:-c4} --steps 5 --configs ${CONFIGS:-scan_variant=0 scan_variant=5 scan_variant=6 scan_variant=7 scan_variant=8 scan_variant=0} > $OUT/study_v7_${W:-c4}.jsonl 2> $OUT/study_v7.log
