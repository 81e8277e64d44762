#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python scripts/scan_study.py --workload c4 --steps 5 --configs "scan_sel_agg=0" "scan_sel_agg=1" "scan_sel_agg=0,scan_slots=104" "scan_sel_agg=1,scan_slots=104" "scan_sel_agg=0,scan_slots=6" > $OUT/study_selkeep_c4.jsonl 2> $OUT/study_selkeep_c4.log
timeout 1200 python scripts/shard_probe.py --workload c4 --shards 8:3 --configs "" "scan_sel_agg=1" "scan_sel_agg=0,scan_slots=104" "scan_sel_agg=1,scan_slots=104" "scan_sel_agg=0,scan_slots=6" > $OUT/shard_probe_selkeep.jsonl 2> $OUT/shard_probe_selkeep.log
