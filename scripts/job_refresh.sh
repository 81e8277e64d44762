#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
for w in c1 c2 c3; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > $OUT/bench_$w.json 2> $OUT/bench_$w.log
done
timeout 2000 python scripts/shard_probe.py --workload c4 --shards 8:0,8:5,8:3,4:0,2:0 > $OUT/shard_probe_c4_final.jsonl 2> $OUT/shard_probe_c4_final.log
