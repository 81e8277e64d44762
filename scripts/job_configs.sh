#!/bin/bash
# bench lines for the other BASELINE configs (ours + the reference arm on the same box)
OUT=gpurun_out; mkdir -p $OUT
for w in c1 c2 c3; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > $OUT/bench_$w.json 2> $OUT/bench_$w.log
  timeout 900 python bench.py --workload $w --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_$w.json 2> $OUT/bench_ref_$w.log
done
