#!/bin/bash
# GPU parity suite + single-GPU gloo rehearsal of the N = 2 bench path (select-split schedule).
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log
VLQ_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --workload c2 --steps 4 --warmup 3 > $OUT/bench_c2_x2_gloo.json 2> $OUT/bench_c2_x2_gloo.log
timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c2_x1.json 2> $OUT/bench_c2_x1.log
