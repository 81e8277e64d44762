# host resources + a first 1B-scale (C4) run
OUT=gpurun_out
free -g > $OUT/host_mem.txt; df -h /tmp /dev/shm >> $OUT/host_mem.txt; nproc >> $OUT/host_mem.txt
( timeout 1500 python bench.py --workload ${W:-c4} --steps 10 --warmup 3 ${EXTRA} > $OUT/bench_${W:-c4}.json 2> $OUT/bench_${W:-c4}.log ) 
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> $OUT/host_mem.txt
