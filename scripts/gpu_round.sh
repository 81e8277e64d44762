#!/bin/bash
# One GPU-box session: parity tests, smoke, bench lines, ncu launch list +
# full capture of the scan kernel.  Everything lands in gpurun_out/.
# usage: scripts/gpu_round.sh [workload] [what...]   what in {tests,smoke,bench,ref,ncu}
W=${1:-c2}; shift
WHAT=${@:-tests bench ref ncu}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_info.txt 2>&1
nproc > $OUT/host_cores.txt; lscpu | grep "Model name" >> $OUT/host_cores.txt
for w in $WHAT; do
  case $w in
    tests)
      timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log ;;
    bench)
      timeout 1500 python bench.py --workload $W --steps 10 --warmup 3 ${EXTRA} > $OUT/bench_$W.json 2> $OUT/bench_$W.log ;;
    ref)
      timeout 1500 python bench.py --workload $W --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_$W.json 2> $OUT/bench_ref_$W.log ;;
    ncu)
      timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $OUT/launches_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --profile > $OUT/ncu_list_$W.log 2>&1
      timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_scan -c 1 \
        -f -o $OUT/scan_$W python bench.py --workload $W --steps 1 --warmup 3 --profile > $OUT/ncu_full_$W.log 2>&1 ;;
    ncu_tc)
      # tensor-pipe utilisation of the tcgen05 coarse GEMM passes (not part of --set full on B200)
      timeout 900 ncu --profile-from-start off --clock-control none -k regex:k_coarse_tc -c 2 \
        --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32.sum,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__inst_executed_pipe_tmem.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum \
        --csv --log-file $OUT/coarse_tc_$W.csv python bench.py --workload $W --steps 1 --warmup 3 --profile > $OUT/ncu_tc_$W.log 2>&1 ;;
    ncu_coarse)
      timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_coarse_tc|k_exact_needed|k_refine" -c 6 \
        -f -o $OUT/coarse_$W python bench.py --workload $W --steps 1 --warmup 3 --profile > $OUT/ncu_coarse_$W.log 2>&1 ;;
  esac
done
ls -la $OUT
