#!/bin/bash
# Round-2 measurement pass (run on the GPU box from the repo root): bench lines for configs[0..2], the ncu launch
# list of one C3 iteration (application replay: the cooperative CTA-pair weight-gradient kernel included),
# achieved occupancy of the environment kernels, counters of the shipped k_gemm_dw2, compute-sanitizer passes.
set -u
O=gpurun_out/m02
mkdir -p $O
for w in rough flat c1; do
  timeout 300 python bench.py --workload $w > $O/bench_$w.txt 2>&1
done
timeout 600 ncu --replay-mode application --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 600 ncu --metrics sm__warps_active.avg.pct_of_peak_sustained_active,sm__maximum_warps_per_active_cycle_pct,launch__occupancy_limit_registers,launch__occupancy_limit_blocks,launch__registers_per_thread,launch__block_size,launch__grid_size,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum \
  --clock-control none -k regex:k_env --launch-skip 48 -c 4 --csv --log-file $O/env_occupancy.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_env.log 2>&1
timeout 900 ncu --replay-mode application --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum \
  --clock-control none -k regex:k_gemm_dw2 --launch-skip 6 -c 3 --csv --log-file $O/dw2.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_dw2.log 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_iteration.py > $O/sanitizer_$t.txt 2>&1
  echo "rc=$?" >> $O/sanitizer_$t.txt
done
