# A/B the walker variants under paper_0805_1827_b200/lib/variants (plus the default build)
V=paper_0805_1827_b200/lib/variants
M="--metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,launch__grid_size,smsp__inst_executed.sum,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"
{
timeout 600 python tools/walk_bench.py 3
for v in "$@"; do BRM_LIB_PATH=$PWD/$V/libbermuda_b200_$v.so timeout 600 python tools/walk_bench.py 3; done
} 2>&1 | grep -v "^+" > gpurun_out/ab_walk_bench.log
cat gpurun_out/ab_walk_bench.log
for v in default "$@"; do
  L=$PWD/$V/libbermuda_b200_$v.so; [ $v = default ] && L=$PWD/paper_0805_1827_b200/lib/libbermuda_b200.so
  BRM_LIB_PATH=$L ncu $M --clock-control none -k regex:walk_units -s 8 -c 1 python tools/prof_c5.py parity 2>&1 | grep -E "walk_units|duration|warps_active|issue_active|fp64|occupancy|grid|inst_executed|stalled" > gpurun_out/ab_ncu_$v.log
  echo "== $v"; cat gpurun_out/ab_ncu_$v.log
done
