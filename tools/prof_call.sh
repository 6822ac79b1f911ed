# Round profile set (run under gpurun from the repo root): bench launch list,
# ncu --set full of the C5 walker launches and of one C5 AdaBoost fit.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-fast-line"
$B > gpurun_out/b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv $B > gpurun_out/ncu_launch.log 2>&1
python tools/prof_c5.py parity > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:walk_units -s 8 -c 2 -o gpurun_out/walk_c5 -f python tools/prof_c5.py parity > gpurun_out/ncu_walk.log 2>&1
$B > gpurun_out/b_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:boost_kernel -s 3 -c 1 -o gpurun_out/boost_c5 -f $B > gpurun_out/ncu_boost.log 2>&1
ls -la gpurun_out
