# Round-2 (e) measurement set, run under gpurun from the repo root: GPU tests, smoke, the five
# bench configs, the reference arm, the C5 launch list and the walker's full ncu capture.
set -x
O=gpurun_out/r02e; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_c5.json.log 2>&1
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-fast-line"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_c5.csv $B > $O/launches_c5.log 2>&1 || \
  BRM_NCU_SAFE=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_c5.csv $B > $O/launches_c5.log 2>&1
python tools/prof_c5.py parity > $O/prof_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:walk_units -s 8 -c 2 -o $O/walk_log_c5 -f python tools/prof_c5.py parity > $O/ncu_walk.log 2>&1
tail -3 $O/gpu_tests.log
