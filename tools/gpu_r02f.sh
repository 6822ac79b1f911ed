# Round-2 (f) measurement set, run under gpurun from the repo root: GPU tests, smoke, the five
# bench configs, the reference arm, the C5 launch list and the walker's full ncu capture.
set -x
O=gpurun_out/r02f; mkdir -p $O
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
for f in "" 1; do echo "BRM_IZ_NO_CACHE=$f"; BRM_IZ_NO_CACHE=$f ncu --metrics gpu__time_duration.sum --clock-control none -k regex:iz_probes -c 9 python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline 2>&1 | grep -E "gpu__time_duration" | awk '{print $NF, $(NF-1)}' | tr '\n' ' '; echo; done > $O/iz_c2_per_date.txt 2>&1
BRM_IZ_NO_CACHE=1 timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c2_nocache.json.log 2>&1
BRM_WALK_LOG=0 timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c2_pricestepper.json.log 2>&1
BRM_WALK_LOG=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fast-line > $O/bench_c5_pricestepper.json.log 2>&1
