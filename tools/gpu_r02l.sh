# Round-2 (l) measurement set, run under gpurun from the repo root: GPU tests, smoke, the five
# bench configs, the reference arm, the C5 launch list, the C5 walker's full ncu capture and the
# C4 walker's (column-constant fast step).
set -x
O=gpurun_out/r02l; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c5.json.log 2>&1
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json.log 2>&1; done
BRM_WALK_COLCONST=0 timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4_triangular.json.log 2>&1
BRM_NO_PRESORT=1 timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4_nopresort.json.log 2>&1
BRM_NO_PRESORT=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fast-line > $O/bench_c5_nopresort.json.log 2>&1
BRM_NO_PRESORT=1 timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c3_nopresort.json.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-fast-line"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_c5.csv $B > $O/launches_c5.log 2>&1 || \
  BRM_NCU_SAFE=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_c5.csv $B > $O/launches_c5.log 2>&1
python tools/summarize_launches.py $O/launches_c5.csv > $O/launches_c5_summary.txt 2>&1
python tools/prof_c5.py parity > $O/prof_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:walk_units -s 8 -c 2 -o $O/walk_log_c5 -f python tools/prof_c5.py parity > $O/ncu_walk.log 2>&1
python tools/ncu_summary.py $O/walk_log_c5.ncu-rep > $O/walk_log_c5_summary.txt 2>&1
python tools/prof_c5.py fast 1 c4 > $O/prof_c4_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:walk_units -s 19 -c 1 -o $O/walk_c4 -f python tools/prof_c5.py fast 1 c4 > $O/ncu_walk_c4.log 2>&1
python tools/ncu_summary.py $O/walk_c4.ncu-rep > $O/walk_c4_fast_summary.txt 2>&1
python tools/ncu_lines.py $O/walk_c4.ncu-rep 0 1.2335e10 60 > $O/walk_c4_fast_lines.txt 2>&1
tail -3 $O/gpu_tests.log; tail -1 $O/smoke.log
for f in $O/bench_c?.json.log $O/bench_c4_triangular.json.log $O/bench_c?_nopresort.json.log; do tail -1 $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'], d['value'], d['e2e']['value'], d['price'], d['ci95'], d.get('kernel_ms_per_step'), d['roofline']['frac'], (d.get('fast_mode') or {}).get('ms_per_step'))"; done
