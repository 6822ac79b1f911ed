# Fast-mode walker after the lean Box-Muller / ex2 step / packed rows: tests, C4 A/B, C3, C5 fast line.
set -x
O=gpurun_out/r02h; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
tail -3 $O/gpu_tests.log
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4.json.log 2>&1
BRM_WALK_COLCONST=0 timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4_triangular.json.log 2>&1
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c3.json.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c5_nocpu.json.log 2>&1
for f in $O/bench_c4.json.log $O/bench_c4_triangular.json.log $O/bench_c3.json.log $O/bench_c5_nocpu.json.log; do tail -1 $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['price'], d['ci95'], d.get('kernel_ms_per_step'), d.get('fast_mode'))"; done
