# C4 walker A/B: the column-constant prefix step against the triangular product, then the new test and C4 bench.
set -x
O=gpurun_out/r02h; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_colconst.py tests/test_gpu_parity.py -m gpu -x -q > $O/colconst_tests.log 2>&1; echo "tests rc=$?" >> $O/colconst_tests.log
tail -3 $O/colconst_tests.log
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4.json.log 2>&1
BRM_WALK_COLCONST=0 timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4_triangular.json.log 2>&1
for f in $O/bench_c4.json.log $O/bench_c4_triangular.json.log; do tail -1 $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['price'], d['ci95'], d.get('kernel_ms_per_step'))"; done
