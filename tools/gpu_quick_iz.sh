# quick GPU check of the I&Z path: C2 / C1 bench lines with and without the log-price probe walker, then the tests
for f in 1 0; do for c in c2 c1; do
  BRM_WALK_LOG=$f timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); print('log=$f', '$c', round(l['ms_per_step'],3), {k:round(v,3) for k,v in l['kernel_ms_per_step'].items()}, 'frac', round(l['roofline']['frac'],3), repr(l['price']), l['ci95'])"
done; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/quick_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/quick_gpu_tests.log
tail -15 gpurun_out/quick_gpu_tests.log
