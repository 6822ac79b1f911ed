# quick GPU check of the I&Z path: C2 / C1 bench lines (draw cache on / off / price stepper), then the tests
run() { timeout 600 python bench.py --config $2 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); print('$1', '$2', round(l['ms_per_step'],3), {k:round(v,3) for k,v in l['kernel_ms_per_step'].items()}, 'frac', round(l['roofline']['frac'],3), repr(l['price']), l['ci95'])"; }
run cache c2
BRM_IZ_NO_CACHE=1 run nocache c2
BRM_WALK_LOG=0 run pricestep c2
run cache c1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/quick_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/quick_gpu_tests.log
tail -15 gpurun_out/quick_gpu_tests.log
