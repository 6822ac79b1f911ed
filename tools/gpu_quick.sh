# quick GPU check: walker A/B bench, then the parity tests that exercise the walker
{
timeout 600 python tools/walk_bench.py 3
BRM_WALK_LOG=0 timeout 600 python tools/walk_bench.py 3
} 2>&1 | grep -v "^+" > gpurun_out/quick_walk_bench.log
cat gpurun_out/quick_walk_bench.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/quick_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/quick_gpu_tests.log
tail -15 gpurun_out/quick_gpu_tests.log
