set -x
V=paper_0805_1827_b200/lib/variants
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
{
timeout 600 python tools/walk_bench.py 3
BRM_WALK_LOG=0 timeout 600 python tools/walk_bench.py 3
for v in minb3 minb4; do BRM_LIB_PATH=$PWD/$V/libbermuda_b200_$v.so timeout 600 python tools/walk_bench.py 3; done
} > gpurun_out/r02d_walk_bench.log 2>&1
cat gpurun_out/r02d_walk_bench.log | grep -v "^+"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02d_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02d_gpu_tests.log
tail -15 gpurun_out/r02d_gpu_tests.log
