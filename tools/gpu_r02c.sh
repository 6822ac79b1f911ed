set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02c_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02c_bench_c5.json.log 2>&1
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_bench_$c.json.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02c_bench_ref.json.log 2>&1
tail -3 gpurun_out/r02c_gpu_tests.log
