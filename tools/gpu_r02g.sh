# Round-2 (g) confirmation after the container was re-created: GPU tests, smoke, C5 bench and the reference arm.
set -x
O=gpurun_out/r02g; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c5.json.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json.log 2>&1
tail -3 $O/gpu_tests.log; tail -2 $O/smoke.log; tail -c 600 $O/bench_c5.json.log
