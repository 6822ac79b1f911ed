# column sort beside the label walk (brm_fit_presort): tests, then C5 / C3 / C4 with and without
set -x
O=gpurun_out/r02k; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_config_parity.py tests/test_gpu_device_loop.py -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
tail -3 $O/gpu_tests.log
for v in "" 1; do
  BRM_NO_PRESORT=$v timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fast-line > $O/bench_c5_nopresort$v.json.log 2>&1
  BRM_NO_PRESORT=$v timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c3_nopresort$v.json.log 2>&1
  BRM_NO_PRESORT=$v timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4_nopresort$v.json.log 2>&1
done
for f in $O/bench_c*.json.log; do echo $f; tail -1 $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'], d['price'], d.get('kernel_ms_per_step'), d['gpu_launches'])"; done
