# fast-mode AdaBoost after the analytic weight sum: timing, the fast-mode tests, C3 / C4 / C5 benches
set -x
O=gpurun_out/r02j; mkdir -p $O
for a in "5000 6 150 fast" "10000 11 100 fast" "20000 41 200 fast" "10000 11 100 parity"; do python tools/boost_timing.py $a 2>&1 | tail -1; done > $O/boost_timing.log 2>&1
cat $O/boost_timing.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
tail -3 $O/gpu_tests.log
for c in c3 c4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json.log 2>&1; done
timeout 900 python bench.py > $O/bench_c5.json.log 2>&1
for f in $O/bench_c?.json.log; do tail -1 $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'], d['value'], d['e2e']['value'], d['price'], d['ci95'], d.get('kernel_ms_per_step'), d['roofline']['frac'], d.get('fast_mode'))"; done
