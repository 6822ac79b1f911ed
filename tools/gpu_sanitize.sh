# compute-sanitizer over small runs of the new kernels (log-price walker, search trees, draw cache)
set -x
O=gpurun_out/sanitize; mkdir -p $O
S=/usr/local/cuda/bin/compute-sanitizer
T="python -m pytest tests/test_gpu_logwalk.py -x -q -k 'vs_oracle and 5-0 or draw_cache and 5 or single_date or too_large'"
timeout 1500 $S --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_logwalk.py -x -q -k "single_date or draw_cache" > $O/memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/memcheck.log
timeout 1500 $S --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_logwalk.py -x -q -k "single_date or draw_cache" > $O/racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/racecheck.log
timeout 1500 $S --tool memcheck --error-exitcode 9 python bench.py --config c5 --scale 0.01 --steps 1 --warmup 0 --no-cpu-baseline --no-fast-line > $O/memcheck_c5.log 2>&1; echo "memcheck c5 rc=$?" >> $O/memcheck_c5.log
timeout 1500 $S --tool racecheck --error-exitcode 9 python bench.py --config c5 --scale 0.005 --steps 1 --warmup 0 --no-cpu-baseline --no-fast-line > $O/racecheck_c5.log 2>&1; echo "racecheck c5 rc=$?" >> $O/racecheck_c5.log
timeout 1500 $S --tool memcheck --error-exitcode 9 python bench.py --config c2 --scale 0.25 --steps 1 --warmup 0 --no-cpu-baseline > $O/memcheck_c2.log 2>&1; echo "memcheck c2 rc=$?" >> $O/memcheck_c2.log
for f in $O/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rc=|passed|failed|Error|hazard" $f | head -8; done
