# per-date durations of the C2 probe kernel (ncu launch list), draw cache on and off
for f in "" 1; do
  echo "== BRM_IZ_NO_CACHE=$f"
  BRM_IZ_NO_CACHE=$f ncu --metrics gpu__time_duration.sum --clock-control none -k regex:iz_probes -c 9 python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline 2>&1 | grep -E "gpu__time_duration" | awk '{print $NF, $(NF-1)}' | tr '\n' ' '
  echo
done
