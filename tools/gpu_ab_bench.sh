# A/B whole-bench lines (C5 parity + fast line, C4) for library variants
V=paper_0805_1827_b200/lib/variants
for v in default "$@"; do
  L=$PWD/$V/libbermuda_b200_$v.so; [ $v = default ] && L=$PWD/paper_0805_1827_b200/lib/libbermuda_b200.so
  for c in c5 c4 c3; do
    BRM_LIB_PATH=$L timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); print('$v', '$c', round(l['ms_per_step'],3), {k:round(v,2) for k,v in l['kernel_ms_per_step'].items()}, 'fast', (l.get('fast_mode') or {}).get('ms_per_step'), l['price'])"
  done
done
