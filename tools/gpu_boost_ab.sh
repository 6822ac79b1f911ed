# AdaBoost CTA-size / cluster-size A/B (fast and parity): CUDA-event time per fit.
V=$PWD/paper_0805_1827_b200/lib/variants
for shape in "5000 6 150" "10000 11 100"; do
  for mode in fast parity; do
    for lib in default t512 t1024; do
      for cl in 8 4 2 1; do
        [ $lib = default ] && L=$PWD/paper_0805_1827_b200/lib/libbermuda_b200.so || L=$V/libbermuda_b200_$lib.so
        [ $lib = t1024 ] && [ $mode = parity ] && continue
        echo -n "lib=$lib cl<=$cl: "; BRM_LIB_PATH=$L BRM_BOOST_CL=$cl timeout 300 python tools/boost_timing.py $shape $mode 2>&1 | tail -1
      done
    done
  done
done > gpurun_out/boost_ab_r02h.log 2>&1
cat gpurun_out/boost_ab_r02h.log
