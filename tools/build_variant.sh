#!/bin/bash
# Build a variant library: recompile the listed csrc/*.cu files with extra nvcc
# defines and link them with the default build's other objects.
#   tools/build_variant.sh NAME "-DFOO=1 -DBAR=2" brm_kern_d10 [more stems...]
# -> paper_0805_1827_b200/lib/variants/libbermuda_b200_NAME.so (load with BRM_LIB_PATH)
set -e
name=$1; defs=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
obj=$root/paper_0805_1827_b200/lib/obj
out=$root/paper_0805_1827_b200/lib/variants
mkdir -p $out/obj_$name
objs=""
for o in $obj/*.o; do
  stem=$(basename $o .o)
  if [[ " $* " == *" $stem "* ]]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
      -Xcompiler -fvisibility=hidden -I $root/include -I $root/paper_0805_1827_b200/csrc $defs \
      -c $root/paper_0805_1827_b200/csrc/$stem.cu -o $out/obj_$name/$stem.o &
    objs="$objs $out/obj_$name/$stem.o"
  else
    objs="$objs $o"
  fi
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libbermuda_b200_$name.so $objs -Xcompiler -fPIC -lcudart
echo $out/libbermuda_b200_$name.so
