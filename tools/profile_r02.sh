#!/usr/bin/env bash
# ncu captures for profiles/ (run on the GPU box from the repo root):
#   launch list of the C5 bench step, full sections of the top kernels.
set -x
mkdir -p gpurun_out/prof
NCU="ncu --clock-control none"
export BRM_NCU_SAFE=1  # no cooperative cluster launches under ncu (boost: 1 CTA per feature; I&Z: no bisection tree)
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-fast-line"
$NCU --metrics gpu__time_duration.sum -c 2000 --csv --log-file gpurun_out/prof/launches_c5.csv $B > gpurun_out/prof/launches_c5.log 2>&1
$NCU --metrics gpu__time_duration.sum -c 2000 --csv --log-file gpurun_out/prof/launches_c2.csv $B --config c2 > gpurun_out/prof/launches_c2.log 2>&1
$NCU --metrics gpu__time_duration.sum -c 2000 --csv --log-file gpurun_out/prof/launches_c1.csv $B --config c1 > gpurun_out/prof/launches_c1.log 2>&1
# full sections: the C5 label walker (date 8 labels), the C2 probe clusters, the LS fit, the sampler
$NCU --set full --import-source on -k regex:walk_units -c 1 -o gpurun_out/prof/walk_c5 -f $B > gpurun_out/prof/walk_c5.log 2>&1
$NCU --set full --import-source on -k regex:iz_probes -c 1 -o gpurun_out/prof/iz_c2 -f $B --config c2 > gpurun_out/prof/iz_c2.log 2>&1
$NCU --set full --import-source on -k regex:ls_fit -c 1 -o gpurun_out/prof/lsfit_c2 -f $B --config c2 > gpurun_out/prof/lsfit_c2.log 2>&1
$NCU --set full --import-source on -k regex:sample_points -c 1 -o gpurun_out/prof/sample_c5 -f $B > gpurun_out/prof/sample_c5.log 2>&1
$NCU --set full --import-source on -k regex:iz_probes -c 1 -o gpurun_out/prof/iz_c1 -f $B --config c1 > gpurun_out/prof/iz_c1.log 2>&1
ls -la gpurun_out/prof
