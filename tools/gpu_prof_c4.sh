# full ncu capture of one C4 label launch (fast mode, d = 40) and one pricing launch
python tools/prof_c5.py fast 1 c4 > gpurun_out/prof_c4_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:walk_units -s 19 -c 1 -o gpurun_out/walk_c4 -f python tools/prof_c5.py fast 1 c4 > gpurun_out/ncu_walk_c4.log 2>&1
tail -n 2 gpurun_out/prof_c4_plain.log; tail -n 3 gpurun_out/ncu_walk_c4.log
