# full ncu capture of the C5 label + pricing walker launches (default library), plus variants A/B
python tools/prof_c5.py parity > gpurun_out/prof_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:walk_units -s 8 -c 2 -o gpurun_out/walk_log_c5 -f python tools/prof_c5.py parity > gpurun_out/ncu_walk.log 2>&1
tail -n 2 gpurun_out/prof_plain.log
bash tools/gpu_ab.sh "$@"
