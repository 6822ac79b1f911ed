# C4 after the column-constant step: rule statistics and a full ncu capture of the date-1 label launch.
set -x
O=gpurun_out/r02h; mkdir -p $O
timeout 600 python tools/c4_rule_stats.py c4 > $O/c4_rule_stats.txt 2>&1
python tools/prof_c5.py fast 1 c4 > $O/prof_c4_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:walk_units -s 19 -c 1 -o $O/walk_c4 -f python tools/prof_c5.py fast 1 c4 > $O/ncu_walk_c4.log 2>&1
tail -n 2 $O/prof_c4_plain.log; tail -n 3 $O/ncu_walk_c4.log
python tools/ncu_summary.py $O/walk_c4.ncu-rep > $O/walk_c4_fast_summary.txt 2>&1
python tools/ncu_lines.py $O/walk_c4.ncu-rep 0 1.52e10 60 > $O/walk_c4_fast_lines.txt 2>&1
cat $O/c4_rule_stats.txt
