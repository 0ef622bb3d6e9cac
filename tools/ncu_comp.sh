# source-level ncu capture of one kernel of the C3 frame (developer tool): tools/ncu_comp.sh <kernel regex> <skip> <count>
out=gpurun_out; mkdir -p $out
k=${1:-wf_composite}; s=${2:-1}; c=${3:-2}
PERF_QUICK=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c -f -o /tmp/src_$k python tools/frame_perf.py c3 > $out/ncu_src_$k.log 2>&1; echo "rc=$?"
ncu -i /tmp/src_$k.ncu-rep --page source --csv > $out/src_$k.csv 2>/dev/null
ncu -i /tmp/src_$k.ncu-rep --page source --csv --print-source cuda > $out/srccu_$k.csv 2>/dev/null
ncu -i /tmp/src_$k.ncu-rep --page raw --csv > $out/raw_$k.csv
python tools/ncu_table.py $out/raw_$k.csv --by-launch | cut -c1-250
ls -la $out/src_$k.csv $out/srccu_$k.csv
