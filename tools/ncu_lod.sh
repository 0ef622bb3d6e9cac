# ncu of the LoD kernels at C3, record and packed density (developer tool)
out=gpurun_out; mkdir -p $out
for mode in ${LOD_MODES:-rec packed}; do
LVX_DENSITY=$mode timeout 600 ncu --set full --clock-control none --import-source on -k regex:'density|mip' -s 4 -c 4 -f -o /tmp/lod_$mode python tools/lod_perf.py 100000 > $out/ncu_lod_$mode.log 2>&1; echo "rc=$?"
ncu -i /tmp/lod_$mode.ncu-rep --page raw --csv > $out/lod_$mode.csv
python tools/ncu_table.py $out/lod_$mode.csv --by-launch --title "LoD $mode" > $out/lod_$mode.txt
ncu -i /tmp/lod_$mode.ncu-rep --page source --csv -k regex:density > $out/lod_${mode}_src.csv 2>/dev/null
done
cat $out/lod_rec.txt $out/lod_packed.txt
