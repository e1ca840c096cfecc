OUT=gpurun_out/r1s2f; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_chain|k_size_next|k_bounds_small|k_size_describe|k_size_outcome|k_size_prep|k_size_offsets" -c 7 -f -o /tmp/k5 python tools/stage_profile.py --config c2 --steps 1 > $OUT/ncu.log 2>&1
python tools/ncu_summary.py /tmp/k5.ncu-rep --json $OUT/k5_summary.json > $OUT/k5_summary.txt 2>&1
for k in k_chain k_size_next k_bounds_small k_size_describe k_size_outcome; do python tools/ncu_source.py /tmp/k5.ncu-rep $k 30 > $OUT/src_$k.txt 2>&1; done
ncu -i /tmp/k5.ncu-rep --page raw --csv > $OUT/raw.csv 2>&1
cut -c1-250 $OUT/k5_summary.txt
