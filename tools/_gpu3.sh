OUT=gpurun_out/r1s2h; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:"k_bounds_small|k_size_next|k_sort_pass|k_histogram|k_size_describe" -c 6 -f -o /tmp/k2 python tools/stage_profile.py --config c2 --steps 1 > $OUT/ncu.log 2>&1
for k in k_bounds_small k_size_next k_sort_pass k_histogram k_size_describe; do python tools/ncu_source.py /tmp/k2.ncu-rep $k 40 > $OUT/src_$k.txt 2>&1; done
python tools/ncu_summary.py /tmp/k2.ncu-rep --json $OUT/k2_summary.json > $OUT/k2_summary.txt 2>&1
cut -c1-200 $OUT/k2_summary.txt
