set -u
OUT=gpurun_out/r1s2g; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for c in c2 c3 c4; do timeout 300 python tools/stage_profile.py --config $c --dispatch > $OUT/stages_$c.json 2>&1; done
tail -3 $OUT/pytest_gpu.log; cat $OUT/stages_*.json | cut -c1-330
