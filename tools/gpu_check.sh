#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench lines, ncu launch list and a full
# capture of the main kernels (summaries land in gpurun_out/TAG; copy the ones to
# keep into profiles/).   usage: tools/gpu_check.sh TAG [skip-tests]
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
if [ "${2:-}" != "skip-tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
fi
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 300 python tools/timeline.py --out $OUT/timeline_c2.json > $OUT/timeline_c2.txt 2>&1
timeout 600 python bench.py --dispatch --steps 50 --no-cpu-baseline --no-e2e > $OUT/bench_dispatch.json 2> $OUT/bench_dispatch.err
timeout 600 python bench.py --config c3 --steps 20 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 600 python bench.py --config c4 --steps 20 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 python bench.py --config c1 --steps 200 > $OUT/bench_c1.json 2> $OUT/bench_c1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 300 python tools/small_timing.py 2 > $OUT/k0_phases.txt 2>&1
timeout 600 python tools/ref_python_bench.py --out $OUT/reference_python_host.jsonl > /dev/null 2> $OUT/reference_python_host.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:"k_pack_bulk|k_sort_pass|k_histogram|k_dispatch|k_bounds_small|k_size_next|k_chain_walk|k_size_outcome" -c 9 -f -o /tmp/full \
   python tools/stage_profile.py --config c2 --steps 1 --dispatch > $OUT/ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/full.ncu-rep --json $OUT/full_summary.json > $OUT/full_summary.txt 2>&1
for c in c1 c3 c4; do  # the other configs' pack launch: DRAM bytes for their roofline.traffic
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
     --clock-control none -k regex:"k_pack_(bulk|rows)" --launch-skip 1 -c 1 --csv \
     python tools/stage_profile.py --config $c --steps 1 > $OUT/pack_traffic_$c.csv 2>/dev/null
done
for k in k_pack_bulk k_histogram k_sort_pass k_dispatch k_size_next k_chain_walk; do
  python tools/ncu_source.py /tmp/full.ncu-rep $k 25 > $OUT/src_$k.txt 2>&1
done
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; cat $OUT/bench.json
