python -m pytest tests/test_gpu_parity.py -q -x -k "pack_variants or alignment" 2>&1 | tail -2
for v in 20 34 32 30 17 20 34 32 30 17; do
  BS_PACK_VARIANT=$v python bench.py --steps 60 --warmup 5 --no-e2e --no-cpu-baseline 2>/tmp/e.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('V$v', d['inflight'], round(d['ms_per_step'],4), round(d['stages_ms']['pack'],4), round(d['roofline']['frac'],4), round(d['window_latency_ms'],4))" || tail -3 /tmp/e.log
done
