python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in c1 c2 c4; do
python bench.py --config $c --steps 100 --warmup 5 --no-e2e --no-cpu-baseline 2>/tmp/e.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['inflight'], round(d['ms_per_step'],4), round(d['window_latency_ms'],4), round(d['stages_ms']['pack'],4), round(d['roofline']['frac'],4))" || tail -3 /tmp/e.log
done
