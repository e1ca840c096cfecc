python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for v in 1 14; do for c in c2 c3 c4; do echo -n "$c variant $v: "; BS_PACK_VARIANT=$v python tools/stage_profile.py --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stage_us']['pack'])"; done; done
BS_PACK_VARIANT=14 python -m pytest tests/test_gpu_parity.py -q -x -k "fixture or c2 or c4" 2>&1 | tail -1
