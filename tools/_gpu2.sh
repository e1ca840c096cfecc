python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for agg in 1 0; do for e in 2 4 8 16; do echo -n "agg $agg ept $e: "; BS_HIST_AGG=$agg BS_HIST_EPT=$e python tools/stage_profile.py --config c2 | python -c "import json,sys; print(json.loads(sys.stdin.read())['stage_us']['histogram'])"; done; done
for agg in 1 0; do for e in 4 16; do echo -n "c3 agg $agg ept $e: "; BS_HIST_AGG=$agg BS_HIST_EPT=$e python tools/stage_profile.py --config c3 | python -c "import json,sys; print(json.loads(sys.stdin.read())['stage_us']['histogram'])"; done; done
for agg in 1 0; do echo -n "c4 agg $agg: "; BS_HIST_AGG=$agg BS_HIST_EPT=4 python tools/stage_profile.py --config c4 | python -c "import json,sys; print(json.loads(sys.stdin.read())['stage_us']['histogram'])"; done
