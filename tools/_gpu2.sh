python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for c in c2 c3; do echo -n "$c align32: "; python tools/stage_profile.py --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['summary']; print(d['stage_us']['pack'], s['packed_elems'], s['admitted_tokens'])"; done
