python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_dispatch.py -q -x -k "multi_cta" 2>&1 | tail -3
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_dispatch.py -q -x -k "multi_cta and 2-0" 2>&1 | tail -3
done
