python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for v in 1 17; do BS_PACK_VARIANT=$v python tools/_probe_pipe.py; done
