OUT=gpurun_out/r1s2c; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file $OUT/launches.csv python tools/stage_profile.py --config c2 --dispatch --steps 1 > $OUT/ncu.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/r1s2c/launches.csv")))
hdr=None
for r in rows:
    if r and r[0]=="ID": hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); print(d["Kernel Name"][:60], d["Grid Size"], d["Metric Value"])
PY
