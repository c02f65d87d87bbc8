mkdir -p gpurun_out/s4v
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4v/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4v/smoke_ncu.log 2>&1; echo "ncu smoke rc=$?"; tail -2 gpurun_out/s4v/smoke_ncu.log
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/s4v/smoke_launches.csv')))
hdr=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[hdr]; ki=h.index('Kernel Name')
c=collections.Counter(r[ki][:48] for r in rows[hdr+1:] if len(r)>ki)
for k,v in c.most_common(30): print(v, k)
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4v/c0_launches.csv python bench.py --config c0 --steps 2 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/s4v/c0_ncu.log 2>&1; echo "ncu c0 rc=$?"; tail -1 gpurun_out/s4v/c0_ncu.log | cut -c1-200
