# decode: ms per token (graph) and the kernel launch list of one decode step (ncu, serialised)
mkdir -p gpurun_out/dec
timeout 600 python tools/decode_bench.py > gpurun_out/dec/decode_bench.json 2>&1
cat gpurun_out/dec/decode_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv -s 900 -c 40 --log-file gpurun_out/dec/launches.csv python tools/decode_bench.py > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/dec/launches.csv')))
i=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
h=rows[i]; k=h.index('Kernel Name'); v=h.index('Metric Value'); g=h.index('Grid Size')
for r in rows[i+1:i+41]:
    print(r[k][:50], r[g], r[v])
PY
