#!/bin/bash
# per-kernel launch list of one refinement evaluation (K=N=4096, M=128)
mkdir -p gpurun_out/rfn
timeout 600 python -m pytest tests/test_refine.py -q -x -m gpu --timeout 300 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rfn/launches.csv python tools/perf_refine.py 4096 4096 128 > gpurun_out/rfn/perf.txt 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/rfn/launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
for r in rows[1:]: print(r[ki][:60], r[vi], r[ui])
PY
