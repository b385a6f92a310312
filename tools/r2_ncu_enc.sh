#!/bin/bash
export PYTHONPATH=$PWD
export QZ_NO_WARMUP=1
O=gpurun_out/ne; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size -k regex:k_enc_lossy --csv python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 1 > $O/list.csv 2>&1
IDX=$(python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/ne/list.csv')) if len(r)>10 and r[-3]=='gpu__time_duration.sum']
d=[float(r[-1]) for r in rows]
print(max(range(len(d)), key=lambda i:d[i]) if d else 0)
PY
)
echo "idx $IDX" > $O/idx.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_lossy --launch-skip $IDX --launch-count 1 \
   -o $O/sup_encode -f python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 1 > $O/ncu_enc.log 2>&1
