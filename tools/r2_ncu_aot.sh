#!/bin/bash
# AOT tile_pass_reg: list launches of one QFT-30 run, full capture (with source) of the longest
export PYTHONPATH=$PWD
O=gpurun_out/na; mkdir -p $O
export QZ_JIT=0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_pass_reg --csv \
  python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 1 > $O/list.csv 2> $O/list.err
IDX=$(python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/na/list.csv')) if len(r)>10 and r[-1].replace('.','',1).isdigit()]
d=[float(r[-1]) for r in rows]
print(max(range(len(d)), key=lambda i:d[i]))
PY
)
echo "longest launch index $IDX" > $O/idx.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tile_pass_reg --launch-skip $IDX --launch-count 1 \
   -o $O/qft_aot_longest -f python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 1 > $O/ncu.log 2>&1
echo done
