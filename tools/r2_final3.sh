#!/bin/bash
# round-2 closing measurement: bench (default), launch list, ncu captures of the dominant pass and the encoder
export PYTHONPATH=$PWD
O=gpurun_out/f3b; mkdir -p $O
( time python bench.py ) > $O/bench.json 2> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-companions > $O/ncu_list.log 2>&1
QZ_JIT_SYNC=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:qz_jit_pass --launch-skip 4 --launch-count 1 \
   -o $O/qft_fused_pass -f python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 1 > $O/ncu_pass.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_lossy --launch-skip 1 --launch-count 1 \
   -o $O/qft_encode -f python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 1 > $O/ncu_enc.log 2>&1
echo done
