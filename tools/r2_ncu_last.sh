#!/bin/bash
export PYTHONPATH=$PWD
export QZ_NO_WARMUP=1
O=gpurun_out/nl; mkdir -p $O
QZ_JIT_SYNC=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:qz_jit_pass --launch-skip 9 --launch-count 1 \
   -o $O/qft_last -f python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 1 > $O/ncu.log 2>&1
