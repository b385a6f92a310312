#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/ct3; mkdir -p $O
for C in 3 4 6; do
  QZ_JIT_MIN_CTAS=$C python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 4 --kprof > $O/qft_$C.log 2>&1
done
