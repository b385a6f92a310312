#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/ct; mkdir -p $O
for C in 2 3; do
  QZ_JIT_MIN_CTAS=$C python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 3 --kprof > $O/qft_$C.log 2>&1
  QZ_JIT_MIN_CTAS=$C python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 3 --kprof > $O/sup_$C.log 2>&1
done
