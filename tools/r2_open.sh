#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/op5; mkdir -p $O
for F in 1 2 3; do
  QZ_FRESH_OPEN=$F python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 5 --kprof > $O/qft_$F.log 2>&1
done
