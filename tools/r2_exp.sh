#!/bin/bash
# A/B of JIT source options: QZ_JIT_DEFINE=<macro> per run
export PYTHONPATH=$PWD
O=gpurun_out/exp; mkdir -p $O
for D in QZ_X QZ_L2_PREFETCH; do
  QZ_JIT_DEFINE=$D python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 3 --kprof > $O/qft_$D.log 2>&1
  QZ_JIT_DEFINE=$D python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 3 --kprof > $O/sup_$D.log 2>&1
done
