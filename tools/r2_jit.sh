#!/bin/bash
# JIT vs AOT gate passes: digests and per-pass times (QFT-30 bench config, supremacy-30 d20)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
: # tests already run
echo "tests rc=$?" >> gpurun_out/jit_tests.log
for J in 0 1; do
  QZ_JIT=$J python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 3 --kprof > gpurun_out/jit_qft_$J.log 2>&1
  QZ_JIT=$J python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 2 --kprof > gpurun_out/jit_sup_$J.log 2>&1
done
