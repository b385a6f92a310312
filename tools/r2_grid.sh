#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/grid; mkdir -p $O
for G in 3 6 16; do
QZ_PASS_GRID=$G python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 5 --kprof > $O/qft_$G.log 2>&1
QZ_PASS_GRID=$G python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 2 > $O/sup_$G.log 2>&1
done
