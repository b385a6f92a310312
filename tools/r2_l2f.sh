#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/l2f; mkdir -p $O
for G in 128 32 64 0; do
QZ_L2_FETCH=$G python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 5 --kprof > $O/qft_$G.log 2>&1
QZ_L2_FETCH=$G python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 2 --kprof > $O/sup_$G.log 2>&1
done
python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 5 --kprof > $O/qft_unset.log 2>&1
