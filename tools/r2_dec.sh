#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/dec; mkdir -p $O
for K in seg warp thread; do
QZ_DEC_KERNEL=$K python tools/probe_dense.py supremacy 30 --m 28 --depth 8 --eb 1e-7 --reps 2 --kprof > $O/sup_$K.log 2>&1
done
