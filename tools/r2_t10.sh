#!/bin/bash
# tile 2^10 x 6 CTAs/SM variant library vs the default build
export PYTHONPATH=$PWD
O=gpurun_out/t10; mkdir -p $O
QZC_LIB=$PWD/build/var_t10/libqzcuda.so python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 3 --kprof > $O/qft_t10.log 2>&1
QZC_LIB=$PWD/build/var_t10/libqzcuda.so python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 3 --kprof > $O/sup_t10.log 2>&1
