#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/encd; mkdir -p $O
QZ_ENC_KERNEL=direct python -m pytest tests/test_gpu_codec.py tests/test_gpu_sim.py -q -x > $O/tests_direct.log 2>&1; echo "rc=$?" >> $O/tests_direct.log
for K in staged direct; do
QZ_ENC_KERNEL=$K python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 2 --kprof > $O/sup_$K.log 2>&1
QZ_ENC_KERNEL=$K python tools/probe_dense.py supremacy 30 --m 28 --depth 8 --eb 1e-7 --reps 2 --kprof > $O/sup28_$K.log 2>&1
QZ_ENC_KERNEL=$K python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 3 --kprof > $O/qft_$K.log 2>&1
done
