#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/flush; mkdir -p $O
QZ_ENC_KERNEL=staged python -m pytest tests/test_gpu_codec.py -q -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
QZ_ENC_KERNEL=staged python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 2 --kprof > $O/sup.log 2>&1
python tools/probe_dense.py supremacy 30 --m 28 --depth 8 --eb 1e-7 --reps 2 --kprof > $O/sup28.log 2>&1
