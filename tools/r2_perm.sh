#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/pm; mkdir -p $O
python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 4 --kprof > $O/qft.log 2>&1
QZ_NO_PERM_FUSE=1 python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 4 --kprof > $O/qft_nofuse.log 2>&1
python -m pytest tests/test_gpu_fresh.py -q > $O/fresh_tests.log 2>&1; echo "rc=$?" >> $O/fresh_tests.log
python -m pytest tests -m gpu -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
