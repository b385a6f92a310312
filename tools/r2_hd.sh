#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/hd; mkdir -p $O
python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 6 --kprof > $O/qft.log 2>&1
python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 2 > $O/sup.log 2>&1
python -m pytest tests -m gpu -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
