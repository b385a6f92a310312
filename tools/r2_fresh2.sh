#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/fr2; mkdir -p $O
python -m pytest tests -m gpu -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
python tools/probe_dense.py qft 30 --c 16 --m 20 --eb 1e-5 --reps 2 --kprof > $O/qft_m20.log 2>&1
python tools/probe_dense.py qft 30 --c 16 --m 26 --eb 1e-5 --reps 2 > $O/qft_m26.log 2>&1
