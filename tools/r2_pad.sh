#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/pad; mkdir -p $O
for F in 3 6; do
  QZ_FRESH_OPEN=$F python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 5 --kprof > $O/qft_$F.log 2>&1
done
python -m pytest tests/test_gpu_sim.py -q -x -k "qft or large or relax or random or golden or r2" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
