#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/dir; mkdir -p $O
for D in 0 1; do
  if [ $D = 1 ]; then export QZ_NO_DIRECT=1; fi
  python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 5 --kprof > $O/qft_$D.log 2>&1
  python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 2 > $O/sup_$D.log 2>&1
  python tools/probe_dense.py grover 28 --c 16 --m 28 --eb 1e-5 --reps 2 > $O/grover_$D.log 2>&1
done
unset QZ_NO_DIRECT
python -m pytest tests -m gpu -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
