#!/bin/bash
# static fresh-qubit skipping in the specialised passes: tests + timing (QZ_NO_FRESH=1 control)
export PYTHONPATH=$PWD
O=gpurun_out/fr; mkdir -p $O
python -m pytest tests/test_jit.py tests/test_gpu_sim.py -q -m gpu -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for F in 0 1; do
  if [ $F = 1 ]; then export QZ_NO_FRESH=1; fi
  python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 3 --kprof > $O/qft_$F.log 2>&1
  python tools/probe_dense.py ghz 30 --c 16 --m 30 --eb 1e-5 --reps 3 --kprof > $O/ghz_$F.log 2>&1
  python tools/probe_dense.py grover 28 --c 16 --m 28 --eb 1e-5 --reps 2 --kprof > $O/grover_$F.log 2>&1
  python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 2 --kprof > $O/sup_$F.log 2>&1
done
