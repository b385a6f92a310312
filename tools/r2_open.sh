#!/bin/bash
# pass splitting at fresh-bit openings: QZ_FRESH_OPEN sweep on QFT-30 (bench config)
export PYTHONPATH=$PWD
O=gpurun_out/op3; mkdir -p $O
for F in 3 4 5 6 8; do
  QZ_FRESH_OPEN=$F python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 5 --kprof > $O/qft_$F.log 2>&1
done
