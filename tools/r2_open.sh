#!/bin/bash
# pass splitting at fresh-bit openings: QZ_FRESH_OPEN sweep on QFT-30 (bench config)
export PYTHONPATH=$PWD
O=gpurun_out/op2; mkdir -p $O
for F in 5 6 7 8 6; do
  QZ_FRESH_OPEN=$F python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 5 > $O/qft_$F.log 2>&1
done
