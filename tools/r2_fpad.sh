#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/fpad; mkdir -p $O
for P in 0 1 2; do for F in 3 6; do
QZ_FUSE_PAD=$P QZ_FRESH_OPEN=$F python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 5 --kprof > $O/qft_${P}_$F.log 2>&1
done; done
