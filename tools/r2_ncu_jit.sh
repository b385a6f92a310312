#!/bin/bash
# ncu full capture of QFT-30 pass #3 as the runtime-specialised kernel
export PYTHONPATH=$PWD
O=gpurun_out/nj; mkdir -p $O
QZ_JIT_SYNC=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:qz_jit_pass --launch-skip 3 --launch-count 1 \
   -o $O/qft_jit_p3 -f python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 1 > $O/ncu.log 2>&1
QZ_JIT_SYNC=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:qz_jit_pass --launch-skip 2 --launch-count 1 \
   -o $O/qft_jit_p2 -f python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 1 > $O/ncu2.log 2>&1
QZ_JIT_SYNC=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:qz_jit_pass --launch-skip 20 --launch-count 1 \
   -o $O/sup_jit_p20 -f python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 1 > $O/ncu3.log 2>&1
echo done
