#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/ex; mkdir -p $O
for i in 1 2; do
QZ_JIT=0 python -m pytest tests/test_gpu_sim.py -q -x -k "qft or large or relax or random" > $O/nojit_$i.log 2>&1; echo "rc=$?" >> $O/nojit_$i.log
python -m pytest tests/test_gpu_sim.py -q -x -k "qft or large or relax or random" > $O/jit_$i.log 2>&1; echo "rc=$?" >> $O/jit_$i.log
done
