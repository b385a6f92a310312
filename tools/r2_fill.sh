#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/fill; mkdir -p $O
QZ_DEBUG_COUNTERS=1 QZ_COUNTERS_PER_PASS=1 QZ_JIT_SYNC=1 QZ_JIT_DEFINE=QZ_COUNT_FILL python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 1 > $O/qft.log 2>&1
QZ_DEBUG_COUNTERS=1 QZ_COUNTERS_PER_PASS=1 QZ_JIT=0 python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 1 > $O/qft_aot.log 2>&1
