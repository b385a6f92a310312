#!/bin/bash
# per-pass, per-group CTA cycle split of the specialised passes (inspection build)
export PYTHONPATH=$PWD
O=gpurun_out/gclk; mkdir -p $O
QZ_DEBUG_COUNTERS=1 QZ_COUNTERS_PER_PASS=1 QZ_JIT_SYNC=1 QZ_JIT_DEFINE=QZ_GROUP_CLOCKS python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 2 > $O/qft.log 2>&1
QZ_DEBUG_COUNTERS=1 QZ_COUNTERS_PER_PASS=1 QZ_JIT_SYNC=1 QZ_JIT_DEFINE=QZ_GROUP_CLOCKS python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --depth 8 --reps 1 > $O/sup.log 2>&1
