#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/gclk2; mkdir -p $O
for F in 3 6; do
QZ_FRESH_OPEN=$F QZ_DEBUG_COUNTERS=1 QZ_COUNTERS_PER_PASS=1 QZ_JIT_SYNC=1 QZ_JIT_DEFINE=QZ_GROUP_CLOCKS python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 2 > $O/qft_$F.log 2>&1
QZ_FRESH_OPEN=$F QZ_TRACE=2 python -c "
from paper_2309_16979_b200 import circuits, engine
sim = engine.Engine().simulator(30, 16, 30, 1e-5)
sim.run(circuits.qft(30))
" > $O/plan_$F.log 2>&1
done
