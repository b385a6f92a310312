#!/bin/bash
# error-bound sweep: supremacy-30 (HBM, fidelity) and supremacy-34 host-staged at eb 1e-7..1e-9
export PYTHONPATH=$PWD
O=gpurun_out/sweep; mkdir -p $O
timeout 1200 python tools/eb_sweep.py --circuit supremacy --n 30 --eb 1e-5 1e-6 1e-7 1e-8 1e-9 > $O/sup30.jsonl 2> $O/sup30.err
for EB in 1e-8 1e-9; do
  timeout 1500 python tools/run_large.py --circuit supremacy --n 34 --m 30 --eb $EB --residency host > $O/sup34_host_$EB.json 2> $O/sup34_host_$EB.err
done
echo done
