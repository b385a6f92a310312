#!/bin/bash
# QFT-30 / supremacy-30 pass times (JIT on) + the GPU sim / jit tests
mkdir -p gpurun_out
export PYTHONPATH=$PWD
python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 3 --kprof > gpurun_out/pq_qft.log 2>&1
python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 2 --kprof > gpurun_out/pq_sup.log 2>&1
python tools/probe_dense.py ghz 30 --c 16 --m 30 --eb 1e-5 --reps 2 --kprof > gpurun_out/pq_ghz.log 2>&1
python tools/probe_dense.py grover 24 --c 16 --m 24 --eb 1e-5 --reps 2 --kprof > gpurun_out/pq_grover.log 2>&1
python -m pytest tests/test_gpu_sim.py tests/test_jit.py -q -m gpu -x > gpurun_out/pq_tests.log 2>&1
echo "rc=$?" >> gpurun_out/pq_tests.log
