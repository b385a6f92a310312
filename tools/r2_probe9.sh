set -u
export PYTHONPATH=$PWD
O=gpurun_out/p9; mkdir -p $O
timeout 300 python tools/probe_dense.py qft 30 --m 30 --eb 1e-5 --reps 3 --kprof > $O/qft30.log 2>&1
timeout 300 python tools/probe_dense.py supremacy 30 --m 30 --eb 1e-7 --reps 2 --kprof > $O/sup30.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
echo probe-done
