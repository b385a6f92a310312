set -u
export PYTHONPATH=$PWD
O=gpurun_out/p12; mkdir -p $O
timeout 300 python tools/probe_dense.py qft 30 --m 30 --eb 1e-5 --reps 3 --kprof > $O/qft30.log 2>&1
timeout 300 python tools/probe_dense.py supremacy 30 --m 30 --eb 1e-7 --reps 2 --kprof > $O/sup30.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_sim.py tests/test_gpu_kernels.py tests/test_gpu_store_io.py -x -q > $O/pytest.log 2>&1
echo probe-done
