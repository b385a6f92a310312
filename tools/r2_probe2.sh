set -u
export PYTHONPATH=$PWD
O=gpurun_out/p2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_kernels.py -x -q > $O/pytest_codec.log 2>&1
timeout 600 python tools/probe_dense.py supremacy 30 --eb 1e-7 > $O/sup30.log 2>&1
timeout 600 python tools/probe_dense.py supremacy 30 --m 28 --depth 8 --eb 1e-7 --reps 1 > $O/sup30m28.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 2 > $O/bench.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_sim.py -x -q > $O/pytest_sim.log 2>&1
echo probe-done
