set -u
export PYTHONPATH=$PWD
O=gpurun_out/p6; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_store_io.py tests/test_gpu_dropin.py tests/test_gpu_codec.py -x -q > $O/pytest.log 2>&1
timeout 600 python tools/probe_dense.py supremacy 30 --eb 1e-7 --reps 2 --kprof > $O/sup30.log 2>&1
timeout 900 ./build/tools/bench_transfer 20,25 5 16 25 > $O/table1.json 2> $O/table1.err
timeout 1500 python bench.py --steps 10 --warmup 3 > $O/bench.log 2>&1
echo probe-done
