set -u
export PYTHONPATH=$PWD
O=gpurun_out/p3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_kernels.py tests/test_gpu_store_io.py -x -q > $O/pytest_a.log 2>&1
timeout 600 python tools/probe_dense.py supremacy 30 --eb 1e-7 > $O/sup30.log 2>&1
timeout 600 python tools/probe_dense.py supremacy 30 --m 28 --depth 8 --eb 1e-7 --reps 2 > $O/sup30m28.log 2>&1
timeout 600 python tools/probe_dense.py qft 30 --m 20 --eb 1e-5 --reps 2 > $O/qft30m20.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_sim.py -x -q > $O/pytest_sim.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_enc_lossy --launch-skip 1 --launch-count 1 \
   -o $O/enc_sup30 -f python tools/probe_dense.py supremacy 30 --eb 1e-7 --reps 1 > $O/ncu_enc.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_dec_lossy_coop --launch-skip 2 --launch-count 1 \
   -o $O/dec_sup30 -f python tools/probe_dense.py supremacy 30 --m 28 --depth 8 --eb 1e-7 --reps 1 > $O/ncu_dec.log 2>&1
echo probe-done
