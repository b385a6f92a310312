set -u
export PYTHONPATH=$PWD
O=gpurun_out/p11; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_codec.py -x -q > $O/pytest_codec.log 2>&1
timeout 600 python tools/probe_dense.py supremacy 30 --m 28 --depth 8 --eb 1e-7 --reps 2 > $O/sup30m28.log 2>&1
QZ_DEC_KERNEL=warp timeout 600 python tools/probe_dense.py supremacy 30 --m 28 --depth 8 --eb 1e-7 --reps 2 > $O/sup30m28_warp.log 2>&1
timeout 600 python tools/probe_dense.py qft 30 --m 20 --eb 1e-5 --reps 2 > $O/qft30m20.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_dec_lossy_seg --launch-skip 2 --launch-count 1 \
   -o $O/dec_seg -f python tools/probe_dense.py supremacy 30 --m 28 --depth 8 --eb 1e-7 --reps 1 > $O/ncu_dec.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_sim.py -x -q > $O/pytest_sim.log 2>&1
echo probe-done
