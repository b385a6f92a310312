set -u
export PYTHONPATH=$PWD
mkdir -p gpurun_out/p1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/p1/smi.txt
QZ_DEBUG_COUNTERS=1 timeout 300 python tools/probe_timing.py qft relaxed > gpurun_out/p1/qft_counters.log 2>&1
timeout 600 python tools/probe_dense.py supremacy 30 --eb 1e-7 > gpurun_out/p1/sup30.log 2>&1
timeout 600 python tools/probe_dense.py qaoa 30 --eb 1e-7 > gpurun_out/p1/qaoa30.log 2>&1
timeout 600 python tools/probe_dense.py supremacy 30 --m 28 --depth 8 --eb 1e-7 --reps 1 > gpurun_out/p1/sup30m28.log 2>&1
timeout 600 python tools/probe_dense.py qft 30 --m 20 --eb 1e-5 --reps 1 > gpurun_out/p1/qft30m20.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_enc_lossy --launch-skip 1 --launch-count 1 \
   -o gpurun_out/p1/enc_sup30 -f python tools/probe_dense.py supremacy 30 --eb 1e-7 --reps 1 > gpurun_out/p1/ncu_enc.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_dec_lossy_warp --launch-skip 1 --launch-count 1 \
   -o gpurun_out/p1/dec_sup30 -f python tools/probe_dense.py supremacy 30 --m 28 --depth 8 --eb 1e-7 --reps 1 > gpurun_out/p1/ncu_dec.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tile_pass_reg --launch-skip 3 --launch-count 1 \
   -o gpurun_out/p1/pass4_qft30 -f python tools/probe_timing.py qft relaxed > gpurun_out/p1/ncu_pass.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/p1/pytest_gpu.log 2>&1
echo probe-done
